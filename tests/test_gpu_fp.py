"""GPU parity of the feature processing layer (NEXT#4, include/dhen.h dhen_fp_*, csrc/fp.cu) against the fp64
oracle (oracle/fp_oracle.py) on the same seeded inputs (synth.make_fp_batch): X0, and after one backward +
SGD every table and bottom-MLP parameter.

Tolerances: fp32 runs -- the lookups, sums and GEMMs are fp32 (SIMT GEMMs, exact fp32): 1e-5 normwise;
bf16 runs -- the oracle emulates the same storage points (dense input, W copies, hidden activations, X0, dZ):
X0 element error <= 1 bf16 ulp of the element (<= |x| 2^-7) + 1e-6 (an fp32 vs fp64 sum can round to the
neighbouring bf16 value), MLP parameter steps 2e-2 normwise (BASELINE G3), table steps 1e-5 (the dX0 rows
are exact bf16 values summed in fp32)."""
import numpy as np
import pytest

import synth
from oracle import fp_oracle as FO
from tests.helpers import norm_err

pytestmark = pytest.mark.gpu


def _run(rows, n_dense, hidden, n_dtok, d, B, dtype, seed=1, mean_bag=3.0, lr=0.5, empty_frac=0.1, bad=None):
    import torch
    from paper_2203_11014_b200.binding import FeatureProcessing
    bf = dtype == "bf16"
    ids, off, dense = synth.make_fp_batch(seed, B, rows, n_dense, mean_bag, bf16=bf, empty_frac=empty_frac)
    if bad is not None:   # out-of-range ids: skipped by both sides' definition (the oracle drops them here)
        ids = ids.copy()
        ids[bad] = rows[0] + 5
    spec = FO.FPSpec(list(rows), n_dense, list(hidden), n_dtok, d)
    fp = FeatureProcessing(rows, n_dense, hidden, n_dtok, d, dtype=dtype, max_batch=B, max_nnz=max(1, len(ids)),
                           seed=seed)
    P = {"tables": [fp.get(t).reshape(R, d).astype(np.float64) for t, R in enumerate(rows)], "W": [], "b": []}
    dims = spec.mlp_dims()
    if n_dtok:
        for k in range(len(dims) - 1):
            P["W"].append(fp.get(len(rows) + 2 * k).reshape(dims[k + 1], dims[k]).astype(np.float64))
            P["b"].append(fp.get(len(rows) + 2 * k + 1).astype(np.float64))
    tdt = torch.bfloat16 if bf else torch.float32
    t_ids = torch.tensor(ids, device="cuda")
    t_off = torch.tensor(off, device="cuda")
    t_dense = torch.tensor(dense, device="cuda").to(tdt).contiguous() if n_dense else torch.zeros(B, 8, device="cuda", dtype=tdt)
    x0 = torch.empty(B, spec.m0, d, device="cuda", dtype=tdt)
    fp.forward(t_ids, t_off, t_dense, x0)
    G = synth.make_x0(seed + 5, B, spec.m0, d, bf16=bf).astype(np.float64) * 0.1   # an upstream dX0
    if bf:
        G = FO.round_bf16(G)
    fp.backward_sgd(torch.tensor(G, dtype=torch.float32, device="cuda").to(tdt), lr)
    torch.cuda.synchronize()
    got = {"X0": x0.float().cpu().numpy().astype(np.float64),
           "tables": [fp.get(t).reshape(R, d).astype(np.float64) for t, R in enumerate(rows)],
           "W": [fp.get(len(rows) + 2 * k).astype(np.float64) for k in range(len(P["W"]))],
           "b": [fp.get(len(rows) + 2 * k + 1).astype(np.float64) for k in range(len(P["b"]))],
           "bad": fp.bad_ids()}
    o_ids = ids.astype(np.int64)
    o_off = off.astype(np.int64)
    if bad is not None:   # the oracle's reading of a skipped id: the bag without it
        keep = np.ones(len(ids), bool)
        keep[bad] = False
        cnt = np.concatenate([[0], np.cumsum(keep)])
        o_off, o_ids = cnt[o_off], o_ids[keep]
    prec = FO.FPPrecision(bf)
    X0, cache = FO.fp_fwd(spec, P, o_ids, o_off, dense.astype(np.float64), prec)
    newP = FO.fp_sgd(P, FO.fp_bwd(spec, P, cache, G, prec), lr)
    return got, X0, P, newP


def _check(got, X0, P, newP, bf, nd):
    if bf:   # pooled tokens: within one bf16 ulp; dense tokens (two bf16 GEMM layers deep): G3-style normwise
        err = np.abs(got["X0"][:, nd:] - X0[:, nd:])
        assert np.all(err <= np.abs(X0[:, nd:]) * 2.0 ** -7 + 1e-6), err.max()
        if nd:
            assert norm_err(got["X0"][:, :nd], X0[:, :nd]) <= 1e-2
    else:
        assert norm_err(got["X0"], X0) <= 1e-5
    for a, o, p in zip(got["tables"], newP["tables"], P["tables"]):
        assert norm_err(a - p, o - p) <= 1e-5
        assert np.array_equal(a[np.all(o == p, axis=1)], p[np.all(o == p, axis=1)])   # untouched rows unchanged
    for a, o, p in zip(got["W"], newP["W"], P["W"]):
        assert norm_err(a - p.reshape(-1), (o - p).reshape(-1)) <= (2e-2 if bf else 1e-5)
    for a, o, p in zip(got["b"], newP["b"], P["b"]):
        assert norm_err(a - p, o - p) <= (2e-2 if bf else 1e-5)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("shape", [
    ((50, 7, 300), 16, (32,), 2, 128, 24),       # several tables, one hidden layer, 2 dense tokens
    ((1000, 40), 13, (64, 32), 1, 256, 33),      # DLRM's 13 dense features (K not a multiple of 8), d = 256
    ((9,), 8, (), 1, 16, 5),                     # C1-sized d = 16, no hidden layer
])
def test_fp_matches_oracle(dtype, shape):
    rows, n_dense, hidden, n_dtok, d, B = shape
    got, X0, P, newP = _run(rows, n_dense, hidden, n_dtok, d, B, dtype)
    _check(got, X0, P, newP, dtype == "bf16", n_dtok)
    assert got["bad"] == 0


def test_fp_sparse_only_and_dense_only():
    got, X0, P, newP = _run((20, 30), 0, (), 0, 128, 16, "fp32")       # no bottom MLP
    _check(got, X0, P, newP, False, 0)
    got, X0, P, newP = _run((), 24, (48,), 3, 128, 16, "bf16")          # no tables
    _check(got, X0, P, newP, True, 3)


def test_fp_out_of_range_ids_skipped():
    got, X0, P, newP = _run((40, 40), 8, (16,), 1, 128, 12, "fp32", bad=[0, 3, 7])
    _check(got, X0, P, newP, False, 1)
    assert got["bad"] == 3


@pytest.mark.parametrize("rows,B,mean_bag", [((64,), 64, 20.0), ((3, 5), 256, 8.0)])
def test_fp_hot_rows_deterministic(rows, B, mean_bag):
    """Power-law ids with long bags (a few rows hit hundreds of times per batch; with 3- and 5-row tables every
    run is hundreds of occurrences long): the sorted-run SGD is deterministic -- two runs give bit-identical
    tables -- and matches the oracle."""
    a = _run(rows, 8, (16,), 1, 256, B, "bf16", seed=3, mean_bag=mean_bag, empty_frac=0.0)
    b = _run(rows, 8, (16,), 1, 256, B, "bf16", seed=3, mean_bag=mean_bag, empty_frac=0.0)
    _check(*a, True, 1)
    for x, y in zip(a[0]["tables"], b[0]["tables"]):
        assert np.array_equal(x, y)


def test_fp_timed_size_sampled():
    """The bench's feature-processing shape (C4F) at a reduced batch: 120 tables x 100k rows,
    d = 256, 8 dense tokens from 64 features; X0 of 4 sampled samples and the touched rows of 3 tables."""
    import torch
    from paper_2203_11014_b200.binding import FeatureProcessing
    rows, n_dense, hidden, n_dtok, d, B = [100_000] * 120, 64, (512,), 8, 256, 256
    ids, off, dense = synth.make_fp_batch(11, B, rows, n_dense, 20.0, bf16=True)
    fp = FeatureProcessing(rows, n_dense, hidden, n_dtok, d, dtype="bf16", max_batch=B, max_nnz=len(ids), seed=11)
    x0 = torch.empty(B, n_dtok + len(rows), d, device="cuda", dtype=torch.bfloat16)
    fp.forward(torch.tensor(ids, device="cuda"), torch.tensor(off, device="cuda"),
               torch.tensor(dense, device="cuda").to(torch.bfloat16), x0)
    torch.cuda.synchronize()
    X = x0.float().cpu().numpy().astype(np.float64)
    ns = len(rows)
    for t in (0, 57, 119):
        T = fp.get(t).reshape(rows[t], d).astype(np.float64)
        for b in (0, 1, 128, 255):
            lo, hi = off[b * ns + t], off[b * ns + t + 1]
            ref = FO.round_bf16(FO.embedding_bag_sum(T, ids[lo:hi]))
            assert np.all(np.abs(X[b, n_dtok + t] - ref) <= np.abs(ref) * 2.0 ** -7 + 1e-6)


def _sharded(rows, n_dense, hidden, n_dtok, d, B, world, dtype="bf16", seed=5, lr=0.5):
    """One forward + backward/SGD of the column-sharded layer at `world` loopback ranks (B samples each) and the
    same global batch on one unsharded object."""
    import threading
    import torch
    from paper_2203_11014_b200 import binding
    from paper_2203_11014_b200.binding import FeatureProcessing
    bf = dtype == "bf16"
    tdt = torch.bfloat16 if bf else torch.float32
    Bg, ns = world * B, len(rows)
    ids, off, dense = synth.make_fp_batch(seed, Bg, rows, n_dense, 6.0, bf16=bf, empty_frac=0.1)
    G = synth.make_x0(seed + 5, Bg, n_dtok + ns, d, bf16=bf) * 0.1
    G = FO.round_bf16(G.astype(np.float64)) if bf else G
    # world 1 on the whole global batch
    ref = FeatureProcessing(rows, n_dense, hidden, n_dtok, d, dtype=dtype, max_batch=Bg, max_nnz=len(ids), seed=seed)
    x_ref = torch.empty(Bg, n_dtok + ns, d, device="cuda", dtype=tdt)
    ref.forward(torch.tensor(ids, device="cuda"), torch.tensor(off, device="cuda"),
                torch.tensor(dense, device="cuda").to(tdt).contiguous(), x_ref)
    ref.backward_sgd(torch.tensor(G, dtype=torch.float32, device="cuda").to(tdt), lr)
    torch.cuda.synchronize()
    nP = ns + 2 * (len(hidden) + 1)
    P_ref = [ref.get(w) for w in range(nP)]
    X_ref = x_ref.float().cpu().numpy()
    nid = binding.loopback_id()
    out, errs = [None] * world, []

    def work(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                probe = FeatureProcessing(rows, n_dense, hidden, n_dtok, d, dtype=dtype, max_batch=B, max_nnz=1, seed=seed)
                S, own = probe.plan(world)
                probe.close()
                owned = sorted({t for t in range(ns) for k in range(S[t]) if own[sum(S[:t]) + k] == r})
                rid, roff = [], [0]   # the global batch's bags of the owned tables, (sample, owned table) order
                for b in range(Bg):
                    for t in owned:
                        seg = ids[off[b * ns + t]:off[b * ns + t + 1]]
                        rid.extend(seg.tolist())
                        roff.append(roff[-1] + len(seg))
                fp = FeatureProcessing(rows, n_dense, hidden, n_dtok, d, dtype=dtype, max_batch=B,
                                       max_nnz=max(1, len(rid)), seed=seed, rank=r, world=world, comm_id=nid,
                                       backend=binding.LOOPBACK)
                assert fp.owned_tables() == owned
                x0 = torch.empty(B, n_dtok + ns, d, device="cuda", dtype=tdt)
                fp.forward(torch.tensor(np.array(rid, np.int32), device="cuda"),
                           torch.tensor(np.array(roff, np.int32), device="cuda"),
                           torch.tensor(dense[r * B:(r + 1) * B], device="cuda").to(tdt).contiguous(), x0)
                fp.backward_sgd(torch.tensor(G[r * B:(r + 1) * B], dtype=torch.float32, device="cuda").to(tdt), lr)
                s.synchronize()
                out[r] = {"X0": x0.float().cpu().numpy(), "P": [fp.get(w) for w in range(nP)], "owned": owned, "fp": fp}
        except Exception as e:  # pragma: no cover - reported below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return X_ref, P_ref, out, ns


@pytest.mark.parametrize("world", [2, 4])
def test_fp_sharded_matches_single(world):
    """Column-sharded tables over `world` loopback ranks (LPT plan, pooled all-to-all forward and backward,
    data-parallel bottom MLP with an all-reduce) against one object holding every table, on the same global
    batch: X0 of every rank's samples and every table after the sparse SGD are bit-identical (the same sums in
    the same order), the bottom MLP within fp32 rounding of the split batch (rank-order all-reduce)."""
    rows, d = (300, 40, 1000, 7, 64), 128      # a large table is cut into column shards, small ones stay whole
    X_ref, P_ref, out, ns = _sharded(rows, 16, (32,), 2, d, 12, world)
    B = 12
    for r, o in enumerate(out):
        assert np.array_equal(o["X0"], X_ref[r * B:(r + 1) * B]), r
    for t in range(ns):   # each rank fills the columns of its shards; together they cover the table once
        merged = np.zeros_like(P_ref[t])
        for o in out:
            merged += o["P"][t]
        assert np.array_equal(merged, P_ref[t]), t
    for w in range(ns, len(P_ref)):
        for o in out:
            assert norm_err(o["P"][w].astype(np.float64), P_ref[w].astype(np.float64)) <= 1e-5, w
