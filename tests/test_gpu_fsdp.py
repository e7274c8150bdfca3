"""The FSDP path executed on one GPU (§8(a) F0 parameter all-gather, B11 gradient
reduce-scatter, B12 SGD on the local shard; PAPER P:142 / P:161 / P:171).

Each test runs `world` virtual ranks in this process through the library's loopback collective backend
(include/dhen.h, dhen_dist.backend = 1): one host thread, one dhen_ctx and one stream per rank, every rank
holding its 1/world shard of every parameter group and its 1/world slice of the global batch.  The
collectives go through the same seam as NCCL (comm.h) -- the runtime's prefetch / slot-release events,
communication stream, reduce-scatter and sharded SGD all run for real; only the transport is in-process
copies and fixed-order sums.  Gate G4: the world-G step equals the world-1 step on the same
global batch -- loss, dL/dX0, every reduced gradient and every updated parameter -- within G1 (fp32 mode,
1e-5) / G3 (bf16, 2e-2), and each rank's collective bytes equal the FSDP byte count of DESIGN.md §10.
"""
import threading

import numpy as np
import pytest

import synth
from oracle import dhen_oracle as O
from tests.gpu_common import t2np, to_binding
from tests.helpers import elem_err, make_flat_params, norm_err, small

pytestmark = pytest.mark.gpu


def _inputs(net, B, dtype, seed):
    X0 = synth.make_x0(seed, B, net.m0, net.d, bf16=(dtype == "bf16"))
    y = synth.make_labels(seed, B)
    return X0, y


def _rank_step(cfg, flats, X0, y, lr, B, rank, world, nid, fsdp, backend, out):
    import torch
    from paper_2203_11014_b200 import binding
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        m = binding.DHEN(cfg, rank=rank, world=world, nccl_id=nid, fsdp=fsdp, backend=backend, stream=s)
        for gi, f in enumerate(flats):
            m.set_params(gi, f, stream=s)
        Bl = B // world
        tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
        x0 = torch.tensor(X0[rank * Bl:(rank + 1) * Bl], device="cuda").to(tdt).contiguous()
        lab = torch.tensor(y[rank * Bl:(rank + 1) * Bl], device="cuda")
        loss = torch.zeros(1, device="cuda")
        dx0 = torch.empty_like(x0)
        s.synchronize()
        b0 = m.comm_bytes()
        m.train_step(x0, lab, lr, B_global=B, loss=loss, dx0=dx0, stream=s)
        s.synchronize()
        b1 = m.comm_bytes()
        grads = [m.get_grads(g, stream=s).astype(np.float64) for g in range(len(flats))]
        params = [m.get_params(g, stream=s).astype(np.float64) for g in range(len(flats))]
        out[rank] = {"loss": float(loss.item()), "dX0": t2np(dx0), "grads": grads, "params": params,
                     "bytes": b1 - b0, "model": m}


def run(net, dtype, B, world, seed=3, lr=0.05, fsdp=True):
    """One training step at `world` virtual ranks (world 1 = the plain single-GPU context)."""
    from paper_2203_11014_b200 import binding
    flats = make_flat_params(net, seed)
    X0, y = _inputs(net, B, dtype, seed)
    cfg = to_binding(net, dtype, B // world)
    nid = binding.loopback_id() if world > 1 else None
    out, errs = [None] * world, []

    def work(r):
        try:
            _rank_step(cfg, flats, X0, y, lr, B, r, world, nid, fsdp, binding.LOOPBACK, out)
        except Exception as e:  # pragma: no cover - reported below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert all(o is not None for o in out), "a rank did not finish"
    res = {"loss": sum(o["loss"] for o in out), "dX0": np.concatenate([o["dX0"] for o in out]),
           "grads": out[0]["grads"], "params": out[0]["params"], "bytes": [o["bytes"] for o in out],
           "ranks": out, "cfg": cfg}
    return res


def expected_bytes(cfg, world, es, n_layers):
    """Per-rank bytes of one FSDP step: every group (layers + head) all-gathered once for the
    forward, layers 0 .. L-2 again for the backward (layer L-1 is still resident in its slot when its backward
    starts), every group reduce-scattered once (fp32)."""
    from paper_2203_11014_b200 import binding
    dist = binding.make_dist(0, world)
    sh = [binding.group_numel(cfg, g, dist)[1] for g in range(n_layers + 1)]
    ag = sum(sh) + sum(sh[:max(0, n_layers - 1)])
    return (world - 1) * (ag * es + sum(sh) * 4)


def _compare(one, many, tol_out, tol_grad, label):
    errs = {"loss": elem_err(many["loss"], one["loss"]), "dX0": norm_err(many["dX0"], one["dX0"])}
    for g, (a, b) in enumerate(zip(many["grads"], one["grads"])):
        errs[f"grad{g}"] = norm_err(a, b)
    for g, (a, b) in enumerate(zip(many["params"], one["params"])):
        errs[f"param{g}"] = elem_err(a, b)
    worst = max(errs.items(), key=lambda kv: kv[1])
    print(f"{label}: worst {worst[0]} {worst[1]:.3g}; " + " ".join(f"{k}={v:.2g}" for k, v in errs.items()))
    for k, v in errs.items():
        tol = tol_grad if (k.startswith("grad") or k == "dX0") else tol_out
        assert v <= tol, (label, k, v, tol)


CASES = [  # (config, dtype, global B, world)
    ("C2", "fp32", 16, 2),
    ("C2", "bf16", 64, 2),
    ("C2", "bf16", 64, 4),
    ("C4", "bf16", 64, 2),
    ("C3", "bf16", 64, 2),
    ("C5", "fp32", 16, 4),
]


@pytest.mark.parametrize("name,dtype,B,world", CASES)
def test_fsdp_world_matches_world1(name, dtype, B, world):
    net = small(name)
    one = run(net, dtype, B, 1)
    many = run(net, dtype, B, world)
    tol = 1e-5 if dtype == "fp32" else 2e-2
    _compare(one, many, tol, tol, f"{name} {dtype} world {world}")
    # every rank holds the same reduced gradients and updated parameters (gathered from the shards)
    for o in many["ranks"][1:]:
        for a, b in zip(o["params"], many["ranks"][0]["params"]):
            assert np.array_equal(a, b)
    es = 2 if dtype == "bf16" else 4
    exp = expected_bytes(many["cfg"], world, es, len(net.layers))
    assert many["bytes"] == [exp] * world, (many["bytes"], exp)


def test_replicated_dp_matches_fsdp():
    """dhen_dist.fsdp = 0 (replicated parameters, gradient all-reduce) equals the sharded step."""
    net = small("C2")
    a = run(net, "fp32", 16, 2, fsdp=True)
    b = run(net, "fp32", 16, 2, fsdp=False)
    _compare(a, b, 1e-6, 1e-6, "DP vs FSDP world 2")


def test_fsdp_matches_oracle_bf16():
    """World 2 against the fp64 oracle emulating the bf16 storage points (G3 through the sharded path)."""
    net = small("C2")
    B, seed, lr = 64, 5, 0.05
    many = run(net, "bf16", B, 2, seed=seed, lr=lr)
    flats = make_flat_params(net, seed)
    params = [O.unflatten(g, f.astype(np.float64)) for g, f in zip(O.param_groups(net), flats)]
    X0, y = _inputs(net, B, "bf16", seed)
    o = O.train_step(net, params, X0.astype(np.float64), y.astype(np.float64), lr, pr=O.Precision(bf16=True))
    assert elem_err(many["loss"], o["loss"]) <= 2e-2
    for g, grp in enumerate(O.param_groups(net)):
        e = norm_err(many["grads"][g], O.flatten(grp, o["grads"][g]))
        assert e <= 2e-2, (g, e)


def test_bf16_reduce_scatter():
    """The paper's quantized gradient collective (dhen_dist.grad_bf16): gradients cast to bf16,
    reduce-scattered in bf16 and widened into the fp32 shard.  Against the fp32 reduce-scatter of the same step:
    every reduced gradient within bf16 rounding (norm 1e-2), parameters within lr times that, and the reduce-scatter
    moves half the bytes."""
    import threading as th
    from paper_2203_11014_b200 import binding
    net = small("C4")
    B, world, seed, lr = 64, 2, 3, 0.05
    flats = make_flat_params(net, seed)
    X0, y = _inputs(net, B, "bf16", seed)
    cfg = to_binding(net, "bf16", B // world)
    outs = {}
    for q in (False, True):
        nid = binding.loopback_id()
        out = [None] * world

        def work(r):
            import torch
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                m = binding.DHEN(cfg, rank=r, world=world, nccl_id=nid, backend=binding.LOOPBACK, grad_bf16=q,
                                 stream=s)
                for gi, f in enumerate(flats):
                    m.set_params(gi, f, stream=s)
                Bl = B // world
                x0 = torch.tensor(X0[r * Bl:(r + 1) * Bl], device="cuda").to(torch.bfloat16).contiguous()
                lab = torch.tensor(y[r * Bl:(r + 1) * Bl], device="cuda")
                s.synchronize()
                b0 = m.comm_bytes()
                m.train_step(x0, lab, lr, B_global=B, stream=s)
                s.synchronize()
                b1 = m.comm_bytes()
                out[r] = {"grads": [m.get_grads(g, stream=s) for g in range(len(flats))],
                          "params": [m.get_params(g, stream=s) for g in range(len(flats))], "bytes": b1 - b0, "m": m}

        ts = [th.Thread(target=work, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(timeout=600)
        assert all(o is not None for o in out)
        outs[q] = out
    eg = max(norm_err(a, b) for a, b in zip(outs[True][0]["grads"], outs[False][0]["grads"]))
    ep = max(elem_err(a, b) for a, b in zip(outs[True][0]["params"], outs[False][0]["params"]))
    print(f"\nbf16 reduce-scatter vs fp32: grads {eg:.2e} params {ep:.2e}")
    gmax = max(float(np.abs(g).max()) for g in outs[False][0]["grads"])
    assert eg <= 1e-2 and ep <= lr * 1e-2 * max(1.0, gmax)
    from paper_2203_11014_b200 import binding as bd
    sh = [bd.group_numel(cfg, g, bd.make_dist(0, world))[1] for g in range(len(net.layers) + 1)]
    ag = sum(sh) + sum(sh[:len(net.layers) - 1])
    assert outs[True][0]["bytes"] == (world - 1) * (ag * 2 + sum(sh) * 2)
    assert outs[False][0]["bytes"] == (world - 1) * (ag * 2 + sum(sh) * 4)
