"""Pins of the feature-processing oracle (oracle/fp_oracle.py, NEXT#4) against things other than
itself: torch's embedding_bag (sum pooling, offsets form) and autograd in fp64, torch.optim.SGD with sparse
embedding gradients, brute force on tiny inputs, FlopCounterMode.  CPU only."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F
from torch.utils.flop_counter import FlopCounterMode

from oracle import fp_oracle as FO
from oracle.dhen_oracle import round_bf16


def _case(seed=0, B=5, rows=(7, 3, 11), n_dense=6, hidden=(8, 5), n_dtok=2, d=4, max_bag=4):
    rng = np.random.default_rng(seed)
    spec = FO.FPSpec(list(rows), n_dense, list(hidden), n_dtok, d)
    P = FO.fp_init(spec, rng)
    lens = rng.integers(0, max_bag + 1, B * spec.n_sparse)          # includes empty bags
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = np.concatenate([rng.integers(0, rows[i % spec.n_sparse], n) for i, n in enumerate(lens)]).astype(np.int64)
    dense = rng.standard_normal((B, n_dense))
    return spec, P, idx, offsets, dense, rng


def _torch_fwd(spec, P, idx, offsets, dense, tabs, Ws, bs):
    B, ns = dense.shape[0], spec.n_sparse
    h = torch.tensor(dense)
    for W, b in zip(Ws, bs):
        h = F.relu(F.linear(h, W, b))
    toks = [h.reshape(B, spec.n_dtok, spec.d)]
    pooled = []
    for t in range(ns):   # per table: the bags of feature t across the batch, in the offsets form
        ids, offs = [], [0]
        for b in range(B):
            lo, hi = offsets[b * ns + t], offsets[b * ns + t + 1]
            ids += list(idx[lo:hi])
            offs.append(offs[-1] + hi - lo)
        pooled.append(F.embedding_bag(torch.tensor(ids, dtype=torch.long), tabs[t],
                                      torch.tensor(offs[:-1], dtype=torch.long), mode="sum"))
    toks.append(torch.stack(pooled, dim=1))
    return torch.cat(toks, dim=1)


def _params_t(P, grad=True):
    tabs = [torch.tensor(T, requires_grad=grad) for T in P["tables"]]
    Ws = [torch.tensor(W, requires_grad=grad) for W in P["W"]]
    bs = [torch.tensor(b, requires_grad=grad) for b in P["b"]]
    return tabs, Ws, bs


def test_embedding_bag_brute_force():
    T = np.arange(12, dtype=np.float64).reshape(4, 3)
    assert FO.embedding_bag_sum(T, np.array([], np.int64)).tolist() == [0, 0, 0]
    assert FO.embedding_bag_sum(T, np.array([1, 1, 3])).tolist() == [3 + 3 + 9, 4 + 4 + 10, 5 + 5 + 11]


@pytest.mark.parametrize("seed", [0, 1])
def test_forward_matches_torch(seed):
    spec, P, idx, offsets, dense, _ = _case(seed)
    X0, _ = FO.fp_fwd(spec, P, idx, offsets, dense)
    tabs, Ws, bs = _params_t(P, grad=False)
    ref = _torch_fwd(spec, P, idx, offsets, dense, tabs, Ws, bs).numpy()
    assert X0.shape == (dense.shape[0], spec.m0, spec.d)
    assert np.abs(X0 - ref).max() < 1e-12


@pytest.mark.parametrize("seed", [0, 3])
def test_backward_matches_autograd(seed):
    spec, P, idx, offsets, dense, rng = _case(seed)
    X0, cache = FO.fp_fwd(spec, P, idx, offsets, dense)
    G = rng.standard_normal(X0.shape)
    grads = FO.fp_bwd(spec, P, cache, G)
    tabs, Ws, bs = _params_t(P)
    (_torch_fwd(spec, P, idx, offsets, dense, tabs, Ws, bs) * torch.tensor(G)).sum().backward()
    for a, tt in zip(grads["tables"], tabs):
        assert np.abs(a - tt.grad.numpy()).max() < 1e-12
    for a, tt in zip(grads["W"], Ws):
        assert np.abs(a - tt.grad.numpy()).max() < 1e-12
    for a, tt in zip(grads["b"], bs):
        assert np.abs(a - tt.grad.numpy()).max() < 1e-12


def test_sparse_sgd_matches_torch_optimizer():
    """One SGD step with sparse embedding gradients (torch.nn.EmbeddingBag(sparse=True) + optim.SGD): the
    same tables as the oracle's dense-equivalent update, and never-looked-up rows unchanged."""
    spec, P, idx, offsets, dense, rng = _case(4, rows=(9, 13))
    lr = 0.3
    X0, cache = FO.fp_fwd(spec, P, idx, offsets, dense)
    G = rng.standard_normal(X0.shape)
    newP = FO.fp_sgd(P, FO.fp_bwd(spec, P, cache, G), lr)
    B, ns = dense.shape[0], spec.n_sparse
    for t in range(ns):
        bag = torch.nn.EmbeddingBag(spec.rows[t], spec.d, mode="sum", sparse=True).double()
        with torch.no_grad():
            bag.weight.copy_(torch.tensor(P["tables"][t]))
        ids, offs = [], [0]
        for b in range(B):
            lo, hi = offsets[b * ns + t], offsets[b * ns + t + 1]
            ids += list(idx[lo:hi])
            offs.append(offs[-1] + hi - lo)
        out = bag(torch.tensor(ids, dtype=torch.long), torch.tensor(offs[:-1], dtype=torch.long))
        opt = torch.optim.SGD(bag.parameters(), lr=lr)
        (out * torch.tensor(G[:, spec.n_dtok + t])).sum().backward()
        assert bag.weight.grad.is_sparse
        opt.step()
        assert np.abs(newP["tables"][t] - bag.weight.detach().numpy()).max() < 1e-12
        untouched = sorted(set(range(spec.rows[t])) - set(int(i) for i in ids))
        assert np.array_equal(newP["tables"][t][untouched], P["tables"][t][untouched])


def test_bf16_storage_points():
    """bf16 mode: X0 and the stored hidden activations are bf16 values, and the result is within bf16
    rounding of the fp64 one (the tables and every sum stay fp64)."""
    spec, P, idx, offsets, dense, _ = _case(5)
    X64, _ = FO.fp_fwd(spec, P, idx, offsets, dense)
    Xb, cache = FO.fp_fwd(spec, P, idx, offsets, dense, FO.FPPrecision(True))
    assert np.array_equal(Xb, round_bf16(Xb))
    for H in cache["H"][:-1]:
        assert np.array_equal(H, round_bf16(H))
    assert np.abs(Xb - X64).max() <= 0.05 * np.abs(X64).max()


def test_mlp_flops_pinned():
    spec, P, idx, offsets, dense, _ = _case(6, hidden=(16, 12))
    tabs, Ws, bs = _params_t(P, grad=False)
    with FlopCounterMode(display=False) as fc:
        h = torch.tensor(dense)
        for W, b in zip(Ws, bs):
            h = F.relu(F.linear(h, W, b))
    assert fc.get_total_flops() == FO.fp_forward_flops_per_sample(spec) * dense.shape[0]
