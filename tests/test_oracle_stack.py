"""Pins of the oracle's layer (Eq.(1)(2)), stack, head and SGD step:
central finite differences, SPEC layer examples
(S:276-278), the north-star 1-module reduction, batch independence,
determinism and the DP loss-scaling identity (R21). CPU only."""
import numpy as np
import pytest

from oracle import dhen_oracle as O
from tests.helpers import M, make_flat_params, oracle_params, small

RNG = np.random.default_rng(1)


def _loss(net, params, X0, y):
    YN, _ = O.forward(net, params, X0)
    z, _ = O.head_fwd(YN, params[-1])
    return O.bce_with_logits(z, y).mean()


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_stack_gradients_vs_finite_differences(name):
    net = small(name)
    if name in ("C3", "C4"):            # keep FD cheap: 1 layer / small mlp
        net = O.NetSpec(net.m0, net.d, net.layers[:1])
    B = 3
    params = oracle_params(net, make_flat_params(net, 11))
    X0 = RNG.standard_normal((B, net.m0, net.d))
    y = (RNG.random(B) < 0.5).astype(np.float64)
    out = O.train_step(net, params, X0, y, lr=0.0)
    h = 1e-6
    for gi, grp in enumerate(params):
        for k, v in grp.items():
            flat = v.reshape(-1)
            idx = RNG.choice(flat.size, size=min(4, flat.size), replace=False)
            for j in idx:
                old = flat[j]
                flat[j] = old + h
                lp = _loss(net, params, X0, y)
                flat[j] = old - h
                lm = _loss(net, params, X0, y)
                flat[j] = old
                fd = (lp - lm) / (2 * h)
                an = out["grads"][gi][k].reshape(-1)[j]
                assert abs(fd - an) <= 1e-4 * max(1e-2, abs(fd)) + 1e-7, (name, k, j, fd, an)
    # dX0
    for _ in range(4):
        b, i, c = RNG.integers(B), RNG.integers(net.m0), RNG.integers(net.d)
        old = X0[b, i, c]
        X0[b, i, c] = old + h
        lp = _loss(net, params, X0, y)
        X0[b, i, c] = old - h
        lm = _loss(net, params, X0, y)
        X0[b, i, c] = old
        fd = (lp - lm) / (2 * h)
        assert abs(fd - out["dX0"][b, i, c]) <= 1e-4 * max(1e-2, abs(fd)) + 1e-7


def test_layer_spec_examples():
    # k = 2, l = 4 each, concat, m_in = 6 -> m_out = 8, W_n is 6 x 8
    net = O.NetSpec(6, 8, [O.LayerSpec([M("linear", 4), M("dcn", 4)])])
    assert O.layer_dims(net) == [(6, 8)]
    names = dict((n, s) for n, s, _ in O.param_groups(net)[0])
    assert names["W_n"] == (6, 8)
    # identity shortcut iff counts match
    net2 = O.NetSpec(8, 8, [O.LayerSpec([M("linear", 4), M("dcn", 4)])])
    assert "W_n" not in dict((n, s) for n, s, _ in O.param_groups(net2)[0])
    # k = 1 linear, l = m, W = I, identity shortcut -> Norm(2X)
    m, d = 5, 6
    net3 = O.NetSpec(m, d, [O.LayerSpec([M("linear", m)])])
    X = RNG.standard_normal((2, m, d))
    g, b = 1 + 0.1 * RNG.standard_normal(d), 0.1 * RNG.standard_normal(d)
    Y, _ = O.layer_fwd(net3, 0, X, {"0.linear.W": np.eye(m), "gamma": g, "beta": b})
    ref, _, _ = O.ln_fwd(2 * X, g, b, 1e-5)
    assert np.abs(Y - ref).max() < 1e-14


@pytest.mark.parametrize("kind", ["dot", "attn", "conv", "dcn", "linear", "mlp"])
def test_one_module_ensemble_reduces_to_module(kind):
    """North-star invariant: a 1-module ensemble with l = m is LN(M(X) + X)."""
    m, d = 6, 8
    s = M(kind, m, heads=2, mlp_hidden=(12, 10))
    net = O.NetSpec(m, d, [O.LayerSpec([s])])
    P = oracle_params(net, make_flat_params(net, 5))[0]
    X = RNG.standard_normal((3, m, d))
    Y, _ = O.layer_fwd(net, 0, X, P)
    p = {k.split(".", 2)[2]: v for k, v in P.items() if k.startswith("0.")}
    if kind == "attn":
        U, _ = O.attn_fwd(X, p, s, O.FP64, 1e-5)
    else:
        U, _ = getattr(O, f"{kind}_fwd")(X, p, s, O.FP64)
    ref, _, _ = O.ln_fwd(U + X, P["gamma"], P["beta"], 1e-5)
    assert np.abs(Y - ref).max() < 1e-14


def test_batch_independence_and_determinism():
    net = small("C4")
    params = oracle_params(net, make_flat_params(net, 3))
    X0 = RNG.standard_normal((4, net.m0, net.d))
    Y, _ = O.forward(net, params, X0)
    Y1, _ = O.forward(net, params, X0[1:2])
    assert np.abs(Y[1:2] - Y1).max() < 1e-12
    Y2, _ = O.forward(net, params, X0)
    assert np.array_equal(Y, Y2)


def test_sgd_step_and_lr_zero():
    net = small("C2")
    params = oracle_params(net, make_flat_params(net, 4))
    X0 = RNG.standard_normal((4, net.m0, net.d))
    y = np.array([0.0, 1.0, 0.0, 0.0])
    o0 = O.train_step(net, params, X0, y, lr=0.0)
    for a, b in zip(o0["params"], params):                 # lr = 0 -> unchanged
        for k in a:
            assert np.array_equal(a[k], b[k])
    o1 = O.train_step(net, params, X0, y, lr=0.25)
    for gi, (a, b) in enumerate(zip(o1["params"], params)):
        for k in a:
            assert np.allclose(a[k], b[k] - 0.25 * o1["grads"][gi][k], rtol=0, atol=1e-15)


def test_data_parallel_split_equals_full_batch():
    """R21: each rank scales by 1/B_global; summing the per-rank grads of two
    half batches gives the full-batch grads (the reduce-scatter semantics)."""
    net = small("C2")
    params = oracle_params(net, make_flat_params(net, 6))
    X0 = RNG.standard_normal((6, net.m0, net.d))
    y = (RNG.random(6) < 0.5).astype(np.float64)
    full = O.train_step(net, params, X0, y, lr=0.0)
    a = O.train_step(net, params, X0[:3], y[:3], lr=0.0, B_global=6)
    b = O.train_step(net, params, X0[3:], y[3:], lr=0.0, B_global=6)
    assert abs(a["loss"] + b["loss"] - full["loss"]) < 1e-14
    for gi in range(len(params)):
        for k in params[gi]:
            assert np.abs(a["grads"][gi][k] + b["grads"][gi][k] - full["grads"][gi][k]).max() < 1e-13


def test_bf16_emulation_is_close_and_exercised():
    net = small("C3")
    params = oracle_params(net, make_flat_params(net, 9))
    X0 = RNG.standard_normal((4, net.m0, net.d))
    y = np.array([0.0, 1.0, 0.0, 1.0])
    ref = O.train_step(net, params, X0, y, lr=0.0)
    emu = O.train_step(net, params, X0, y, lr=0.0, pr=O.Precision(bf16=True))
    d = np.abs(emu["Y_N"] - ref["Y_N"]).max()
    assert 1e-4 < d < 0.1          # rounding happened, and stayed bf16-sized
    # rounded tensors are exactly bf16-representable
    _, caches = O.forward(net, O.compute_params(params, O.Precision(bf16=True)), X0, O.Precision(bf16=True))
    R = caches[0]["R"]
    assert np.array_equal(O.round_bf16(R), R)


# ------------------------------------------------------------------- ensemble variants (R27; NEXT#3)
def _ens_net(ens, shortcut_proj=False):
    m0 = 6
    l = 5 if shortcut_proj else 6                     # 6 -> 5 exercises W_n with a sum ensemble
    mods = [M("dot", l), M("dcn", l), M("attn", l, heads=2), M("mlp", l, mlp_hidden=(12, 10)), M("dcn_lit", l)]
    return O.NetSpec(m0, 8, [O.LayerSpec(mods, ensemble=ens), O.LayerSpec([M("linear", l), M("conv", l)],
                                                                            ensemble=ens)])


@pytest.mark.parametrize("ens", ["sum", "wsum"])
@pytest.mark.parametrize("proj", [False, True])
def test_ensemble_gradients_vs_finite_differences(ens, proj):
    """Sum / weighted-sum ensembles: every gradient (the ensemble weights included) and dX0 against
    central finite differences of the loss."""
    net = _ens_net(ens, proj)
    O.validate(net)
    B = 3
    params = oracle_params(net, make_flat_params(net, 12))
    X0 = RNG.standard_normal((B, net.m0, net.d))
    y = (RNG.random(B) < 0.5).astype(np.float64)
    out = O.train_step(net, params, X0, y, lr=0.0)
    h = 1e-6
    for gi, grp in enumerate(params):
        for k, v in grp.items():
            flat = v.reshape(-1)
            idx = RNG.choice(flat.size, size=min(3, flat.size), replace=False)
            for j in idx:
                old = flat[j]
                flat[j] = old + h
                lp = _loss(net, params, X0, y)
                flat[j] = old - h
                lm = _loss(net, params, X0, y)
                flat[j] = old
                fd = (lp - lm) / (2 * h)
                an = out["grads"][gi][k].reshape(-1)[j]
                assert abs(fd - an) <= 1e-4 * max(1e-2, abs(fd)) + 1e-7, (ens, k, j, fd, an)
    b, i, c = 1, 2, 3
    old = X0[b, i, c]
    X0[b, i, c] = old + h
    lp = _loss(net, params, X0, y)
    X0[b, i, c] = old - h
    lm = _loss(net, params, X0, y)
    X0[b, i, c] = old
    assert abs((lp - lm) / (2 * h) - out["dX0"][b, i, c]) <= 1e-4 * max(1e-2, abs((lp - lm) / (2 * h))) + 1e-7


def test_ensemble_reductions():
    """A 1-module sum / weighted-sum (w = 1) layer is the 1-module concat layer; a weighted sum with all w = 1
    is the sum (outputs and every shared gradient); scaling one module's weight to 0 removes that module."""
    X = RNG.standard_normal((3, 6, 8))
    one = [M("dcn", 6)]
    outs = []
    for ens in ("concat", "sum", "wsum"):
        net = O.NetSpec(6, 8, [O.LayerSpec(one, ensemble=ens)])
        P = oracle_params(net, make_flat_params(net, 5, perturb_ln=False))[0]
        outs.append(O.layer_fwd(net, 0, X, P)[0])
    assert np.array_equal(outs[0], outs[1]) and np.allclose(outs[1], outs[2], atol=0, rtol=0)
    mods = [M("linear", 6), M("dcn", 6), M("conv", 6)]
    ns, nw = (O.NetSpec(6, 8, [O.LayerSpec(mods, ensemble=e)]) for e in ("sum", "wsum"))
    Ps = oracle_params(ns, make_flat_params(ns, 6, perturb_ln=False))[0]
    Pw = dict(Ps, ens_w=np.ones(3))
    Ys, cs = O.layer_fwd(ns, 0, X, Ps)
    Yw, cw = O.layer_fwd(nw, 0, X, Pw)
    assert np.allclose(Ys, Yw, rtol=0, atol=1e-13)
    dY = RNG.standard_normal(Ys.shape)
    dXs, gs = O.layer_bwd(ns, 0, cs, dY, Ps)
    dXw, gw = O.layer_bwd(nw, 0, cw, dY, Pw)
    assert np.allclose(dXs, dXw, rtol=0, atol=1e-12)
    for k, v in gs.items():
        assert np.allclose(v, gw[k], rtol=0, atol=1e-12), k
    # w_1 = 0: the layer equals the sum of modules 0 and 2
    P0 = dict(Pw, ens_w=np.array([1.0, 0.0, 1.0]))
    n2 = O.NetSpec(6, 8, [O.LayerSpec([mods[0], mods[2]], ensemble="sum")])
    P2 = {k: v for k, v in Ps.items() if not k.startswith("1.")}
    P2 = {k.replace("2.conv", "1.conv"): v for k, v in P2.items()}
    assert np.allclose(O.layer_fwd(nw, 0, X, P0)[0], O.layer_fwd(n2, 0, X, P2)[0], rtol=0, atol=1e-13)


def _inj_net():
    """Dense-token injection (R38): 2 dense tokens of X0 fed to every module of layers 0 and 2 (several kinds),
    layer 1 without; layer 2 maps 9 -> 7 tokens (W_n)."""
    l0 = O.LayerSpec([M("dot", 4), M("dcn", 2), M("attn", 3, heads=2)], dense_in=True)
    l1 = O.LayerSpec([M("linear", 5), M("conv", 4)])
    l2 = O.LayerSpec([M("mlp", 3, mlp_hidden=(12, 10)), M("dcn_full", 4)], dense_in=True)
    return O.NetSpec(9, 8, [l0, l1, l2], dense_tokens=2)


def test_dense_injection_gradients_vs_finite_differences():
    """Every sampled gradient and dX0 -- the injected dense tokens (X0[:, :2]: their gradient comes through the
    layer-0 input path and both injected layers) and ordinary tokens -- against central finite differences."""
    net = _inj_net()
    O.validate(net)
    B = 3
    params = oracle_params(net, make_flat_params(net, 13))
    X0 = RNG.standard_normal((B, net.m0, net.d))
    y = (RNG.random(B) < 0.5).astype(np.float64)
    out = O.train_step(net, params, X0, y, lr=0.0)
    h = 1e-6
    for gi, grp in enumerate(params):
        for k, v in grp.items():
            flat = v.reshape(-1)
            for j in RNG.choice(flat.size, size=min(2, flat.size), replace=False):
                old = flat[j]
                flat[j] = old + h
                lp = _loss(net, params, X0, y)
                flat[j] = old - h
                lm = _loss(net, params, X0, y)
                flat[j] = old
                fd = (lp - lm) / (2 * h)
                an = out["grads"][gi][k].reshape(-1)[j]
                assert abs(fd - an) <= 1e-4 * max(1e-2, abs(fd)) + 1e-7, (gi, k, j, fd, an)
    for (b, i, c) in [(0, 0, 1), (1, 1, 5), (2, 4, 3), (1, 8, 7)]:   # dense tokens 0, 1 and two ordinary ones
        old = X0[b, i, c]
        X0[b, i, c] = old + h
        lp = _loss(net, params, X0, y)
        X0[b, i, c] = old - h
        lm = _loss(net, params, X0, y)
        X0[b, i, c] = old
        fd = (lp - lm) / (2 * h)
        assert abs(fd - out["dX0"][b, i, c]) <= 1e-4 * max(1e-2, abs(fd)) + 1e-7, (b, i, c)


def test_dense_injection_reduces_to_explicit_concat():
    """A one-layer net with injection equals the same modules on the explicitly widened input [X ; D] whose
    extra tokens are dropped from the shortcut: with a 1-module concat layer that is the module on [X ; D] plus X,
    and the module's gradient w.r.t. D is what the injected net adds to dX0's dense tokens."""
    d, m, nD, l = 6, 5, 2, 5
    X0 = RNG.standard_normal((2, m, d))
    s = M("linear", l)
    net = O.NetSpec(m, d, [O.LayerSpec([s], dense_in=True)], dense_tokens=nD)
    p = oracle_params(net, make_flat_params(net, 14))
    Y, cache = O.layer_fwd(net, 0, X0, p[0], O.FP64, X0[:, :nD])
    U, _ = O.linear_fwd(np.concatenate([X0, X0[:, :nD]], 1), {"W": p[0]["0.linear.W"]}, s, O.FP64)
    ref, _, _ = O.ln_fwd(U + X0, p[0]["gamma"], p[0]["beta"], net.ln_eps)
    assert np.abs(Y - ref).max() < 1e-12
    assert p[0]["0.linear.W"].shape == (m + nD, l)
