"""Pins of the fp64 oracle's modules against things other than itself:
PyTorch fp64 library routines + autograd (an independent derivation of every
backward), SPEC hand examples (S:<line>), closed forms and invariants.
CPU only (not gpu)."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import dhen_oracle as O


RNG = np.random.default_rng(0)


def rnd(*shape, scale=1.0):
    return RNG.standard_normal(shape) * scale


def t(a, grad=False):
    return torch.tensor(np.asarray(a, np.float64), requires_grad=grad)


# ---------------------------------------------------------------- Dot (Eq.3)
def test_dot_spec_examples():
    s = O.ModuleSpec("dot", 1)
    # orthogonal tokens -> dot vector [0]; W_m all ones -> zero output
    X = np.array([[[1.0, 0.0], [0.0, 1.0]]])
    U, c = O.dot_fwd(X, {"W_m": np.ones((2, 1))}, s, O.FP64)
    assert c["Z"].tolist() == [[0.0]] and np.all(U == 0)
    # e1 = e2 = (1,1) -> [2]
    X = np.array([[[1.0, 1.0], [1.0, 1.0]]])
    _, c = O.dot_fwd(X, {"W_m": np.ones((2, 1))}, s, O.FP64)
    assert c["Z"].tolist() == [[2.0]]
    # m = 4 -> h = 6, row-major pair order = torch.triu_indices
    ii, jj = O.triu_pairs(4)
    ref = torch.triu_indices(4, 4, 1)
    assert len(ii) == 6 and ii.tolist() == ref[0].tolist() and jj.tolist() == ref[1].tolist()


def test_dot_brute_force_and_autograd():
    B, m, d, l = 3, 5, 4, 2
    s = O.ModuleSpec("dot", l)
    h = m * (m - 1) // 2
    X, W = rnd(B, m, d), rnd(l * d, h)
    U, c = O.dot_fwd(X, {"W_m": W}, s, O.FP64)
    # brute force loops
    for b in range(B):
        p = 0
        for i in range(m):
            for j in range(i + 1, m):
                assert abs(c["Z"][b, p] - sum(X[b, i, k] * X[b, j, k] for k in range(d))) < 1e-12
                p += 1
    # autograd through torch.bmm + torch.triu_indices + F.linear
    Xt, Wt = t(X, True), t(W, True)
    iu = torch.triu_indices(m, m, 1)
    G = torch.bmm(Xt, Xt.transpose(1, 2))[:, iu[0], iu[1]]
    Ut = F.linear(G, Wt).reshape(B, l, d)
    assert np.allclose(Ut.detach().numpy(), U, atol=1e-12)
    dU = rnd(B, l, d)
    (Ut * t(dU)).sum().backward()
    dX, g = O.dot_bwd(X, {"W_m": W}, s, c, dU, O.FP64)
    assert np.abs(dX - Xt.grad.numpy()).max() < 1e-12
    assert np.abs(g["W_m"] - Wt.grad.numpy()).max() < 1e-12


def test_dot_gram_symmetry_and_rotation_invariance():
    B, m, d = 2, 6, 5
    X = rnd(B, m, d)
    G = X @ X.transpose(0, 2, 1)
    assert np.array_equal(G, G.transpose(0, 2, 1)) or np.abs(G - G.transpose(0, 2, 1)).max() < 1e-14
    Q, _ = np.linalg.qr(rnd(d, d))
    s = O.ModuleSpec("dot", 2)
    W = rnd(2 * d, m * (m - 1) // 2)
    U1, _ = O.dot_fwd(X, {"W_m": W}, s, O.FP64)
    U2, _ = O.dot_fwd(X @ Q, {"W_m": W}, s, O.FP64)     # S:231, within 1e-9
    assert np.abs(U1 - U2).max() < 1e-9


# ------------------------------------------------------- Linear / token mix
def test_linear_spec_examples():
    s = O.ModuleSpec("linear", 1)
    # X = [[1,2],[3,4]] as d x m (d=2, m=2), W = [[1],[1]] -> [[3],[7]];
    # our layout is tokens x dims, i.e. the transpose.
    X = np.array([[[1.0, 3.0], [2.0, 4.0]]])
    U, _ = O.linear_fwd(X, {"W": np.array([[1.0], [1.0]])}, s, O.FP64)
    assert U.tolist() == [[[3.0, 7.0]]]
    # identity passthrough
    X = rnd(2, 4, 3)
    U, _ = O.linear_fwd(X, {"W": np.eye(4)}, O.ModuleSpec("linear", 4), O.FP64)
    assert np.array_equal(U, X)


def test_tokmix_autograd():
    B, m, d, l = 3, 5, 4, 3
    T, W, dU = rnd(B, m, d), rnd(m, l), rnd(B, l, d)
    Tt, Wt = t(T, True), t(W, True)
    Ut = torch.matmul(Wt.t(), Tt)          # per sample Wᵀ T
    assert np.allclose(Ut.detach().numpy(), O.tokmix_fwd(T, W), atol=1e-13)
    (Ut * t(dU)).sum().backward()
    dT, dW = O.tokmix_bwd(T, W, dU)
    assert np.abs(dT - Tt.grad.numpy()).max() < 1e-12
    assert np.abs(dW - Wt.grad.numpy()).max() < 1e-12


# ----------------------------------------------------------------- DCN (Eq.7)
def test_dcn_identities():
    B, m, d, l = 2, 4, 3, 4
    s = O.ModuleSpec("dcn", l)
    X = rnd(B, m, d)
    # north-star invariant: W = 0, b = 0 => T = X exactly (W_u = I => U = X)
    U, c = O.dcn_fwd(X, {"W": np.zeros((d, d)), "b": np.zeros(d), "W_u": np.eye(m)}, s, O.FP64)
    assert np.array_equal(c["T"], X) and np.array_equal(U, X)
    b = rnd(d)
    _, c = O.dcn_fwd(X, {"W": np.zeros((d, d)), "b": b, "W_u": np.eye(m)}, s, O.FP64)
    assert np.abs(c["T"] - X * (1 + b)).max() < 1e-14
    U, _ = O.dcn_fwd(np.zeros((B, m, d)), {"W": rnd(d, d), "b": b, "W_u": rnd(m, l)}, s, O.FP64)
    assert np.all(U == 0)


def test_dcn_autograd():
    B, m, d, l = 3, 4, 5, 3
    s = O.ModuleSpec("dcn", l)
    X, W, b, Wu, dU = rnd(B, m, d), rnd(d, d), rnd(d), rnd(m, l), rnd(B, l, d)
    p = {"W": W, "b": b, "W_u": Wu}
    U, c = O.dcn_fwd(X, p, s, O.FP64)
    Xt, Wt, bt, Wut = t(X, True), t(W, True), t(b, True), t(Wu, True)
    A = F.linear(Xt, Wt, bt)
    Ut = torch.matmul(Wut.t(), Xt * A + Xt)
    assert np.allclose(Ut.detach().numpy(), U, atol=1e-12)
    (Ut * t(dU)).sum().backward()
    dX, g = O.dcn_bwd(X, p, s, c, dU, O.FP64)
    assert np.abs(dX - Xt.grad.numpy()).max() < 1e-12
    for k, tt in (("W", Wt), ("b", bt), ("W_u", Wut)):
        assert np.abs(g[k] - tt.grad.numpy()).max() < 1e-12, k


# ---------------------------------------------------------------- Conv (Eq.5)
def test_conv_vs_torch_conv2d_and_autograd():
    B, m, d, l, C = 2, 6, 7, 3, 4
    s = O.ModuleSpec("conv", l, conv_channels=C, conv_k=3)
    X, K, Wu, dU = rnd(B, m, d), rnd(C, 3, 3), rnd(m, l), rnd(B, l, d)
    p = {"K": K, "W_u": Wu}
    U, c = O.conv_fwd(X, p, s, O.FP64)
    Xt, Kt, Wut = t(X, True), t(K, True), t(Wu, True)
    Tt = F.conv2d(Xt[:, None], Kt[:, None], padding=1).mean(1)     # library routine
    assert np.abs(Tt.detach().numpy() - c["T"]).max() < 1e-12
    Ut = torch.matmul(Wut.t(), Tt)
    (Ut * t(dU)).sum().backward()
    dX, g = O.conv_bwd(X, p, s, c, dU, O.FP64)
    assert np.abs(dX - Xt.grad.numpy()).max() < 1e-12
    assert np.abs(g["K"] - Kt.grad.numpy()).max() < 1e-12
    assert np.abs(g["W_u"] - Wut.grad.numpy()).max() < 1e-12
    # R12: every channel receives the identical filter gradient
    assert np.abs(g["K"] - g["K"][0:1]).max() < 1e-12


def test_conv_5x5_vs_torch():
    B, m, d, C = 1, 7, 6, 2
    s = O.ModuleSpec("conv", 2, conv_channels=C, conv_k=5)
    X, K = rnd(B, m, d), rnd(C, 5, 5)
    _, c = O.conv_fwd(X, {"K": K, "W_u": rnd(m, 2)}, s, O.FP64)
    ref = F.conv2d(t(X)[:, None], t(K)[:, None], padding=2).mean(1).numpy()
    assert np.abs(ref - c["T"]).max() < 1e-12


def test_conv_spec_examples():
    B, m, d = 2, 5, 4
    X = rnd(B, m, d)
    delta = np.zeros((1, 3, 3))
    delta[0, 1, 1] = 1.0
    # delta kernel, C=1, W = identity -> output equals input
    U, _ = O.conv_fwd(X, {"K": delta, "W_u": np.eye(m)}, O.ModuleSpec("conv", m, conv_channels=1), O.FP64)
    assert np.array_equal(U, X)
    # all-zero filters -> all-zero pre-projection map
    _, c = O.conv_fwd(X, {"K": np.zeros((4, 3, 3)), "W_u": rnd(m, 2)}, O.ModuleSpec("conv", 2), O.FP64)
    assert np.all(c["T"] == 0)


# ----------------------------------------------------------- Attention (Eq.4)
def _attn_params(d, m, l, H, f):
    return {"W_q": rnd(d, d, scale=0.4), "W_k": rnd(d, d, scale=0.4), "W_v": rnd(d, d, scale=0.4),
            "W_o": rnd(d, d, scale=0.4), "b_q": rnd(d, scale=0.1), "b_v": rnd(d, scale=0.1),
            "b_o": rnd(d, scale=0.1), "g1": 1 + rnd(d, scale=0.1), "be1": rnd(d, scale=0.1),
            "g2": 1 + rnd(d, scale=0.1), "be2": rnd(d, scale=0.1), "W_1": rnd(f, d, scale=0.3),
            "b_1": rnd(f, scale=0.1), "W_2": rnd(d, f, scale=0.3), "b_2": rnd(d, scale=0.1),
            "W_u": rnd(m, l)}


def _torch_tel(p, d, H, f):
    tel = torch.nn.TransformerEncoderLayer(d, H, f, dropout=0.0, activation="relu",
                                           batch_first=True, norm_first=False, layer_norm_eps=1e-5)
    tel = tel.double()
    with torch.no_grad():
        tel.self_attn.in_proj_weight.copy_(t(np.concatenate([p["W_q"], p["W_k"], p["W_v"]])))
        tel.self_attn.in_proj_bias.copy_(t(np.concatenate([p["b_q"], np.zeros(d), p["b_v"]])))
        tel.self_attn.out_proj.weight.copy_(t(p["W_o"]))
        tel.self_attn.out_proj.bias.copy_(t(p["b_o"]))
        tel.linear1.weight.copy_(t(p["W_1"]))
        tel.linear1.bias.copy_(t(p["b_1"]))
        tel.linear2.weight.copy_(t(p["W_2"]))
        tel.linear2.bias.copy_(t(p["b_2"]))
        tel.norm1.weight.copy_(t(p["g1"]))
        tel.norm1.bias.copy_(t(p["be1"]))
        tel.norm2.weight.copy_(t(p["g2"]))
        tel.norm2.bias.copy_(t(p["be2"]))
    tel.train()   # dropout=0: identical math, but keeps the reference (non-fastpath) kernels
    return tel


@pytest.mark.parametrize("H", [1, 2])
def test_attention_vs_torch_encoder_layer(H):
    B, m, d, l, f = 3, 5, 8, 3, 16
    s = O.ModuleSpec("attn", l, heads=H, ffn_mult=2)
    p = _attn_params(d, m, l, H, f)
    X, dU = rnd(B, m, d), rnd(B, l, d)
    U, c = O.attn_fwd(X, p, s, O.FP64, 1e-5)
    tel = _torch_tel(p, d, H, f)
    Xt = t(X, True)
    Tt = tel(Xt)
    assert np.abs(Tt.detach().numpy() - c["T"]).max() < 1e-12
    Wut = t(p["W_u"], True)
    Ut = torch.matmul(Wut.t(), Tt)
    assert np.abs(Ut.detach().numpy() - U).max() < 1e-12
    (Ut * t(dU)).sum().backward()
    dX, g = O.attn_bwd(X, p, s, c, dU, O.FP64)
    assert np.abs(dX - Xt.grad.numpy()).max() < 1e-11
    d_ = d
    ipw = tel.self_attn.in_proj_weight.grad.numpy()
    ipb = tel.self_attn.in_proj_bias.grad.numpy()
    pairs = {"W_q": ipw[:d_], "W_k": ipw[d_:2 * d_], "W_v": ipw[2 * d_:], "b_q": ipb[:d_], "b_v": ipb[2 * d_:],
             "W_o": tel.self_attn.out_proj.weight.grad, "b_o": tel.self_attn.out_proj.bias.grad,
             "W_1": tel.linear1.weight.grad, "b_1": tel.linear1.bias.grad,
             "W_2": tel.linear2.weight.grad, "b_2": tel.linear2.bias.grad,
             "g1": tel.norm1.weight.grad, "be1": tel.norm1.bias.grad,
             "g2": tel.norm2.weight.grad, "be2": tel.norm2.bias.grad, "W_u": Wut.grad}
    for k, v in pairs.items():
        v = v if isinstance(v, np.ndarray) else v.numpy()
        assert np.abs(g[k] - v).max() < 1e-11, k
    # R10: the (removed) key bias has identically zero gradient
    assert np.abs(ipb[d_:2 * d_]).max() < 1e-12


def test_attention_single_token_and_permutation():
    d, H = 4, 2
    p = _attn_params(d, 1, 1, H, 8)
    s = O.ModuleSpec("attn", 1, heads=H, ffn_mult=2)
    _, c = O.attn_fwd(rnd(2, 1, d), p, s, O.FP64, 1e-5)
    assert np.all(c["P"] == 1.0)               # m = 1 -> [[1]] exactly
    m, l = 5, 3
    p = _attn_params(d, m, l, H, 8)
    X = rnd(2, m, d)
    perm = RNG.permutation(m)
    U1, _ = O.attn_fwd(X, p, s, O.FP64, 1e-5)
    p2 = dict(p, W_u=p["W_u"][perm])
    U2, _ = O.attn_fwd(X[:, perm], p2, s, O.FP64, 1e-5)
    assert np.abs(U1 - U2).max() < 1e-12


# ------------------------------------------------------------------------ MLP
def test_mlp_vs_torch_autograd():
    B, m, d, l, h1, h2 = 4, 3, 4, 2, 10, 7
    s = O.ModuleSpec("mlp", l, mlp_hidden=(h1, h2))
    p = {"W_1": rnd(h1, m * d, scale=0.5), "b_1": rnd(h1, scale=0.3), "W_2": rnd(h2, h1, scale=0.5),
         "b_2": rnd(h2, scale=0.3), "W_m": rnd(l * d, h2)}
    X, dU = rnd(B, m, d), rnd(B, l, d)
    U, c = O.mlp_fwd(X, p, s, O.FP64)
    Xt = t(X, True)
    pt = {k: t(v, True) for k, v in p.items()}
    v = F.linear(F.relu(F.linear(F.relu(F.linear(Xt.reshape(B, -1), pt["W_1"], pt["b_1"])),
                                 pt["W_2"], pt["b_2"])), pt["W_m"])
    Ut = v.reshape(B, l, d)
    assert np.abs(Ut.detach().numpy() - U).max() < 1e-12
    (Ut * t(dU)).sum().backward()
    dX, g = O.mlp_bwd(X, p, s, c, dU, O.FP64)
    assert np.abs(dX - Xt.grad.numpy()).max() < 1e-12
    for k in p:
        assert np.abs(g[k] - pt[k].grad.numpy()).max() < 1e-12, k


# ------------------------------------------------------------------ LayerNorm
def test_layernorm_vs_torch():
    R, g, b, dY = rnd(3, 4, 6), 1 + rnd(6, scale=0.2), rnd(6, scale=0.2), rnd(3, 4, 6)
    Y, mu, rstd = O.ln_fwd(R, g, b, 1e-5)
    Rt, gt, bt = t(R, True), t(g, True), t(b, True)
    Yt = F.layer_norm(Rt, (6,), gt, bt, 1e-5)
    assert np.abs(Yt.detach().numpy() - Y).max() < 1e-13
    (Yt * t(dY)).sum().backward()
    dR, dg, db = O.ln_bwd(dY, R, mu, rstd, g)
    assert np.abs(dR - Rt.grad.numpy()).max() < 1e-12
    assert np.abs(dg - gt.grad.numpy()).max() < 1e-12
    assert np.abs(db - bt.grad.numpy()).max() < 1e-12
    # LN of a constant vector -> 0 ; mean 0 / var 1 within 1e-6
    Yc, _, _ = O.ln_fwd(np.full((1, 1, 4), 5.0), np.ones(4), np.zeros(4), 1e-5)
    assert np.all(Yc == 0)
    Yn, _, _ = O.ln_fwd(rnd(5, 7, 32), np.ones(32), np.zeros(32), 1e-5)
    assert np.abs(Yn.mean(-1)).max() < 1e-6 and np.abs(Yn.var(-1) - 1).max() < 1e-3


# ----------------------------------------------------------------- head, loss
def test_head_loss_vs_torch():
    B, m, d = 6, 3, 5
    Y, w, b = rnd(B, m, d), rnd(d), rnd(1)
    y = (RNG.random(B) < 0.5).astype(np.float64)
    z, pooled = O.head_fwd(Y, {"w_h": w, "b_h": b})
    Yt, wt, bt = t(Y, True), t(w, True), t(b, True)
    zt = Yt.mean(1) @ wt + bt
    lt = F.binary_cross_entropy_with_logits(zt, t(y))      # mean over batch
    assert abs(lt.item() - O.bce_with_logits(z, y).mean()) < 1e-14
    lt.backward()
    dY, g = O.head_bwd(Y, pooled, z, y, {"w_h": w, "b_h": b}, B)
    assert np.abs(dY - Yt.grad.numpy()).max() < 1e-14
    assert np.abs(g["w_h"] - wt.grad.numpy()).max() < 1e-14
    assert abs(g["b_h"][0] - bt.grad.item()) < 1e-14
    # zero head -> sigmoid(0) = 0.5; sigma'(0) = 1/4
    z0, _ = O.head_fwd(Y, {"w_h": np.zeros(d), "b_h": np.zeros(1)})
    assert np.all(O.sigmoid(z0) == 0.5)
    assert O.sigmoid(0.0) * (1 - O.sigmoid(0.0)) == 0.25
    # extreme logits stay finite (stable BCE form)
    assert np.isfinite(O.bce_with_logits(np.array([800.0, -800.0]), np.array([0.0, 1.0]))).all()


# ------------------------------------------------------------------- bf16 RNE
def test_round_bf16_matches_torch():
    x = np.concatenate([rnd(10000) * 10 ** RNG.uniform(-6, 6, 10000),
                        np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -(1.0 + 2 ** -8), 0.0])])
    x32 = x.astype(np.float32).astype(np.float64)     # fp32-representable inputs
    ref = torch.tensor(x32, dtype=torch.float32).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(O.round_bf16(x32), ref)


def test_flop_formula_vs_torch_counter():
    from torch.utils.flop_counter import FlopCounterMode
    from tests.helpers import small
    # C2-shaped small net (dot + dcn); torch counts matmuls / bmm / einsum
    net = small("C2")
    m, d = net.m0, net.d
    B = 1
    from tests.helpers import make_flat_params, oracle_params
    P = oracle_params(net, make_flat_params(net, 1))
    X = t(rnd(B, m, d))
    with FlopCounterMode(display=False) as fc:
        for n, L in enumerate(net.layers):
            outs = []
            for i, s in enumerate(L.modules):
                pp = {k.split(".")[-1]: t(v) for k, v in P[n].items() if k.startswith(f"{i}.")}
                if s.kind == "dot":
                    iu = torch.triu_indices(m, m, 1)
                    G = torch.bmm(X, X.transpose(1, 2))[:, iu[0], iu[1]]
                    outs.append(F.linear(G, pp["W_m"]).reshape(B, s.l, d))
                else:
                    A = F.linear(X, pp["W"], pp["b"])
                    outs.append(torch.matmul(pp["W_u"].t(), X * A + X))
            X = torch.cat(outs, 1)
    assert fc.get_total_flops() == O.forward_flops_per_sample(net)


# ------------------------------------------------------------------- Adam (NEXT#3)
def test_adam_matches_torch():
    """oracle.adam_update against the library routine torch.optim.Adam (fp64, 4 steps, several tensors)."""
    rng = np.random.default_rng(3)
    params = [{"a": rng.standard_normal((5, 7)), "b": rng.standard_normal(3)}, {"c": rng.standard_normal(11)}]
    tp = [torch.tensor(v, dtype=torch.float64, requires_grad=True) for g in params for v in g.values()]
    opt = torch.optim.Adam(tp, lr=0.01, betas=(0.8, 0.95), eps=1e-6)
    st = O.adam_init(params)
    for _ in range(4):
        grads = [{k: rng.standard_normal(v.shape) for k, v in g.items()} for g in params]
        flat = [gr for g in grads for gr in g.values()]
        for t_, gr in zip(tp, flat):
            t_.grad = torch.tensor(gr)
        opt.step()
        params, st = O.adam_update(params, grads, st, 0.01, 0.8, 0.95, 1e-6)
        got = [v for g in params for v in g.values()]
        for a, b in zip(got, tp):
            assert np.abs(a - b.detach().numpy()).max() <= 1e-12
    assert st["t"] == 4


def test_adam_bf16_state_matches_torch_bf16_loop():
    """The BF16 optimizer (R35): Adam whose moments live in torch.bfloat16 tensors (torch's own RNE conversion),
    fp32-free fp64 math for the update -- the oracle's bf16_state rounding must give the same parameters and
    bf16-representable moments; with the moments left unrounded it differs (the rounding is live)."""
    rng = np.random.default_rng(4)
    params = [{"a": rng.standard_normal((6, 5))}]
    th = torch.tensor(params[0]["a"])
    m = torch.zeros(6, 5, dtype=torch.bfloat16)
    v = torch.zeros(6, 5, dtype=torch.bfloat16)
    st, st32 = O.adam_init(params), O.adam_init(params)
    p32 = params
    b1, b2, eps, lr = 0.9, 0.99, 1e-3, 0.01
    for t in range(1, 5):
        g = rng.standard_normal((6, 5))
        mt = b1 * m.double() + (1 - b1) * torch.tensor(g)
        vt = b2 * v.double() + (1 - b2) * torch.tensor(g) ** 2
        th = th - lr * (mt / (1 - b1 ** t)) / ((vt / (1 - b2 ** t)).sqrt() + eps)
        m, v = mt.to(torch.bfloat16), vt.to(torch.bfloat16)
        params, st = O.adam_update(params, [{"a": g}], st, lr, b1, b2, eps, bf16_state=True)
        p32, st32 = O.adam_update(p32, [{"a": g}], st32, lr, b1, b2, eps)
        assert np.abs(params[0]["a"] - th.numpy()).max() <= 1e-12
        assert np.array_equal(st["m"][0]["a"], m.double().numpy()) and np.array_equal(st["v"][0]["a"], v.double().numpy())
    assert np.abs(p32[0]["a"] - params[0]["a"]).max() > 1e-9


# ------------------------------------------------------------------- flattened full-rank DCN-v2 (R37; NEXT#3)
def test_dcn_full_vs_torch_autograd():
    B, m, d, l = 3, 4, 5, 3
    s = O.ModuleSpec("dcn_full", l)
    X, W, b, Wu = rnd(B, m, d), rnd(m * d, m * d, scale=0.2), rnd(m * d), rnd(m, l)
    p = {"W": W, "b": b, "W_u": Wu}
    U, cache = O.dcn_full_fwd(X, p, s, O.FP64)
    dU = rnd(B, l, d)
    dX, g = O.dcn_full_bwd(X, p, s, cache, dU, O.FP64)
    Xt, Wt, bt, Wut = t(X, True), t(W, True), t(b, True), t(Wu, True)
    x = Xt.reshape(B, m * d)
    A = F.linear(x, Wt, bt)
    Ut = torch.matmul(Wut.t(), (x * A + x).reshape(B, m, d))
    assert np.abs(U - Ut.detach().numpy()).max() < 1e-12
    (Ut * t(dU)).sum().backward()
    for a, ref in ((dX, Xt), (g["W"], Wt), (g["b"], bt), (g["W_u"], Wut)):
        assert np.abs(a - ref.grad.numpy()).max() < 1e-10


def test_dcn_full_reduces_to_per_token_dcn():
    """A block-diagonal W = I_m (x) W_tok and b = (b_tok, .., b_tok) make the flattened cross the per-token
    north-star DCN (R13): same output, same dX, and the diagonal blocks of dW sum to the per-token dW."""
    B, m, d, l = 2, 3, 4, 2
    Wt, bt, Wu = rnd(d, d, scale=0.3), rnd(d), rnd(m, l)
    X, dU = rnd(B, m, d), rnd(B, l, d)
    pf = {"W": np.kron(np.eye(m), Wt), "b": np.tile(bt, m), "W_u": Wu}
    pt = {"W": Wt, "b": bt, "W_u": Wu}
    Uf, cf = O.dcn_full_fwd(X, pf, O.ModuleSpec("dcn_full", l), O.FP64)
    Ut, ct = O.dcn_fwd(X, pt, O.ModuleSpec("dcn", l), O.FP64)
    assert np.abs(Uf - Ut).max() < 1e-12
    dXf, gf = O.dcn_full_bwd(X, pf, O.ModuleSpec("dcn_full", l), cf, dU, O.FP64)
    dXt, gt = O.dcn_bwd(X, pt, O.ModuleSpec("dcn", l), ct, dU, O.FP64)
    assert np.abs(dXf - dXt).max() < 1e-12
    assert np.abs(sum(gf["W"][i * d:(i + 1) * d, i * d:(i + 1) * d] for i in range(m)) - gt["W"]).max() < 1e-12
    assert np.abs(gf["b"].reshape(m, d).sum(0) - gt["b"]).max() < 1e-12


# ------------------------------------------------------------------- paper-literal DCN, Eq.(7) (R31; NEXT#3)
def _dcnl(X, W, b):
    net = O.NetSpec(X.shape[1], X.shape[2], [O.LayerSpec([O.ModuleSpec("dcn_lit", W.shape[1])])])
    return O.dcn_lit_fwd(X, {"W": W, "b": b}, net.layers[0].modules[0], O.FP64)


def test_dcn_lit_spec_examples():
    """identity tokens -> G = I, u = W + b; all-zero X -> u = b (columns of u = the l embeddings)."""
    W = RNG.standard_normal((2, 3))
    b = RNG.standard_normal((3, 2))
    U, _ = _dcnl(np.eye(2)[None], W, b)
    assert np.allclose(U[0], W.T + b, atol=1e-14)
    U0, _ = _dcnl(np.zeros((1, 4, 2)), W, b)
    assert np.array_equal(U0[0], b)


def test_dcn_lit_vs_torch_autograd():
    """u = (X_nX_nᵀ) W + b in torch fp64 (bmm + matmul), outputs and every gradient by autograd."""
    B, m, d, l = 3, 5, 4, 6
    X = RNG.standard_normal((B, m, d))
    W = RNG.standard_normal((d, l))
    b = RNG.standard_normal((l, d))
    U, cache = _dcnl(X, W, b)
    Xt, Wt, bt = (torch.tensor(a, requires_grad=True) for a in (X, W, b))
    Xn = Xt.transpose(1, 2)                                     # X_n = d x m
    u = torch.matmul(torch.bmm(Xn, Xn.transpose(1, 2)), Wt)     # [B][d][l]
    Ut = u.transpose(1, 2) + bt
    assert np.abs(Ut.detach().numpy() - U).max() <= 1e-12
    dU = RNG.standard_normal(U.shape)
    Ut.backward(torch.tensor(dU))
    net = O.NetSpec(m, d, [O.LayerSpec([O.ModuleSpec("dcn_lit", l)])])
    dX, g = O.dcn_lit_bwd(X, {"W": W, "b": b}, net.layers[0].modules[0], cache, dU, O.FP64)
    assert np.abs(dX - Xt.grad.numpy()).max() <= 1e-11
    assert np.abs(g["W"] - Wt.grad.numpy()).max() <= 1e-11
    assert np.abs(g["b"] - bt.grad.numpy()).max() <= 1e-12


def test_dcn_lit_flops_spec_example():
    """cross-net d = 8, m = 6, l = 4 -> Gram 2·8·8·6 = 768 + projection 2·8·8·4 = 512 = 1280 (plus the
    concat layer's nothing else: one module, m_in != m_out brings W_n: 2·6·4·8)."""
    net = O.NetSpec(6, 8, [O.LayerSpec([O.ModuleSpec("dcn_lit", 4)])])
    assert O.forward_flops_per_sample(net) == 1280 + 2 * 6 * 4 * 8
