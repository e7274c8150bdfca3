"""DHEN CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 numpy implementation of what the DHEN layer-stack training
step computes (arXiv 2203.11014, /root/reference/PAPER.md = "P:<line>").
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` leg may import this module.  The product path
(`paper_2203_11014_b200`, `libdhen.so`) never imports, links or executes it,
and this file imports nothing from the product.

Every forward and backward is written out from its definition; backward
passes are hand-derived (no autograd).  A library primitive (matmul / einsum)
serves as a step; there is no blocking, fusion or reordering beyond the
definition.  Readings of silent / ambiguous passages follow SURVEY.md §8(c)
and are listed in DESIGN.md §3 ("R<n>").

Layout: X is [B][m][d]; row t of a sample is the paper's column x^t.

bf16 storage emulation (R20/R24): the GPU path stores some
intermediates in bf16 and computes in fp32.  `Precision(bf16=True)` rounds
(round-to-nearest-even) at the named storage points via `q(name, x)`; every
name used is listed in STORAGE_POINTS.  Arithmetic between storage points is
fp64.  `Precision()` (default) rounds nowhere (fp64 everywhere).

Pins: tests/test_oracle_*.py (torch fp64 autograd and library routines,
central finite differences, SPEC hand examples, closed forms, invariants).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

import numpy as np

# --------------------------------------------------------------------------
# configuration (the oracle's own; the product has its own C structs)
# --------------------------------------------------------------------------
KINDS = ("dot", "attn", "conv", "dcn", "linear", "mlp", "dcn_lit", "dcn_full")


@dataclass
class ModuleSpec:
    kind: str
    l: int                      # output token count l_i
    heads: int = 2              # attn (R10)
    ffn_mult: int = 4           # attn (R10)
    conv_channels: int = 4      # conv (R12)
    conv_k: int = 3             # conv (R12)
    mlp_hidden: Tuple[int, int] = (1024, 1024)   # mlp (R14)


@dataclass
class LayerSpec:
    modules: List[ModuleSpec]
    # Ensemble of Eq.(1) ("it can be concatenation, sum, or weighted sum"): "concat" along tokens (R5,
    # the configs' reading), "sum" of the modules' outputs, or "wsum" = sum with one learnable scalar weight
    # per module (R27; initialised to 1, so a fresh wsum layer computes the sum).  sum / wsum need equal l_i.
    ensemble: str = "concat"
    # Dense-token injection ("the raw numerical (dense) features can be part of the input to any modules for
    # ensembling in every layer", NEXT#3, R38): every module of the layer reads [X_n ; D] (m_in + n_dense tokens),
    # D = the first NetSpec.dense_tokens tokens of X0 (the feature processing layer's dense tokens, R32); the
    # shortcut and the LayerNorm still see X_n.
    dense_in: bool = False


@dataclass
class NetSpec:
    m0: int
    d: int
    layers: List[LayerSpec]
    ln_eps: float = 1e-5
    dense_tokens: int = 0       # R38: X0[:, :dense_tokens] are the dense tokens D injected into dense_in layers


def module_in(net: NetSpec, n: int) -> int:
    """Tokens every module of layer n reads: m_in, plus the dense tokens when the layer injects them (R38)."""
    return layer_dims(net)[n][0] + (net.dense_tokens if net.layers[n].dense_in else 0)


def layer_dims(net: NetSpec) -> List[Tuple[int, int]]:
    """(m_in, m_out) per layer; m_out = Σ l_i (concat ensemble, R5), or the common l_i (sum / wsum)."""
    dims, m = [], net.m0
    for L in net.layers:
        mo = sum(s.l for s in L.modules) if L.ensemble == "concat" else L.modules[0].l
        dims.append((m, mo))
        m = mo
    return dims


def validate(net: NetSpec) -> None:
    """Preconditions of SURVEY §8(b)."""
    if net.m0 < 1 or net.d < 1 or not net.layers:
        raise ValueError("bad net dims")
    if not 0 <= net.dense_tokens <= net.m0 or (any(L.dense_in for L in net.layers) and net.dense_tokens == 0):
        raise ValueError("dense injection needs 1 <= dense_tokens <= m0 (R38)")
    for (m_in, _), L in zip(layer_dims(net), net.layers):
        if not L.modules:
            raise ValueError("empty layer")
        if L.ensemble not in ("concat", "sum", "wsum"):
            raise ValueError(f"unknown ensemble {L.ensemble}")
        if L.ensemble != "concat" and len({s.l for s in L.modules}) != 1:
            raise ValueError("sum / weighted-sum ensembles need equal module output counts l_i")
        for s in L.modules:
            if s.kind not in KINDS:
                raise ValueError(f"unknown kind {s.kind}")
            if s.l < 1:
                raise ValueError("l < 1")
            if s.kind == "dot" and m_in < 2:
                raise ValueError("dot needs m >= 2 (S:186)")
            if s.kind == "attn" and net.d % s.heads != 0:
                raise ValueError("d % heads != 0 (S:195)")
            if s.kind == "conv" and s.conv_k % 2 == 0:
                raise ValueError("even conv kernel (S:204)")


def module_param_shapes(s: ModuleSpec, m: int, d: int) -> List[Tuple[str, Tuple[int, ...], int]]:
    """Canonical parameter order of one module: (name, shape, fan_in).

    SURVEY §8(b) "Canonical param order"; dense maps use [out, in], token
    maps the paper's [m, l].
    """
    l = s.l
    if s.kind == "dot":
        h = m * (m - 1) // 2
        return [("W_m", (l * d, h), h)]
    if s.kind == "linear":
        return [("W", (m, l), m)]
    if s.kind == "dcn_lit":   # Eq.(7) literally (R31): W ∈ R^{d×l}, the bias of the l output embeddings [l, d]
        return [("W", (d, l), d), ("b", (l, d), d)]
    if s.kind == "dcn":
        return [("W", (d, d), d), ("b", (d,), d), ("W_u", (m, l), m)]
    if s.kind == "dcn_full":   # the flattened full-rank DCN-v2 (R37): W ∈ R^{md×md} on vec(X)
        return [("W", (m * d, m * d), m * d), ("b", (m * d,), m * d), ("W_u", (m, l), m)]
    if s.kind == "conv":
        k = s.conv_k
        return [("K", (s.conv_channels, k, k), k * k), ("W_u", (m, l), m)]
    if s.kind == "attn":
        f = s.ffn_mult * d
        return [("W_q", (d, d), d), ("W_k", (d, d), d), ("W_v", (d, d), d), ("W_o", (d, d), d),
                ("b_q", (d,), d), ("b_v", (d,), d), ("b_o", (d,), d),
                ("g1", (d,), 0), ("be1", (d,), 0), ("g2", (d,), 0), ("be2", (d,), 0),
                ("W_1", (f, d), d), ("b_1", (f,), d), ("W_2", (d, f), f), ("b_2", (d,), f),
                ("W_u", (m, l), m)]
    if s.kind == "mlp":
        h1, h2 = s.mlp_hidden
        return [("W_1", (h1, m * d), m * d), ("b_1", (h1,), m * d),
                ("W_2", (h2, h1), h1), ("b_2", (h2,), h1),
                ("W_m", (l * d, h2), h2)]
    raise ValueError(s.kind)


def param_groups(net: NetSpec) -> List[List[Tuple[str, Tuple[int, ...], int]]]:
    """Groups 0..N-1 = layers, group N = head.  Names are '<i>.<kind>.<p>'."""
    groups = []
    for n, ((m_in, m_out), L) in enumerate(zip(layer_dims(net), net.layers)):
        g = []
        for i, s in enumerate(L.modules):
            for name, shp, fan in module_param_shapes(s, module_in(net, n), net.d):
                g.append((f"{i}.{s.kind}.{name}", shp, fan))
        if L.ensemble == "wsum":
            g.append(("ens_w", (len(L.modules),), 0))         # R27, initialised to 1
        if m_in != m_out:
            g.append(("W_n", (m_in, m_out), m_in))      # Eq.(2), R4
        g.append(("gamma", (net.d,), 0))
        g.append(("beta", (net.d,), 0))
        groups.append(g)
    groups.append([("w_h", (net.d,), net.d), ("b_h", (1,), net.d)])   # R17
    return groups


def group_size(group) -> int:
    return int(sum(int(np.prod(shp)) for _, shp, _ in group))


def unflatten(group, flat: np.ndarray) -> Dict[str, np.ndarray]:
    out, o = {}, 0
    for name, shp, _ in group:
        n = int(np.prod(shp))
        out[name] = np.asarray(flat[o:o + n], dtype=np.float64).reshape(shp)
        o += n
    assert o == flat.size, (o, flat.size)
    return out


def flatten(group, params: Dict[str, np.ndarray]) -> np.ndarray:
    return np.concatenate([np.asarray(params[n], np.float64).reshape(-1) for n, _, _ in group])


# --------------------------------------------------------------------------
# precision emulation
# --------------------------------------------------------------------------
STORAGE_POINTS = (
    # compute copy of every parameter (the bf16 shard / gathered buffer, R20)
    "params",
    # layer level
    "Y", "R", "dR", "dX",
    # weighted-sum ensemble: each module's dU = w_i dR (R27)
    "ens.dU",
    # paper-literal DCN (R31): the per-sample d x d Gram and the symmetrised dG
    "dcnl.G", "dcnl.S",
    # head
    "head.dY",
    # modules
    "dot.Z", "dot.dZ",
    "dcn.A", "dcn.T", "dcn.dT", "dcn.dA",
    "conv.T", "conv.dT",
    "attn.QKV", "attn.P", "attn.O", "attn.R1", "attn.Z1", "attn.F", "attn.R2", "attn.T",
    "attn.dT", "attn.dR2", "attn.dF", "attn.dR1", "attn.dO", "attn.dS", "attn.dQKV",
    "mlp.h1", "mlp.h2", "mlp.dh2", "mlp.dh1",
)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp64 values to the nearest bfloat16 (8 significant bits), ties to
    even (R24).  Normal range only (values here never approach 2^-126)."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                     # x = m * 2^e, 0.5 <= |m| < 1
    r = np.rint(m * 256.0)                 # 8 significant bits, RNE
    return np.ldexp(r, e - 8)


# Where the CUDA path stores bf16.  dcn.dT is not one: the DCN backward is fused into
# the token-projection dgrad epilogue, which keeps dT in fp32 registers.
GPU_POINTS = tuple(p for p in STORAGE_POINTS if p != "dcn.dT")


@dataclass
class Precision:
    bf16: bool = False
    points: Sequence[str] = GPU_POINTS

    def q(self, name: str, x: np.ndarray) -> np.ndarray:
        assert name in STORAGE_POINTS, name
        if self.bf16 and name in self.points:
            return round_bf16(x)
        return x


FP64 = Precision()

# --------------------------------------------------------------------------
# LayerNorm (R6: per token over d, biased variance, eps, shared gamma/beta)
# --------------------------------------------------------------------------


def ln_fwd(R: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float):
    mu = R.mean(axis=-1, keepdims=True)
    var = ((R - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xh = (R - mu) * rstd
    return xh * g + b, mu, rstd


def ln_bwd(dY: np.ndarray, R_saved: np.ndarray, mu, rstd, g: np.ndarray):
    """B2: dR = rstd·(gy − mean(gy) − x̂·mean(gy⊙x̂)), gy = dY⊙γ.
    x̂ is recomputed from the stored pre-norm tensor R_saved (which may be the
    bf16-rounded copy) and the fp statistics of the forward."""
    xh = (R_saved - mu) * rstd
    gy = dY * g
    dR = rstd * (gy - gy.mean(-1, keepdims=True) - xh * (gy * xh).mean(-1, keepdims=True))
    red = tuple(range(dY.ndim - 1))
    return dR, (dY * xh).sum(axis=red), dY.sum(axis=red)


# --------------------------------------------------------------------------
# token projection (Eq.(4)-(6): u = W·T with W ∈ R^{m×l} on the token axis, R11)
# --------------------------------------------------------------------------


def tokmix_fwd(T: np.ndarray, W: np.ndarray) -> np.ndarray:
    # U[b,t,c] = Σ_i W[i,t] T[b,i,c]
    return np.einsum("it,bic->btc", W, T)


def tokmix_bwd(T: np.ndarray, W: np.ndarray, dU: np.ndarray):
    dT = np.einsum("it,btc->bic", W, dU)
    dW = np.einsum("bic,btc->it", T, dU)
    return dT, dW


# --------------------------------------------------------------------------
# modules
# --------------------------------------------------------------------------


def triu_pairs(m: int):
    """Strict upper triangle, row-major: p(i,j) = i·m − i(i+1)/2 + (j−i−1) (R7)."""
    ii, jj = [], []
    for i in range(m):
        for j in range(i + 1, m):
            ii.append(i)
            jj.append(j)
    return np.array(ii, dtype=np.int64), np.array(jj, dtype=np.int64)


def dot_fwd(X, p, s: ModuleSpec, pr: Precision):
    """Eq.(3) with the public DLRM dot (R7) and the single-tensor
    map W_m: z = triu(X Xᵀ), v = W_m z, U = reshape(v, l, d) (R9)."""
    B, m, d = X.shape
    G = X @ X.transpose(0, 2, 1)
    iu, ju = triu_pairs(m)
    Z = pr.q("dot.Z", G[:, iu, ju])
    V = Z @ p["W_m"].T
    return V.reshape(B, s.l, d), {"Z": Z}


def dot_bwd(X, p, s, c, dU, pr):
    B, m, d = X.shape
    dV = dU.reshape(B, s.l * d)
    dWm = dV.T @ c["Z"]
    dZ = pr.q("dot.dZ", dV @ p["W_m"])
    iu, ju = triu_pairs(m)
    S = np.zeros((B, m, m))
    S[:, iu, ju] = dZ
    S = S + S.transpose(0, 2, 1)              # symmetric, zero diagonal
    dX = S @ X
    return dX, {"W_m": dWm}


def linear_fwd(X, p, s, pr):
    """Eq.(6): u = X·W on the token axis (R11)."""
    return tokmix_fwd(X, p["W"]), {}


def linear_bwd(X, p, s, c, dU, pr):
    dX, dW = tokmix_bwd(X, p["W"], dU)
    return dX, {"W": dW}


def dcn_fwd(X, p, s, pr):
    """North-star DCN-v2 cross per token (R13): A = X Wᵀ + b; T = X ⊙ A + X;
    then the unify map W_u ∈ R^{m×l} (Eq.(7) reading)."""
    A = X @ p["W"].T + p["b"]
    T = pr.q("dcn.T", X * A + X)
    A = pr.q("dcn.A", A)
    return tokmix_fwd(T, p["W_u"]), {"A": A, "T": T}


def dcn_bwd(X, p, s, c, dU, pr):
    dT, dWu = tokmix_bwd(c["T"], p["W_u"], dU)
    dT = pr.q("dcn.dT", dT)          # not a storage point of the fused GPU path (kept for emulation studies)
    dA = pr.q("dcn.dA", dT * X)
    dX = dT * c["A"] + dT + dA @ p["W"]
    dW = dA.reshape(-1, dA.shape[-1]).T @ X.reshape(-1, X.shape[-1])
    db = dA.reshape(-1, dA.shape[-1]).sum(0)
    return dX, {"W": dW, "b": db, "W_u": dWu}


def dcn_full_fwd(X, p, s, pr):
    """Flattened full-rank DCN-v2 (NEXT#3, SURVEY ledger 13, R37): the sample x = vec(X) ∈ R^{m·d} (token rows in
    order), A = x Wᵀ + b with W ∈ R^{md×md}, T = x ⊙ A + x, read back as m tokens; then the unify map W_u."""
    B, m, d = X.shape
    A = (X.reshape(B, m * d) @ p["W"].T + p["b"]).reshape(B, m, d)
    T = pr.q("dcn.T", X * A + X)
    A = pr.q("dcn.A", A)
    return tokmix_fwd(T, p["W_u"]), {"A": A, "T": T}


def dcn_full_bwd(X, p, s, c, dU, pr):
    B, m, d = X.shape
    dT, dWu = tokmix_bwd(c["T"], p["W_u"], dU)
    dA = pr.q("dcn.dA", dT * X)
    dAf, Xf = dA.reshape(B, m * d), X.reshape(B, m * d)
    dX = dT * c["A"] + dT + (dAf @ p["W"]).reshape(B, m, d)
    return dX, {"W": dAf.T @ Xf, "b": dAf.sum(0), "W_u": dWu}


def dcn_lit_fwd(X, p, s, pr):
    """Eq.(7) read literally (NEXT#3; R31 after SPEC S:219-222 / S:235): per sample the d x d
    Gram over tokens G = X_n X_nᵀ (X_n = Xᵀ is d x m, so G[c][k] = Σ_i X[i][c] X[i][k]), u = G W + b with
    W ∈ R^{d×l}; the columns of u are the l output embeddings, U[t][c] = (G W)[c][t] + b[t][c]."""
    G = pr.q("dcnl.G", np.einsum("bic,bik->bck", X, X))
    U = np.einsum("bck,kt->btc", G, p["W"]) + p["b"]
    return U, {"G": G}


def dcn_lit_bwd(X, p, s, c, dU, pr):
    """dW[k][t] = Σ_b Σ_c G[c][k] dU[t][c];  db = Σ_b dU;  dG[c][k] = Σ_t dU[t][c] W[k][t];
    dX = X (dG + dGᵀ)  (G = XᵀX)."""
    G = c["G"]
    dW = np.einsum("bck,btc->kt", G, dU)
    db = dU.sum(0)
    dG = np.einsum("btc,kt->bck", dU, p["W"])
    S = pr.q("dcnl.S", dG + dG.transpose(0, 2, 1))
    return X @ S, {"W": dW, "b": db}


def _corr2d_same(img, ker):
    """Zero-padded 'same' 2-D cross-correlation of [B,m,d] with a k×k kernel:
    O[i][j] = Σ_{a,e=-r..r} K[a+r][e+r]·X[i+a][j+e] (R12)."""
    B, m, d = img.shape
    k = ker.shape[0]
    r = (k - 1) // 2
    P = np.zeros((B, m + 2 * r, d + 2 * r))
    P[:, r:r + m, r:r + d] = img
    out = np.zeros((B, m, d))
    for a in range(k):
        for e in range(k):
            out += ker[a, e] * P[:, a:a + m, e:e + d]
    return out


def conv_fwd(X, p, s, pr):
    """Eq.(5), reading R12: 1-channel m×d image, C k×k filters,
    same zero padding, channel mean, no bias; then W_u."""
    C = s.conv_channels
    T = sum(_corr2d_same(X, p["K"][ch]) for ch in range(C)) / C
    T = pr.q("conv.T", T)
    return tokmix_fwd(T, p["W_u"]), {"T": T}


def conv_bwd(X, p, s, c, dU, pr):
    dT, dWu = tokmix_bwd(c["T"], p["W_u"], dU)
    dT = pr.q("conv.dT", dT)
    C, k = s.conv_channels, s.conv_k
    r = (k - 1) // 2
    B, m, d = X.shape
    Xp = np.zeros((B, m + 2 * r, d + 2 * r))
    Xp[:, r:r + m, r:r + d] = X
    dTp = np.zeros((B, m + 2 * r, d + 2 * r))
    dTp[:, r:r + m, r:r + d] = dT
    dK = np.zeros((C, k, k))
    dX = np.zeros_like(X)
    for ch in range(C):
        for a in range(k):
            for e in range(k):
                # dK_c[a][e] = (1/C) Σ dT[i][j] X[i+a-r][j+e-r]
                dK[ch, a, e] = (dT * Xp[:, a:a + m, e:e + d]).sum() / C
                # dX[i'][j'] += (1/C) K_c[a][e] dT[i'-a+r][j'-e+r]
                dX += p["K"][ch, a, e] * dTp[:, 2 * r - a:2 * r - a + m, 2 * r - e:2 * r - e + d] / C
    return dX, {"K": dK, "W_u": dWu}


def _softmax_rows(S):
    S = S - S.max(axis=-1, keepdims=True)
    E = np.exp(S)
    return E / E.sum(axis=-1, keepdims=True)


def attn_fwd(X, p, s, pr, eps):
    """Eq.(4): u = W · TransformerEncoderLayer(X), read as PyTorch
    nn.TransformerEncoderLayer (post-norm, ReLU, dropout 0, H heads, FFN f·d,
    no key bias) then the unify map W_u (R10, R11)."""
    B, m, d = X.shape
    H = s.heads
    dh = d // H
    Wqkv = np.concatenate([p["W_q"], p["W_k"], p["W_v"]], 0)
    bqkv = np.concatenate([p["b_q"], np.zeros(d), p["b_v"]])
    QKV = pr.q("attn.QKV", X @ Wqkv.T + bqkv)
    Q, K, V = QKV[..., :d], QKV[..., d:2 * d], QKV[..., 2 * d:]
    Qh = Q.reshape(B, m, H, dh).transpose(0, 2, 1, 3)
    Kh = K.reshape(B, m, H, dh).transpose(0, 2, 1, 3)
    Vh = V.reshape(B, m, H, dh).transpose(0, 2, 1, 3)
    S = (Qh @ Kh.transpose(0, 1, 3, 2)) / math.sqrt(dh)
    P = pr.q("attn.P", _softmax_rows(S))
    O = pr.q("attn.O", (P @ Vh).transpose(0, 2, 1, 3).reshape(B, m, d))
    R1 = X + O @ p["W_o"].T + p["b_o"]
    Z1, mu1, rs1 = ln_fwd(R1, p["g1"], p["be1"], eps)
    R1 = pr.q("attn.R1", R1)
    Z1 = pr.q("attn.Z1", Z1)
    F = pr.q("attn.F", np.maximum(Z1 @ p["W_1"].T + p["b_1"], 0.0))
    R2 = Z1 + F @ p["W_2"].T + p["b_2"]
    T, mu2, rs2 = ln_fwd(R2, p["g2"], p["be2"], eps)
    R2 = pr.q("attn.R2", R2)
    T = pr.q("attn.T", T)
    c = dict(QKV=QKV, P=P, O=O, R1=R1, mu1=mu1, rs1=rs1, Z1=Z1, F=F, R2=R2, mu2=mu2, rs2=rs2, T=T)
    return tokmix_fwd(T, p["W_u"]), c


def attn_bwd(X, p, s, c, dU, pr):
    B, m, d = X.shape
    H = s.heads
    dh = d // H
    g = {}
    dT, g["W_u"] = tokmix_bwd(c["T"], p["W_u"], dU)
    dT = pr.q("attn.dT", dT)
    # LN2 and FFN
    dR2, g["g2"], g["be2"] = ln_bwd(dT, c["R2"], c["mu2"], c["rs2"], p["g2"])
    dR2 = pr.q("attn.dR2", dR2)
    g["W_2"] = dR2.reshape(-1, d).T @ c["F"].reshape(-1, c["F"].shape[-1])
    g["b_2"] = dR2.reshape(-1, d).sum(0)
    dF = pr.q("attn.dF", (dR2 @ p["W_2"]) * (c["F"] > 0))          # ReLU'(0) = 0 (R22)
    g["W_1"] = dF.reshape(-1, dF.shape[-1]).T @ c["Z1"].reshape(-1, d)
    g["b_1"] = dF.reshape(-1, dF.shape[-1]).sum(0)
    dZ1 = dR2 + dF @ p["W_1"]
    # LN1 and out-projection
    dR1, g["g1"], g["be1"] = ln_bwd(dZ1, c["R1"], c["mu1"], c["rs1"], p["g1"])
    dR1 = pr.q("attn.dR1", dR1)
    g["W_o"] = dR1.reshape(-1, d).T @ c["O"].reshape(-1, d)
    g["b_o"] = dR1.reshape(-1, d).sum(0)
    dO = pr.q("attn.dO", dR1 @ p["W_o"])
    # attention core (B6)
    QKV, P = c["QKV"], c["P"]
    Qh = QKV[..., :d].reshape(B, m, H, dh).transpose(0, 2, 1, 3)
    Kh = QKV[..., d:2 * d].reshape(B, m, H, dh).transpose(0, 2, 1, 3)
    Vh = QKV[..., 2 * d:].reshape(B, m, H, dh).transpose(0, 2, 1, 3)
    dOh = dO.reshape(B, m, H, dh).transpose(0, 2, 1, 3)
    dVh = P.transpose(0, 1, 3, 2) @ dOh
    dP = dOh @ Vh.transpose(0, 1, 3, 2)
    dS = P * (dP - (P * dP).sum(-1, keepdims=True))
    dS = pr.q("attn.dS", dS / math.sqrt(dh))
    dQh = dS @ Kh
    dKh = dS.transpose(0, 1, 3, 2) @ Qh

    def merge(t):
        return t.transpose(0, 2, 1, 3).reshape(B, m, d)

    dQKV = pr.q("attn.dQKV", np.concatenate([merge(dQh), merge(dKh), merge(dVh)], -1))
    Wqkv = np.concatenate([p["W_q"], p["W_k"], p["W_v"]], 0)
    dX = dR1 + dQKV @ Wqkv
    dW = dQKV.reshape(-1, 3 * d).T @ X.reshape(-1, d)
    g["W_q"], g["W_k"], g["W_v"] = dW[:d], dW[d:2 * d], dW[2 * d:]
    col = dQKV.reshape(-1, 3 * d).sum(0)
    g["b_q"], g["b_v"] = col[:d], col[2 * d:]
    return dX, g


def mlp_fwd(X, p, s, pr):
    """P:96 single-tensor rule with an MLP (R14): flatten → [Linear+ReLU]×2 →
    W_m → l tokens."""
    B, m, d = X.shape
    Xf = X.reshape(B, m * d)
    h1 = pr.q("mlp.h1", np.maximum(Xf @ p["W_1"].T + p["b_1"], 0.0))
    h2 = pr.q("mlp.h2", np.maximum(h1 @ p["W_2"].T + p["b_2"], 0.0))
    v = h2 @ p["W_m"].T
    return v.reshape(B, s.l, d), {"h1": h1, "h2": h2}


def mlp_bwd(X, p, s, c, dU, pr):
    B, m, d = X.shape
    Xf = X.reshape(B, m * d)
    dv = dU.reshape(B, s.l * d)
    g = {"W_m": dv.T @ c["h2"]}
    dh2 = pr.q("mlp.dh2", (dv @ p["W_m"]) * (c["h2"] > 0))
    g["W_2"] = dh2.T @ c["h1"]
    g["b_2"] = dh2.sum(0)
    dh1 = pr.q("mlp.dh1", (dh2 @ p["W_2"]) * (c["h1"] > 0))
    g["W_1"] = dh1.T @ Xf
    g["b_1"] = dh1.sum(0)
    dX = (dh1 @ p["W_1"]).reshape(B, m, d)
    return dX, g


# --------------------------------------------------------------------------
# layer (Eq.(1)(2))
# --------------------------------------------------------------------------


def _module_params(P: Dict[str, np.ndarray], i: int, kind: str):
    pre = f"{i}.{kind}."
    return {k[len(pre):]: v for k, v in P.items() if k.startswith(pre)}


def layer_fwd(net: NetSpec, n: int, X: np.ndarray, P: Dict[str, np.ndarray], pr: Precision = FP64, D=None):
    """Y = Norm(Concat_i Interaction_i(X_n) + ShortCut(X_n)) (Eq.(1)); ShortCut
    = X_n if len(X_n) == len(Y) else W_nᵀ X_n on the token axis (Eq.(2), R2-R4).
    With dense injection (R38) the modules read [X_n ; D].  Returns (Y, cache)."""
    L = net.layers[n]
    m_in, m_out = layer_dims(net)[n]
    assert X.shape[1] == m_in
    Xm = np.concatenate([X, D], axis=1) if L.dense_in else X
    us, caches = [], []
    for i, s in enumerate(L.modules):
        p = _module_params(P, i, s.kind)
        if s.kind == "attn":
            U, c = attn_fwd(Xm, p, s, pr, net.ln_eps)
        else:
            U, c = {"dot": dot_fwd, "linear": linear_fwd, "dcn": dcn_fwd, "dcn_lit": dcn_lit_fwd, "dcn_full": dcn_full_fwd,
                    "conv": conv_fwd, "mlp": mlp_fwd}[s.kind](Xm, p, s, pr)
        us.append(U)
        caches.append(c)
    if L.ensemble == "concat":
        Ucat = np.concatenate(us, axis=1)
    elif L.ensemble == "sum":
        Ucat = sum(us)
    else:
        Ucat = sum(w * u for w, u in zip(P["ens_w"], us))
    R = Ucat + (X if m_in == m_out else tokmix_fwd(X, P["W_n"]))
    Y, mu, rstd = ln_fwd(R, P["gamma"], P["beta"], net.ln_eps)
    cache = {"X": X, "Xm": Xm, "mods": caches, "R": pr.q("R", R), "mu": mu, "rstd": rstd,
             "us": us if L.ensemble == "wsum" else None}
    return pr.q("Y", Y), cache


def layer_bwd(net: NetSpec, n: int, cache, dY: np.ndarray, P, pr: Precision = FP64, add=None, with_dD: bool = False):
    """Backward of layer_fwd.  Returns (dX, grads dict in canonical names).  Dense injection (R38): the modules'
    gradient w.r.t. the injected tokens D is returned as a third value when with_dD; `add` (fp64, the layer input's
    shape) is added before dX is rounded (the stack adds every layer's dD to dX0's dense tokens that way)."""
    L = net.layers[n]
    m_in, m_out = layer_dims(net)[n]
    X = cache["X"]
    Xm = cache["Xm"]
    g = {}
    dR, g["gamma"], g["beta"] = ln_bwd(dY, cache["R"], cache["mu"], cache["rstd"], P["gamma"])
    dR = pr.q("dR", dR)
    if m_in == m_out:
        dX = dR.copy()
    else:
        dX, g["W_n"] = tokmix_bwd(X, P["W_n"], dR)
    off = 0
    dD = None
    if L.ensemble == "wsum":   # d(sum_i w_i U_i)/dw_i = <U_i, dR>
        g["ens_w"] = np.array([(u * dR).sum() for u in cache["us"]])
    for i, s in enumerate(L.modules):
        p = _module_params(P, i, s.kind)
        if L.ensemble == "concat":
            dU = dR[:, off:off + s.l, :]
            off += s.l
        elif L.ensemble == "sum":
            dU = dR
        else:
            dU = pr.q("ens.dU", P["ens_w"][i] * dR)
        fn = {"dot": dot_bwd, "linear": linear_bwd, "dcn": dcn_bwd, "dcn_lit": dcn_lit_bwd, "dcn_full": dcn_full_bwd,
              "conv": conv_bwd,
              "attn": attn_bwd, "mlp": mlp_bwd}[s.kind]
        dXi, gi = fn(Xm, p, s, cache["mods"][i], dU, pr)
        dX = dX + dXi[:, :m_in]
        if L.dense_in:
            dD = dXi[:, m_in:] if dD is None else dD + dXi[:, m_in:]
        for k, v in gi.items():
            g[f"{i}.{s.kind}.{k}"] = v
    if add is not None:
        dX = dX + add
    return (pr.q("dX", dX), g, dD) if with_dD else (pr.q("dX", dX), g)


# --------------------------------------------------------------------------
# head, loss (R17) and the training step (SGD, R18; DP loss scaling, R21)
# --------------------------------------------------------------------------


def head_fwd(Y: np.ndarray, ph):
    pooled = Y.mean(axis=1)
    z = pooled @ ph["w_h"] + ph["b_h"][0]
    return z, pooled


def bce_with_logits(z: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Stable form max(z,0) − y·z + log(1 + e^{−|z|})."""
    return np.maximum(z, 0.0) - y * z + np.log1p(np.exp(-np.abs(z)))


def sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def head_bwd(Y, pooled, z, y, ph, B_global: int, pr: Precision = FP64):
    B, m, d = Y.shape
    dz = (sigmoid(z) - y) / B_global
    dY = pr.q("head.dY", np.broadcast_to((dz[:, None] * ph["w_h"][None, :] / m)[:, None, :], Y.shape).copy())
    return dY, {"w_h": pooled.T @ dz, "b_h": np.array([dz.sum()])}


def compute_params(params: List[Dict[str, np.ndarray]], pr: Precision = FP64):
    """The parameter values the arithmetic sees: the master values, rounded to
    bf16 in bf16 mode (the gathered compute copy, R20)."""
    return [{k: pr.q("params", v) for k, v in g.items()} for g in params]


def forward(net: NetSpec, params: List[Dict[str, np.ndarray]], X0: np.ndarray, pr: Precision = FP64):
    """Forward of the stack; `params` are the compute values (see compute_params)."""
    X = X0
    D = X0[:, :net.dense_tokens]   # R38: the dense tokens injected into dense_in layers
    caches = []
    for n in range(len(net.layers)):
        X, c = layer_fwd(net, n, X, params[n], pr, D)
        caches.append(c)
    return X, caches


def train_step(net: NetSpec, params: List[Dict[str, np.ndarray]], X0: np.ndarray, y: np.ndarray,
               lr: float, B_global: int | None = None, pr: Precision = FP64):
    """One SGD step: θ ← θ − lr·g (R18).  The loss is the mean BCE over the
    GLOBAL batch (R21); with B_global = B this is the single-process step."""
    B = X0.shape[0]
    Bg = B if B_global is None else B_global
    cparams = compute_params(params, pr)
    YN, caches = forward(net, cparams, X0, pr)
    ph = cparams[-1]
    z, pooled = head_fwd(YN, ph)
    loss_sum = bce_with_logits(z, y).sum()
    dY, gh = head_bwd(YN, pooled, z, y, ph, Bg, pr)
    grads: List[Dict[str, np.ndarray]] = [None] * len(params)
    grads[-1] = gh
    dD = np.zeros(X0[:, :net.dense_tokens].shape)   # R38: the injected tokens' gradient, summed over layers
    for n in reversed(range(1, len(net.layers))):
        dY, grads[n], dDn = layer_bwd(net, n, caches[n], dY, cparams[n], pr, with_dD=True)
        if dDn is not None:
            dD = dD + dDn
    if net.layers:
        # layer 0: dX0's dense tokens (X0[:, :dense_tokens]) also take dD -- every layer's, layer 0's own included --
        # added before dX0 is rounded (the GPU adds it in the same fp32 step)
        if net.layers[0].dense_in:
            dD = dD + layer_bwd(net, 0, caches[0], dY, cparams[0], pr, with_dD=True)[2]
        add = None
        if net.dense_tokens:
            add = np.zeros(caches[0]["X"].shape)
            add[:, :net.dense_tokens] = dD
        dY, grads[0] = layer_bwd(net, 0, caches[0], dY, cparams[0], pr, add)
    new = [{k: v - lr * grads[gi][k] for k, v in grp.items()} for gi, grp in enumerate(params)]
    return {"loss": loss_sum / Bg, "loss_sum": loss_sum, "logits": z, "Y_N": YN, "dX0": dY,
            "grads": grads, "params": new}


# --------------------------------------------------------------------------
# Adam (NEXT#3; P:158 names the paper's optimizer only as a "BF16 optimizer"): the method variant the
# library offers beside SGD (R18).  Kingma & Ba's update with PyTorch's torch.optim.Adam conventions
# (bias-corrected moments, eps added to sqrt(v_hat), no weight decay), written out per element.
# Pin: tests/test_oracle_modules.py::test_adam_matches_torch (the library routine, several steps).
# --------------------------------------------------------------------------


def adam_init(params: List[Dict[str, np.ndarray]]):
    return {"t": 0, "m": [{k: np.zeros_like(v) for k, v in g.items()} for g in params],
            "v": [{k: np.zeros_like(v) for k, v in g.items()} for g in params]}


def adam_update(params, grads, state, lr: float, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8,
                bf16_state: bool = False):
    """Step t = state.t + 1:  m = b1 m + (1 - b1) g;  v = b2 v + (1 - b2) g^2;
    theta -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps).  Returns (new params, new state).
    bf16_state (the "BF16 optimizer", R35): the moments are STORED rounded to bf16 (RNE) after each step;
    this step's update uses the unrounded m, v."""
    t = state["t"] + 1
    c1, c2 = 1.0 - b1 ** t, 1.0 - b2 ** t
    new_p, new_m, new_v = [], [], []
    for gi, grp in enumerate(params):
        P, M, V = {}, {}, {}
        for k, th in grp.items():
            g = grads[gi][k]
            M[k] = b1 * state["m"][gi][k] + (1.0 - b1) * g
            V[k] = b2 * state["v"][gi][k] + (1.0 - b2) * g * g
            P[k] = th - lr * (M[k] / c1) / (np.sqrt(V[k] / c2) + eps)
            if bf16_state:
                M[k], V[k] = round_bf16(M[k]), round_bf16(V[k])
        new_p.append(P); new_m.append(M); new_v.append(V)
    return new_p, {"t": t, "m": new_m, "v": new_v}


# --------------------------------------------------------------------------
# FLOP accounting (A18; 2·M·N·K per contraction, forward only)
# --------------------------------------------------------------------------


def forward_flops_per_sample(net: NetSpec) -> int:
    d, tot = net.d, 0
    for (m_in, m_out), L in zip(layer_dims(net), net.layers):
        for s in L.modules:
            l = s.l
            if s.kind == "dot":
                h = m_in * (m_in - 1) // 2
                tot += 2 * m_in * m_in * d + 2 * h * l * d
            elif s.kind == "linear":
                tot += 2 * m_in * l * d
            elif s.kind == "dcn_lit":
                tot += 2 * d * d * m_in + 2 * d * d * l
            elif s.kind == "dcn":
                tot += 2 * m_in * d * d + 2 * m_in * l * d
            elif s.kind == "dcn_full":
                tot += 2 * (m_in * d) ** 2 + 2 * m_in * l * d
            elif s.kind == "conv":
                tot += 2 * m_in * d * s.conv_k * s.conv_k + 2 * m_in * l * d
            elif s.kind == "attn":
                f = s.ffn_mult * d
                tot += (2 * m_in * d * 3 * d + 2 * 2 * m_in * m_in * d + 2 * m_in * d * d
                        + 2 * 2 * m_in * d * f + 2 * m_in * l * d)
            elif s.kind == "mlp":
                h1, h2 = s.mlp_hidden
                tot += 2 * m_in * d * h1 + 2 * h1 * h2 + 2 * h2 * l * d
        if m_in != m_out:
            tot += 2 * m_in * m_out * d
    return tot
