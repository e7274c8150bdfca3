"""Feature processing layer oracle (NEXT#4) — TEST INFRASTRUCTURE ONLY.

Plain fp64 numpy implementation of the step before the DHEN stack: the feature processing layer
"the same ... in DLRM" ("In this work, we use the same feature processing layer in DLRM"):
  * sparse features: each categorical feature t has a lookup table E_t in R^{R_t x d}; a sample's
    (multi-hot) list of ids for feature t is pooled by SUM into one d-vector (DLRM's EmbeddingBag, mode
    "sum"; reading R32 in DESIGN.md §3);
  * dense features: the numerical values go through "several MLPs" (the DLRM bottom MLP: Linear + ReLU
    at every layer, R32) whose output of n_dtok * d values is read as n_dtok d-dimensional tokens;
  * X0 = concat(dense tokens, sparse tokens) in R^{m0 x d}, m0 = n_dtok + n_sparse (DLRM concatenates
    the dense output first: R32).
Backward and the optimizer (R34): dL/dE_t[r] = sum over the occurrences of row r of dL/dX0[b, n_dtok + t];
SGD E <- E - lr dE touches exactly the looked-up rows (every other row has a zero gradient); the bottom
MLP's parameters take plain SGD like the stack's.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s baseline legs may import this module; it imports
nothing from the product.  bf16 storage points (R33, mirrored from the CUDA path): the dense input, the MLP
parameters' compute copies (W_k and b_k), the hidden activations H_k, X0, and the MLP backward's dZ_k; the tables and every
sum stay fp32 / fp64.  Pins: tests/test_oracle_fp.py (torch embedding_bag / autograd / SGD, brute force).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List

import numpy as np

from oracle.dhen_oracle import round_bf16

FP_POINTS = ("fp.dense", "fp.W", "fp.H", "fp.X0", "fp.dZ")


@dataclass
class FPSpec:
    rows: List[int]           # R_t: rows of table t (one table per sparse feature)
    n_dense: int              # numerical features per sample
    hidden: List[int]         # bottom-MLP hidden widths
    n_dtok: int               # dense tokens: the MLP's output width is n_dtok * d
    d: int

    @property
    def n_sparse(self) -> int:
        return len(self.rows)

    @property
    def m0(self) -> int:
        return self.n_dtok + self.n_sparse

    def mlp_dims(self) -> List[int]:
        return [self.n_dense] + list(self.hidden) + [self.n_dtok * self.d]


@dataclass
class FPPrecision:
    bf16: bool = False

    def q(self, name: str, x: np.ndarray) -> np.ndarray:
        assert name in FP_POINTS, name
        return round_bf16(x) if self.bf16 else x


def fp_init(spec: FPSpec, rng: np.random.Generator) -> Dict[str, list]:
    """Tables U(+-sqrt(1/R_t)) (DLRM's embedding init), MLP weights / biases U(+-1/sqrt(fan_in))."""
    tables = [rng.uniform(-1, 1, (R, spec.d)) * np.sqrt(1.0 / R) for R in spec.rows]
    dims = spec.mlp_dims()
    W = [rng.uniform(-1, 1, (dims[k + 1], dims[k])) / np.sqrt(dims[k]) for k in range(len(dims) - 1)]
    b = [rng.uniform(-1, 1, dims[k + 1]) / np.sqrt(dims[k]) for k in range(len(dims) - 1)]
    return {"tables": tables, "W": W, "b": b}


def embedding_bag_sum(table: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """One bag: sum of the looked-up rows, in list order (an empty bag pools to zero)."""
    out = np.zeros(table.shape[1])
    for r in ids:
        out = out + table[r]
    return out


def fp_fwd(spec: FPSpec, P, indices: np.ndarray, offsets: np.ndarray, dense: np.ndarray,
           prec: FPPrecision = FPPrecision()):
    """indices: all ids, bag (b, t) = indices[offsets[b n_sparse + t] : offsets[b n_sparse + t + 1]]
    (sample-major CSR, ids relative to table t); dense: [B][n_dense].  Returns X0 [B][m0][d] and the cache."""
    B = dense.shape[0]
    d, ns, nd = spec.d, spec.n_sparse, spec.n_dtok
    h = prec.q("fp.dense", dense.astype(np.float64))
    Hs, Zs = [h], []
    for k, (W, b) in enumerate(zip(P["W"], P["b"])):
        z = h @ prec.q("fp.W", W).T + prec.q("fp.W", b)   # the compute copies of W_k and b_k (R33)
        a = np.maximum(z, 0.0)                     # ReLU after every bottom-MLP layer (R32)
        Zs.append(z)
        last = k == len(P["W"]) - 1
        h = a if last else prec.q("fp.H", a)
        Hs.append(h)
    X0 = np.zeros((B, spec.m0, d))
    X0[:, :nd, :] = Hs[-1].reshape(B, nd, d)
    for b in range(B):
        for t in range(ns):
            lo, hi = offsets[b * ns + t], offsets[b * ns + t + 1]
            X0[b, nd + t] = embedding_bag_sum(P["tables"][t], indices[lo:hi])
    X0 = prec.q("fp.X0", X0)
    return X0, {"H": Hs, "Z": Zs, "X0": X0, "indices": indices, "offsets": offsets, "B": B}


def fp_bwd(spec: FPSpec, P, cache, dX0: np.ndarray, prec: FPPrecision = FPPrecision()):
    """dX0 [B][m0][d] -> gradients {"tables": dense arrays like the tables, "W": [...], "b": [...]}.
    The last layer's ReLU derivative is taken from the stored output (X0's dense tokens > 0)."""
    B = cache["B"]
    d, ns, nd = spec.d, spec.n_sparse, spec.n_dtok
    L = len(P["W"])
    out = cache["X0"][:, :nd, :].reshape(B, nd * d)
    dZ = prec.q("fp.dZ", dX0[:, :nd, :].reshape(B, nd * d) * (out > 0))
    gW, gb = [None] * L, [None] * L
    for k in range(L - 1, -1, -1):
        gW[k] = dZ.T @ cache["H"][k]
        gb[k] = dZ.sum(axis=0)
        if k > 0:
            dH = dZ @ prec.q("fp.W", P["W"][k])
            dZ = prec.q("fp.dZ", dH * (cache["H"][k] > 0))
    gT = [np.zeros_like(T) for T in P["tables"]]
    idx, off = cache["indices"], cache["offsets"]
    for b in range(B):
        for t in range(ns):
            for e in range(off[b * ns + t], off[b * ns + t + 1]):
                gT[t][idx[e]] += dX0[b, nd + t]
    return {"tables": gT, "W": gW, "b": gb}


def fp_sgd(P, G, lr: float):
    """theta <- theta - lr g for every table and MLP parameter (rows with no occurrence are unchanged)."""
    return {"tables": [T - lr * g for T, g in zip(P["tables"], G["tables"])],
            "W": [W - lr * g for W, g in zip(P["W"], G["W"])],
            "b": [b - lr * g for b, g in zip(P["b"], G["b"])]}


def fp_forward_flops_per_sample(spec: FPSpec) -> int:
    """Bottom-MLP contraction FLOPs 2 * in * out per layer (pooling adds are not contractions)."""
    dims = spec.mlp_dims()
    return sum(2 * dims[k] * dims[k + 1] for k in range(len(dims) - 1))
