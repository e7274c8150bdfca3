"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

Holds NONE of the method's arithmetic: only random numbers of the shapes and
distributions DESIGN.md §5 states (SURVEY §8(d) "Concrete synthetic inputs"):

* X0 ~ N(0, 1), rounded to bf16 (RNE) for bf16 runs, fp32 otherwise;
* labels ~ Bernoulli(0.05) ("CTR-shaped"; the paper never states its CTR);
* parameters: U(±1/sqrt(fan_in)) for weights, LN gamma = 1 (+0.1·N(0,1) when
  perturbed) and beta = 0 (+0.1·N(0,1) when perturbed), so LN grads are exercised.

All draws use numpy's PCG64 with explicit seeds; seeds are 2203011014 + config
index by convention (bench.py / tests pass them in).
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 2203011014


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def to_bf16_f32(a: np.ndarray) -> np.ndarray:
    """fp32 -> nearest bf16 (ties to even), returned as fp32 values (bit trick
    on the fp32 representation; inputs are finite)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def make_x0(seed: int, B: int, m: int, d: int, bf16: bool) -> np.ndarray:
    x = _rng(seed).standard_normal((B, m, d), dtype=np.float32)
    return to_bf16_f32(x) if bf16 else x


def make_labels(seed: int, B: int, ctr: float = 0.05) -> np.ndarray:
    return (_rng(seed + 7919).random(B) < ctr).astype(np.float32)


def make_params(seed: int, entries, perturb_ln: bool = True) -> np.ndarray:
    """entries: list of (size, init) with init in {('u', fan_in), ('one',), ('zero',)}.
    Returns one flat fp32 vector in the given order."""
    rng = _rng(seed + 104729)
    out = []
    for size, init in entries:
        if init[0] == "u":
            bound = 1.0 / np.sqrt(init[1])
            out.append(rng.uniform(-bound, bound, size).astype(np.float32))
        elif init[0] == "one":
            v = np.ones(size, np.float32)
            if perturb_ln:
                v += (0.1 * rng.standard_normal(size)).astype(np.float32)
            out.append(v)
        elif init[0] == "zero":
            v = np.zeros(size, np.float32)
            if perturb_ln:
                v += (0.1 * rng.standard_normal(size)).astype(np.float32)
            out.append(v)
        else:
            raise ValueError(init)
    return np.concatenate(out).astype(np.float32) if out else np.zeros(0, np.float32)


def make_fp_batch(seed: int, B: int, rows, n_dense: int, mean_bag: float, alpha: float = 3.0,
                  bf16: bool = True, empty_frac: float = 0.0):
    """Feature-processing inputs (NEXT#4): per (sample, table) a bag of
    1 + Poisson(mean_bag - 1) ids (a fraction `empty_frac` of bags empty), ids skewed towards the head of
    each table (floor(R u^alpha), u ~ U(0, 1): power-law-like row popularity, as in click logs), CSR in
    sample-major order (int32 ids relative to their table, int32 offsets); dense features ~ N(0, 1)
    (bf16-rounded for bf16 runs).  Returns (ids, offsets, dense)."""
    rng = _rng(seed + 15485863)
    ns = len(rows)
    lens = 1 + rng.poisson(max(mean_bag - 1.0, 0.0), B * ns)
    if empty_frac > 0:
        lens[rng.random(B * ns) < empty_frac] = 0
    offsets = np.zeros(B * ns + 1, np.int64)
    offsets[1:] = np.cumsum(lens)
    R = np.tile(np.asarray(rows, np.int64), B)
    ids = np.floor(np.repeat(R, lens) * rng.random(int(offsets[-1])) ** alpha).astype(np.int64)
    ids = np.minimum(ids, np.repeat(R, lens) - 1)
    dense = rng.standard_normal((B, n_dense), dtype=np.float32)
    if bf16:
        dense = to_bf16_f32(dense)
    return ids.astype(np.int32), offsets.astype(np.int32), dense
