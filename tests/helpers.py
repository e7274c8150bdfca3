"""Test helpers: config builders and oracle-side parameter generation.

The configs mirror BASELINE.json's C1-C5 (module choices from SURVEY §8(d));
`scale` shrinks them for CPU-speed oracle runs while keeping the structure.
"""
from __future__ import annotations

import numpy as np

import synth
from oracle import dhen_oracle as O


def M(kind, l, **kw):
    return O.ModuleSpec(kind, l, **kw)


def config(name: str) -> O.NetSpec:
    """Full-size BASELINE.json configs."""
    if name == "C1":
        return O.NetSpec(8, 16, [O.LayerSpec([M("dot", 4), M("linear", 4)])])
    if name == "C2":
        return O.NetSpec(64, 128, [O.LayerSpec([M("dot", 32), M("dcn", 32)]) for _ in range(2)])
    if name == "C3":
        L0 = O.LayerSpec([M("attn", 64), M("linear", 32), M("mlp", 32)])
        return O.NetSpec(100, 128, [L0] + [O.LayerSpec([M("attn", 64), M("linear", 32), M("mlp", 32)])
                                            for _ in range(3)])
    if name == "C4":
        return O.NetSpec(128, 256, [O.LayerSpec([M("dot", 32), M("attn", 32), M("conv", 16),
                                                 M("dcn", 32), M("linear", 16)]) for _ in range(8)])
    if name == "C5":
        return O.NetSpec(128, 256, [O.LayerSpec([M("dcn", 128)]) for _ in range(8)])
    raise KeyError(name)


def small(name: str) -> O.NetSpec:
    """Structure-preserving reduced configs the oracle finishes in well under a second."""
    if name == "C1":
        return config("C1")
    if name == "C2":
        return O.NetSpec(12, 16, [O.LayerSpec([M("dot", 6), M("dcn", 6)]) for _ in range(2)])
    if name == "C3":
        mk = lambda: O.LayerSpec([M("attn", 6, heads=2), M("linear", 3), M("mlp", 3, mlp_hidden=(24, 20))])
        return O.NetSpec(10, 16, [mk(), mk()])          # 10 -> 12 exercises W_n
    if name == "C4":
        return O.NetSpec(12, 16, [O.LayerSpec([M("dot", 3), M("attn", 3), M("conv", 2),
                                               M("dcn", 2), M("linear", 2)]) for _ in range(2)])
    if name == "C5":
        return O.NetSpec(12, 16, [O.LayerSpec([M("dcn", 12)]) for _ in range(3)])
    raise KeyError(name)


def init_entries(group):
    ent = []
    for name, shp, fan in group:
        size = int(np.prod(shp))
        base = name.split(".")[-1]
        if base in ("gamma", "g1", "g2", "ens_w"):
            ent.append((size, ("one",)))
        elif base in ("beta", "be1", "be2"):
            ent.append((size, ("zero",)))
        else:
            ent.append((size, ("u", fan)))
    return ent


def make_flat_params(net: O.NetSpec, seed: int, perturb_ln: bool = True):
    """One flat fp32 vector per group (layers then head), canonical order."""
    return [synth.make_params(seed + 31 * gi, init_entries(g), perturb_ln)
            for gi, g in enumerate(O.param_groups(net))]


def oracle_params(net: O.NetSpec, flats):
    return [O.unflatten(g, f.astype(np.float64)) for g, f in zip(O.param_groups(net), flats)]


def elem_err(a, o):
    """max_i |a_i − o_i| / max(1, |o_i|) (SURVEY §8(c) parity metric)."""
    a = np.asarray(a, np.float64)
    o = np.asarray(o, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - o) / np.maximum(1.0, np.abs(o))))


def norm_err(a, o):
    """max_i |a_i − o_i| / max_i |o_i| (per tensor)."""
    a = np.asarray(a, np.float64)
    o = np.asarray(o, np.float64)
    if a.size == 0:
        return 0.0
    den = np.max(np.abs(o))
    return float(np.max(np.abs(a - o)) / (den if den > 0 else 1.0))
