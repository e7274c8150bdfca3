"""BASELINE.json configurations C1-C5 (module choices: SURVEY §8(d) table)."""
from __future__ import annotations

from .binding import Config, Module

DESCR = {
    "C1": "1-layer DHEN {DotProduct, Linear}, 8 features x dim 16, batch 32, fp32",
    "C2": "2-layer DHEN {DotProduct, DCN}, 64 features x dim 128, batch 2048, bf16",
    "C3": "4-layer DHEN {SelfAttention, Linear, MLP}, 100 features x dim 128, batch 8192, bf16",
    "C4": "8-layer DHEN {DotProduct, SelfAttention, Conv, DCN, Linear}, 128 features x dim 256, 8192/GPU, bf16",
    "C5": "8-layer DCN-only stack, 128 features x dim 256, 8192/GPU, bf16",
}
BATCH = {"C1": 32, "C2": 2048, "C3": 8192, "C4": 8192, "C5": 8192}


def make(name: str, batch: int | None = None, seed: int = 2203011014) -> Config:
    B = batch or BATCH[name]
    if name == "C1":
        return Config(8, 16, [[Module("dot", 4), Module("linear", 4)]], dtype="fp32", batch_max_local=B, seed=seed + 1)
    if name == "C2":
        return Config(64, 128, [[Module("dot", 32), Module("dcn", 32)] for _ in range(2)], dtype="bf16",
                      batch_max_local=B, seed=seed + 2)
    if name == "C3":
        return Config(100, 128, [[Module("attn", 64), Module("linear", 32), Module("mlp", 32)] for _ in range(4)],
                      dtype="bf16", batch_max_local=B, seed=seed + 3)
    if name == "C4":
        return Config(128, 256, [[Module("dot", 32), Module("attn", 32), Module("conv", 16), Module("dcn", 32),
                                  Module("linear", 16)] for _ in range(8)], dtype="bf16", batch_max_local=B,
                      seed=seed + 4)
    if name == "C5":
        return Config(128, 256, [[Module("dcn", 128)] for _ in range(8)], dtype="bf16", batch_max_local=B,
                      seed=seed + 5)
    raise KeyError(name)


# Feature processing fronts (NEXT#4, `bench.py --fp`): (tables, rows per table, dense features, bottom-MLP
# hidden widths, dense tokens, mean ids per bag).  Tables + dense tokens = the config's m0; ids per bag
# 1 + Poisson(mean - 1), power-law row popularity (synth.make_fp_batch).
FP = {
    "C1": (6, 1_000, 8, (), 2, 4.0),
    "C2": (56, 100_000, 64, (512,), 8, 20.0),
    "C3": (92, 100_000, 64, (512,), 8, 20.0),
    "C4": (120, 100_000, 64, (512,), 8, 20.0),
    "C5": (120, 100_000, 64, (512,), 8, 20.0),
}
