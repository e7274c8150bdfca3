"""Time the feature processing layer alone (forward, backward + SGD) at a bench shape (configs.FP):
    python tools/fp_bench.py [--config C4] [--iters 5]
Prints ms per call (CUDA events, L2 flushed before each).  Run under ncu for the per-kernel split."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2203_11014_b200 import binding, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--lib", default="", help="load this libdhen build instead of the default (A/B runs)")
a = ap.parse_args()
if a.lib:
    binding.load(a.lib)
cfg = configs.make(a.config, a.batch or None)
B = cfg.batch_max_local
ntab, R, nden, hid, ndtok, mbag = configs.FP[a.config]
ids, offs, dense = synth.make_fp_batch(7, B, [R] * ntab, nden, mbag)
fp = binding.FeatureProcessing([R] * ntab, nden, hid, ndtok, cfg.d, dtype=cfg.dtype, max_batch=B, max_nnz=len(ids))
tdt = torch.bfloat16
ti, to = torch.tensor(ids, device="cuda"), torch.tensor(offs, device="cuda")
td = torch.tensor(dense, device="cuda").to(tdt)
x0 = torch.empty(B, cfg.m0, cfg.d, device="cuda", dtype=tdt)
dx0 = (torch.randn(B, cfg.m0, cfg.d, device="cuda") * 0.01).to(tdt)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
f = b = 0.0
for it in range(a.iters + 2):
    flush.zero_()
    ev[0].record()
    fp.forward(ti, to, td, x0)
    ev[1].record()
    flush.zero_()
    ev[2].record()
    fp.backward_sgd(dx0, 0.01)
    ev[3].record()
    torch.cuda.synchronize()
    if it >= 2:
        f += ev[0].elapsed_time(ev[1])
        b += ev[2].elapsed_time(ev[3])
print(f"{a.config} B={B} ids={len(ids)} fwd {f / a.iters:.3f} ms  bwd+sgd {b / a.iters:.3f} ms")
