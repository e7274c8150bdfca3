"""Child process of tests/test_gpu_attn.py::test_attn_bwd_barrier_race_probe: one attention-only DHEN layer
(m = 100, d = 128, H = 2 -> dh = 64, the C3 shape) forward + backward through the library build given on the
command line; prints a checksum of dX and the layer gradients.  A race-probe build whose protocol deadlocks
traps in its bounded mbarrier wait (the process then fails with the watchdog's report on stdout)."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(lib):
    import numpy as np
    import torch

    from paper_2203_11014_b200 import binding
    binding.load(lib)
    m, d, B = 100, 128, 600
    cfg = binding.Config(m, d, [[binding.Module("attn", m, heads=2)]], dtype="bf16", batch_max_local=B, seed=7)
    model = binding.DHEN(cfg)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(B, m, d, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(B, m, d, device="cuda", generator=g) / 30).to(torch.bfloat16)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        model.zero_grad()
        model.layer_fwd(0, x, y)
        model.layer_bwd(0, dy, dx)
    torch.cuda.synchronize()
    h = hashlib.sha256(dx.view(torch.int16).cpu().numpy().tobytes())
    h.update(model.get_grads(0).astype(np.float32).tobytes())
    print("CHECKSUM", h.hexdigest(), flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
