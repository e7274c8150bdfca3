"""HBM bandwidth probes (CUDA events): write-only fill, read-only reduction, copy.  Usage: python tools/membw.py
Note: torch's fill_ / zero_ of a uint8 tensor measure torch's byte-fill kernel (3.9 TB/s here), not the HBM write
ceiling; tools/micro/write_bw.cu measures plain, streaming and TMA bulk stores (6.2-7.4 TB/s)."""
import torch


def t(fn, it=20):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(it)]
    fn()
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[it // 2]


x = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
y = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
n = x.numel()
print(f"write (fill)   {n / t(lambda: x.fill_(1)) / 1e6:8.1f} GB/s")
print(f"write (memset) {n / t(lambda: x.zero_()) / 1e6:8.1f} GB/s")
xf = x.view(torch.float32)
print(f"read (sum)     {n / t(lambda: xf.sum()) / 1e6:8.1f} GB/s")
print(f"copy           {2 * n / t(lambda: y.copy_(x)) / 1e6:8.1f} GB/s")
