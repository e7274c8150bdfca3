"""cuBLAS (torch.matmul) timings of plain row-major GEMMs with the same M, N, K as the DHEN step's
shapes: a calibration of what the hardware / library reaches (not part of the product)."""
import torch

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, M, N, K, odt in [("tok-like", 262144, 32, 64, torch.float32), ("n128", 262144, 128, 64, torch.bfloat16),
                           ("k256", 65536, 128, 256, torch.bfloat16), ("dcn.cross", 131072, 128, 128, torch.bfloat16),
                           ("dot.proj", 2048, 4096, 2016, torch.float32), ("C4 dot.proj", 8192, 8192, 8128, torch.bfloat16),
                           ("C4 dcn", 1048576, 256, 256, torch.bfloat16), ("C4 ffn1", 1048576, 1024, 256, torch.bfloat16)]:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=odt)
    for _ in range(3):
        torch.matmul(A, B.t(), out=out) if odt == torch.bfloat16 else out.copy_(torch.matmul(A, B.t()))
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(A, B.t(), out=out) if odt == torch.bfloat16 else torch.matmul(A, B.t())
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[5]
    byts = (M * K + N * K) * 2 + M * N * (4 if odt == torch.float32 else 2)
    print(f"{name:12s} M={M} N={N} K={K}: {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:8.1f} TF/s {byts/ms/1e6:8.1f} GB/s")
