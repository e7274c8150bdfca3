"""Time single library GEMMs of the DHEN step's shapes through the C-ABI test hook
(CUDA events, L2 flushed before each launch).  Usage:
    python tools/gemm_bench.py [--cfg C2] [--only name] [--iters 20]
Prints one line per shape: ms, TFLOP/s, GB/s (algorithmic bytes)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def shapes(cfg):
    # (name, M, N, K, batch, A(s_mn,s_k,bs0,bs1,zdiv,kdiv,s_ko), B(...), C(rs,cs,bs0,bs1,zdiv), acc, a2, b2, c2, cdt)
    if cfg == "C2":
        B, m, d, l, mo = 2048, 64, 128, 32, 64
        h = m * (m - 1) // 2
    else:
        B, m, d, l, mo = 8192, 128, 256, 32, 128
        h = m * (m - 1) // 2
    R = B * m
    f32, bf = torch.float32, torch.bfloat16
    return [
        ("dot.gram", m, m, d, B, (d, 1, m * d, 0, 1, 0, 0), (d, 1, m * d, 0, 1, 0, 0), (m, 1, m * m, 0, 1), 0,
         (0, 0), (0, 0), (0, 0), f32),
        ("dot.proj", B, l * d, h, 1, (h, 1, 0, 0, 1, 0, 0), (h, 1, 0, 0, 1, 0, 0), (mo * d, 1, 0, 0, 1), 0,
         (0, 0), (0, 0), (0, 0), f32),
        ("dot.proj_dgrad", B, h, l * d, 1, (mo * d, 1, 0, 0, 1, 0, 0), (1, h, 0, 0, 1, 0, 0), (h, 1, 0, 0, 1), 0,
         (0, 0), (0, 0), (0, 0), bf),
        ("dot.proj_wgrad", l * d, h, B, 1, (1, mo * d, 0, 0, 1, 0, 0), (1, h, 0, 0, 1, 0, 0), (h, 1, 0, 0, 1), 1,
         (0, 0), (0, 0), (0, 0), f32),
        ("dot.gram_bwd", m, d, m, B, (m, 1, m * m, 0, 1, 0, 0), (1, d, m * d, 0, 1, 0, 0), (d, 1, m * d, 0, 1), 1,
         (0, 0), (0, 0), (0, 0), f32),
        ("dcn.cross", R, d, d, 1, (d, 1, 0, 0, 1, 0, 0), (d, 1, 0, 0, 1, 0, 0), (d, 1, 0, 0, 1), 0,
         (0, 0), (0, 0), (0, 0), bf),
        ("dcn.wgrad", d, d, R, 1, (1, d, 0, 0, 1, 0, 0), (1, d, 0, 0, 1, 0, 0), (d, 1, 0, 0, 1), 1,
         (0, 0), (0, 0), (0, 0), f32),
        ("tokmix.fwd", B * d, l, m, 1, (1, d, 0, 0, 1, 0, 0), (1, l, 0, 0, 1, 0, 0), (1, d, 0, 0, 1), 0,
         (d, m * d), (0, 0), (d, mo * d), f32),
        ("tokmix.dgrad", B * d, m, l, 1, (1, d, 0, 0, 1, 0, 0), (l, 1, 0, 0, 1, 0, 0), (1, d, 0, 0, 1), 0,
         (d, mo * d), (0, 0), (d, m * d), bf),
        ("tokmix.wgrad", m, l, B * d, 1, (d, 1, 0, 0, 1, d, m * d), (d, 1, 0, 0, 1, d, mo * d), (l, 1, 0, 0, 1), 1,
         (0, 0), (0, 0), (0, 0), f32),
        ("attn.ffn1", R, 4 * d, d, 1, (d, 1, 0, 0, 1, 0, 0), (d, 1, 0, 0, 1, 0, 0), (4 * d, 1, 0, 0, 1), 0,
         (0, 0), (0, 0), (0, 0), bf),
        ("attn.ffn2_dgrad", R, 4 * d, d, 1, (d, 1, 0, 0, 1, 0, 0), (1, 4 * d, 0, 0, 1, 0, 0), (4 * d, 1, 0, 0, 1), 0,
         (0, 0), (0, 0), (0, 0), bf),
        ("attn.ffn2", R, d, 4 * d, 1, (4 * d, 1, 0, 0, 1, 0, 0), (4 * d, 1, 0, 0, 1, 0, 0), (d, 1, 0, 0, 1), 0,
         (0, 0), (0, 0), (0, 0), f32),
        ("mlp.fc2_wgrad", 1024, 1024, 8192, 1, (1, 1024, 0, 0, 1, 0, 0), (1, 1024, 0, 0, 1, 0, 0), (1024, 1, 0, 0, 1), 1,
         (0, 0), (0, 0), (0, 0), f32),
        # weight gradients (K = B m rows, both operands MN-major, split-K)
        ("attn.ffn1_wgrad", 4 * d, d, R, 1, (1, 4 * d, 0, 0, 1, 0, 0), (1, d, 0, 0, 1, 0, 0), (d, 1, 0, 0, 1), 1,
         (0, 0), (0, 0), (0, 0), f32),
        ("attn.ffn2_wgrad", d, 4 * d, R, 1, (1, d, 0, 0, 1, 0, 0), (1, 4 * d, 0, 0, 1, 0, 0), (4 * d, 1, 0, 0, 1), 1,
         (0, 0), (0, 0), (0, 0), f32),
        # experiments: same M, N, K as tokmix.fwd with plain layouts
        ("x.kmaj_rowmajor", B * d, l, m, 1, (m, 1, 0, 0, 1, 0, 0), (m, 1, 0, 0, 1, 0, 0), (l, 1, 0, 0, 1), 0,
         (0, 0), (0, 0), (0, 0), f32),
        ("x.kmaj_n128", B * d, 128, m, 1, (m, 1, 0, 0, 1, 0, 0), (m, 1, 0, 0, 1, 0, 0), (128, 1, 0, 0, 1), 0,
         (0, 0), (0, 0), (0, 0), bf),
        ("x.kmaj_k256", B * d // 4, 128, 256, 1, (256, 1, 0, 0, 1, 0, 0), (256, 1, 0, 0, 1, 0, 0), (128, 1, 0, 0, 1), 0,
         (0, 0), (0, 0), (0, 0), bf),
        ("x.mnA_rowmajor", B * d, l, m, 1, (1, d, 0, 0, 1, 0, 0), (1, l, 0, 0, 1, 0, 0), (l, 1, 0, 0, 1), 0,
         (d, m * d), (0, 0), (0, 0), f32),
    ]


def extent(r, K, z, s_mn, s_k, bs0, bs1, zdiv, kdiv, s_ko, mdiv=0, s_mo=0):
    rows = ((r - 1) // mdiv) * s_mo + ((r - 1) % mdiv) * s_mn if mdiv else (r - 1) * s_mn
    kk = ((K - 1) % kdiv) * s_k + ((K - 1) // kdiv) * s_ko if kdiv else (K - 1) * s_k
    zz = ((z - 1) // zdiv) * bs0 + ((z - 1) % zdiv) * bs1
    return rows + kk + zz + 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C2")
    ap.add_argument("--only", default="")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--path", type=int, default=0)
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--flush", default="write", choices=["write", "read", "none"])
    ap.add_argument("--lib", default="", help="load this libdhen build instead of the default (A/B runs)")
    ap.add_argument("--epi", type=int, default=0, help="fused epilogue mode (1 mask, 2 resid, 3 cross, 4 relu, 5 relu+bits out, 6 bits in)")
    args = ap.parse_args()
    if args.lib:
        from paper_2203_11014_b200 import binding
        binding.load(args.lib)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for (name, M, N, K, Z, a, b, c, acc, a2, b2, c2, cdt) in shapes(args.cfg):
        if args.only and args.only not in name:
            continue
        A = torch.randn(extent(M, K, Z, *a, *a2), device="cuda").to(torch.bfloat16)
        Bm = torch.randn(extent(N, K, Z, *b, *b2), device="cuda").to(torch.bfloat16)
        rs, cs, cb0, cb1, czd = c
        cext = extent(M, N, Z, rs, cs, cb0, cb1, czd, 0, 0, *c2)
        Cm = torch.zeros(cext, device="cuda", dtype=cdt)
        q = [M, N, K, Z] + list(a) + list(b) + list(c) + [acc] + list(a2) + list(b2) + list(c2)
        E = torch.randn(cext, device="cuda").to(torch.bfloat16) if args.epi else None
        aux = torch.empty(cext, device="cuda", dtype=torch.bfloat16) if args.epi == 3 else None
        if args.epi in (5, 6):   # ReLU bitmask [N / 32][M] words
            aux = torch.randint(-2**31, 2**31 - 1, (((N + 31) // 32) * M * Z,), device="cuda", dtype=torch.int32)
        if args.epi:
            from paper_2203_11014_b200.binding import debug_gemm_epi

            def debug_gemm(q, A, Bm, Cm, path=0, ws=None):  # noqa: F811
                return debug_gemm_epi(q, A, Bm, Cm, args.epi, E=E, aux=aux, path=path, ws=ws)
        else:
            from paper_2203_11014_b200.binding import debug_gemm
        tc = debug_gemm(q, A, Bm, Cm, path=args.path, ws=ws)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.iters)]
        for e0, e1 in ev:
            if args.flush == "write":
                flush.zero_()
            elif args.flush == "read":
                flush_sum = flush.view(torch.int32).sum()  # noqa: F841  (read-only flush: clean lines)
            e0.record()
            debug_gemm(q, A, Bm, Cm, path=args.path, ws=ws)
            e1.record()
        torch.cuda.synchronize()
        ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)[len(ev) // 2]
        if args.trace:
            from paper_2203_11014_b200.binding import load
            import ctypes
            tr = torch.zeros(512, dtype=torch.int64, device="cuda")
            load().dhen_debug_gemm_trace(ctypes.c_void_p(tr.data_ptr()))
            flush.zero_()
            debug_gemm(q, A, Bm, Cm, path=args.path, ws=ws)
            torch.cuda.synchronize()
            load().dhen_debug_gemm_trace(None)
            t = tr.cpu().tolist()
            t0 = min(x for x in t if x > 0)
            names = ["load_issue", "mma_start", "data_ready", "epi_start", "tmem_read", "epi_end", "arrived"]
            for i in range(16):
                print("  item/iter %2d: " % i + " ".join(f"{nm}={(t[64 * k + i] - t0) if t[64 * k + i] else -1:7d}"
                                                      for k, nm in enumerate(names)))
        fl = 2.0 * M * N * K * Z
        es_c = 4 if cdt == torch.float32 else 2
        byts = A.numel() * 2 + Bm.numel() * 2 + M * N * Z * es_c * (2 if acc else 1)
        print(f"{name:16s} tc={int(tc)} M={M:7d} N={N:5d} K={K:6d} Z={Z:5d} {ms * 1e3:9.1f} us "
              f"{fl / ms / 1e9:8.1f} TF/s {byts / ms / 1e6:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
