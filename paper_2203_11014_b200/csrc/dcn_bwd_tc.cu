// dcn_bwd_tc.cu — B8, the DCN cross backward, as ONE kernel per 128-row tile (north-star reading R13 of Eq.(7),
// P:123-128):
//
//   forward   A = X W^T + b,   T = X (.) A + X,   U = W_u^T T
//   backward  dT = W_u dU   (MMA 1: K = l tokens, spt samples per tile through the block-diagonal W_u)
//             dA = dT (.) X                          (bf16: the weight / bias gradients' operand, and MMA 2's A)
//             dX = [dR or acc] + dT (.) A + dT + dA W  (MMA 2: K = d)
//
// The two-GEMM form moves an fp32 [B m][d] partial dX through HBM between the dT GEMM and the dA W GEMM (8 B per
// element, 2 GB per C4 / C5 layer).  Here the partial P = base + dT (.) A + dT never leaves the SM: it is written
// back into MMA 1's TMEM columns, dA goes to shared memory as MMA 2's K-major A operand (and from there to HBM by
// TMA store for the weight gradients), MMA 2 accumulates dA W into the other d TMEM columns, and the epilogue emits
// P + dA W once.  Per item only dU arrives for the MMAs; W streams through a two-slot ring of 64-row k-blocks (it is
// the same every item, so its loads run ahead); X, A and the base arrive as per-warp 32 x 32 TMA boxes (the next
// pass's boxes fly while this pass is combined); dA and dX leave by TMA store from the warp's own 32-row slices of
// the dA tile.  Same arithmetic in the same order as the two-GEMM path: dX and dA bit-identical.  The bias
// gradient db = sum_rows dA is read down the stored dA slices (lane = column, rows in order) into one partial row
// per CTA quadrant; the runtime adds the partial rows in order.
//
// Warps: 0 TMA producer (W_u once, dU per item, the W ring), 1 MMA issuer (+ TMEM), 2-9 epilogue (warp w: TMEM lanes
// 32 (w % 4) .., column half (w - 2) / 4), each issuing its own operand-box loads.  Persistent CTAs, items strided.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "dcn_bwd.h"
#include "gemm_tc_kernel.cuh"
#include "tuning.h"

namespace dhen {
namespace dcnb {

using namespace tc;

struct Params {
  int m, l, d, spt, K1, items;
  int rin_f32, out_f32;      // base: bf16 dR (first writer) or fp32 accumulator; out: fp32 accumulator or bf16 dX
  float* bsum;               // [grid * 4][d] partial column sums of the stored dA
};
struct Maps {
  CUtensorMap wu, du, w;     // MMA operands (128-B swizzle)
  CUtensorMap x, a, rin;     // per-warp operand boxes 32 rows x 32 columns (bf16: 64-B swizzle, fp32 base: 128-B)
  CUtensorMap da, out;       // stores: dA 32 x 64 bf16 (128-B); out 32 x 64 bf16 or 32 x 32 fp32 (128-B), or in
                             // the shared-tile form 32 x 32 bf16 (64-B)
};

__device__ __forceinline__ void tma_load2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tma_store2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0), "r"(c1),
               "r"(src)
               : "memory");
}
__device__ __forceinline__ void arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

// barrier indices
// (BDA + c: 64-column chunk c of dA is in shared memory -- MMA 2's k-block c may start)
enum { BC = 0, BUF = 1, BUE = 2, BD1 = 3, BD2 = 4, BTF = 5, BWF = 6, BWE = 8, BOP = 10, BSR = 18, BDA = 19, NBAR = 23 };

// SH (the shared-tile form, K1 up to 128): the dU tile and the dA tile share one 128 x D buffer (dU is consumed by
// MMA 1 before dA is written; the next dU lands once MMA 2 and the dA stores have read it), W_u' takes two chunks,
// and the dX boxes go through the spare 2 KB of each warp's operand slot (bf16 base and bf16 dX only).
template <int D, bool SH> struct Smem {
  static constexpr int NCH = D / 64;
  static constexpr int WU = SH ? 32768 : 16384;    // W_u' [128][K1], K-major 64-column chunks (K1 <= 128 / 64)
  static constexpr int U = SH ? 0 : 16384;         // dU tile: NCH chunks of K1 rows x 64 columns (K1 D 2 <= 16 KB)
  static constexpr int A = 128 * D * 2;            // dA tile: NCH K-major chunks of 128 rows x 64 columns
  static constexpr int W = NCH * 8192;             // one W k-block: 64 rows x D, NCH MN-major 64 x 64 boxes
  static constexpr int OPW = 8192;                 // per epilogue warp: X 2 KB | A 2 KB | base <= 4 KB
  static constexpr int oWU = 0, oA = oWU + WU, oU = SH ? oA : oA + A, oW = oA + A + U, oOP = oW + 2 * W,
                       oBAR = oOP + 8 * OPW;
  static constexpr int BYTES = oBAR + 256 + 1024;
};

template <int D, bool SH>
__global__ void __launch_bounds__(320, 1) dcn_bwd_kernel(const __grid_constant__ Maps mp, const __grid_constant__ Params p) {
  pdl_release();
  using S = Smem<D, SH>;
  constexpr int NCH = S::NCH;
  constexpr int HC = D / 2, NP = HC / 32;   // epilogue columns per warp, 32-column passes
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t s0 = smem_u32(smem);
  const uint32_t sWu = s0 + S::oWU, sU = s0 + S::oU, sA = s0 + S::oA, sW = s0 + S::oW, sOP = s0 + S::oOP;
  uint64_t* bars = (uint64_t*)(smem + S::oBAR);
  auto B_ = [&](int i) { return smem_u32(bars + i); };
  uint32_t* tslot = (uint32_t*)(bars + NBAR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mp.wu) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mp.du) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mp.w) : "memory");
    for (int i = 0; i < NBAR; ++i) mbar_init(B_(i), (i >= BDA || i == BTF || i == BSR) ? 8 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(2 * D));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  pdl_wait();
  const int n = (int)blockIdx.x < p.items ? (p.items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const int K1 = p.K1;

  if (warp == 0) {
    if (lane == 0) {   // ---------------- producer
      const int kc1 = (K1 + 63) / 64;
      mbar_expect_tx(B_(BC), (uint32_t)(kc1 * 16384));
      for (int c = 0; c < kc1; ++c) tma_load2d(sWu + (uint32_t)(c * 16384), &mp.wu, 64 * c, 0, B_(BC));
      int wc = 0;   // W k-blocks issued (ring position)
      for (int it = 0; it < n; ++it) {
        const int item = blockIdx.x + it * gridDim.x;
        // the dU buffer is free: MMA 1 of item it - 1 has read it (SH: MMA 2 and the dA stores of item it - 1 too)
        if (it >= 1) mbar_wait(B_(SH ? BSR : BUE), (it - 1) & 1);
        mbar_expect_tx(B_(BUF), (uint32_t)(NCH * K1 * 128));
        for (int c = 0; c < NCH; ++c) {   // box 64 d x l tokens x spt samples -> K1 rows x 64 columns
          const uint32_t dst = sU + (uint32_t)(c * K1 * 128);
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
              "l"(&mp.du), "r"(64 * c), "r"(0), "r"(item * p.spt), "r"(B_(BUF))
              : "memory");
        }
        for (int kb = 0; kb < NCH; ++kb, ++wc) {   // W k-block kb: NCH boxes of 64 columns x 64 rows
          const int s = wc & 1;
          if (wc >= 2) mbar_wait(B_(BWE + s), ((wc >> 1) - 1) & 1);
          mbar_expect_tx(B_(BWF + s), (uint32_t)S::W);
          for (int c = 0; c < NCH; ++c) tma_load2d(sW + (uint32_t)(s * S::W + c * 8192), &mp.w, 64 * c, 64 * kb, B_(BWF + s));
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer
      // MMA 1: D1[128 x D] = W_u'[128 x K1] (K-major) dU[K1 x D] (MN-major, chunks of K1 rows x 64 columns)
      // MMA 2: D2[128 x D] = dA[128 x D] (K-major, 64-column chunks of 128 rows) W[D x D] (MN-major ring k-blocks)
      const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) | ((uint32_t)(D >> 3) << 17) |
                          ((uint32_t)(128 >> 4) << 24);
      mbar_wait(B_(BC), 0);
      int wc = 0;
      for (int it = 0; it < n; ++it) {
        const uint32_t ph = it & 1;
        mbar_wait(B_(BUF), ph);                              // dU landed
        if (it >= 1) mbar_wait(B_(BTF), (it - 1) & 1);      // item it - 1's epilogue read both accumulators
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kk = 0; kk < K1 / 16; ++kk) {
          const uint64_t ad = sdesc(sWu + (uint32_t)((kk >> 2) * 16384 + (kk & 3) * 32), 16, 1024);
          const uint64_t bd = sdesc(sU + (uint32_t)kk * 2048u, (uint32_t)(K1 * 128), 1024);
          mma_f16(tmem, ad, bd, id, kk > 0 ? 1u : 0u);
        }
        mma_commit(B_(BUE));
        mma_commit(B_(BD1));
        for (int kb = 0; kb < NCH; ++kb, ++wc) {   // k-block kb as soon as dA chunk kb is written (K in order)
          const int s = wc & 1;
          mbar_wait(B_(BDA + kb), ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          mbar_wait(B_(BWF + s), (wc >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const uint64_t ad = sdesc(sA + (uint32_t)(kb * 16384 + k4 * 32), 16, 1024);
            const uint64_t bd = sdesc(sW + (uint32_t)(s * S::W + k4 * 2048), 8192, 1024);
            mma_f16(tmem + (uint32_t)D, ad, bd, id, (kb > 0 || k4 > 0) ? 1u : 0u);
          }
          mma_commit(B_(BWE + s));                           // ring slot free once these MMAs complete
        }
        mma_commit(B_(BD2));
      }
    }
  } else {   // ---------------- epilogue warps 2-9
    // warp (q4, hh) owns rows 32 q4 .. and, in pass j, columns 64 j + 32 hh .. (chunk j's half hh): after pass j of
    // all eight warps dA chunk j is complete and MMA 2 runs its k-block j while the next passes are combined.  The
    // two warps of a quadrant share its 32-row slices of the dA tile (named barrier 1 + q4 before a slice is stored).
    const int q4 = warp & 3, hh = (warp - 2) >> 2;
    const uint32_t tq = tmem + ((uint32_t)(q4 * 32) << 16);
    auto colj = [&](int j) { return 64 * j + 32 * hh; };
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(1 + q4) : "memory"); };
    const uint32_t op = sOP + (uint32_t)((warp - 2) * S::OPW), opb = B_(BOP + warp - 2);
    const uint32_t swx = (uint32_t)((lane >> 1) & 3), sw8 = (uint32_t)(lane & 7);
    // the warp's slice of the dA tile for its 64-column chunk c: rows 32 q4.., a 32 x 64 bf16 box (128-B swizzle)
    auto slice = [&](int c) { return sA + (uint32_t)(c * 16384 + q4 * 4096); };
    const uint32_t base_bytes = p.rin_f32 ? 4096u : 2048u;
    auto issue = [&](int item, int j) {   // lane 0: operand boxes of (item, pass j)
      const int row0 = item * 128 + q4 * 32, col = colj(j);
      mbar_expect_tx(opb, 4096u + base_bytes);
      tma_load2d(op, &mp.x, col, row0, opb);
      tma_load2d(op + 2048u, &mp.a, col, row0, opb);
      tma_load2d(op + 4096u, &mp.rin, col, row0, opb);
    };
    float bs[NP];   // running column sums of dA: lane = column colj(j) + lane
#pragma unroll
    for (int j = 0; j < NP; ++j) bs[j] = 0.f;
    uint32_t oph = 0;
    if (lane == 0 && n > 0) issue(blockIdx.x, 0);
    for (int it = 0; it < n; ++it) {
      const int item = blockIdx.x + it * gridDim.x;
      const uint32_t ph = it & 1;
      mbar_wait(B_(BD1), ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) bulk_wait_read<0>();   // the previous item's dX stores have read the quadrant's dA slices
      __syncwarp();
      pair_sync();
      // ---- phase 1: dA = dT (.) X -> the dA tile; P = base + dT (.) A + dT -> MMA 1's TMEM columns
#pragma unroll 1
      for (int j = 0; j < NP; ++j) {
        uint32_t v[32];
        ld_tmem32(tq + colj(j), v);
        mbar_wait(opb, oph);
        oph ^= 1u;
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float pv[32];
        const int col = colj(j);
        const uint32_t drow = slice(col >> 6) + (uint32_t)(lane * 128);
#pragma unroll
        for (int g = 0; g < 4; ++g) {   // 8 columns at a time
          const uint32_t ox = op + (uint32_t)(lane * 64) + ((((uint32_t)g) ^ swx) << 4);
          float xv[8], av[8], bv[8];
          unpack_bf8(lds16_(ox), xv);
          unpack_bf8(lds16_(ox + 2048u), av);
          if (p.rin_f32) {
            const uint32_t rb = op + 4096u + (uint32_t)(lane * 128);
            const float4 b0 = lds4(rb + ((((uint32_t)(2 * g)) ^ sw8) << 4));
            const float4 b1 = lds4(rb + ((((uint32_t)(2 * g + 1)) ^ sw8) << 4));
            bv[0] = b0.x; bv[1] = b0.y; bv[2] = b0.z; bv[3] = b0.w; bv[4] = b1.x; bv[5] = b1.y; bv[6] = b1.z; bv[7] = b1.w;
          } else {
            unpack_bf8(lds16_(ox + 4096u), bv);
          }
          uint32_t da[4];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float t = __uint_as_float(v[8 * g + e]);
            pv[8 * g + e] = bv[e] + (t * av[e] + t);   // the first-writer / accumulator base + dT (.) A + dT
          }
#pragma unroll
          for (int e = 0; e < 4; ++e)
            da[e] = pack_bf2(__uint_as_float(v[8 * g + 2 * e]) * xv[2 * e], __uint_as_float(v[8 * g + 2 * e + 1]) * xv[2 * e + 1]);
          const uint32_t gg = (uint32_t)(((col & 63) >> 3) + g);   // 16-B granule within the 64-column chunk
          sts4u(drow + ((gg ^ sw8) << 4), da[0], da[1], da[2], da[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // dA chunk j visible to MMA 2
        __syncwarp();   // every lane has read the operand slot: refill it (next pass, or the next item's first)
        if (lane == 0) {
          arrive(B_(BDA + j));
          if (j + 1 < NP) issue(item, j + 1);
          else if (it + 1 < n) issue(item + gridDim.x, 0);
        }
        tmem_st32f(tq + colj(j), pv);   // P replaces dT in MMA 1's columns
      }
      __syncwarp();
      // the bias gradient: column sums of the STORED dA over this warp's rows (lane = column, rows in order)
      if (p.bsum) {
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          const int col = colj(j) + lane;
          const uint32_t sl = slice(col >> 6);
          const uint32_t cb = (uint32_t)((col & 63) >> 3), ce = (uint32_t)((col & 7) * 2);
          float s_ = 0.f;
#pragma unroll 8
          for (int rr = 0; rr < 32; ++rr) {
            unsigned short h_;
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h_) : "r"(sl + (uint32_t)(rr * 128) + ((cb ^ (uint32_t)(rr & 7)) << 4) + ce)
                         : "memory");
            s_ += __uint_as_float((uint32_t)h_ << 16);
          }
          bs[j] += s_;
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      pair_sync();   // both halves of every slice of the quadrant are written: the hh = 0 warp stores them
      if (hh == 0 && lane == 0) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) tma_store2d(&mp.da, slice(c), 64 * c, item * 128 + q4 * 32);
        bulk_commit();
      }
      // ---- phase 2: out = P + dA W, through the warp's dA slices (free once MMA 2 is done and dA is stored)
      mbar_wait(B_(BD2), ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        bulk_wait_read<0>();              // the dA stores have read the dA tile
        if (SH) arrive(B_(BSR));          // (SH: the next dU may land in it)
      }
      __syncwarp();
      pair_sync();
#pragma unroll 1
      for (int j = 0; j < NP; ++j) {
        uint32_t pv[32], w2[32];
        ld_tmem32(tq + colj(j), pv);
        ld_tmem32(tq + (uint32_t)D + colj(j), w2);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (j + 1 == NP) {   // both accumulators read: MMA 1 of the next item may start
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) arrive(B_(BTF));
        }
        float o[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = __uint_as_float(pv[e]) + __uint_as_float(w2[e]);
        const int col = colj(j);
        if (SH) {          // bf16, one 32 x 32 box per pass in the operand slot's spare 2 KB
          const uint32_t ob = op + 6144u;
          if (j > 0) {
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
          }
#pragma unroll
          for (int g = 0; g < 4; ++g)
            sts4u(ob + (uint32_t)(lane * 64) + ((((uint32_t)g) ^ swx) << 4), pack_bf2(o[8 * g], o[8 * g + 1]),
                  pack_bf2(o[8 * g + 2], o[8 * g + 3]), pack_bf2(o[8 * g + 4], o[8 * g + 5]), pack_bf2(o[8 * g + 6], o[8 * g + 7]));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store2d(&mp.out, ob, col, item * 128 + q4 * 32);
            bulk_commit();
          }
        } else if (p.out_f32) {   // one 32 x 32 fp32 box per pass, cycling through the warp's slices (chunks = hh mod 2)
          constexpr int NSL = NCH / 2;
          const uint32_t box = slice(2 * (j % NSL) + hh) + (uint32_t)(lane * 128);
          if (j >= NSL) {   // the store that last read this slice is done with it
            if (lane == 0) bulk_wait_read<NSL - 1>();
            __syncwarp();
          }
#pragma unroll
          for (int g = 0; g < 8; ++g) sts4(box + ((((uint32_t)g) ^ sw8) << 4), o[4 * g], o[4 * g + 1], o[4 * g + 2], o[4 * g + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store2d(&mp.out, slice(2 * (j % NSL) + hh), col, item * 128 + q4 * 32);
            bulk_commit();
          }
        } else {           // bf16: the quadrant's two warps fill chunk j's 32 x 64 slice, the hh = 0 warp stores it
          const uint32_t rowb = slice(col >> 6) + (uint32_t)(lane * 128);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const uint32_t gg = (uint32_t)(((col & 63) >> 3) + g);
            sts4u(rowb + ((gg ^ sw8) << 4), pack_bf2(o[8 * g], o[8 * g + 1]), pack_bf2(o[8 * g + 2], o[8 * g + 3]),
                  pack_bf2(o[8 * g + 4], o[8 * g + 5]), pack_bf2(o[8 * g + 6], o[8 * g + 7]));
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          pair_sync();
          if (hh == 0 && lane == 0) {
            tma_store2d(&mp.out, slice(j), 64 * j, item * 128 + q4 * 32);
            bulk_commit();
          }
        }
      }
    }
    if (lane == 0) bulk_wait_all();
    if (p.bsum) {   // this warp's partial column sums -> row (blockIdx * 4 + q4), columns colj(j) + lane
#pragma unroll
      for (int j = 0; j < NP; ++j) p.bsum[((int64_t)blockIdx.x * 4 + q4) * p.d + colj(j) + lane] = bs[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * D));
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn encode() {
  static EncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)f;
  }
  return fn;
}
// tensor map: `rank` dims (innermost first), strides in bytes of dims 1.., box
static bool mapn(CUtensorMap* mp, const void* ptr, bool f32, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                 const cuuint32_t* box, CUtensorMapSwizzle sw) {
  EncodeFn fn = encode();
  if (!fn || ((uintptr_t)ptr & 15)) return false;
  for (int i = 0; i < rank - 1; ++i)
    if (strides[i] % 16) return false;
  cuuint32_t e[3] = {1, 1, 1};
  return fn(mp, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr),
            dims, strides, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the form a shape takes: 0 none, 1 separate dU / dA tiles (K1 d 2 <= 16 KB), 2 shared tile (K1 <= 128; bf16 base
// and bf16 dX, the operand slot holding the dX box)
static int form(int B, int m, int l, int d, int64_t ldu, int rin_f32, int out_f32) {
  if (d != 128 && d != 256) return 0;
  if (m > 128 || 128 % m != 0) return 0;
  const int spt = 128 / m, K1 = spt * l;
  if (B % spt != 0 || K1 % 16 != 0 || l > 256 || ldu % 8 != 0) return 0;
  if (K1 * d * 2 <= 16384) return 1;
  return (K1 <= 128 && !rin_f32 && !out_f32) ? 2 : 0;
}
bool supported(int B, int m, int l, int d, int64_t ldu, int rin_f32, int out_f32) {
  return form(B, m, l, d, ldu, rin_f32, out_f32) != 0;
}

cudaError_t bwd(const void* Wu, const void* dU, int64_t ldu, const void* W, const void* X, const void* A, const void* rin,
                int rin_f32, void* out, int out_f32, void* dA, float* bsum, int B, int m, int l, int d, cudaStream_t st,
                int* rows_out) {
  const int fm = form(B, m, l, d, ldu, rin_f32, out_f32);
  if (!fm) return cudaErrorNotSupported;
  Params p;
  p.m = m; p.l = l; p.d = d; p.spt = 128 / m; p.K1 = p.spt * l; p.items = B / p.spt;
  p.rin_f32 = rin_f32; p.out_f32 = out_f32; p.bsum = bsum;
  const cuuint64_t R = (cuuint64_t)B * m;
  Maps mp;
  {   // W_u' = W_u [m][l] (spt = 1) or its block-diagonal form [128][spt l]: K-major A, one 64-column chunk
    cuuint64_t dims[2] = {(cuuint64_t)p.K1, 128};
    cuuint64_t str[1] = {(cuuint64_t)p.K1 * 2};
    cuuint32_t box[2] = {64, 128};   // (a second 64-column chunk for K1 > 64)
    if (!mapn(&mp.wu, Wu, false, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorNotSupported;
  }
  {   // dU [B][l][d] (sample stride ldu): box 64 columns x l tokens x spt samples = K1 rows
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)l, (cuuint64_t)B};
    cuuint64_t str[2] = {(cuuint64_t)d * 2, (cuuint64_t)ldu * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)l, (cuuint32_t)p.spt};
    if (!mapn(&mp.du, dU, false, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorNotSupported;
  }
  {   // W [d][d] row-major = MN-major B: boxes of 64 columns x 64 rows
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)d};
    cuuint64_t str[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, 64};
    if (!mapn(&mp.w, W, false, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorNotSupported;
  }
  {   // [B m][d] row-major tensors: operand boxes 32 x 32, store boxes 32 rows x 64 bf16 / 32 fp32
    cuuint64_t dims[2] = {(cuuint64_t)d, R};
    cuuint64_t s2[1] = {(cuuint64_t)d * 2}, s4[1] = {(cuuint64_t)d * 4};
    cuuint32_t b32[2] = {32, 32}, b64[2] = {64, 32};
    if (!mapn(&mp.x, X, false, 2, dims, s2, b32, CU_TENSOR_MAP_SWIZZLE_64B) ||
        !mapn(&mp.a, A, false, 2, dims, s2, b32, CU_TENSOR_MAP_SWIZZLE_64B) ||
        !mapn(&mp.rin, rin, rin_f32 != 0, 2, dims, rin_f32 ? s4 : s2, b32,
              rin_f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B) ||
        !mapn(&mp.da, dA, false, 2, dims, s2, b64, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !mapn(&mp.out, out, out_f32 != 0, 2, dims, out_f32 ? s4 : s2, (out_f32 || fm == 2) ? b32 : b64,
              fm == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorNotSupported;
  }
  static int sms = 0;
  if (!sms) { int dev = 0; cudaGetDevice(&dev); cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev); }
  const int grid = std::min(p.items, sms);
  *rows_out = bsum ? grid * 4 : 0;
  auto go = [&](auto kern, int bytes, int idx) -> cudaError_t {
    static int attr[4] = {0, 0, 0, 0};
    if (!attr[idx]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      attr[idx] = 1;
    }
    pdl_launch(kern, grid, 320, bytes, st, mp, p);
    ++g_launches;
    return cudaGetLastError();
  };
  static_assert(Smem<256, false>::BYTES <= 227 * 1024 && Smem<256, true>::BYTES <= 227 * 1024, "smem");
  if (fm == 1)
    return d == 128 ? go(dcn_bwd_kernel<128, false>, Smem<128, false>::BYTES, 0)
                    : go(dcn_bwd_kernel<256, false>, Smem<256, false>::BYTES, 1);
  return d == 128 ? go(dcn_bwd_kernel<128, true>, Smem<128, true>::BYTES, 2)
                  : go(dcn_bwd_kernel<256, true>, Smem<256, true>::BYTES, 3);
}

}  // namespace dcnb
}  // namespace dhen
