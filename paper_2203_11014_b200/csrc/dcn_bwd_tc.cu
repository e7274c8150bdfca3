// dcn_bwd_tc.cu — B8, the DCN cross backward, as ONE kernel per 128-row tile (north-star reading R13 of Eq.(7),
// P:123-128):
//
//   forward   A = X W^T + b,   T = X (.) A + X,   U = W_u^T T
//   backward  dT = W_u dU   (MMA 1: K = l tokens)
//             dA = dT (.) X                          (bf16: the weight / bias gradients' operand, and MMA 2's A)
//             dX = [dR or acc] + dT (.) A + dT + dA W  (MMA 2: K = d)
//
// Round 1 ran this as two GEMMs with an fp32 [B, m, d] partial dX between them (written, then re-read: 2 GB of
// HBM traffic per C4 / C5 layer).  Here the partial P = base + dT (.) A + dT never leaves the SM: it is written
// back into MMA 1's TMEM columns, dA goes to shared memory as MMA 2's K-major A operand (and to HBM for the
// weight gradients), MMA 2 accumulates dA W into the other 256 TMEM columns, and the epilogue emits
// P + dA W once.  W (d x d, 128 KB at d = 256) and W_u (or its block-diagonal form when several samples share a
// tile) stay resident in shared memory for the whole launch; per item only dU arrives (TMA) and X, A, base are
// read by the epilogue warps.  Same arithmetic, same order as the two-GEMM path (bit-identical dX and dA).
// The bias gradient db = sum_rows dA is summed per warp (fixed xor tree, fixed item order) into one partial
// row per CTA quadrant; the runtime adds the partial rows in order.
//
// Warps: 0 producer (TMA), 1 MMA issuer (+ TMEM), 2-9 epilogue (warp w: TMEM lanes 32 (w % 4) .., column half
// (w - 2) / 4).  Persistent CTAs, one per SM, items strided.
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
  int64_t ldu;               // elements between samples of dU (its layer's m_out d)
  const __nv_bfloat16* X;    // [B m][d]
  const __nv_bfloat16* A;    // [B m][d] saved pre-cross A
  const void* rin;           // [B m][d]
  void* out;                 // [B m][d]
  __nv_bfloat16* dA;         // [B m][d]
  float* bsum;               // [grid * 4][d] partial column sums of the stored dA
};

__device__ __forceinline__ void tma_load2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tma_load3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void ld_tmem16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void st_tmem16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}
__device__ __forceinline__ void arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

template <int D>
__global__ void __launch_bounds__(320, 1) dcn_bwd_kernel(const __grid_constant__ CUtensorMap wumap,
                                                const __grid_constant__ CUtensorMap dumap,
                                                const __grid_constant__ CUtensorMap wmap,
                                                const __grid_constant__ Params p) {
  pdl_release();
  constexpr int NCH = D / 64;               // 64-column chunks of a row
  constexpr int WB = NCH * NCH * 8192;      // W: NCH K blocks x NCH boxes of 64 x 64
  constexpr int UB = 128 * D * 2;           // dU tile (<= 128 K rows x D) / dA tile (128 rows x D)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sW = smem_u32(smem), sWu = sW + WB, sU = sWu + 2 * 16384;   // W_u: up to 2 chunks of 64 K
  uint64_t* bars = (uint64_t*)(smem + WB + 2 * 16384 + UB);
  auto B_ = [&](int i) { return smem_u32(bars + i); };
  // 0 consts (W, W_u) landed, 1 ufull, 2 d1 (MMA 1 done: dU read), 3 a2 ready (8), 4 d2 (MMA 2 done: dA read),
  // 5 tmem free (8)
  uint32_t* tslot = (uint32_t*)(bars + 6);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&wumap) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&dumap) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&wmap) : "memory");
    for (int i = 0; i < 6; ++i) mbar_init(B_(i), (i == 3 || i == 5) ? 8 : 1);
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
  const int K1 = p.K1, kc1 = (K1 + 63) / 64;   // MMA 1's K and its 64-column chunks of W_u

  if (warp == 0) {
    if (lane == 0) {   // ---------------- producer
      mbar_expect_tx(B_(0), (uint32_t)(WB + kc1 * 16384));
      for (int kb = 0; kb < NCH; ++kb)
        for (int c = 0; c < NCH; ++c) tma_load2d(sW + (uint32_t)((kb * NCH + c) * 8192), &wmap, 64 * c, 64 * kb, B_(0));
      for (int c = 0; c < kc1; ++c) tma_load2d(sWu + (uint32_t)(c * 16384), &wumap, 64 * c, 0, B_(0));
      for (int it = 0; it < n; ++it) {
        const int item = blockIdx.x + it * gridDim.x;
        if (it >= 1) mbar_wait(B_(4), (it - 1) & 1);   // dA of item it - 1 (same bytes) read by its MMA 2
        mbar_expect_tx(B_(1), (uint32_t)(NCH * K1 * 128));
        for (int c = 0; c < NCH; ++c)   // box 64 d x l tokens x spt samples -> K1 rows x 64 columns
          tma_load3d(sU + (uint32_t)(c * K1 * 128), &dumap, 64 * c, 0, item * p.spt, B_(1));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer
      // MMA 1: D1[128 x D] = W_u'[128 x K1] (K-major) dU[K1 x D] (MN-major, chunks of K1 rows x 64 columns)
      // MMA 2: D2[128 x D] = dA[128 x D] (K-major, 64-column chunks of 128 rows) W[D x D] (MN-major)
      const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) | ((uint32_t)(D >> 3) << 17) |
                          ((uint32_t)(128 >> 4) << 24);
      mbar_wait(B_(0), 0);
      for (int it = 0; it < n; ++it) {
        const uint32_t ph = it & 1;
        mbar_wait(B_(1), ph);                        // dU landed
        if (it >= 1) mbar_wait(B_(5), (it - 1) & 1); // item it - 1's epilogue read both accumulators
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kk = 0; kk < K1 / 16; ++kk) {
          const uint64_t ad = sdesc(sWu + (uint32_t)((kk >> 2) * 16384 + (kk & 3) * 32), 16, 1024);
          const uint64_t bd = sdesc(sU + (uint32_t)kk * 2048u, (uint32_t)(K1 * 128), 1024);
          mma_f16(tmem, ad, bd, id, kk > 0 ? 1u : 0u);
        }
        mma_commit(B_(2));
        mbar_wait(B_(3), ph);                        // dA written into shared memory, P back in TMEM
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = sdesc(sU + (uint32_t)((kk >> 2) * 16384 + (kk & 3) * 32), 16, 1024);
          const uint64_t bd = sdesc(sW + (uint32_t)((kk >> 2) * NCH * 8192 + (kk & 3) * 2048), 8192, 1024);
          mma_f16(tmem + (uint32_t)D, ad, bd, id, kk > 0 ? 1u : 0u);
        }
        mma_commit(B_(4));
      }
    }
  } else {   // ---------------- epilogue warps 2-9
    const int q4 = warp & 3, hh = (warp - 2) >> 2;
    constexpr int HC = D / 2;
    const uint32_t tq = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(hh * HC);
    float bs[HC / 16];   // running column sums of dA: lane keeps column 16 q + (lane & 15) (lanes 16-31 duplicate)
#pragma unroll
    for (int q = 0; q < HC / 16; ++q) bs[q] = 0.f;
    for (int it = 0; it < n; ++it) {
      const int item = blockIdx.x + it * gridDim.x;
      const uint32_t ph = it & 1;
      const int64_t row = (int64_t)item * 128 + q4 * 32 + lane;   // R = spt m = 128 rows per item
      const int64_t ro = row * p.d;
      // X / A / base of 16-column piece q, raw (packed): issued one piece ahead of its use -- the first piece
      // before the MMA-1 wait -- so every epilogue warp keeps two pieces of loads in flight
      struct Pre { uint4 x[2], a[2], r[4]; };
      auto fetch = [&](int q, Pre& f) {
        const int col = hh * HC + 16 * q;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          f.x[g] = __ldg(reinterpret_cast<const uint4*>(p.X + ro + col) + g);
          f.a[g] = __ldg(reinterpret_cast<const uint4*>(p.A + ro + col) + g);
        }
        if (p.rin_f32) {
#pragma unroll
          for (int g = 0; g < 4; ++g) f.r[g] = __ldcg(reinterpret_cast<const uint4*>((const float*)p.rin + ro + col) + g);
        } else {
#pragma unroll
          for (int g = 0; g < 2; ++g) f.r[g] = __ldg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)p.rin + ro + col) + g);
        }
      };
      Pre pf[2];
      fetch(0, pf[0]);
      mbar_wait(B_(2), ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int q = 0; q < HC / 16; ++q) {   // 16-column pieces (register budget of a 320-thread CTA: 168)
        const int col = hh * HC + 16 * q;
        uint32_t v[16];
        ld_tmem16(tq + 16 * q, v);
        if (q + 1 < HC / 16) fetch(q + 1, pf[(q + 1) & 1]);
        const Pre& f = pf[q & 1];
        float xv[16], av[16], bv[16];
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          unpack_bf8(f.x[g], xv + 8 * g);
          unpack_bf8(f.a[g], av + 8 * g);
          if (!p.rin_f32) unpack_bf8(f.r[g], bv + 8 * g);
        }
        if (p.rin_f32) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            bv[4 * g] = __uint_as_float(f.r[g].x); bv[4 * g + 1] = __uint_as_float(f.r[g].y);
            bv[4 * g + 2] = __uint_as_float(f.r[g].z); bv[4 * g + 3] = __uint_as_float(f.r[g].w);
          }
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t da[8];
        float pv[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float t = __uint_as_float(v[e]);
          pv[e] = bv[e] + (t * av[e] + t);   // the first-writer / accumulator base + dT (.) A + dT
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) da[e] = pack_bf2(__uint_as_float(v[2 * e]) * xv[2 * e], __uint_as_float(v[2 * e + 1]) * xv[2 * e + 1]);
        // dA -> HBM (weight / bias gradients) and -> the K-major shared tile of MMA 2 (row = q4 * 32 + lane)
        uint4* dg = reinterpret_cast<uint4*>(p.dA + ro + col);
        dg[0] = make_uint4(da[0], da[1], da[2], da[3]);
        dg[1] = make_uint4(da[4], da[5], da[6], da[7]);
        const int r = q4 * 32 + lane;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const int gg = ((col & 63) >> 3) + g;   // 16-B granule within the 64-column chunk
          sts4u(sU + (uint32_t)((col >> 6) * 16384 + r * 128 + ((gg ^ (r & 7)) << 4)), da[4 * g], da[4 * g + 1],
                da[4 * g + 2], da[4 * g + 3]);
        }
        // the bias gradient: column sums of the STORED dA over this warp's 32 rows (fixed xor tree: lanes l and
        // l ^ 16 fold first, then within each half; lane keeps column lane & 15)
        float cs[16];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          cs[2 * e] = __uint_as_float(da[e] << 16);
          cs[2 * e + 1] = __uint_as_float(da[e] & 0xffff0000u);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int e = 0; e < 16; ++e) cs[e] += __shfl_xor_sync(0xffffffffu, cs[e], o);
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (e == (lane & 15)) bs[q] += cs[e];
        st_tmem16(tq + 16 * q, pv);   // P replaces dT in MMA 1's columns
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) arrive(B_(3));
      mbar_wait(B_(4), ph);   // MMA 2 done
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int q = 0; q < HC / 32; ++q) {
        const int col = hh * HC + 32 * q;
        uint32_t pv[32], w2[32];
        ld_tmem32(tq + 32 * q, pv);
        ld_tmem32(tq + (uint32_t)D + 32 * q, w2);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float o[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = __uint_as_float(pv[e]) + __uint_as_float(w2[e]);
        if (p.out_f32) {
          float4* dst = reinterpret_cast<float4*>((float*)p.out + ro + col);
#pragma unroll
          for (int g = 0; g < 8; ++g) dst[g] = make_float4(o[4 * g], o[4 * g + 1], o[4 * g + 2], o[4 * g + 3]);
        } else {
          uint4* dst = reinterpret_cast<uint4*>((__nv_bfloat16*)p.out + ro + col);
#pragma unroll
          for (int g = 0; g < 4; ++g)
            dst[g] = make_uint4(pack_bf2(o[8 * g], o[8 * g + 1]), pack_bf2(o[8 * g + 2], o[8 * g + 3]),
                                pack_bf2(o[8 * g + 4], o[8 * g + 5]), pack_bf2(o[8 * g + 6], o[8 * g + 7]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) arrive(B_(5));
    }
    if (p.bsum && lane < 16) {   // this warp's partial column sums -> row (blockIdx * 4 + q4), column hh HC + 16 q + lane
#pragma unroll
      for (int q = 0; q < HC / 16; ++q) p.bsum[((int64_t)blockIdx.x * 4 + q4) * p.d + hh * HC + 16 * q + lane] = bs[q];
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
// bf16 tensor map, 128-B swizzle: `rank` dims (innermost first), strides in bytes of dims 1.., box
static bool mapn(CUtensorMap* mp, const void* ptr, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                 const cuuint32_t* box) {
  EncodeFn fn = encode();
  if (!fn || ((uintptr_t)ptr & 15)) return false;
  for (int i = 0; i < rank - 1; ++i)
    if (strides[i] % 16) return false;
  cuuint32_t e[3] = {1, 1, 1};
  return fn(mp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims, strides, box, e,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool supported(int B, int m, int l, int d, int64_t ldu) {
  if (d != 128 && d != 256) return false;
  if (m > 128 || 128 % m != 0) return false;
  const int spt = 128 / m, K1 = spt * l;
  return B % spt == 0 && K1 % 16 == 0 && K1 <= 128 && l <= 256 && ldu % 8 == 0;
}

cudaError_t bwd(const void* Wu, const void* dU, int64_t ldu, const void* W, const void* X, const void* A, const void* rin,
                int rin_f32, void* out, int out_f32, void* dA, float* bsum, int B, int m, int l, int d, cudaStream_t st,
                int* rows_out) {
  if (!supported(B, m, l, d, ldu)) return cudaErrorNotSupported;
  Params p;
  p.m = m; p.l = l; p.d = d; p.spt = 128 / m; p.K1 = p.spt * l; p.items = B / p.spt;
  p.rin_f32 = rin_f32; p.out_f32 = out_f32; p.ldu = ldu;
  p.X = (const __nv_bfloat16*)X; p.A = (const __nv_bfloat16*)A; p.rin = rin; p.out = out;
  p.dA = (__nv_bfloat16*)dA; p.bsum = bsum;
  CUtensorMap wum, dum, wm;
  {   // W_u' = W_u [m][l] (spt = 1) or its block-diagonal form [128][spt l]: K-major A, chunks of 64 columns
    cuuint64_t dims[2] = {(cuuint64_t)p.K1, 128};
    cuuint64_t str[1] = {(cuuint64_t)p.K1 * 2};
    cuuint32_t box[2] = {64, 128};
    if (!mapn(&wum, Wu, 2, dims, str, box)) return cudaErrorNotSupported;
  }
  {   // dU [B][l][d] (sample stride ldu): box 64 columns x l tokens x spt samples = K1 rows
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)l, (cuuint64_t)B};
    cuuint64_t str[2] = {(cuuint64_t)d * 2, (cuuint64_t)ldu * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)l, (cuuint32_t)p.spt};
    if (!mapn(&dum, dU, 3, dims, str, box)) return cudaErrorNotSupported;
  }
  {   // W [d][d] row-major = MN-major B: boxes of 64 columns x 64 rows
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)d};
    cuuint64_t str[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, 64};
    if (!mapn(&wm, W, 2, dims, str, box)) return cudaErrorNotSupported;
  }
  static int sms = 0;
  if (!sms) { int dev = 0; cudaGetDevice(&dev); cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev); }
  const int grid = std::min(p.items, sms);
  *rows_out = bsum ? grid * 4 : 0;
  auto go = [&](auto kern, int D) -> cudaError_t {
    const int smem = (D / 64) * (D / 64) * 8192 + 2 * 16384 + 128 * D * 2 + 6 * 8 + 16 + 1024;
    static int attr[5] = {0, 0, 0, 0, 0};   // (indexed by d / 64)
    if (!attr[D / 64]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr[D / 64] = 1;
    }
    pdl_launch(kern, grid, 320, smem, st, wum, dum, wm, p);
    ++g_launches;
    return cudaGetLastError();
  };
  return d == 128 ? go(dcn_bwd_kernel<128>, 128) : go(dcn_bwd_kernel<256>, 256);
}

}  // namespace dcnb
}  // namespace dhen
