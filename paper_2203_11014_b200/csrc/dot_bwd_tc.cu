// dot_bwd_tc.cu — B5's last step, the Gram backward, with S built on chip:
//
//   dX_b (+)= S_b X_b,   S_b[i][j] = S_b[j][i] = dz_b[p(i, j)] (i < j),  S_b[i][i] = 0
//   p(i, j) = i m - i (i + 1) / 2 + (j - i - 1)        (Eq.(3); R7: strict upper triangle, row-major)
//
// The symmetric S is never stored: per item (one sample, or 128 / m samples stacked when m <= 64, so every MMA
// row carries data) the packed triangle(s) arrive with one cp.async.bulk (16 KB at m = 128), eight warps scatter
// them into the 128-B-swizzled K-major A tile in shared memory (block-diagonal when several samples share the
// tile), and one tcgen05.mma chain D[128 x d] = S[128 x R] X[R x d] runs with X's rows as the MN-major B operand
// (TMA, 64 x 64 boxes).  The epilogue leaves TMEM lane = row and writes the layer's dX contribution in one of the
// four forms the runtime's first / last dX-writer schedule needs (B3, B10):
//   ACC        acc (fp32) += S X                 (TMA reduce-add, 32 x 32 fp32 boxes)
//   FIRST      acc (fp32)  = dR (bf16) + S X     (TMA store)
//   EMIT       dX (bf16)   = acc (fp32) + S X    (TMA store, 32 x 64 bf16 boxes)
//   FIRST_EMIT dX (bf16)   = dR (bf16) + S X
// Per item the kernel moves the triangle and X in and the dX rows out: the step's algorithmic bytes (the dense
// [B, m, m] S of the unfused path, written and re-read, is gone).
//
// Warps: 0 producer (TMA / bulk copies), 1 MMA issuer (+ TMEM allocation), 2-9 build S and run the epilogue
// (warp w reads TMEM lanes 32 (w % 4) .., column half (w - 2) / 4).  Persistent CTAs, items strided.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "dot_bwd.h"
#include "gemm_tc_kernel.cuh"
#include "tuning.h"

namespace dhen {
namespace dotb {

using namespace tc;

constexpr int CH = 128 * 128;   // one 64-column (128-B) swizzled chunk of 128 rows: 16 KB

struct Params {
  int B, m, d, spt, R, items, mode;
  int64_t ldz;                  // elements between samples' triangles (>= h)
  const __nv_bfloat16* dZ;      // [B][ldz] packed triangles
  const void* rin;              // FIRST*: dR (bf16), EMIT: acc (fp32); row-major [B m][d]
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
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
__device__ __forceinline__ void tma_radd2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
}
__device__ __forceinline__ void arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}

// D[128 x N] = A[128 x K] B[K x N]: A K-major 128-B swizzled chunks of 64 K (CH bytes apart); B MN-major, per
// 64-row K block (N / 64) boxes of 64 N x 64 K (8 KB apart), K blocks kbs bytes apart.
__device__ __forceinline__ void mma_sx(uint32_t d, uint32_t a, uint32_t b, uint32_t kbs, uint32_t id, int ksteps) {
  for (int kk = 0; kk < ksteps; ++kk) {
    const uint64_t ad = sdesc(a + (uint32_t)((kk >> 2) * CH + (kk & 3) * 32), 16, 1024);
    const uint64_t bd = sdesc(b + (uint32_t)(kk >> 2) * kbs + (uint32_t)(kk & 3) * 2048u, 64 * 64 * 2, 1024);
    mma_f16(d, ad, bd, id, kk > 0 ? 1u : 0u);
  }
}

template <int D>
__global__ void __launch_bounds__(320, 1) gram_bwd_kernel(const __grid_constant__ CUtensorMap xmap,
                                                          const __grid_constant__ CUtensorMap omap,
                                                          const __grid_constant__ Params p) {
  pdl_release();
  constexpr int NCH = D / 64;                 // 64-column chunks of a row
  constexpr int XB = 2 * NCH * 8192;          // X tile: 2 K blocks (128 rows) x NCH boxes of 8 KB
  constexpr int ZB = 16384;                   // one staged triangle buffer
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sX = smem_u32(smem), sS = sX + XB, sZ = sS + 2 * CH, sO = sZ + 2 * ZB;   // sO: 8 warps x 2 x 4 KB
  uint64_t* bars = (uint64_t*)(smem + XB + 2 * CH + 2 * ZB + 8 * 2 * 4096);
  auto B_ = [&](int i) { return smem_u32(bars + i); };
  // 0 xfull, 1 xfree, 2,3 zfull[s], 4,5 zfree[s] (8), 6 s_ready (8), 7 sfree, 8,9 tfull[ab], 10,11 tempty[ab] (8)
  uint32_t* tslot = (uint32_t*)(bars + 12);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&omap) : "memory");
    for (int i = 0; i < 12; ++i) mbar_init(B_(i), (i == 4 || i == 5 || i == 6 || i == 10 || i == 11) ? 8 : 1);
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
  const int m = p.m, R = p.R, spt = p.spt;
  const int h = m * (m - 1) / 2;
  const int n = (int)blockIdx.x < p.items ? (p.items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const uint32_t zbytes = (uint32_t)(spt * h * 2);
  const int kblocks = (R + 63) / 64;

  if (warp == 0) {
    if (lane == 0) {   // ---------------- producer
      for (int it = 0; it < n; ++it) {
        const int item = blockIdx.x + it * gridDim.x, s = it & 1;
        if (it >= 2) mbar_wait(B_(4 + s), ((it >> 1) - 1) & 1);   // triangle buffer s read by the S builders
        mbar_expect_tx(B_(2 + s), zbytes);
        bulk_g2s(sZ + s * ZB, p.dZ + (int64_t)item * spt * p.ldz, zbytes, B_(2 + s));
        if (it >= 1) mbar_wait(B_(1), (it - 1) & 1);               // X of item it - 1 read by its MMAs
        mbar_expect_tx(B_(0), (uint32_t)(kblocks * NCH * 8192));
        for (int kb = 0; kb < kblocks; ++kb)
          for (int c = 0; c < NCH; ++c)
            tma_load2d(sX + (uint32_t)((kb * NCH + c) * 8192), &xmap, 64 * c, item * R + 64 * kb, B_(0));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer
      const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) | ((uint32_t)(D >> 3) << 17) |
                          ((uint32_t)(128 >> 4) << 24);
      const int ksteps = (R + 15) / 16;
      for (int it = 0; it < n; ++it) {
        const int ab = it & 1;
        mbar_wait(B_(6), it & 1);                                  // S built
        mbar_wait(B_(0), it & 1);                                  // X landed
        if (it >= 2) mbar_wait(B_(10 + ab), ((it >> 1) - 1) & 1);  // accumulator ab drained (item it - 2)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        mma_sx(tmem + (uint32_t)(ab * D), sS, sX, (uint32_t)(NCH * 8192), id, ksteps);
        mma_commit(B_(7));        // S free
        mma_commit(B_(1));        // X free
        mma_commit(B_(8 + ab));   // accumulator ready
      }
    }
  } else {   // ---------------- warps 2-9: S builders, then epilogue
    const int t = threadIdx.x - 64;   // 0..255
    const int q4 = warp & 3, hh = (warp - 2) >> 2;
    auto build = [&](int it) {
      const int s = it & 1;
      mbar_wait(B_(2 + s), (it >> 1) & 1);                    // triangle(s) landed
      if (it >= 1) mbar_wait(B_(7), (it - 1) & 1);            // previous S consumed by its MMAs
      const uint32_t zs = sZ + (uint32_t)(s * ZB);
      // thread t fills row r = t / 2, columns [c0, c0 + 64) of the 128 x 128 tile (8 granules of 8 bf16): only
      // the row's own diagonal block [sr m, sr m + m) is nonzero; i < j reads the packed row i contiguously,
      // i > j reads column i of the triangle (index j m - j (j + 1) / 2 + i - j - 1)
      const int r = t >> 1, c0 = (t & 1) * 64;
      int sr = 0, i = 0;
      if (r < R) { sr = r / m; i = r - sr * m; }
      const int kb0 = sr * m;
      const uint32_t zb = zs + (uint32_t)(sr * h * 2);
      const int up0 = i * m - i * (i + 1) / 2 - i - 1;   // p(i, j) = up0 + j for j > i
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = c0 + 8 * g + e - kb0;
          uint32_t v = 0u;
          if (r < R && j >= 0 && j < m && j != i && c0 + 8 * g + e < R) {
            const int idx = j > i ? up0 + j : j * m - j * (j + 1) / 2 + i - j - 1;
            v = lds_u16(zb + (uint32_t)(idx * 2));
          }
          w[e >> 1] |= v << (16 * (e & 1));
        }
        const int k0 = c0 + 8 * g;
        const uint32_t dst = sS + (uint32_t)((k0 >> 6) * CH + r * 128 + ((((k0 & 63) >> 3) ^ (r & 7)) << 4));
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy smem writes -> the MMA's reads
      __syncwarp();
      if (lane == 0) { arrive(B_(6)); arrive(B_(4 + s)); }
    };
    uint32_t tsel = 0;   // this warp's output box parity (alternating over all passes of all items)
    const uint32_t boxes = sO + (uint32_t)((warp - 2) * 2 * 4096);
    const int rbase = q4 * 32;
    if (n > 0) build(0);
    for (int it = 0; it < n; ++it) {
      const int item = blockIdx.x + it * gridDim.x, ab = it & 1;
      const bool rows_ok = rbase < R;
      const int64_t grow = (int64_t)item * R + rbase + lane;   // this lane's row of [B m][d]
      const bool out_bf16 = p.mode >= 2;
      constexpr int HC = D / 2;
      // the first NPRE columns' dR / accumulator row segment is loaded before the next item's S is built and
      // the accumulator is ready (its latency hides under both); every later 32-column piece loads its own
      constexpr int NPRE = D == 128 ? 64 : 32;
      float pre[NPRE];
      auto load_rin = [&](int col, float* f) {   // 32 columns of this lane's row of rin, as fp32
        if (p.mode == 2) {
          const float4* src = reinterpret_cast<const float4*>((const float*)p.rin + grow * p.d + col);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 x = __ldcg(src + q);
            f[4 * q] = x.x; f[4 * q + 1] = x.y; f[4 * q + 2] = x.z; f[4 * q + 3] = x.w;
          }
        } else {
          const uint4* src = reinterpret_cast<const uint4*>((const __nv_bfloat16*)p.rin + grow * p.d + col);
#pragma unroll
          for (int q = 0; q < 4; ++q) unpack_bf8(__ldg(src + q), f + 8 * q);
        }
      };
      if (p.mode != 0 && rows_ok) {
        load_rin(hh * HC, pre);
        if (NPRE == 64) load_rin(hh * HC + 32, pre + 32);
      }
      if (it + 1 < n) build(it + 1);
      mbar_wait(B_(8 + ab), (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tq = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * D + hh * (D / 2));
      uint32_t pk[32];   // the current box row, packed (32 fp32 values, or 64 bf16 as pairs)
#pragma unroll
      for (int q = 0; q < HC / 32; ++q) {   // 32-column chunks; a box row holds 1 (fp32) or 2 (bf16) chunks
        const int col = hh * HC + 32 * q;
        uint32_t v[32];
        ld_tmem32(tq + 32 * q, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (q == HC / 32 - 1) {   // accumulator read: hand it back
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) arrive(B_(10 + ab));
        }
        if (!rows_ok) continue;
        float* a = reinterpret_cast<float*>(v);
        if (p.mode != 0) {
          float f[32];
          if (32 * q < NPRE) {
#pragma unroll
            for (int e = 0; e < 32; ++e) f[e] = pre[(32 * q) % NPRE + e];
          } else {
            load_rin(col, f);
          }
#pragma unroll
          for (int e = 0; e < 32; ++e) a[e] += f[e];
        }
        if (out_bf16) {
#pragma unroll
          for (int e = 0; e < 16; ++e) pk[16 * (q & 1) + e] = pack_bf2(a[2 * e], a[2 * e + 1]);
          if ((q & 1) == 0) continue;   // the box row is complete after the odd chunk
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) pk[e] = v[e];
        }
        const int bcol = out_bf16 ? col - 32 : col;   // first column of this box
        const uint32_t box = boxes + (uint32_t)((tsel & 1) * 4096);
        ++tsel;
        if (lane == 0) bulk_wait_read<1>();   // the store that last read this box is done with it
        __syncwarp();
        const uint32_t rowa = box + (uint32_t)(lane * 128);
#pragma unroll
        for (int gq = 0; gq < 8; ++gq)
          sts4u(rowa + (uint32_t)(((gq ^ (lane & 7)) & 7) << 4), pk[4 * gq], pk[4 * gq + 1], pk[4 * gq + 2], pk[4 * gq + 3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const int row0 = item * R + rbase;
          if (p.mode == 0) tma_radd2d(&omap, box, bcol, row0);
          else tma_store2d(&omap, box, bcol, row0);
          bulk_commit();
        }
      }
    }
    if (lane == 0) bulk_wait_all();
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
static bool map2(CUtensorMap* mp, const void* ptr, bool f32, int cols, int64_t rows, int bc, int br) {
  EncodeFn fn = encode();
  const int es = f32 ? 4 : 2;
  if (!fn || ((uintptr_t)ptr & 15) || (cols * es) % 16) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * es};
  cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br}, e[2] = {1, 1};
  return fn(mp, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
            strides, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int samples_per_item(int m) { return (m <= 64 && 128 % m == 0) ? 128 / m : 1; }

bool supported(int B, int m, int d, int64_t ldz) {
  if (m < 2 || m > 128 || (d != 128 && d != 256)) return false;   // (TMEM: 2 d columns, a power of two)
  const int spt = samples_per_item(m), R = spt * m, h = m * (m - 1) / 2;
  return R % 32 == 0 && B % spt == 0 && ldz == h && (spt * h * 2) % 16 == 0 && spt * h * 2 <= 16384;
}

cudaError_t gram_bwd(const void* dZ, int64_t ldz, const void* X, int B, int m, int d, int mode, const void* rin, void* out,
                     cudaStream_t st) {
  if (!supported(B, m, d, ldz) || ((uintptr_t)dZ & 15) || mode < 0 || mode > 3) return cudaErrorNotSupported;
  Params p;
  p.B = B; p.m = m; p.d = d; p.spt = samples_per_item(m); p.R = p.spt * m; p.items = B / p.spt; p.mode = mode;
  p.ldz = ldz; p.dZ = (const __nv_bfloat16*)dZ; p.rin = rin;
  CUtensorMap xm, om;
  const bool of32 = mode < 2;
  if (!map2(&xm, X, false, d, (int64_t)B * m, 64, 64) || !map2(&om, out, of32, d, (int64_t)B * m, of32 ? 32 : 64, 32))
    return cudaErrorNotSupported;
  static int sms = 0;
  if (!sms) { int dev = 0; cudaGetDevice(&dev); cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev); }
  const int grid = std::min(p.items, sms);
  auto go = [&](auto kern, int D) -> cudaError_t {
    const int smem = 2 * (D / 64) * 8192 + 2 * CH + 2 * 16384 + 8 * 2 * 4096 + 12 * 8 + 16 + 1024;
    static int attr_set[5] = {0, 0, 0, 0, 0};   // (indexed by d / 64)
    if (!attr_set[D / 64]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr_set[D / 64] = 1;
    }
    pdl_launch(kern, grid, 320, smem, st, xm, om, p);
    ++g_launches;
    return cudaGetLastError();
  };
  return d == 128 ? go(gram_bwd_kernel<128>, 128) : go(gram_bwd_kernel<256>, 256);
}

}  // namespace dotb
}  // namespace dhen
