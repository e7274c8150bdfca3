// gemm_tc.cu — bf16 GEMM on the 5th-generation tensor cores (sm_100a):
// TMA (cp.async.bulk.tensor, 128B swizzle) fills a multi-stage shared-memory
// ring guarded by mbarriers; one elected thread issues tcgen05.mma
// (kind::f16, M = 128, N = BN, K = 16 per instruction) accumulating in TMEM;
// tcgen05.commit releases ring slots and finally signals the epilogue; four
// warps read the fp32 accumulator back with tcgen05.ld and apply the fused
// epilogue (bias / DCN cross / ReLU / mask / residual / +=).
//
// Operands may be K-major or MN-major (transposed views of row-major tensors,
// so dgrad / wgrad need no transpose kernels), batched through up to two
// batch strides, and may have a two-level K (k -> (k / kdiv, k % kdiv)) so the
// token-mixing weight gradients reduce over (sample, dim) in one GEMM.  Long K
// with few output tiles is split across CTAs with a deterministic fixed-order
// second pass.
#include <cuda.h>

#include <algorithm>

#include "gemm.h"
#include "gemm_epi.cuh"

namespace dhen {
namespace tc {

constexpr int BM = 128, BK = 64;

struct OpMap {
  int mn_major;   // 1: MN contiguous (boxes of 64 MN x 64 K), 0: K contiguous (box 64 K x tile rows)
  int has_ko;     // coordinate slot 2 holds k / kdiv
  int kdiv;
  int mo;         // coordinate slot of row / mdiv (-1: single-level rows)
  int mdiv;
  int z1, z0;     // coordinate slots of z % zdiv and z / zdiv (-1: operand not batched there)
  int zdiv;
};

struct Params {
  Gemm g;
  OpMap a, b;
  int tiles_m, tiles_n;
  int kblocks, splits, kb_per_split;
  int zbase;
  int lanes_rows;   // epilogue: consecutive lanes on consecutive rows (output column-contiguous)
  float* ws;
  uint32_t idesc;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load5(uint32_t dst, const CUtensorMap* map, const int c[5], uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;   // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}

template <int TILE>
__device__ __forceinline__ void load_operand(const CUtensorMap* map, const OpMap& om, uint32_t dst, int mn0, int k,
                                             int z, uint32_t mbar) {
  int c[5] = {0, 0, 0, 0, 0};
  const int kin = om.has_ko ? k % om.kdiv : k;
  if (om.has_ko) c[2] = k / om.kdiv;
  if (om.mo >= 0) { c[om.mo] = mn0 / om.mdiv; mn0 = mn0 % om.mdiv; }
  if (om.z1 >= 0) c[om.z1] = z % om.zdiv;
  if (om.z0 >= 0) c[om.z0] = z / om.zdiv;
  if (!om.mn_major) {
    c[0] = kin;
    c[1] = mn0;
    tma_load5(dst, map, c, mbar);
  } else {
#pragma unroll
    for (int j = 0; j < TILE / 64; ++j) {
      c[0] = mn0 + 64 * j;
      c[1] = kin;
      tma_load5(dst + j * 64 * BK * 2, map, c, mbar);
    }
  }
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(128, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   const __grid_constant__ Params p) {
  constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* bars = (uint64_t*)(sB + STAGES * B_BYTES);   // full[STAGES], empty[STAGES], tfull
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * STAGES + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int tile = blockIdx.x;
  const int tm = tile % p.tiles_m, tn = tile / p.tiles_m;
  const int z = p.zbase + blockIdx.y / p.splits, sp = blockIdx.y % p.splits;
  const int m0 = tm * BM, n0 = tn * BN;
  const int kb0 = sp * p.kb_per_split;
  const int nk = min(p.kblocks, kb0 + p.kb_per_split) - kb0;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
    for (int s = 0; s < 2 * STAGES + 1; ++s) mbar_init(smem_u32(bars + s), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int i = 0; i < nk; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      mbar_wait(smem_u32(bars + STAGES + s), ph ^ 1);
      const uint32_t fb = smem_u32(bars + s);
      mbar_expect_tx(fb, A_BYTES + B_BYTES);
      const int k = (kb0 + i) * BK;
      load_operand<BM>(&tma_a, p.a, smem_u32(sA + s * A_BYTES), m0, k, z, fb);
      load_operand<BN>(&tma_b, p.b, smem_u32(sB + s * B_BYTES), n0, k, z, fb);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread)
    const uint32_t a_step = p.a.mn_major ? 16 * 128 : 32;   // bytes per K = 16 slice
    const uint32_t b_step = p.b.mn_major ? 16 * 128 : 32;
    const uint32_t a_lbo = p.a.mn_major ? 64 * BK * 2 : 16, b_lbo = p.b.mn_major ? 64 * BK * 2 : 16;
    for (int i = 0; i < nk; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      mbar_wait(smem_u32(bars + s), ph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ab = smem_u32(sA + s * A_BYTES), bb = smem_u32(sB + s * B_BYTES);
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk) {
        const uint64_t ad = sdesc(ab + kk * a_step, a_lbo, 1024);
        const uint64_t bd = sdesc(bb + kk * b_step, b_lbo, 1024);
        mma_f16(tmem, ad, bd, p.idesc, (i > 0 || kk > 0) ? 1u : 0u);
      }
      mma_commit(smem_u32(bars + STAGES + s));   // slot free once these MMAs complete
    }
    mma_commit(smem_u32(bars + 2 * STAGES));     // accumulator complete
  }
  __syncwarp();

  // ---------------- epilogue: TMEM -> registers -> smem (the idle ring) -> fused epilogue -> global.
  // Each warp owns TMEM lanes / tile rows [32w, 32w+32).  Pass 1 parks its rows in shared memory
  // (row stride BN+1: conflict-free both ways); pass 2 walks them with consecutive lanes on
  // consecutive memory (columns, or rows when the output is column-contiguous) so every global
  // access of the epilogue is coalesced.
  if (nk > 0) mbar_wait(smem_u32(bars + 2 * STAGES), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  constexpr int SROW = BN + 1;
  float* stage = reinterpret_cast<float*>(smem) + warp * 32 * SROW;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) stage[lane * SROW + c0 + j] = nk > 0 ? __uint_as_float(v[j]) : 0.f;
  }
  __syncwarp();
  const Gemm& g = p.g;
  const int rbase = m0 + warp * 32;
  if (!p.lanes_rows) {
#pragma unroll 1
    for (int r = 0; r < 32; ++r) {
      const int row = rbase + r;
      if (row >= g.M) break;
#pragma unroll
      for (int q = 0; q < BN / 32; ++q) {
        const int col = n0 + lane + 32 * q;
        if (col < g.N) {
          const float acc = stage[r * SROW + lane + 32 * q];
          if (p.splits == 1) epi_apply(g, z, row, col, acc);
          else p.ws[((int64_t)(z * p.splits + sp) * g.M + row) * g.N + col] = acc;
        }
      }
    }
  } else {
    const int row = rbase + lane;
    if (row < g.M) {
#pragma unroll 4
      for (int cc = 0; cc < BN; ++cc) {
        const int col = n0 + cc;
        if (col >= g.N) break;
        epi_apply(g, z, row, col, stage[lane * SROW + cc]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
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

// Build the TMA map of one operand (rows = M for A, N for B).  Returns false if
// the layout is not TMA-expressible (the GEMM then runs on the SIMT path).
static bool make_map(CUtensorMap* map, OpMap* om, const Operand& o, int rows, int K, int batch, int tile_rows) {
  const int64_t es = 2;
  const bool kmaj = (o.s_k == 1), mnmaj = (o.s_mn == 1);
  if (!kmaj && !mnmaj) return false;
  if (((uintptr_t)o.ptr & 15) != 0) return false;
  om->mn_major = kmaj ? 0 : 1;
  om->has_ko = o.kdiv ? 1 : 0;
  om->kdiv = o.kdiv ? o.kdiv : 1;
  om->zdiv = o.zdiv;
  om->z0 = om->z1 = om->mo = -1;
  om->mdiv = o.mdiv ? o.mdiv : 1;
  if (o.kdiv && (o.kdiv % BK != 0 || K % o.kdiv != 0)) return false;
  if (o.mdiv && (o.mdiv % tile_rows != 0 || rows % o.mdiv != 0)) return false;
  cuuint64_t dims[5] = {1, 1, 1, 1, 1}, strides[4] = {0, 0, 0, 0};
  cuuint32_t box[5] = {1, 1, 1, 1, 1}, estr[5] = {1, 1, 1, 1, 1};
  const int kin = o.kdiv ? o.kdiv : K;
  int64_t s1;
  const int rin = o.mdiv ? o.mdiv : rows;
  if (!om->mn_major) {
    dims[0] = kin; dims[1] = rin; s1 = o.s_mn;
    box[0] = BK; box[1] = tile_rows;
  } else {
    dims[0] = rin; dims[1] = kin; s1 = o.s_k;
    box[0] = 64; box[1] = BK;
  }
  strides[0] = s1 * es;
  int r = 2;
  if (o.kdiv) { dims[r] = K / o.kdiv; strides[r - 1] = o.s_ko * es; ++r; }
  if (o.mdiv) { dims[r] = rows / o.mdiv; strides[r - 1] = o.s_mo * es; om->mo = r; ++r; }
  if (o.zdiv > 1 && o.bs1 != 0) { dims[r] = o.zdiv; strides[r - 1] = o.bs1 * es; om->z1 = r; ++r; }
  const int nb0 = (batch + o.zdiv - 1) / o.zdiv;
  if (nb0 > 1 && o.bs0 != 0) {
    if (r >= 5) return false;
    dims[r] = nb0; strides[r - 1] = o.bs0 * es; om->z0 = r; ++r;
  }
  if (r > 5) return false;
  for (int i = 0; i < 4; ++i) {
    if (i + 1 >= r) strides[i] = (i == 0 ? 16 : strides[i - 1]) ;
    if (strides[i] % 16 != 0 || strides[i] == 0 || strides[i] >= (1ull << 40)) return false;
  }
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  CUresult res = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(o.ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS;
}

template <int BN, int STAGES>
static cudaError_t launch(const Params& p0, const CUtensorMap& ma, const CUtensorMap& mb, cudaStream_t st) {
  constexpr int SMEM = STAGES * (BM * BK * 2 + BN * BK * 2) + (2 * STAGES + 1) * 8 + 16 + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  const int ntiles = p0.tiles_m * p0.tiles_n;
  const int zmax = 65535 / p0.splits;
  for (int zb = 0; zb < p0.g.batch; zb += zmax) {
    Params p = p0;
    p.zbase = zb;
    const int nz = std::min(zmax, p0.g.batch - zb);
    gemm_tc_kernel<BN, STAGES><<<dim3(ntiles, nz * p.splits), 128, SMEM, st>>>(ma, mb, p);
    ++g_launches;
  }
  return cudaGetLastError();
}

}  // namespace tc

cudaError_t gemm_tc(const Gemm& g, const Workspace& ws, cudaStream_t st) {
  using namespace tc;
  if (g.a.dt != BF16 || g.b.dt != BF16 || g.M <= 0 || g.N <= 0 || g.K <= 0 || g.batch <= 0) return cudaErrorNotSupported;
  if (g.N < 16) return cudaErrorNotSupported;
  const int BN = g.N <= 64 ? 64 : 128;
  Params p;
  p.g = g;
  CUtensorMap ma, mb;
  if (!make_map(&ma, &p.a, g.a, g.M, g.K, g.batch, BM)) return cudaErrorNotSupported;
  if (!make_map(&mb, &p.b, g.b, g.N, g.K, g.batch, BN)) return cudaErrorNotSupported;
  p.tiles_m = (g.M + BM - 1) / BM;
  p.tiles_n = (g.N + BN - 1) / BN;
  p.kblocks = (g.K + BK - 1) / BK;
  const int64_t tiles = (int64_t)p.tiles_m * p.tiles_n * g.batch;
  int splits = 1;
  if (tiles < 148 && p.kblocks >= 8) {
    splits = (int)std::min<int64_t>((2 * 148 + tiles - 1) / tiles, p.kblocks / 4);
    while (splits > 1 && (int64_t)splits * g.batch * g.M * g.N * 4 > (int64_t)ws.bytes) --splits;
  }
  p.kb_per_split = (p.kblocks + splits - 1) / splits;
  p.splits = (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;   // no empty splits
  p.ws = ws.ptr;
  p.zbase = 0;
  p.lanes_rows = (g.c.cs != 1 && g.c.rs == 1 && splits == 1) ? 1 : 0;
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)p.a.mn_major << 15) | ((uint32_t)p.b.mn_major << 16) |
            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  cudaError_t e = BN == 64 ? launch<64, 4>(p, ma, mb, st) : launch<128, 3>(p, ma, mb, st);
  if (e != cudaSuccess) return e;
  if (p.splits > 1) return splitk_reduce(g, p.splits, ws.ptr, st);
  return cudaSuccess;
}

}  // namespace dhen
