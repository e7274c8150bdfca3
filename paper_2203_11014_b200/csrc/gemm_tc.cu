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
  int zbase, nz;    // batch indices [zbase, zbase + nz) in this launch
  int lanes_rows;   // epilogue: consecutive lanes on consecutive rows (output column-contiguous)
  int fast;         // vectorised epilogue: 4 consecutive columns per lane (all views row-major, aligned)
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

__device__ __forceinline__ void ld4(const void* p, int64_t off, int dt, float* o) {
  if (dt == F32) {
    const float4 v = *reinterpret_cast<const float4*>(static_cast<const float*>(p) + off);
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  } else {
    const uint2 v = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(p) + off);
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&v.x);
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&v.y);
    const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
    o[0] = fa.x; o[1] = fa.y; o[2] = fb.x; o[3] = fb.y;
  }
}
__device__ __forceinline__ void st4(void* p, int64_t off, int dt, const float* v) {
  if (dt == F32) {
    *reinterpret_cast<float4*>(static_cast<float*>(p) + off) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p) + off) = u;
  }
}
// Per-row base offsets of every epilogue view (the column term is added per element).
struct RowBase {
  int64_t c, cross, aux, mask, resid;
};
__device__ __forceinline__ RowBase row_base(const Gemm& g, int z, int row) {
  RowBase rb;
  rb.c = g.c.off(z, row, 0);
  rb.cross = g.e.cross.ptr ? g.e.cross.off(z, row, 0) : 0;
  rb.aux = g.e.aux.ptr ? g.e.aux.off(z, row, 0) : 0;
  rb.mask = g.e.mask.ptr ? g.e.mask.off(z, row, 0) : 0;
  rb.resid = g.e.resid.ptr ? g.e.resid.off(z, row, 0) : 0;
  return rb;
}
__device__ __forceinline__ float bias_at(const Epilogue& e, int j) {
  if (!e.bias) return 0.f;
  if (e.bias_gap_hi > e.bias_gap_lo) {
    if (j >= e.bias_gap_lo && j < e.bias_gap_hi) return 0.f;
    if (j >= e.bias_gap_hi) j -= e.bias_gap_hi - e.bias_gap_lo;
  }
  return ld_as_f32(e.bias, j, e.bias_dt);
}
// The fused epilogue of one element given its row bases (same math as epi_apply).
__device__ __forceinline__ void epi_elem(const Gemm& g, const RowBase& rb, int col, float acc) {
  const Epilogue& e = g.e;
  float v = acc * e.alpha + bias_at(e, col);
  if (e.cross.ptr) {
    if (e.aux.ptr) st_from_f32(e.aux.ptr, rb.aux + col * e.aux.cs, e.aux.dt, v);
    const float x = ld_as_f32(e.cross.ptr, rb.cross + col * e.cross.cs, e.cross.dt);
    v = x * v + x;
  } else if (e.aux.ptr) {
    st_from_f32(e.aux.ptr, rb.aux + col * e.aux.cs, e.aux.dt, v);
  }
  if (e.relu) v = fmaxf(v, 0.f);
  if (e.mask.ptr) v = ld_as_f32(e.mask.ptr, rb.mask + col * e.mask.cs, e.mask.dt) > 0.f ? v : 0.f;
  if (e.resid.ptr) v += ld_as_f32(e.resid.ptr, rb.resid + col * e.resid.cs, e.resid.dt);
  const int64_t co = rb.c + col * g.c.cs;
  if (e.accumulate) v += ld_as_f32(g.c.ptr, co, g.c.dt);
  st_from_f32(g.c.ptr, co, g.c.dt, v);
}

// Vectorised epilogue of 4 consecutive columns [col, col + 4) of one row (all views cs == 1).
// Operands of a 4-column chunk are loaded first (epi4_load) for several rows, then combined and
// stored (epi4_store): keeps several independent global loads in flight per lane.
struct Chunk4 {
  float x[4], m[4], r[4], c[4];
};
__device__ __forceinline__ void epi4_load(const Gemm& g, const RowBase& rb, int col, Chunk4& k) {
  const Epilogue& e = g.e;
  if (e.cross.ptr) ld4(e.cross.ptr, rb.cross + col, e.cross.dt, k.x);
  if (e.mask.ptr) ld4(e.mask.ptr, rb.mask + col, e.mask.dt, k.m);
  if (e.resid.ptr) ld4(e.resid.ptr, rb.resid + col, e.resid.dt, k.r);
  if (e.accumulate) ld4(g.c.ptr, rb.c + col, g.c.dt, k.c);
}
__device__ __forceinline__ void epi4_store(const Gemm& g, const RowBase& rb, int col, float* a, const float* bias4,
                                           const Chunk4& k) {
  const Epilogue& e = g.e;
#pragma unroll
  for (int t = 0; t < 4; ++t) a[t] = a[t] * e.alpha + bias4[t];
  if (e.aux.ptr) st4(e.aux.ptr, rb.aux + col, e.aux.dt, a);
  if (e.cross.ptr) {
#pragma unroll
    for (int t = 0; t < 4; ++t) a[t] = k.x[t] * a[t] + k.x[t];
  }
  if (e.relu) {
#pragma unroll
    for (int t = 0; t < 4; ++t) a[t] = fmaxf(a[t], 0.f);
  }
  if (e.mask.ptr) {
#pragma unroll
    for (int t = 0; t < 4; ++t) a[t] = k.m[t] > 0.f ? a[t] : 0.f;
  }
  if (e.resid.ptr) {
#pragma unroll
    for (int t = 0; t < 4; ++t) a[t] += k.r[t];
  }
  if (e.accumulate) {
#pragma unroll
    for (int t = 0; t < 4; ++t) a[t] += k.c[t];
  }
  st4(g.c.ptr, rb.c + col, g.c.dt, a);
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

// Persistent, warp-specialised kernel: warp 0 = TMA producer, warp 1 = MMA issuer,
// warps 2-9 = epilogue.  Work items (tile, batch index, K split) are strided over
// the grid.  The TMEM accumulator is double-buffered (2 x BN columns) so the
// epilogue of item i overlaps the MMAs of item i+1 and the loads of item i+2.
template <int BN, int STAGES>
__global__ void __launch_bounds__(320, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   const __grid_constant__ Params p) {
  constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
  constexpr int SC = BN / 2 < 64 ? BN / 2 : 64;   // columns staged per epilogue pass
  constexpr int SROW = SC + 4;              // float4 rows; 16-B granules conflict-free both ways
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  float* stage_all = (float*)(sB + STAGES * B_BYTES);
  uint64_t* bars = (uint64_t*)(stage_all + 8 * 32 * SROW);   // full[S], empty[S], tfull[2], tempty[2]
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * STAGES + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = p.tiles_m * p.tiles_n;
  const int total = ntiles * p.nz * p.splits;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
    for (int s = 0; s < 2 * STAGES + 2; ++s) mbar_init(smem_u32(bars + s), 1);
    for (int s = 0; s < 2; ++s) mbar_init(smem_u32(tempty + s), 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  auto decode = [&](int item, int& m0, int& n0, int& z, int& sp, int& kb0, int& nk) {
    const int tile = item % ntiles;
    const int zs = item / ntiles;
    sp = zs % p.splits;
    z = p.zbase + zs / p.splits;
    m0 = (tile % p.tiles_m) * BM;
    n0 = (tile / p.tiles_m) * BN;
    kb0 = sp * p.kb_per_split;
    nk = min(p.kblocks, kb0 + p.kb_per_split) - kb0;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int it = 0;
      for (int item = blockIdx.x; item < total; item += gridDim.x) {
        int m0, n0, z, sp, kb0, nk;
        decode(item, m0, n0, z, sp, kb0, nk);
        for (int i = 0; i < nk; ++i, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(smem_u32(empty + s), ph ^ 1);
          const uint32_t fb = smem_u32(full + s);
          mbar_expect_tx(fb, A_BYTES + B_BYTES);
          const int k = (kb0 + i) * BK;
          load_operand<BM>(&tma_a, p.a, smem_u32(sA + s * A_BYTES), m0, k, z, fb);
          load_operand<BN>(&tma_b, p.b, smem_u32(sB + s * B_BYTES), n0, k, z, fb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (single thread)
      const uint32_t a_step = p.a.mn_major ? 16 * 128 : 32;   // bytes per K = 16 slice
      const uint32_t b_step = p.b.mn_major ? 16 * 128 : 32;
      const uint32_t a_lbo = p.a.mn_major ? 64 * BK * 2 : 16, b_lbo = p.b.mn_major ? 64 * BK * 2 : 16;
      int it = 0, li = 0;
      for (int item = blockIdx.x; item < total; item += gridDim.x, ++li) {
        int m0, n0, z, sp, kb0, nk;
        decode(item, m0, n0, z, sp, kb0, nk);
        const int ab = li & 1;
        const uint32_t aph = (li >> 1) & 1;
        mbar_wait(smem_u32(tempty + ab), aph ^ 1);      // epilogue drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t dacc = tmem + (uint32_t)(ab * BN);
        for (int i = 0; i < nk; ++i, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(smem_u32(full + s), ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t ab_ = smem_u32(sA + s * A_BYTES), bb_ = smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = sdesc(ab_ + kk * a_step, a_lbo, 1024);
            const uint64_t bd = sdesc(bb_ + kk * b_step, b_lbo, 1024);
            mma_f16(dacc, ad, bd, p.idesc, (i > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(smem_u32(empty + s));               // ring slot free once these MMAs complete
        }
        mma_commit(smem_u32(tfull + ab));                // accumulator ready for the epilogue
      }
    }
  } else {
    // ---------------- epilogue warps 2..9: warp w reads TMEM lanes [32 (w % 4), +32) (hardware rule)
    // and column half hh of the accumulator; 8 warps give the epilogue enough loads in flight.
    const int q4 = warp & 3;
    const int hh = (warp - 2) >> 2;
    constexpr int HC = BN / 2;                 // columns per warp
    float* stage = stage_all + (warp - 2) * 32 * SROW;
    const Gemm& g = p.g;
    int li = 0;
    for (int item = blockIdx.x; item < total; item += gridDim.x, ++li) {
      int m0, n0, z, sp, kb0, nk;
      decode(item, m0, n0, z, sp, kb0, nk);
      const int ab = li & 1;
      const uint32_t aph = (li >> 1) & 1;
      mbar_wait(smem_u32(tfull + ab), aph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int rbase = m0 + q4 * 32;
      if (p.lanes_rows) {
        // column-contiguous output: row per lane straight from TMEM; consecutive lanes = consecutive addresses
        const int row = rbase + lane;
        const bool rok = row < g.M;
        RowBase rb;
        if (rok) rb = row_base(g, z, row);
#pragma unroll 1
        for (int c0 = hh * HC; c0 < hh * HC + HC; c0 += 16) {
          uint32_t v[16];
          const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * BN + c0);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                "=r"(v[15])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c0 + 16 >= hh * HC + HC) {
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(tempty + ab)) : "memory");
          }
          if (rok && n0 + c0 < g.N) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int col = n0 + c0 + j;
              if (col < g.N) epi_elem(g, rb, col, __uint_as_float(v[j]));
            }
          }
        }
        continue;
      }
      // row-major output: park this warp's 32 x SC block in smem, then walk it with lanes on columns
#pragma unroll 1
      for (int pc = 0; pc < HC; pc += SC) {
#pragma unroll 1
      for (int c0 = 0; c0 < SC; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * BN + hh * HC + pc + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float4* dst = reinterpret_cast<float4*>(stage + lane * SROW + c0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dst[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]), __uint_as_float(v[4 * j + 2]),
                               __uint_as_float(v[4 * j + 3]));
      }
      if (pc + SC >= HC) {
        // accumulator fully read: hand it back to the MMA warp
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(tempty + ab)) : "memory");
      }
      __syncwarp();
      const int cbase = n0 + hh * HC + pc;
      if (p.fast) {
        constexpr int LPR = SC / 4;            // lanes per row (4 columns each)
        constexpr int RPP = 32 / LPR;          // rows per pass
        constexpr int U = 2;                   // passes whose loads are in flight together
        const int sub = lane / LPR, cl = lane % LPR;
        const int col = cbase + 4 * cl;
        float bias4[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) bias4[t] = (col + t < g.N) ? bias_at(g.e, col + t) : 0.f;
        const bool full4 = col + 3 < g.N;
#pragma unroll 1
        for (int r0 = 0; r0 < 32; r0 += RPP * U) {
          RowBase rb[U];
          Chunk4 k[U];
          bool ok[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int r = r0 + u * RPP + sub;
            const int row = rbase + r;
            ok[u] = (r < 32) && (row < g.M) && (col < g.N);
            if (ok[u]) {
              rb[u] = row_base(g, z, row);
              if (full4) epi4_load(g, rb[u], col, k[u]);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
            const int r = r0 + u * RPP + sub;
            const float4 a4 = *reinterpret_cast<const float4*>(stage + r * SROW + 4 * cl);
            float a[4] = {a4.x, a4.y, a4.z, a4.w};
            if (full4) {
              epi4_store(g, rb[u], col, a, bias4, k[u]);
            } else {
#pragma unroll
              for (int t = 0; t < 4; ++t)
                if (col + t < g.N) epi_elem(g, rb[u], col + t, a[t]);
            }
          }
        }
      } else {
#pragma unroll 1
        for (int r = 0; r < 32; ++r) {
          const int row = rbase + r;
          if (row >= g.M) break;
          RowBase rb;
          if (p.splits == 1) rb = row_base(g, z, row);
#pragma unroll
          for (int q = 0; q < SC / 32; ++q) {
            const int col = cbase + lane + 32 * q;
            if (col < g.N) {
              const float acc = stage[r * SROW + lane + 32 * q];
              if (p.splits == 1) epi_elem(g, rb, col, acc);
              else p.ws[((int64_t)(z * p.splits + sp) * g.M + row) * g.N + col] = acc;
            }
          }
        }
      }
      __syncwarp();
      }
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
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

// a view can take 4-wide vector accesses: column-contiguous rows, every row / batch offset a multiple of 4
// elements and a base aligned to 4 elements of its dtype
static bool vec_ok(const View& v) {
  if (!v.ptr) return true;
  const int es = v.dt == F32 ? 4 : 2;
  if (v.cs != 1) return false;
  if (((uintptr_t)v.ptr) % (4 * es)) return false;
  if (v.rs % 4 || v.bs0 % 4 || v.bs1 % 4 || v.rs_o % 4) return false;
  return true;
}

template <int BN, int STAGES>
static cudaError_t launch(const Params& p0, const CUtensorMap& ma, const CUtensorMap& mb, cudaStream_t st) {
  constexpr int SC = BN / 2 < 64 ? BN / 2 : 64;
  constexpr int SMEM = STAGES * (BM * BK * 2 + BN * BK * 2) + 8 * 32 * (SC + 4) * 4 + (2 * STAGES + 4) * 8 + 16 + 1024;
  static_assert(SMEM <= 227 * 1024, "smem");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  const int ntiles = p0.tiles_m * p0.tiles_n;
  const int zmax = std::max(1, (int)std::min<int64_t>(p0.g.batch, (int64_t)(1 << 30) / ((int64_t)ntiles * p0.splits)));
  for (int zb = 0; zb < p0.g.batch; zb += zmax) {
    Params p = p0;
    p.zbase = zb;
    p.nz = std::min(zmax, p0.g.batch - zb);
    const int64_t items = (int64_t)ntiles * p.nz * p.splits;
    const int grid = (int)std::min<int64_t>(items, 148);
    gemm_tc_kernel<BN, STAGES><<<grid, 320, SMEM, st>>>(ma, mb, p);
    ++g_launches;
  }
  return cudaGetLastError();
}

}  // namespace tc

cudaError_t gemm_tc(const Gemm& g, const Workspace& ws, cudaStream_t st) {
  using namespace tc;
  if (g.a.dt != BF16 || g.b.dt != BF16 || g.M <= 0 || g.N <= 0 || g.K <= 0 || g.batch <= 0) return cudaErrorNotSupported;
  if (g.N < 16) return cudaErrorNotSupported;
  const int BN = g.N <= 64 ? 64 : g.N <= 128 ? 128 : 256;
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
  if (tiles < 148 && p.kblocks >= 8) {   // few output tiles, long K: split K across CTAs
    splits = (int)std::min<int64_t>((2 * 148 + tiles - 1) / tiles, p.kblocks / 4);
    while (splits > 1 && (int64_t)splits * g.batch * g.M * g.N * 4 > (int64_t)ws.bytes) --splits;
  }
  p.kb_per_split = (p.kblocks + splits - 1) / splits;
  p.splits = (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;   // no empty splits
  p.ws = ws.ptr;
  p.zbase = 0;
  p.nz = g.batch;
  p.lanes_rows = (g.c.cs != 1 && g.c.rs == 1 && splits == 1) ? 1 : 0;
  p.fast = (!p.lanes_rows && splits == 1 && vec_ok(g.c) && vec_ok(g.e.cross) && vec_ok(g.e.aux) &&
            vec_ok(g.e.resid) && vec_ok(g.e.mask)) ? 1 : 0;
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)p.a.mn_major << 15) | ((uint32_t)p.b.mn_major << 16) |
            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  cudaError_t e = BN == 64 ? launch<64, 6>(p, ma, mb, st) : BN == 128 ? launch<128, 4>(p, ma, mb, st)
                                                      : launch<256, 3>(p, ma, mb, st);
  if (e != cudaSuccess) return e;
  if (p.splits > 1) return splitk_reduce(g, p.splits, ws.ptr, st);
  return cudaSuccess;
}

}  // namespace dhen
