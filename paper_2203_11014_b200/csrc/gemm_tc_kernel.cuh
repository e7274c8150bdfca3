// gemm_tc_kernel.cuh — device side of the tcgen05 GEMM (see gemm_tc.cu for the host side and the
// design notes).  Included by gemm_tc.cu and by the three per-tile-width instantiation units.
#pragma once
// bf16 GEMM on the 5th-generation tensor cores (sm_100a):
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
#include <cstdlib>

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

// Compact, host-resolved epilogue plan: every present view shares one row geometry
// (offset = row term + batch term + col * cs), operands other than C are bf16.
enum { EF_ACC = 1, EF_RELU = 2, EF_MASK = 4, EF_CROSS = 8, EF_AUX = 16, EF_RESID = 32, EF_BIAS = 64,
       EF_DCNB = 128, EF_TRIU = 256, EF_LN = 512, EF_BITS = 1024, EF_BMASK = 2048,
       EF_R32 = 4096 /* the residual view is fp32 (the dX accumulator; its last writer emits bf16 dX) */ };
struct Lean {
  void* c;
  const void* x;
  void* aux;
  const void* mask;
  const void* resid;
  const void* bias;
  int64_t rs, rs_o, bs0, bs1, cs;
  int rdiv, zdiv;
  int c_f32, flags, gap_lo, gap_hi, hi_off;
  int triu_m;
  float alpha;
  const void* ln_gamma;
  const void* ln_beta;
  float* ln_mu;
  float* ln_rstd;
  float ln_eps;
  int ln_d;
  uint32_t* bits;     // ReLU bitmask, word-major [N / 32][bits_ld = M]: EF_BITS writes (value > 0), EF_BMASK masks
  int64_t bits_ld;
  float* bsum;        // EF_DCNB: per-CTA column sums of dA -> bsum[blockIdx][N] (N <= 256), or nullptr
  float* csum;        // TMA-store bf16 C: column sums of the stored C per 32-row block -> csum[row / 32][N]
};

// TMA maps of the epilogue outputs: c = C, d = the aux output (the LayerNorm epilogue's pre-norm sum R)
struct OutMaps {
  CUtensorMap c;
  CUtensorMap d;
  // DCN-backward operand epilogue (Params::dcnt): X, A, dR loaded and dA stored as 32 x 32 bf16 boxes (64-B
  // swizzle); dX (c) leaves as 32 x 32 fp32 boxes (128-B swizzle) through `c`
  CUtensorMap x, m, r, a;
};

struct Params {
  Gemm g;
  Lean ep;
  int lean;         // 1: use the lean epilogue plan
  int lean_id;      // >0: compile-time specialised pass (8 columns per lane / 16 per row-lane)
  OpMap a, b;
  int tiles_m, tiles_n;
  int n_fast;       // raster: N tiles fastest (tiles_n small) or M tiles fastest
  int kblocks, splits, kb_per_split;
  int zbase, nz;    // batch indices [zbase, zbase + nz) in this launch
  int lanes_rows;   // epilogue: consecutive lanes on consecutive rows (output column-contiguous)
  int fast;         // vectorised epilogue: 4 consecutive columns per lane (all views row-major, aligned)
  int fast8;        // 8 consecutive columns per lane (N % 8 == 0, 16-B aligned rows)
  float* ws;
  uint32_t idesc;
  int pair;           // 1: CTA pairs (cluster of 2) compute 256-row tiles with cta_group::2 MMAs
  long long* trace;   // debug: CTA 0 records clock64 timestamps (nullptr = off)
  int tstore;         // 1: TMA-store epilogue (row-major C, flags within TS_FLAGS; fp32 += is a TMA reduce-add)
  int lnst;           // LayerNorm epilogue with TMA: residual boxes in (tma_o.r), R (tma_o.d) and Y (tma_o.c) out
  int ln_rdiv;        // lnst: rows per group L of the 4-D maps {N, L, M / L, batch}
  int dcnt;           // DCN backward (EF_DCNB): operands staged by TMA into per-warp shared boxes, outputs TMA-stored
  int crosst;         // DCN cross forward (bias + cross + aux, bf16): X by TMA boxes, A and T TMA-stored
  int rst;            // fp32-residual epilogue (EF_RESID | EF_R32, bf16 C): residual by TMA boxes, C TMA-stored
  int pf_dist;        // > 0: the producer prefetches the operand tiles of the item pf_dist items ahead into L2
  int wr;             // W-resident instantiation (gemm_tc_kernel<.., WR = true>): the CTA's B tile stays in shared memory
};
// epilogue flags the TMA-store path implements (any subset; EF_ACC only with fp32 C, as cp.reduce .add)
constexpr int TS_FLAGS = EF_BIAS | EF_RELU | EF_ACC | EF_BITS | EF_BMASK;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
// phase wait (common.cuh: unbounded spin, or the watchdog build's bounded one reporting the call site)
#define mbar_wait(a, parity) mbar_wait_impl<false>((a), (parity), __FILE__, __LINE__)
__device__ __forceinline__ void tma_load5(uint32_t dst, const CUtensorMap* map, const int c[5], uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(mbar)
      : "memory");
}
// --- CTA-pair (cta_group::2) helpers: the pair shares one 256 x BN accumulator tile; each CTA holds
// 128 rows of A and BN / 2 rows of B in its own shared memory and 128 accumulator lanes in its own TMEM.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {   // same offset in CTA `rank` of the cluster
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load5_pair(uint32_t dst, const CUtensorMap* map, const int c[5], uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_pair(uint32_t mbar) {   // arrive on the barrier at this offset in both CTAs
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(mbar),
               "h"((uint16_t)3)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t a) {   // a: shared::cluster address (possibly the peer's)
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
#define mbar_wait_cluster(a, parity) mbar_wait_impl<true>((a), (parity), __FILE__, __LINE__)
__device__ __forceinline__ void tempty_arrive(uint32_t a, bool pair) {   // accumulator drained (rank 0 counts both CTAs)
  if (pair) mbar_arrive_cluster(mapa_u32(a, 0));
  else asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
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

__device__ __forceinline__ void tmem_st32f(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
// ---- TMA-store epilogue helpers
__device__ __forceinline__ void tma_store3(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(c2), "r"(src)
               : "memory");
}
__device__ __forceinline__ void tma_store4(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(c2), "r"(c3), "r"(src)
               : "memory");
}
__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tma_load4(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                          uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tma_reduce_add3(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2), "r"(src)
               : "memory");
}
// fp32 += of 4 consecutive elements in L2 (REDG.ADD.F32x4; subnormal addends flush to zero)
__device__ __forceinline__ void red_add4(float* p, const float* v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3])
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint4 lds16_(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts4u(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ void ld_tmem32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
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
    if (j >= e.bias_gap_hi) j = j - e.bias_gap_hi + e.bias_hi_off;
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

// ---- explicit-state-space memory helpers for the epilogue (no generic addressing)
__device__ __forceinline__ void sts4(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void unpack_bf4(const uint2 u, float* o) {
  o[0] = __uint_as_float(u.x << 16); o[1] = __uint_as_float(u.x & 0xffff0000u);
  o[2] = __uint_as_float(u.y << 16); o[3] = __uint_as_float(u.y & 0xffff0000u);
}
__device__ __forceinline__ void ldg_bf4(const void* base, int64_t off, float* o) {
  unpack_bf4(__ldg(reinterpret_cast<const uint2*>((const __nv_bfloat16*)base + off)), o);
}
__device__ __forceinline__ void ldg_c4(const void* base, int64_t off, int f32, float* o) {
  if (f32) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>((const float*)base + off));
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  } else {
    unpack_bf4(__ldcg(reinterpret_cast<const uint2*>((const __nv_bfloat16*)base + off)), o);
  }
}
__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void stg4(void* base, int64_t off, int f32, const float* v) {
  if (f32) {
    __stwb(reinterpret_cast<float4*>((float*)base + off), make_float4(v[0], v[1], v[2], v[3]));
  } else {
    uint2 u;
    u.x = pack_bf2(v[0], v[1]);
    u.y = pack_bf2(v[2], v[3]);
    __stwb(reinterpret_cast<uint2*>((__nv_bfloat16*)base + off), u);
  }
}
__device__ __forceinline__ float ldg_bf1(const void* base, int64_t off) {
  const unsigned short u = __ldg(reinterpret_cast<const unsigned short*>((const __nv_bfloat16*)base + off));
  return __uint_as_float(((uint32_t)u) << 16);
}
__device__ __forceinline__ float ldg_c1(const void* base, int64_t off, int f32) {
  if (f32) return __ldcg((const float*)base + off);
  const unsigned short u = __ldcg(reinterpret_cast<const unsigned short*>((const __nv_bfloat16*)base + off));
  return __uint_as_float(((uint32_t)u) << 16);
}
__device__ __forceinline__ void stg1(void* base, int64_t off, int f32, float v) {
  if (f32) {
    __stwb((float*)base + off, v);
  } else {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    __stwb(reinterpret_cast<unsigned short*>((__nv_bfloat16*)base + off), *reinterpret_cast<const unsigned short*>(&h));
  }
}
__device__ __forceinline__ int64_t lean_row(const Lean& e, int z, int row) {
  int64_t o;
  if (e.rdiv) {
    const unsigned q = (unsigned)row / (unsigned)e.rdiv;
    o = (int64_t)q * e.rs_o + (int64_t)((unsigned)row - q * (unsigned)e.rdiv) * e.rs;
  } else {
    o = (int64_t)row * e.rs;
  }
  if (e.zdiv == 1) {
    o += (int64_t)z * e.bs0;
  } else {
    const unsigned q = (unsigned)z / (unsigned)e.zdiv;
    o += (int64_t)q * e.bs0 + (int64_t)((unsigned)z - q * (unsigned)e.zdiv) * e.bs1;
  }
  return o;
}
__device__ __forceinline__ float lean_bias(const Lean& e, int j) {
  if (e.gap_hi > e.gap_lo) {
    if (j >= e.gap_lo && j < e.gap_hi) return 0.f;
    if (j >= e.gap_hi) j = j - e.gap_hi + e.hi_off;
  }
  return ldg_bf1(e.bias, j);
}
// one element of the lean epilogue
__device__ __forceinline__ void lean1(const Lean& e, int64_t o, float v, float bias) {
  const int f = e.flags;
  v = v * e.alpha + bias;
  if (f & EF_AUX) stg1(e.aux, o, 0, v);
  if (f & EF_CROSS) { const float x = ldg_bf1(e.x, o); v = x * v + x; }
  if (f & EF_RELU) v = fmaxf(v, 0.f);
  if (f & EF_MASK) v = ldg_bf1(e.mask, o) > 0.f ? v : 0.f;
  if (f & EF_RESID) v += ldg_bf1(e.resid, o);
  if (f & EF_ACC) v += ldg_c1(e.c, o, e.c_f32);
  stg1(e.c, o, e.c_f32, v);
}

// ---- compile-time specialised epilogue passes (one per (flags, C dtype) in use; see lean_variant())
// Global accesses through intrinsics (no asm volatile / memory clobbers) so the compiler can issue
// the loads of several rows ahead of earlier stores.
__device__ __forceinline__ void unpack_bf8(const uint4 u, float* o) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) { o[2 * t] = __uint_as_float(w[t] << 16); o[2 * t + 1] = __uint_as_float(w[t] & 0xffff0000u); }
}
__device__ __forceinline__ void ldg_bf8(const void* base, int64_t off, float* o) {
  unpack_bf8(__ldg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)base + off)), o);
}
template <bool CF32>
__device__ __forceinline__ void ldg_c8(const void* base, int64_t off, float* o) {
  if (CF32) {
    const float4* q = reinterpret_cast<const float4*>((const float*)base + off);
    const float4 a = __ldcg(q), b = __ldcg(q + 1);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
  } else {
    unpack_bf8(__ldcg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)base + off)), o);
  }
}
template <bool CF32>
__device__ __forceinline__ void stg8(void* base, int64_t off, const float* v) {
  if (CF32) {
    float4* q = reinterpret_cast<float4*>((float*)base + off);
    __stwb(q, make_float4(v[0], v[1], v[2], v[3]));
    __stwb(q + 1, make_float4(v[4], v[5], v[6], v[7]));
  } else {
    uint4 u;
    u.x = pack_bf2(v[0], v[1]); u.y = pack_bf2(v[2], v[3]); u.z = pack_bf2(v[4], v[5]); u.w = pack_bf2(v[6], v[7]);
    __stwb(reinterpret_cast<uint4*>((__nv_bfloat16*)base + off), u);
  }
}
__device__ __forceinline__ int64_t shfl64(int64_t v, int src) {
  const int lo = __shfl_sync(0xffffffffu, (int)(v & 0xffffffff), src);
  const int hi = __shfl_sync(0xffffffffu, (int)(v >> 32), src);
  return ((int64_t)hi << 32) | (uint32_t)lo;
}
// Row-major output, 8 consecutive columns per lane (N % 8 == 0, 16-B aligned rows).  Rows are handled
// in groups of G: first every extra operand of the group is loaded (all loads in flight together),
// then the group is combined and stored -- one memory latency per group instead of per row.
template <int F, bool CF32, int SC>
__device__ __forceinline__ void lean_pass8(const Lean& e, int z, int rbase, int M, int N, int cbase, uint32_t stage,
                                           int lane, uint32_t csw = 0u) {
  constexpr int LPR = SC / 8, RPP = 32 / LPR, SROW = SC + 4;
  constexpr int NR = 32 / RPP;                               // rows per lane in this pass
  // operands to prefetch per row: bf16 uint4 slots (X / A / mask / resid / bf16 C) and fp32 C
  constexpr int NB = ((F & (EF_CROSS | EF_DCNB)) ? 1 : 0) + ((F & (EF_MASK | EF_DCNB)) ? 1 : 0) +
                     (((F & EF_RESID) && !(F & EF_R32)) ? 1 : 0) + (((F & EF_ACC) && !CF32) ? 1 : 0);
  // fp32 operand per row: C itself (+=, fp32 C) or an fp32 residual (EF_R32); DCN backward adds with red.global
  constexpr bool F32C = ((F & EF_ACC) && CF32) || ((F & EF_R32) != 0);
  constexpr int REGS = NB * 4 + (F32C ? 8 : 0);               // registers per prefetched row
  constexpr int SLX = 0;                                                     // compile-time slot indices
  constexpr int SLM = SLX + ((F & (EF_CROSS | EF_DCNB)) ? 1 : 0);
  constexpr int SLR = SLM + ((F & (EF_MASK | EF_DCNB)) ? 1 : 0);
  constexpr int SLC = SLR + ((F & EF_RESID) ? 1 : 0);
  constexpr int G0 = REGS == 0 ? NR : (REGS <= 4 ? 8 : REGS <= 8 ? 4 : 2);
  constexpr int G = G0 < NR ? G0 : NR;                          // rows per load group
  const int sub = lane / LPR, cl = lane % LPR;
  const int col = cbase + 8 * cl;
  const bool cok = col < N;
  const int64_t my_off = (rbase + lane < M) ? lean_row(e, z, rbase + lane) : 0;   // row offset of row `lane`
  float bias8[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) bias8[t] = 0.f;
  if ((F & EF_BIAS) && cok) {
#pragma unroll
    for (int t = 0; t < 8; ++t) bias8[t] = lean_bias(e, col + t);
  }
  const float alpha = e.alpha;
  const bool alpha1 = alpha == 1.f;
  float dsum[(F & EF_DCNB) ? 8 : 1];   // EF_DCNB with csw: this lane's column sums of dA over its rows
#pragma unroll
  for (int t = 0; t < ((F & EF_DCNB) ? 8 : 1); ++t) dsum[t] = 0.f;
  // operand loads of row group q (rows sub + (q * G + k) * RPP) into register buffer `buf`; the loads of
  // group q + 1 are issued before group q is combined and stored (two groups in flight per lane)
  constexpr int NG = NR / G;
  int64_t o[2][G];
  bool ok[2][G];
  uint4 ub[2][G][NB > 0 ? NB : 1];
  float cv[2][G][F32C ? 8 : 1];
  auto prefetch = [&](int q, int buf) {
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const int r = sub + (q * G + k) * RPP;
      o[buf][k] = shfl64(my_off, r) + col;
      ok[buf][k] = cok && (rbase + r < M);
      if (ok[buf][k]) {
        if constexpr ((F & (EF_CROSS | EF_DCNB)) != 0)
          ub[buf][k][SLX] = __ldg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)e.x + o[buf][k]));
        if constexpr ((F & (EF_MASK | EF_DCNB)) != 0)
          ub[buf][k][SLM] = __ldg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)e.mask + o[buf][k]));
        if constexpr ((F & EF_RESID) != 0)
          ub[buf][k][SLR] = __ldg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)e.resid + o[buf][k]));
        if constexpr ((F & EF_ACC) != 0 && !CF32)
          ub[buf][k][SLC] = __ldcg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)e.c + o[buf][k]));
        if constexpr (F32C) ldg_c8<true>((F & EF_R32) ? e.resid : e.c, o[buf][k], cv[buf][k]);
      }
    }
  };
  // the 8 lanes of a quarter-warp read one staged row: lanes 4-7 take their two 16-B chunks in the
  // opposite order so each instruction touches 8 distinct bank groups (no 2-way conflict)
  const uint32_t sw = (uint32_t)((cl >> 2) & 1) << 4;
  prefetch(0, 0);
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    const int cb = q & 1;
    if (q + 1 < NG) prefetch(q + 1, cb ^ 1);
    float4 st0[G], st1[G];
#pragma unroll
    for (int k = 0; k < G; ++k) {   // staged accumulator rows of the group
      const int r = sub + (q * G + k) * RPP;
      const uint32_t sa = stage + (uint32_t)((r * SROW + 8 * cl) * 4);
      st0[k] = lds4(sa + sw);
      st1[k] = lds4(sa + (sw ^ 16u));
    }
#pragma unroll
    for (int k = 0; k < G; ++k) {
      if (!ok[cb][k]) continue;
      const int r = sub + (q * G + k) * RPP;
      const int64_t ok_ = o[cb][k];
      const float4 x0 = sw ? st1[k] : st0[k], x1 = sw ? st0[k] : st1[k];
      float a[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
      if (F & EF_TRIU) {
        // strict upper triangle of the per-sample Gram: pairs (i, j > i) row-major (R7)
        const int i = rbase + r, c0 = col;
        const int64_t zb = ok_ - col - (int64_t)i * e.rs;   // = z * bs0 (rs = 0 for this view)
        const int64_t base = zb + (int64_t)i * e.triu_m - (int64_t)i * (i + 1) / 2 - i - 1;
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (c0 + t > i) stg1(e.c, base + c0 + t, CF32, a[t] * alpha);
        continue;
      }
      if (F & EF_DCNB) {
        // B8 fused: dA = dT * X (bf16, aux), dX_acc += dT * A + dT  (dT = the fp32 accumulator)
        // (the fp32 dX accumulator is updated in L2 by vector reductions: one adder per element, fixed order)
        float xv[8], av[8], da[8], dx[8];
        unpack_bf8(ub[cb][k][SLX], xv);
        unpack_bf8(ub[cb][k][SLM], av);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float v = alpha1 ? a[t] : a[t] * alpha;
          da[t] = v * xv[t];
          dx[t] = v * av[t] + v;
        }
        uint4 dau;   // dA as stored (bf16 pairs); the bias gradient sums exactly these values, in row order
        dau.x = pack_bf2(da[0], da[1]); dau.y = pack_bf2(da[2], da[3]);
        dau.z = pack_bf2(da[4], da[5]); dau.w = pack_bf2(da[6], da[7]);
        __stwb(reinterpret_cast<uint4*>((__nv_bfloat16*)e.aux + ok_), dau);
        if constexpr ((F & EF_DCNB) != 0) {
          const uint32_t dw[4] = {dau.x, dau.y, dau.z, dau.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            dsum[2 * t] += __uint_as_float(dw[t] << 16);
            dsum[2 * t + 1] += __uint_as_float(dw[t] & 0xffff0000u);
          }
        }
        if constexpr ((F & EF_RESID) != 0) {
          // first writer of the dX accumulator: dX = dR (identity shortcut, B3) + dT A + dT, a plain store
          float rv8[8];
          unpack_bf8(ub[cb][k][SLR], rv8);
#pragma unroll
          for (int t = 0; t < 8; ++t) dx[t] += rv8[t];
          stg8<true>(e.c, ok_, dx);
        } else {
          red_add4((float*)e.c + ok_, dx);
          red_add4((float*)e.c + ok_ + 4, dx + 4);
        }
        continue;
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) a[t] = a[t] * alpha + bias8[t];
      float t8[8];
      if (F & EF_AUX) stg8<false>(e.aux, ok_, a);
      if constexpr ((F & EF_CROSS) != 0) {
        unpack_bf8(ub[cb][k][SLX], t8);
#pragma unroll
        for (int t = 0; t < 8; ++t) a[t] = t8[t] * a[t] + t8[t];
      }
      if (F & EF_RELU) {
#pragma unroll
        for (int t = 0; t < 8; ++t) a[t] = fmaxf(a[t], 0.f);
      }
      if constexpr ((F & EF_MASK) != 0) {
        unpack_bf8(ub[cb][k][SLM], t8);
#pragma unroll
        for (int t = 0; t < 8; ++t) a[t] = t8[t] > 0.f ? a[t] : 0.f;
      }
      if constexpr ((F & EF_RESID) != 0 && (F & EF_R32) != 0) {
#pragma unroll
        for (int t = 0; t < 8; ++t) a[t] += cv[cb][k][t];
      } else if constexpr ((F & EF_RESID) != 0) {
        unpack_bf8(ub[cb][k][SLR], t8);
#pragma unroll
        for (int t = 0; t < 8; ++t) a[t] += t8[t];
      }
      if (F & EF_ACC) {
        if (CF32) {
#pragma unroll
          for (int t = 0; t < 8; ++t) a[t] += cv[cb][k][t];
        } else {
          unpack_bf8(ub[cb][k][SLC], t8);
#pragma unroll
          for (int t = 0; t < 8; ++t) a[t] += t8[t];
        }
      }
      stg8<CF32>(e.c, ok_, a);
    }
  }
  if constexpr ((F & EF_DCNB) != 0) {
    if (csw) {   // fold the lanes of one column group (fixed xor tree), then one lane adds to the warp's row
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
        for (int t = 0; t < 8; ++t) dsum[t] += __shfl_xor_sync(0xffffffffu, dsum[t], o);
      if (sub == 0 && cok) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const uint32_t a_ = csw + (uint32_t)((col + t) * 4);
          float s_;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(s_) : "r"(a_) : "memory");
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(a_), "f"(s_ + dsum[t]) : "memory");
        }
      }
    }
  }
}
// Column-contiguous output (cs != 1, rs == 1): one row per lane, 16 accumulator columns in registers.
// Every operand of the 16 columns is loaded before the first store (the stores may alias C's loads, so
// the compiler could not hoist them itself): 16 x (operands) independent loads in flight per lane.
template <int F, bool CF32>
__device__ __forceinline__ void lean_rows16(const Lean& e, int64_t lo, int col0, int N, const uint32_t* v) {
  if constexpr ((F & EF_TRIU) != 0) return;   // host never selects the triangle in column-contiguous mode
  constexpr bool LX = (F & (EF_CROSS | EF_DCNB)) != 0, LM = (F & (EF_MASK | EF_DCNB)) != 0;
  constexpr bool LR = (F & EF_RESID) != 0, LC = (F & EF_ACC) != 0;
  constexpr bool C32 = CF32 || (F & EF_DCNB) != 0;
  const float alpha = e.alpha;
  float xs[16], ms[16], rv[16], cv[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int col = col0 + j;
    if (col < N) {
      const int64_t o = lo + (int64_t)col * e.cs;
      if constexpr (LX) xs[j] = ldg_bf1(e.x, o);
      if constexpr (LM) ms[j] = ldg_bf1(e.mask, o);
      if constexpr (LR) rv[j] = (F & EF_R32) ? ldg_c1(e.resid, o, 1) : ldg_bf1(e.resid, o);
      if constexpr (LC) cv[j] = ldg_c1(e.c, o, C32);
    }
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int col = col0 + j;
    if (col >= N) break;
    const int64_t o = lo + (int64_t)col * e.cs;
    float a = __uint_as_float(v[j]) * alpha;
    if constexpr ((F & EF_DCNB) != 0) {
      // B8 fused: dA = dT * X (bf16 aux), dX_acc += dT * A + dT
      stg1(e.aux, o, 0, a * xs[j]);
      if constexpr (LR) stg1(e.c, o, 1, rv[j] + a * ms[j] + a);   // first writer of dX
      else asm volatile("red.global.add.f32 [%0], %1;" ::"l"((float*)e.c + o), "f"(a * ms[j] + a) : "memory");
      continue;
    }
    if (F & EF_BIAS) a += lean_bias(e, col);
    if (F & EF_AUX) stg1(e.aux, o, 0, a);
    if constexpr ((F & EF_CROSS) != 0) a = xs[j] * a + xs[j];
    if (F & EF_RELU) a = fmaxf(a, 0.f);
    if constexpr ((F & EF_MASK) != 0) a = ms[j] > 0.f ? a : 0.f;
    if constexpr (LR) a += rv[j];
    if constexpr ((F & EF_ACC) != 0) a += cv[j];
    stg1(e.c, o, CF32, a);
  }
}
// The (flags, C dtype) combinations the DHEN step uses get a specialised loop; id 0 = none.
#define LEAN_VARIANTS(X)                          \
  X(1, 0, true)                                   \
  X(2, 0, false)                                  \
  X(3, EF_ACC, true)                              \
  X(4, EF_BIAS | EF_RELU, false)                  \
  X(5, EF_BIAS | EF_RESID, true)                  \
  X(6, EF_RESID, true)                            \
  X(7, EF_MASK, false)                            \
  X(8, EF_BIAS | EF_CROSS | EF_AUX, false)        \
  X(9, EF_BIAS, false)                            \
  X(10, EF_BIAS, true)                            \
  X(11, EF_ACC, false)                            \
  X(12, EF_DCNB, true)                            \
  X(13, EF_TRIU, false)                           \
  X(14, EF_TRIU, true)                            \
  X(15, EF_RELU, false)                           \
  X(16, EF_RESID, false)                          \
  X(17, EF_MASK, true)                            \
  X(18, EF_BIAS | EF_CROSS, false)                \
  X(19, EF_BIAS | EF_RESID | EF_AUX | EF_LN, false)      \
  X(20, EF_RESID | EF_AUX | EF_LN, false)               \
  X(21, EF_BIAS | EF_RELU | EF_BITS, false)              \
  X(22, EF_BMASK, false)                                 \
  X(23, EF_DCNB | EF_RESID, true)                       \
  X(24, EF_RESID | EF_R32, false)
static inline int lean_variant(int flags, bool cf32) {
#define LV_ID(id, f, c) if (flags == (f) && cf32 == (c)) return id;
  LEAN_VARIANTS(LV_ID)
#undef LV_ID
  return 0;
}
template <int V> struct VarF {   // variant id -> (flags, fp32 C)
  static constexpr int F = 0;
  static constexpr bool C = false;
};
#define LV_SPEC(i, f, c)                    \
  template <> struct VarF<i> {              \
    static constexpr int F = (f);           \
    static constexpr bool C = (c);          \
  };
LEAN_VARIANTS(LV_SPEC)
#undef LV_SPEC

// Per-item TMA coordinates of one operand: everything except the K position is fixed for the
// item (computed once, with the divisions); the k-loop only advances (kin, ko) by additions.
struct OpCoords {
  int mn;          // inner-row coordinate of the tile start (row % mdiv when two-level)
  int c2, c3, c4;  // slots 2..4 with the K-independent parts filled in (ko added to slot 2 per k-block)
};
__device__ __forceinline__ OpCoords op_coords(const OpMap& om, int mn0, int z) {
  int c[5] = {0, 0, 0, 0, 0};
  if (om.mo >= 0) { c[om.mo] = mn0 / om.mdiv; mn0 = mn0 % om.mdiv; }
  if (om.z1 >= 0) c[om.z1] = z % om.zdiv;
  if (om.z0 >= 0) c[om.z0] = z / om.zdiv;
  OpCoords r;
  r.mn = mn0; r.c2 = c[2]; r.c3 = c[3]; r.c4 = c[4];
  return r;
}
__device__ __forceinline__ void load_tile(const CUtensorMap* map, bool mn_major, const OpCoords& q, int kin, int ko,
                                          uint32_t dst, uint32_t mbar, int chunks, bool pair) {
  int c[5];
  c[2] = q.c2 + ko; c[3] = q.c3; c[4] = q.c4;
  if (!mn_major) {
    c[0] = kin; c[1] = q.mn;
    if (pair) tma_load5_pair(dst, map, c, mbar); else tma_load5(dst, map, c, mbar);
  } else {
    for (int j = 0; j < chunks; ++j) {   // 64-column boxes (MN-major, 128B swizzle)
      c[0] = q.mn + 64 * j; c[1] = kin;
      if (pair) tma_load5_pair(dst + j * 64 * BK * 2, map, c, mbar); else tma_load5(dst + j * 64 * BK * 2, map, c, mbar);
    }
  }
}

// L2 prefetch of one operand's k-block tile (the same boxes load_tile fetches; no shared memory, no barrier)
__device__ __forceinline__ void prefetch_tile(const CUtensorMap* map, bool mn_major, const OpCoords& q, int kin, int ko,
                                              int chunks) {
  int c[5];
  c[2] = q.c2 + ko; c[3] = q.c3; c[4] = q.c4;
  for (int j = 0; j < (mn_major ? chunks : 1); ++j) {
    if (!mn_major) { c[0] = kin; c[1] = q.mn; }
    else { c[0] = q.mn + 64 * j; c[1] = kin; }
    asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(map), "r"(c[0]),
                 "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
                 : "memory");
  }
}

// Persistent, warp-specialised kernel: warp 0 = TMA producer, warp 1 = MMA issuer,
// warps 2-9 = epilogue.  Work items (tile, batch index, K split) are strided over
// the grid.  The TMEM accumulator is double-buffered (2 x BN columns) so the
// epilogue of item i overlaps the MMAs of item i+1 and the loads of item i+2.
template <int BN> struct EpiSmem {
  static constexpr int SC = BN / 2 < 64 ? BN / 2 : 64;   // columns staged per epilogue pass
  static constexpr int SROW = SC + 4;                     // float4 rows; 16-B granules conflict-free both ways
  static constexpr int STAGE = 8 * 32 * SROW * 4;         // fp32 staging of the 8 epilogue warps
  static constexpr int TBOX = 8 * 2 * 4096;               // TMA-store boxes: 2 x (32 rows x 128 B) per warp
  static constexpr int BYTES = STAGE > TBOX ? STAGE : TBOX;
  static constexpr int SBIAS = 2 * BN > 512 ? 2 * BN : 512;   // floats: [2][BN] bias, or the LN (mean, M2) exchange
};

// DCN-backward operand epilogue (Params::dcnt): per epilogue warp two 6-KB operand slots (X | A | dR boxes of
// 32 rows x 32 bf16) and one 4-KB fp32 dX box, in place of the fp32 staging area
constexpr int DCNT_WARP_BYTES = 16384;
// LayerNorm epilogue with TMA (Params::lnst): per warp the residual / R boxes (HC / 64 boxes of 32 rows x 64
// bf16, 128-B swizzle) and one Y box
template <int BN> constexpr int lnt_warp_bytes() { return (BN / 2) * 64; }   // (Y overwrites R in the same boxes)
static_assert(EpiSmem<128>::BYTES >= 8 * 8192, "the cross epilogue's per-warp boxes fit the staging area (BN >= 128)");
template <int BN, int VAR, bool PAIR>
constexpr int epi_bytes() {
  return ((VarF<VAR>::F & EF_DCNB) != 0 && EpiSmem<BN>::BYTES < 8 * DCNT_WARP_BYTES) ? 8 * DCNT_WARP_BYTES
         : ((VarF<VAR>::F & EF_LN) != 0 && !PAIR && EpiSmem<BN>::BYTES < 8 * lnt_warp_bytes<BN>())
             ? 8 * lnt_warp_bytes<BN>()
             : EpiSmem<BN>::BYTES;
}
// operand-ring depth of an instantiation: the DCN-backward dT GEMM (K = l, one k-block) takes one slot, the
// single-CTA LayerNorm GEMMs at BN = 256 two (their epilogue boxes need the rest of shared memory)
template <int BN, int STAGES, int VAR, bool PAIR>
constexpr int eff_stages() {
  return (VarF<VAR>::F & EF_DCNB) != 0 ? 1 : STAGES;
}
// per-warp TMA-arrival barriers of the operand epilogues (DCN backward: 2 slots; LayerNorm: 1)
template <int VAR> constexpr bool has_opbar() {
  return (VarF<VAR>::F & (EF_DCNB | EF_LN | EF_CROSS)) != 0 || (VarF<VAR>::F == (EF_RESID | EF_R32) && !VarF<VAR>::C);
}

// W-resident short-K GEMMs (Params::wr): a CTA keeps the whole K x BN tile of B (the weight, K <= 256) in shared
// memory for all its items -- with N tiles fastest and a grid that is a multiple of tiles_n, every item of a CTA
// has the same N tile -- and the ring streams only A.  Per 128 x 256 tile the CTA then reads 64 KB instead of
// 192 KB through L2 (these GEMMs sit at the L2 throughput cap).  TMA-store epilogues only, with one
// store box per warp (the resident tile takes the second box's shared memory), and the bias row of the CTA's one N
// tile staged once.
constexpr int WR_KB = 4;   // resident B k-blocks (K <= 4 BK = 256)
// A-ring slots: single CTA 4; a CTA pair holds half the B tile each, so 8 (128 KB of A in flight a CTA)
template <bool PAIR> constexpr int wr_na() { return PAIR ? 8 : 4; }
template <int BN, int VAR> constexpr bool wr_ok() {
  return BN == 256 && VAR > 0 && (VarF<VAR>::F & ~TS_FLAGS) == 0 && !VarF<VAR>::C && (VarF<VAR>::F & EF_ACC) == 0;
}
template <int BN, bool PAIR> constexpr int wr_smem() {
  return wr_na<PAIR>() * BM * BK * 2 + WR_KB * (PAIR ? BN * BK : BN * BK * 2) + 8 * 4096 + BN * 4 +
         (2 * wr_na<PAIR>() + 6) * 8 + 16 + 1024;   // bias: 1 tile
}

template <int BN, int STAGES, bool PAIR>
constexpr int ring_stages() {
  return PAIR ? (STAGES * (BM * BK * 2 + BN * BK * 2)) / (BM * BK * 2 + BN * BK) : STAGES;
}

template <int BN, int STAGES, int VAR, bool PAIR, bool WR = false>
__global__ void __launch_bounds__(320, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   const __grid_constant__ OutMaps tma_o, const __grid_constant__ Params p) {
  pdl_release();
  constexpr int A_BYTES = BM * BK * 2;
  // B bytes per ring slot in this CTA (a pair CTA loads BN / 2 rows), and the ring depth the same shared
  // memory holds: a pair kernel gets the deeper ring (BN = 256: 4 slots instead of 3)
  constexpr int B_BYTES = PAIR ? BN * BK : BN * BK * 2;
  constexpr int NST = WR ? wr_na<PAIR>() : ring_stages<BN, STAGES, PAIR>();
  static_assert(!WR || wr_ok<BN, VAR>(), "W-resident: TMA-store variants");
  constexpr int SC = EpiSmem<BN>::SC;
  constexpr int SROW = EpiSmem<BN>::SROW;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + NST * A_BYTES;   // WR: the resident B tile (WR_KB k-blocks), else the ring's B slots
  float* stage_all = (float*)(sB + (WR ? WR_KB : NST) * B_BYTES);   // fp32 staging, or the TMA-store boxes (1024-B aligned)
  float* sbias = (float*)((uint8_t*)stage_all + (WR ? 8 * 4096 : epi_bytes<BN, VAR, PAIR>()));   // [2][BN] bias of the current tiles
  uint64_t* bars = (uint64_t*)(sbias + (WR ? BN : EpiSmem<BN>::SBIAS));   // full[S], empty[S], tfull[2], tempty[2]
  uint64_t* full = bars;
  uint64_t* empty = bars + NST;
  uint64_t* tfull = bars + 2 * NST;
  uint64_t* tempty = bars + 2 * NST + 2;
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * NST + 4);
  uint64_t* wfull = bars + 2 * NST + 5;   // WR: the resident B tile has landed
  // DCN-backward variants: [8 epilogue warps][256 columns] fp32 column sums of dA (Lean::bsum)
  constexpr bool BSV = VAR > 0 && (VarF<VAR>::F & EF_DCNB) != 0;
  float* csum = (float*)(bars + 2 * NST + 6);
  // [8 epilogue warps][2 slots] TMA-arrival barriers of the operand epilogues (after the DCN column sums)
  uint64_t* opbar = (uint64_t*)(csum + (BSV ? 8 * 256 : 0));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = p.tiles_m * p.tiles_n;
  const int total = ntiles * p.nz * p.splits;
  // CTA-pair mode: both CTAs of a cluster walk the same items (256-row tiles); rank 0 issues the MMAs
  constexpr bool pair = PAIR;   // separate instantiation: cta_group::2 code requires a cluster launch
  const uint32_t crank = pair ? cluster_rank() : 0u;
  const int wid = pair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int nwk = pair ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int BMP = pair ? 2 * BM : BM;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
    for (int s = 0; s < 2 * NST + 2; ++s) mbar_init(smem_u32(bars + s), 1);
    for (int s = 0; s < 2; ++s) mbar_init(smem_u32(tempty + s), pair ? 16 : 8);   // epilogue warps of both CTAs
    if constexpr (WR) mbar_init(smem_u32(wfull), 1);
    if constexpr (VAR > 0 && has_opbar<VAR>())
      for (int s = 0; s < 16; ++s) mbar_init(smem_u32(opbar + s), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (pair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(2 * BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(2 * BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if constexpr (BSV) {
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) csum[i] = 0.f;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (pair) cluster_sync_all();   // the peer's barriers are initialised before any remote arrive / TMA
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  pdl_wait();   // prerequisites complete (barrier init / TMEM alloc above overlapped the previous kernel's tail)

  auto decode = [&](int item, int& m0, int& n0, int& z, int& sp, int& kb0, int& nk) {
    const int tile = item % ntiles;
    const int zs = item / ntiles;
    sp = zs % p.splits;
    z = p.zbase + zs / p.splits;
    if (p.n_fast) {   // tall-skinny: the N tiles of one M row-block run together (A read once from DRAM)
      m0 = (tile / p.tiles_n) * BMP;
      n0 = (tile % p.tiles_n) * BN;
    } else {
      m0 = (tile % p.tiles_m) * BMP;
      n0 = (tile / p.tiles_m) * BN;
    }
    kb0 = sp * p.kb_per_split;
    nk = min(p.kblocks, kb0 + p.kb_per_split) - kb0;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int it = 0;
      // short K: the operand tiles of the item pf_dist items ahead are requested into L2 now, so the ring's loads
      // of that item hit L2 instead of waiting out a DRAM round trip with only NST k-blocks in flight
      auto l2_prefetch = [&](int pitem) {
        int m0, n0, z, sp, kb0, nk;
        decode(pitem, m0, n0, z, sp, kb0, nk);
        const OpCoords qa = op_coords(p.a, m0 + (int)crank * BM, z), qb = op_coords(p.b, n0 + (int)crank * (BN / 2), z);
        int ka = p.a.has_ko ? (kb0 * BK) % p.a.kdiv : kb0 * BK, koa = p.a.has_ko ? (kb0 * BK) / p.a.kdiv : 0;
        int kbk = p.b.has_ko ? (kb0 * BK) % p.b.kdiv : kb0 * BK, kob = p.b.has_ko ? (kb0 * BK) / p.b.kdiv : 0;
        const int kda = p.a.has_ko ? p.a.kdiv : 0x7fffffff, kdb = p.b.has_ko ? p.b.kdiv : 0x7fffffff;
        for (int i = 0; i < nk; ++i) {
          prefetch_tile(&tma_a, p.a.mn_major != 0, qa, ka, koa, BM / 64);
          if (!WR) prefetch_tile(&tma_b, p.b.mn_major != 0, qb, kbk, kob, pair ? BN / 128 : BN / 64);   // (WR: resident)
          ka += BK; while (ka >= kda) { ka -= kda; ++koa; }
          kbk += BK; while (kbk >= kdb) { kbk -= kdb; ++kob; }
        }
      };
      if constexpr (WR) {   // the CTA's B tile, once (every item of this CTA has the same N tile and all of K)
        if (wid < total) {
          int m0, n0, z, sp, kb0, nk;
          decode(wid, m0, n0, z, sp, kb0, nk);
          const OpCoords qb = op_coords(p.b, n0 + (int)crank * (BN / 2), z);   // (a pair CTA: its half of B)
          int kbk = p.b.has_ko ? (kb0 * BK) % p.b.kdiv : kb0 * BK, kob = p.b.has_ko ? (kb0 * BK) / p.b.kdiv : 0;
          const int kdb = p.b.has_ko ? p.b.kdiv : 0x7fffffff;
          uint32_t wb = smem_u32(wfull);
          if (!pair) {
            mbar_expect_tx(wb, (uint32_t)(nk * B_BYTES));
          } else {   // both CTAs' halves land on rank 0's barrier
            if (crank == 0) mbar_expect_tx(wb, (uint32_t)(2 * nk * B_BYTES));
            wb = mapa_u32(wb, 0);
          }
          for (int i = 0; i < nk; ++i) {
            load_tile(&tma_b, p.b.mn_major != 0, qb, kbk, kob, smem_u32(sB) + i * B_BYTES, wb, pair ? BN / 128 : BN / 64, pair);
            kbk += BK; while (kbk >= kdb) { kbk -= kdb; ++kob; }
          }
        }
      }
      const bool pf = p.pf_dist > 0 && p.kb_per_split <= 8;
      if (pf)
        for (int d = 1; d < p.pf_dist; ++d)
          if (wid + d * nwk < total) l2_prefetch(wid + d * nwk);
      for (int item = wid; item < total; item += nwk) {
        if (pf && item + p.pf_dist * nwk < total) l2_prefetch(item + p.pf_dist * nwk);
        int m0, n0, z, sp, kb0, nk;
        decode(item, m0, n0, z, sp, kb0, nk);
        const OpCoords qa = op_coords(p.a, m0 + (int)crank * BM, z), qb = op_coords(p.b, n0 + (int)crank * (BN / 2), z);
        // K position: (kin, ko) per operand; both operands share k, but each has its own kdiv
        const int k0 = kb0 * BK;
        int ka = p.a.has_ko ? k0 % p.a.kdiv : k0, koa = p.a.has_ko ? k0 / p.a.kdiv : 0;
        int kbk = p.b.has_ko ? k0 % p.b.kdiv : k0, kob = p.b.has_ko ? k0 / p.b.kdiv : 0;
        const int kda = p.a.has_ko ? p.a.kdiv : 0x7fffffff, kdb = p.b.has_ko ? p.b.kdiv : 0x7fffffff;
        const bool amn = p.a.mn_major != 0, bmn = p.b.mn_major != 0;
        uint32_t s = (uint32_t)(it % NST), ph = (uint32_t)((it / NST) & 1);
        for (int i = 0; i < nk; ++i, ++it) {
          mbar_wait(smem_u32(empty + s), ph ^ 1);
          if (p.trace && blockIdx.x == 0 && it < 64) p.trace[it] = clock64();
          uint32_t fb = smem_u32(full + s);
          if (WR && !pair) {
            mbar_expect_tx(fb, A_BYTES);
          } else if (WR) {
            if (crank == 0) mbar_expect_tx(fb, 2 * A_BYTES);
            fb = mapa_u32(fb, 0);
          } else if (!pair) {
            mbar_expect_tx(fb, A_BYTES + B_BYTES);
          } else {
            if (crank == 0) mbar_expect_tx(fb, 2 * (A_BYTES + B_BYTES));   // both CTAs' halves land on rank 0's barrier
            fb = mapa_u32(fb, 0);
          }
          load_tile(&tma_a, amn, qa, ka, koa, smem_u32(sA) + s * A_BYTES, fb, BM / 64, pair);
          if (!WR) load_tile(&tma_b, bmn, qb, kbk, kob, smem_u32(sB) + s * B_BYTES, fb, pair ? BN / 128 : BN / 64, pair);
          ka += BK; while (ka >= kda) { ka -= kda; ++koa; }     // kdiv < BK: several outer indices per k-block
          kbk += BK; while (kbk >= kdb) { kbk -= kdb; ++kob; }
          if (++s == NST) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {
      // ---------------- MMA issuer (single thread)
      const uint32_t a_step = p.a.mn_major ? 16 * 128 : 32;   // bytes per K = 16 slice
      const uint32_t b_step = p.b.mn_major ? 16 * 128 : 32;
      const uint32_t a_lbo = p.a.mn_major ? 64 * BK * 2 : 16, b_lbo = p.b.mn_major ? 64 * BK * 2 : 16;
      int it = 0, li = 0;
      if constexpr (WR) {
        mbar_wait(smem_u32(wfull), 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
      for (int item = wid; item < total; item += nwk, ++li) {
        int m0, n0, z, sp, kb0, nk;
        decode(item, m0, n0, z, sp, kb0, nk);
        const int ab = li & 1;
        const uint32_t aph = (li >> 1) & 1;
        if (pair) mbar_wait_cluster(smem_u32(tempty + ab), aph ^ 1);   // both CTAs' epilogues drained it
        else mbar_wait(smem_u32(tempty + ab), aph ^ 1);      // epilogue drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (p.trace && blockIdx.x == 0 && li < 64) p.trace[64 + li] = clock64();
        const uint32_t dacc = tmem + (uint32_t)(ab * BN);
        for (int i = 0; i < nk; ++i, ++it) {
          const int s = it % NST;
          const uint32_t ph = (it / NST) & 1;
          mbar_wait(smem_u32(full + s), ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (p.trace && blockIdx.x == 0 && it < 64) p.trace[128 + it] = clock64();
          const uint32_t ab_ = smem_u32(sA + s * A_BYTES), bb_ = smem_u32(sB + (WR ? i : s) * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = sdesc(ab_ + kk * a_step, a_lbo, 1024);
            const uint64_t bd = sdesc(bb_ + kk * b_step, b_lbo, 1024);
            if (pair) mma_f16_pair(dacc, ad, bd, p.idesc, (i > 0 || kk > 0) ? 1u : 0u);
            else mma_f16(dacc, ad, bd, p.idesc, (i > 0 || kk > 0) ? 1u : 0u);
          }
          // ring slot free once these MMAs complete
          if (pair) mma_commit_pair(smem_u32(empty + s)); else mma_commit(smem_u32(empty + s));
        }
        // accumulator ready for the epilogue
        if (pair) mma_commit_pair(smem_u32(tfull + ab)); else mma_commit(smem_u32(tfull + ab));
      }
    }
  } else {
    // ---------------- epilogue warps 2..9: warp w reads TMEM lanes [32 (w % 4), +32) (hardware rule)
    // and column half hh of the accumulator; 8 warps keep enough stores / loads in flight.
    const int q4 = warp & 3;
    const int hh = (warp - 2) >> 2;
    constexpr int HC = BN / 2;                 // columns per warp
    const uint32_t stage = smem_u32(stage_all) + (uint32_t)((warp - 2) * 32 * SROW * 4);
    const Gemm& g = p.g;
    const Lean& e = p.ep;
    uint32_t tsel = 0;   // TMA-store box parity of this warp (running over all passes of all tiles)
    int li = 0;
    // DCN-backward operand epilogue (BSV && p.dcnt).  Per warp and 32-column pass: X, A (and the first writer's
    // dR) arrive as 32 x 32 bf16 boxes by TMA into one of two operand slots -- the next pass's boxes are in
    // flight while this pass is combined, with no registers held for them -- lane = row combines them with the
    // accumulator row from TMEM, dA = bf16(dT X) overwrites X in its box, dX = dT A + dT (+ dR) goes to an fp32
    // box, and both leave by TMA store (dX +=: TMA reduce-add).  The dA column sums are read down the stored box.
    constexpr int NPD = BSV ? HC / 32 : 1;   // 32-column passes per warp and tile
    uint32_t gpass = 0;                      // running pass count of this warp: operand slot gpass & 1
    float dsum_t[NPD];
#pragma unroll
    for (int j = 0; j < NPD; ++j) dsum_t[j] = 0.f;
    // per-warp operand boxes: 16 KB (DCN backward: two 6-KB slots + the dX box) or 8 KB (cross: two 4-KB slots)
    const uint32_t opw = smem_u32(stage_all) + (uint32_t)((warp - 2) * (BSV ? DCNT_WARP_BYTES : 8192));
    const uint32_t obar = smem_u32(opbar) + (uint32_t)((warp - 2) * 16);
    auto op_issue = [&](int item_, int j_, uint32_t slot_) {   // lane 0: the operand boxes of (item_, pass j_)
      int m0_, n0_, z_, sp_, kb0_, nk_;
      decode(item_, m0_, n0_, z_, sp_, kb0_, nk_);
      const int r_ = m0_ + q4 * 32, c_ = n0_ + hh * HC + 32 * j_;
      const uint32_t dst = opw + slot_ * 6144u, b = obar + slot_ * 8u;
      constexpr bool FR = (VarF<VAR>::F & EF_RESID) != 0;
      mbar_expect_tx(b, FR ? 3 * 2048 : 2 * 2048);
      tma_load3(dst, &tma_o.x, c_, r_, z_, b);
      tma_load3(dst + 2048, &tma_o.m, c_, r_, z_, b);
      if (FR) tma_load3(dst + 4096, &tma_o.r, c_, r_, z_, b);
    };
    if (BSV && p.dcnt && lane == 0 && wid < total) op_issue(wid, 0, 0u);
    // DCN cross forward with TMA (XTV && p.crosst): per warp and 32-column pass the X box (32 x 32 bf16) arrives
    // into one of two 4-KB slots -- the next pass's flies while this one is combined -- A = alpha acc + b goes to
    // the slot's second box, T = X (.) A + X overwrites X in place, and both leave by TMA store
    constexpr bool XTV = VAR > 0 && VarF<VAR>::F == (EF_BIAS | EF_CROSS | EF_AUX) && !VarF<VAR>::C;
    auto xt_issue = [&](int item_, int j_, uint32_t slot_) {   // lane 0: the X box of (item_, pass j_)
      int m0_, n0_, z_, sp_, kb0_, nk_;
      decode(item_, m0_, n0_, z_, sp_, kb0_, nk_);
      const uint32_t b = obar + slot_ * 8u;
      mbar_expect_tx(b, 2048u);
      tma_load3(opw + slot_ * 4096u, &tma_o.x, n0_ + hh * HC + 32 * j_, m0_ + q4 * 32, z_, b);
    };
    if (XTV && p.crosst && lane == 0 && wid < total) xt_issue(wid, 0, 0u);
    // fp32-residual epilogue with TMA (RTV && p.rst; the first writer of a token-map dgrad, C = alpha acc + dR):
    // per warp and 32-column pass the fp32 residual box (32 rows x 128 B) arrives into one of two 4-KB slots --
    // the next pass's flies while this one is combined -- lane = row reads its 32 values, then writes the bf16
    // result into the slot's first 2 KB as a 64-B-swizzled 32 x 32 box, which leaves by TMA store
    constexpr bool RTV = VAR > 0 && VarF<VAR>::F == (EF_RESID | EF_R32) && !VarF<VAR>::C;
    auto rt_issue = [&](int item_, int j_, uint32_t slot_) {   // lane 0: the residual box of (item_, pass j_)
      int m0_, n0_, z_, sp_, kb0_, nk_;
      decode(item_, m0_, n0_, z_, sp_, kb0_, nk_);
      const uint32_t b = obar + slot_ * 8u;
      mbar_expect_tx(b, 4096u);
      tma_load3(opw + slot_ * 4096u, &tma_o.r, n0_ + hh * HC + 32 * j_, m0_ + q4 * 32, z_, b);
    };
    if (RTV && p.rst && lane == 0 && wid < total) rt_issue(wid, 0, 0u);
    // LayerNorm epilogue with TMA (LNV && p.lnst): the warp's 32 x HC residual block arrives by TMA into its
    // boxes, R = acc + bias + resid overwrites it in place and leaves by TMA store, then Y overwrites R (once the R
    // stores have read it) and leaves the same way; the next tile's residual is requested as soon as the Y stores
    // have read the boxes, so it lands while the warp waits for the next accumulator.  8 KB a warp fit the staging
    // area, so the operand ring keeps its depth and CTA pairs take it too.
    constexpr bool LNT = VAR > 0 && (VarF<VAR>::F & EF_LN) != 0;
    const uint32_t lnw = smem_u32(stage_all) + (uint32_t)((warp - 2) * lnt_warp_bytes<BN>());
    uint32_t lph = 0;
    auto ln_issue = [&](int item_) {   // lane 0: the residual boxes of item_'s 32 x HC block
      int m0_, n0_, z_, sp_, kb0_, nk_;
      decode(item_, m0_, n0_, z_, sp_, kb0_, nk_);
      const int r_ = m0_ + (int)crank * BM + q4 * 32, c_ = n0_ + hh * HC;
      mbar_expect_tx(obar, (uint32_t)(HC * 64));
#pragma unroll
      for (int j = 0; j < HC / 64; ++j)
        tma_load4(lnw + (uint32_t)(j * 4096), &tma_o.r, c_ + 64 * j, r_ % p.ln_rdiv, r_ / p.ln_rdiv, z_, obar);
    };
    if (LNT && p.lnst && lane == 0 && wid < total) ln_issue(wid);
    for (int item = wid; item < total; item += nwk, ++li) {
      int m0, n0, z, sp, kb0, nk;
      decode(item, m0, n0, z, sp, kb0, nk);
      const int ab = li & 1;
      const uint32_t aph = (li >> 1) & 1;
      if constexpr (BSV) {
        if (p.dcnt) {
          constexpr bool FIRST = (VarF<VAR>::F & EF_RESID) != 0;
          const int rbase = m0 + q4 * 32;
          const float alpha = e.alpha;
          const bool alpha1 = alpha == 1.f;
          mbar_wait(smem_u32(tfull + ab), aph);
          asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
          for (int j = 0; j < NPD; ++j, ++gpass) {
            const uint32_t slot = gpass & 1u, oph = (gpass >> 1) & 1u;
            // the previous pass's stores have read their boxes (dA in the other slot, the dX box): refill the
            // other slot with the next pass's operands (this tile's pass j + 1, else the next tile's pass 0)
            if (lane == 0) {
              bulk_wait_read<0>();
              if (j + 1 < NPD) op_issue(item, j + 1, slot ^ 1u);
              else if (item + nwk < total) op_issue(item + nwk, 0, slot ^ 1u);
            }
            __syncwarp();
            uint32_t v[32];
            ld_tmem32(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * BN + hh * HC + 32 * j), v);
            mbar_wait(obar + slot * 8u, oph);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (j + 1 == NPD) {   // accumulator fully read: hand it back to the MMA warp
              asm volatile("tcgen05.fence::before_thread_sync;");
              __syncwarp();
              if (lane == 0) tempty_arrive(smem_u32(tempty + ab), pair);
            }
            const uint32_t xb = opw + slot * 6144u;
            const uint32_t rowx = xb + (uint32_t)(lane * 64), rowd = opw + 12288u + (uint32_t)(lane * 128);
            const uint32_t swx = (uint32_t)((lane >> 1) & 3), swd = (uint32_t)(lane & 7);
#pragma unroll
            for (int c = 0; c < 4; ++c) {   // 16-B granule c of the 64-B bf16 row (64-B swizzle: c ^ ((row >> 1) & 3))
              const uint32_t off = ((uint32_t)c ^ swx) << 4;
              float xv[8], av[8], rv[8], da[8], dx[8];
              unpack_bf8(lds16_(rowx + off), xv);
              unpack_bf8(lds16_(rowx + 2048u + off), av);
              if (FIRST) unpack_bf8(lds16_(rowx + 4096u + off), rv);
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                const float tv = alpha1 ? __uint_as_float(v[8 * c + t]) : __uint_as_float(v[8 * c + t]) * alpha;
                da[t] = tv * xv[t];
                dx[t] = tv * av[t] + tv;
                if (FIRST) dx[t] += rv[t];
              }
              sts4u(rowx + off, pack_bf2(da[0], da[1]), pack_bf2(da[2], da[3]), pack_bf2(da[4], da[5]),
                    pack_bf2(da[6], da[7]));
              sts4(rowd + ((((uint32_t)(2 * c)) ^ swd) << 4), dx[0], dx[1], dx[2], dx[3]);
              sts4(rowd + ((((uint32_t)(2 * c + 1)) ^ swd) << 4), dx[4], dx[5], dx[6], dx[7]);
            }
            __syncwarp();
            if (e.bsum) {   // column sums of the stored dA: lane = column, rows in order
              float s_ = 0.f;
#pragma unroll 8
              for (int r = 0; r < 32; ++r) {
                unsigned short h_;
                asm volatile("ld.shared.u16 %0, [%1];"
                             : "=h"(h_)
                             : "r"(xb + (uint32_t)(r * 64) + (((uint32_t)(lane >> 3) ^ (uint32_t)((r >> 1) & 3)) << 4) +
                                   (uint32_t)((lane & 7) * 2))
                             : "memory");
                s_ += __uint_as_float((uint32_t)h_ << 16);
              }
              dsum_t[j] += s_;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              const int col = n0 + hh * HC + 32 * j;
              tma_store3(&tma_o.a, xb, col, rbase, z);
              if (FIRST) tma_store3(&tma_o.c, opw + 12288u, col, rbase, z);
              else tma_reduce_add3(&tma_o.c, opw + 12288u, col, rbase, z);
              bulk_commit();
            }
          }
          continue;
        }
      }
      if constexpr (RTV) {
        if (p.rst) {
          const int rbase = m0 + q4 * 32;
          const float alpha = e.alpha;
          mbar_wait(smem_u32(tfull + ab), aph);
          asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
          for (int j = 0; j < HC / 32; ++j, ++gpass) {
            const uint32_t slot = gpass & 1u, oph = (gpass >> 1) & 1u;
            if (lane == 0) {   // the previous pass's store has read the other slot: refill it
              bulk_wait_read<0>();
              if (j + 1 < HC / 32) rt_issue(item, j + 1, slot ^ 1u);
              else if (item + nwk < total) rt_issue(item + nwk, 0, slot ^ 1u);
            }
            __syncwarp();
            uint32_t v[32];
            ld_tmem32(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * BN + hh * HC + 32 * j), v);
            mbar_wait(obar + slot * 8u, oph);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (j + 1 == HC / 32) {   // accumulator fully read: hand it back to the MMA warp
              asm volatile("tcgen05.fence::before_thread_sync;");
              __syncwarp();
              if (lane == 0) tempty_arrive(smem_u32(tempty + ab), pair);
            }
            const uint32_t sl = opw + slot * 4096u;
            const uint32_t rrow = sl + (uint32_t)(lane * 128), swr = (uint32_t)(lane & 7);
            float a[32];
#pragma unroll
            for (int c = 0; c < 8; ++c) {   // 16-B granule c of the 128-B fp32 row (128-B swizzle: c ^ (row & 7))
              const float4 r4 = lds4(rrow + ((((uint32_t)c) ^ swr) << 4));
              a[4 * c] = __uint_as_float(v[4 * c]) * alpha + 0.f + r4.x;
              a[4 * c + 1] = __uint_as_float(v[4 * c + 1]) * alpha + 0.f + r4.y;
              a[4 * c + 2] = __uint_as_float(v[4 * c + 2]) * alpha + 0.f + r4.z;
              a[4 * c + 3] = __uint_as_float(v[4 * c + 3]) * alpha + 0.f + r4.w;
            }
            __syncwarp();   // every lane has read its residual row before the bf16 rows overwrite the slot
            const uint32_t orow = sl + (uint32_t)(lane * 64), swo = (uint32_t)((lane >> 1) & 3);
#pragma unroll
            for (int c = 0; c < 4; ++c)   // 16-B granule c of the 64-B bf16 row (64-B swizzle: c ^ ((row >> 1) & 3))
              sts4u(orow + ((((uint32_t)c) ^ swo) << 4), pack_bf2(a[8 * c], a[8 * c + 1]), pack_bf2(a[8 * c + 2], a[8 * c + 3]),
                    pack_bf2(a[8 * c + 4], a[8 * c + 5]), pack_bf2(a[8 * c + 6], a[8 * c + 7]));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              tma_store3(&tma_o.c, sl, n0 + hh * HC + 32 * j, rbase, z);
              bulk_commit();
            }
          }
          continue;
        }
      }
      if constexpr (XTV) {
        if (p.crosst) {
          const int rbase = m0 + q4 * 32;
          const float alpha = e.alpha;
          mbar_wait(smem_u32(tfull + ab), aph);
          asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
          for (int j = 0; j < HC / 32; ++j, ++gpass) {
            const uint32_t slot = gpass & 1u, oph = (gpass >> 1) & 1u;
            if (lane == 0) {   // the previous pass's stores have read the other slot: refill it
              bulk_wait_read<0>();
              if (j + 1 < HC / 32) xt_issue(item, j + 1, slot ^ 1u);
              else if (item + nwk < total) xt_issue(item + nwk, 0, slot ^ 1u);
            }
            __syncwarp();
            uint32_t v[32];
            ld_tmem32(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * BN + hh * HC + 32 * j), v);
            const int col = n0 + hh * HC + 32 * j;
            float bv[32];
#pragma unroll
            for (int q = 0; q < 4; ++q) ldg_bf8(e.bias, col + 8 * q, bv + 8 * q);
            mbar_wait(obar + slot * 8u, oph);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (j + 1 == HC / 32) {   // accumulator fully read: hand it back to the MMA warp
              asm volatile("tcgen05.fence::before_thread_sync;");
              __syncwarp();
              if (lane == 0) tempty_arrive(smem_u32(tempty + ab), pair);
            }
            const uint32_t xrow = opw + slot * 4096u + (uint32_t)(lane * 64), arow = xrow + 2048u;
            const uint32_t swx = (uint32_t)((lane >> 1) & 3);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint32_t off = ((uint32_t)c ^ swx) << 4;
              float xv[8], a8[8], t8[8];
              unpack_bf8(lds16_(xrow + off), xv);
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                a8[t] = __uint_as_float(v[8 * c + t]) * alpha + bv[8 * c + t];
                t8[t] = xv[t] * a8[t] + xv[t];
              }
              sts4u(arow + off, pack_bf2(a8[0], a8[1]), pack_bf2(a8[2], a8[3]), pack_bf2(a8[4], a8[5]), pack_bf2(a8[6], a8[7]));
              sts4u(xrow + off, pack_bf2(t8[0], t8[1]), pack_bf2(t8[2], t8[3]), pack_bf2(t8[4], t8[5]), pack_bf2(t8[6], t8[7]));
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              tma_store3(&tma_o.a, opw + slot * 4096u + 2048u, col, rbase, z);
              tma_store3(&tma_o.c, opw + slot * 4096u, col, rbase, z);
              bulk_commit();
            }
          }
          continue;
        }
      }
      if constexpr (LNT) {
        if (p.lnst) {
          constexpr int F = VarF<VAR>::F;
          const int rbase = m0 + (int)crank * BM + q4 * 32;
          const int row = rbase + lane;
          const bool rok = row < g.M;
          const int64_t ro = rok ? lean_row(e, z, row) : 0;
          const uint32_t tq = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * BN + hh * HC);
          const bool xch_mode = e.ln_d != HC;
          float* xch = sbias + q4 * 128;
          const int cb0 = n0 + hh * HC;
          const int seg0 = xch_mode ? n0 : cb0;
          const int gofs = cb0 - seg0;
          const float inv_d = 1.f / (float)e.ln_d;
          const uint32_t bar_id = 2 + q4;
          const int gr = rbase % p.ln_rdiv, gq = rbase / p.ln_rdiv;   // the boxes' row coordinates
          const uint32_t sw = (uint32_t)(lane & 7);
          mbar_wait(smem_u32(tfull + ab), aph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          mbar_wait(obar, lph);
          lph ^= 1u;
          // pass 1: v = alpha acc (+ bias) + resid -> TMEM and R (in place of the residual), chunked mean / M2
          float s1 = 0.f, s2 = 0.f;
#pragma unroll
          for (int c = 0; c < HC; c += 32) {
            uint32_t v[32];
            ld_tmem32(tq + c, v);
            float bv[32], rv[32];
            if constexpr ((F & EF_BIAS) != 0) {
#pragma unroll
              for (int q = 0; q < 4; ++q) ldg_bf8(e.bias, cb0 + c + 8 * q, bv + 8 * q);
            } else {
#pragma unroll
              for (int q = 0; q < 32; ++q) bv[q] = 0.f;
            }
            const uint32_t rrow = lnw + (uint32_t)((c >> 6) * 4096 + lane * 128);
            const uint32_t g0 = (uint32_t)((c & 63) >> 3);   // first 16-B granule of these 32 columns
#pragma unroll
            for (int q = 0; q < 4; ++q) unpack_bf8(lds16_(rrow + (((g0 + q) ^ sw) << 4)), rv + 8 * q);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            float f[32];
            float cs_ = 0.f;
#pragma unroll
            for (int q = 0; q < 32; ++q) { f[q] = __uint_as_float(v[q]) * e.alpha + bv[q] + rv[q]; cs_ += f[q]; }
            const float cm = cs_ * (1.f / 32.f);
            float cm2 = 0.f;
#pragma unroll
            for (int q = 0; q < 32; ++q) { const float t_ = f[q] - cm; cm2 = fmaf(t_, t_, cm2); }
            if (c == 0) {
              s1 = cm; s2 = cm2;
            } else {
              const float w_ = 32.f / (float)(c + 32), dl = cm - s1;
              s1 = fmaf(dl, w_, s1);
              s2 += cm2 + dl * dl * ((float)c * w_);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
              sts4u(rrow + (((g0 + q) ^ sw) << 4), pack_bf2(f[8 * q], f[8 * q + 1]), pack_bf2(f[8 * q + 2], f[8 * q + 3]),
                    pack_bf2(f[8 * q + 4], f[8 * q + 5]), pack_bf2(f[8 * q + 6], f[8 * q + 7]));
            tmem_st32f(tq + c, f);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int j = 0; j < HC / 64; ++j) tma_store4(&tma_o.d, lnw + (uint32_t)(j * 4096), cb0 + 64 * j, gr, gq, z);
            bulk_commit();
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          if (xch_mode) {   // [quadrant][hh][32 lanes] of (mean, M2) pairs through the bias scratch
            const uint32_t xa = smem_u32(xch);
            asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(xa + (uint32_t)((hh * 32 + lane) * 8)), "f"(s1), "f"(s2)
                         : "memory");
            asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
            float a1, a2, b1, b2;
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a1), "=f"(a2) : "r"(xa + (uint32_t)(lane * 8)) : "memory");
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(b1), "=f"(b2) : "r"(xa + (uint32_t)((32 + lane) * 8))
                         : "memory");
            const float dl = b1 - a1;
            s1 = 0.5f * (a1 + b1);
            s2 = (a2 + b2) + dl * dl * (0.5f * (float)HC);
            asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
          }
          const float mean = s1;
          const float rs = rsqrtf(s2 * inv_d + e.ln_eps);
          if (rok && (!xch_mode || hh == 0)) {
            const int64_t tok = (ro + seg0) / e.ln_d;
            e.ln_mu[tok] = mean;
            e.ln_rstd[tok] = rs;
          }
          // Y overwrites R in the same boxes once the R stores have read them
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
          // pass 2: Y = gamma (v - mu) rstd + beta, one 64-column box store at a time
#pragma unroll 1
          for (int c = 0; c < HC; c += 32) {
            uint32_t v[32];
            ld_tmem32(tq + c, v);
            float gv[32], be[32];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              ldg_bf8(e.ln_gamma, gofs + c + 8 * q, gv + 8 * q);
              ldg_bf8(e.ln_beta, gofs + c + 8 * q, be + 8 * q);
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (c + 32 >= HC) {   // accumulator fully read: hand it back to the MMA warp
              asm volatile("tcgen05.fence::before_thread_sync;");
              __syncwarp();
              if (lane == 0) tempty_arrive(smem_u32(tempty + ab), pair);
            }
            const uint32_t g0 = (uint32_t)((c & 63) >> 3);
            const uint32_t yrow = lnw + (uint32_t)((c >> 6) * 4096 + lane * 128);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float y[8];
#pragma unroll
              for (int t = 0; t < 8; ++t) y[t] = (__uint_as_float(v[8 * q + t]) - mean) * rs * gv[8 * q + t] + be[8 * q + t];
              sts4u(yrow + (((g0 + q) ^ sw) << 4), pack_bf2(y[0], y[1]), pack_bf2(y[2], y[3]), pack_bf2(y[4], y[5]),
                    pack_bf2(y[6], y[7]));
            }
            if ((c & 63) == 32 || c + 32 >= HC) {   // the 64-column box is complete
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) {
                tma_store4(&tma_o.c, lnw + (uint32_t)((c >> 6) * 4096), cb0 + (c & ~63), gr, gq, z);
                bulk_commit();
              }
            }
          }
          // the boxes are free once the Y stores have read them: the next tile's residual can land (its latency
          // overlaps the wait for the next accumulator)
          if (lane == 0) {
            bulk_wait_read<0>();
            if (item + nwk < total) ln_issue(item + nwk);
          }
          continue;
        }
      }
      // LayerNorm epilogue: the warp's residual block (32 rows x HC bf16) is loaded BEFORE the accumulator is
      // ready -- with lanes along columns (coalesced 16-B loads) into the warp's staging area, where pass 1
      // reads its row back and overwrites it with R -- so its latency hides under the tile's MMAs
      constexpr bool LNV = VAR > 0 && (VarF<VAR>::F & EF_LN) != 0;
      // (measured: the coalesced staging pre-load wins when a warp half is a whole LN segment, ln_d == HC;
      // with the warp-pair exchange, ln_d == BN, a per-row register prefetch is faster)
      const bool ln_stage_x = LNV && e.ln_d == HC && !p.lnst;
      uint4 rpre[LNV ? HC / 8 : 1];
      if (LNV && !ln_stage_x && !p.lnst) {
        const int row_ = m0 + (int)crank * BM + q4 * 32 + lane;
        if (row_ < g.M) {
          const __nv_bfloat16* rp = (const __nv_bfloat16*)e.resid + lean_row(e, z, row_) + n0 + hh * HC;
#pragma unroll
          for (int q = 0; q < (LNV ? HC / 8 : 1); ++q) rpre[q] = __ldg(reinterpret_cast<const uint4*>(rp) + q);
        } else {
#pragma unroll
          for (int q = 0; q < (LNV ? HC / 8 : 1); ++q) rpre[q] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
      if (ln_stage_x) {
        constexpr int PBr = HC * 2 + 16, LPRr = HC / 8, RPIr = 32 / LPRr;
        const uint32_t stgw_ = smem_u32(stage_all) + (uint32_t)((warp - 2) * 32 * SROW * 4);
        const int row_ = m0 + (int)crank * BM + q4 * 32 + lane;
        const int64_t my_ro = row_ < g.M ? lean_row(e, z, row_) : 0;
        const int cl = lane % LPRr, sr = lane / LPRr;
        __syncwarp();   // the previous tile's Y flush has read the staging area
#pragma unroll 4
        for (int r0 = 0; r0 < 32; r0 += RPIr) {
          const int r = r0 + sr;
          const int64_t orow = shfl64(my_ro, r);
          uint4 u = make_uint4(0u, 0u, 0u, 0u);
          if (m0 + (int)crank * BM + q4 * 32 + r < g.M)
            u = __ldg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)e.resid + orow + n0 + hh * HC + cl * 8));
          sts4u(stgw_ + (uint32_t)(r * PBr + cl * 16), u.x, u.y, u.z, u.w);
        }
        __syncwarp();
      }
      // ReLU-bitmask words of the warp's rows x HC columns, also fetched before the accumulator is ready
      constexpr bool BMV = VAR > 0 && (VarF<VAR>::F & EF_BMASK) != 0;
      uint32_t bpre[BMV ? HC / 32 : 1];
      if constexpr (BMV) {
        const int row_ = m0 + (int)crank * BM + q4 * 32 + lane;
        const uint32_t* bp = e.bits + (int64_t)((n0 + hh * HC) / 32) * e.bits_ld + row_;   // word-major: lanes coalesce
#pragma unroll
        for (int q = 0; q < HC / 32; ++q) bpre[q] = row_ < g.M ? __ldg(bp + (int64_t)q * e.bits_ld) : 0u;
      }
      mbar_wait(smem_u32(tfull + ab), aph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (p.trace && blockIdx.x == 0 && li < 64 && warp == 2 && lane == 0) p.trace[192 + li] = clock64();
      const int rbase = m0 + (int)crank * BM + q4 * 32;
      if constexpr (VAR > 0 && (VarF<VAR>::F & EF_LN) != 0) {
        // ---- LayerNorm epilogue over row segments of ln_d columns (each segment one token of d features).
        // Lane = row.  ln_d == HC: a warp's column half is one whole segment; ln_d == BN: the two warps of a
        // TMEM lane quadrant (hh = 0, 1) own the two halves of the segment and exchange row partial sums through
        // shared memory (named barrier per quadrant).  Pass 1: v = alpha acc (+ bias) + resid -> TMEM, R = bf16(v)
        // stored, mean and M2 of v (chunked, Chan-merged); pass 2: Y = gamma (v - mu) rstd + beta.  The segment's
        // statistics index is (element offset of its first column) / ln_d, relative to ln_mu / ln_rstd.
        constexpr int F = VarF<VAR>::F;
        const int row = rbase + lane;
        const bool rok = row < g.M;
        const int64_t ro = rok ? lean_row(e, z, row) : 0;
        const uint32_t tq = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * BN + hh * HC);
        const bool xch_mode = e.ln_d != HC;
        float* xch = sbias + q4 * 128;  // [quadrant][hh][32 lanes] row partial (mean, M2) pairs (the bias scratch)
        const int cb0 = n0 + hh * HC;                       // first column of this warp's half
        const int seg0 = xch_mode ? n0 : cb0;               // first column of the segment
        const int gofs = cb0 - seg0;                        // gamma / beta index of column cb0
        const float inv_d = 1.f / (float)e.ln_d;
        const uint32_t bar_id = 2 + q4;
        // R and Y leave through the warp's staging area (bf16 rows of HC columns, 16-B padded pitch) and are
        // stored with lanes along columns (coalesced 16-B stores) instead of one row per lane
        constexpr int PB = HC * 2 + 16;
        const uint32_t stgw = smem_u32(stage_all) + (uint32_t)((warp - 2) * 32 * SROW * 4);
        static_assert(32 * PB <= 32 * SROW * 4, "LN staging fits the warp's staging area");
        auto stage8 = [&](int col, const float* vals) {   // 8 values of this lane's row at warp-local column col
          sts4u(stgw + (uint32_t)(lane * PB + col * 2), pack_bf2(vals[0], vals[1]), pack_bf2(vals[2], vals[3]),
                pack_bf2(vals[4], vals[5]), pack_bf2(vals[6], vals[7]));
        };
        auto flush = [&](void* base) {   // staged 32 x HC block -> rows rbase.., columns cb0..
          __syncwarp();
          constexpr int LPRr = HC / 8, RPI = 32 / LPRr;
          const int cl = lane % LPRr, sr = lane / LPRr;
#pragma unroll 4
          for (int r0 = 0; r0 < 32; r0 += RPI) {
            const int r = r0 + sr;
            const int64_t orow = shfl64(ro, r);
            const uint4 u = lds16_(stgw + (uint32_t)(r * PB + cl * 16));
            if (rbase + r < g.M)
              *reinterpret_cast<uint4*>((__nv_bfloat16*)base + orow + cb0 + cl * 8) = u;
          }
          __syncwarp();
        };
        // Row statistics without cancellation: per 32-column chunk the mean and the sum of squared deviations
        // from it (two passes over the chunk's registers), merged chunk by chunk with Chan's pairwise update, and
        // across the quadrant warp pair the same way -- a large common offset |mean| >> std costs no precision.
        float s1 = 0.f, s2 = 0.f;   // running mean and M2 (sum of squared deviations) of this thread's columns
#pragma unroll
        for (int c = 0; c < HC; c += 32) {   // unrolled: rpre is indexed with compile-time offsets
          uint32_t v[32];
          ld_tmem32(tq + c, v);
          float rv[32], bv[32];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            unpack_bf8(ln_stage_x ? lds16_(stgw + (uint32_t)(lane * PB + (c + 8 * q) * 2)) : rpre[c / 8 + q], rv + 8 * q);
          if constexpr ((F & EF_BIAS) != 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) ldg_bf8(e.bias, cb0 + c + 8 * q, bv + 8 * q);
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q) bv[q] = 0.f;
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float f[32];
          float cs_ = 0.f;
#pragma unroll
          for (int q = 0; q < 32; ++q) { f[q] = __uint_as_float(v[q]) * e.alpha + bv[q] + rv[q]; cs_ += f[q]; }
          const float cm = cs_ * (1.f / 32.f);
          float cm2 = 0.f;
#pragma unroll
          for (int q = 0; q < 32; ++q) { const float t_ = f[q] - cm; cm2 = fmaf(t_, t_, cm2); }
          if (c == 0) {
            s1 = cm; s2 = cm2;
          } else {   // merge (c columns: s1, s2) with (32 columns: cm, cm2)
            const float w_ = 32.f / (float)(c + 32), dl = cm - s1;
            s1 = fmaf(dl, w_, s1);
            s2 += cm2 + dl * dl * ((float)c * w_);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) stage8(c + 8 * q, f + 8 * q);
          tmem_st32f(tq + c, f);
        }
        flush(e.aux);   // R
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if (xch_mode) {   // [quadrant][hh][32 lanes] of (mean, M2) pairs through the bias scratch
          const uint32_t xa = smem_u32(xch);
          asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(xa + (uint32_t)((hh * 32 + lane) * 8)), "f"(s1), "f"(s2)
                       : "memory");
          asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
          float a1, a2, b1, b2;
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a1), "=f"(a2) : "r"(xa + (uint32_t)(lane * 8)) : "memory");
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(b1), "=f"(b2) : "r"(xa + (uint32_t)((32 + lane) * 8))
                       : "memory");
          const float dl = b1 - a1;   // two halves of HC columns each
          s1 = 0.5f * (a1 + b1);
          s2 = (a2 + b2) + dl * dl * (0.5f * (float)HC);
          asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
        }
        const float mean = s1;
        const float var = s2 * inv_d;
        const float rs = rsqrtf(var + e.ln_eps);
        if (rok && (!xch_mode || hh == 0)) {
          const int64_t tok = (ro + seg0) / e.ln_d;
          e.ln_mu[tok] = mean;
          e.ln_rstd[tok] = rs;
        }
#pragma unroll 1
        for (int c = 0; c < HC; c += 32) {
          uint32_t v[32];
          ld_tmem32(tq + c, v);
          float gv[32], be[32];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            ldg_bf8(e.ln_gamma, gofs + c + 8 * q, gv + 8 * q);
            ldg_bf8(e.ln_beta, gofs + c + 8 * q, be + 8 * q);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c + 32 >= HC) {   // accumulator fully read: hand it back to the MMA warp
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) tempty_arrive(smem_u32(tempty + ab), pair);
          }
          float y[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) y[q] = (__uint_as_float(v[q]) - mean) * rs * gv[q] + be[q];
#pragma unroll
          for (int q = 0; q < 4; ++q) stage8(c + 8 * q, y + 8 * q);
        }
        flush(e.c);     // Y
        continue;
      }
      if constexpr (VAR > 0 && ((VarF<VAR>::F & ~TS_FLAGS) == 0) && (!(VarF<VAR>::F & EF_ACC) || VarF<VAR>::C)) {
        if (p.tstore) {
          // ---- TMA-store epilogue: lane = row; a pass takes 128 B of the row (64 bf16 / 32 fp32 columns) from
          // TMEM, applies alpha / bias / ReLU, writes it into a 128-B-swizzled box (32 rows x 128 B) and one lane
          // stores the box with cp.async.bulk.tensor (fp32 +=: cp.reduce.async.bulk .add).  Two boxes per warp.
          constexpr int F = VarF<VAR>::F;
          constexpr bool CF = VarF<VAR>::C;
          constexpr int CW = CF ? 32 : 64;
          float* sb = WR ? sbias : sbias + ab * BN;
          if constexpr ((F & EF_BIAS) != 0) {
            if (!WR || li == 0) {   // WR: every item of the CTA has the same N tile, so the same bias row
              asm volatile("bar.sync 1, 256;" ::: "memory");   // every epilogue warp finished the tile that used sb
              const int t = threadIdx.x - 64;
              for (int j = t; j < BN; j += 256) sb[j] = (n0 + j < g.N) ? lean_bias(e, n0 + j) : 0.f;
              asm volatile("bar.sync 1, 256;" ::: "memory");
            }
          }
          const uint32_t boxes = smem_u32(stage_all) + (uint32_t)((warp - 2) * (WR ? 1 : 2) * 4096);
          const float alpha = e.alpha;
#pragma unroll 1
          for (int pc = 0; pc < HC; pc += CW) {
            uint32_t v[CW];
            const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * BN + hh * HC + pc);
            ld_tmem32(taddr, v);
            if constexpr (CW == 64) ld_tmem32(taddr + 32, v + 32);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (pc + CW >= HC) {   // accumulator fully read: hand it back to the MMA warp
              asm volatile("tcgen05.fence::before_thread_sync;");
              __syncwarp();
              if (lane == 0) tempty_arrive(smem_u32(tempty + ab), pair);
            }
            const int cl0 = hh * HC + pc;   // tile-local column of v[0]
            const int brow = rbase + lane;
            uint32_t mw[CW / 32];            // ReLU bitmask words of these CW columns (EF_BMASK: read)
            if constexpr ((F & EF_BMASK) != 0) {   // this pass's words from the prefetch, then shift it down
#pragma unroll
              for (int q = 0; q < CW / 32; ++q) mw[q] = bpre[q];
#pragma unroll
              for (int q = 0; q + CW / 32 < HC / 32; ++q) bpre[q] = bpre[q + CW / 32];
            }
            if (alpha != 1.f) {   // (a uniform branch: the plain GEMMs skip the multiply)
#pragma unroll
              for (int j = 0; j < CW; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * alpha);
            }
            if constexpr ((F & EF_BIAS) != 0) {   // the tile's bias row from shared memory, 16 B at a time
              const uint32_t sba = smem_u32(sb + cl0);
#pragma unroll
              for (int j = 0; j < CW; j += 4) {
                const float4 b4 = lds4(sba + (uint32_t)(j * 4));
                v[j] = __float_as_uint(__uint_as_float(v[j]) + b4.x);
                v[j + 1] = __float_as_uint(__uint_as_float(v[j + 1]) + b4.y);
                v[j + 2] = __float_as_uint(__uint_as_float(v[j + 2]) + b4.z);
                v[j + 3] = __float_as_uint(__uint_as_float(v[j + 3]) + b4.w);
              }
            }
#pragma unroll
            for (int j = 0; j < CW; ++j) {
              float a = __uint_as_float(v[j]);
              if constexpr ((F & EF_RELU) != 0) a = fmaxf(a, 0.f);
              if constexpr ((F & EF_BMASK) != 0) a = ((mw[j >> 5] >> (j & 31)) & 1u) ? a : 0.f;
              v[j] = __float_as_uint(a);
            }
            if constexpr ((F & EF_BITS) != 0 && !CF) {
              // bit j = the STORED bf16 value is > 0: round-to-nearest-even maps a float > 0 to a bf16 > 0 exactly
              // when it exceeds half the smallest bf16 subnormal, 2^-134 (R22, R24)
#pragma unroll
              for (int q = 0; q < CW / 32; ++q) {
                uint32_t w = 0;
#pragma unroll
                for (int t = 0; t < 32; ++t) w |= (__uint_as_float(v[32 * q + t]) > 0x1p-134f ? 1u : 0u) << t;
                mw[q] = w;
              }
              if (brow < g.M) {
                uint32_t* bp = e.bits + (int64_t)((n0 + cl0) / 32) * e.bits_ld + brow;
#pragma unroll
                for (int q = 0; q < CW / 32; ++q) bp[(int64_t)q * e.bits_ld] = mw[q];
              }
            }
            const uint32_t box = boxes + (uint32_t)(WR ? 0 : (tsel & 1) * 4096);   // alternate across passes AND tiles
            ++tsel;
            if (lane == 0) {   // the store that last read this box is done with it
              if constexpr (WR) bulk_wait_read<0>(); else bulk_wait_read<1>();
            }
            __syncwarp();
            const uint32_t rowa = box + (uint32_t)(lane * 128);
#pragma unroll
            for (int gq = 0; gq < 8; ++gq) {   // 16-B granule gq of the row -> swizzled slot gq ^ (row & 7)
              const uint32_t a = rowa + (uint32_t)(((gq ^ (lane & 7)) & 7) << 4);
              if constexpr (CF) {
                sts4u(a, v[4 * gq], v[4 * gq + 1], v[4 * gq + 2], v[4 * gq + 3]);
              } else {
                sts4u(a, pack_bf2(__uint_as_float(v[8 * gq]), __uint_as_float(v[8 * gq + 1])),
                      pack_bf2(__uint_as_float(v[8 * gq + 2]), __uint_as_float(v[8 * gq + 3])),
                      pack_bf2(__uint_as_float(v[8 * gq + 4]), __uint_as_float(v[8 * gq + 5])),
                      pack_bf2(__uint_as_float(v[8 * gq + 6]), __uint_as_float(v[8 * gq + 7])));
              }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              if constexpr ((F & EF_ACC) != 0) tma_reduce_add3(&tma_o.c, box, n0 + cl0, rbase, z);
              else tma_store3(&tma_o.c, box, n0 + cl0, rbase, z);
              bulk_commit();
            }
            if constexpr (!CF && (F & EF_ACC) == 0) {
              if (e.csum) {   // column sums of the 32 stored (bf16) rows: lane = 2 columns, read down the box
                // 32 independent loads, four running pairs (rows r % 4) summed at the end: a fixed order
                const int nr = min(32, g.M - rbase);
                float2 sp[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                for (int r = 0; r < 32; ++r) {
                  uint32_t w;
                  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w)
                               : "r"(box + (uint32_t)(r * 128 + ((((lane >> 2) ^ (r & 7)) & 7) << 4) + (lane & 3) * 4))
                               : "memory");
                  if (r >= nr) w = 0u;
                  sp[r & 3].x += __uint_as_float(w << 16);
                  sp[r & 3].y += __uint_as_float(w & 0xffff0000u);
                }
                const float s0 = (sp[0].x + sp[1].x) + (sp[2].x + sp[3].x);
                const float s1 = (sp[0].y + sp[1].y) + (sp[2].y + sp[3].y);
                const int cg = n0 + cl0 + 2 * lane;
                if (cg < g.N) {
                  float* cp = e.csum + ((int64_t)z * ((g.M + 31) / 32) + rbase / 32) * g.N + cg;
                  cp[0] = s0;
                  if (cg + 1 < g.N) cp[1] = s1;
                }
              }
            }
          }
          continue;
        }
      }
      if (p.lanes_rows) {
        // column-contiguous output: row per lane straight from TMEM; consecutive lanes = consecutive addresses
        const int row = rbase + lane;
        const bool rok = row < g.M;
        RowBase rb;
        int64_t lo = 0;
        if (rok) { if (p.lean) lo = lean_row(e, z, row); else rb = row_base(g, z, row); }
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
            if (lane == 0) tempty_arrive(smem_u32(tempty + ab), pair);
          }
          if (rok && n0 + c0 < g.N) {
            if constexpr (VAR > 0) {
              lean_rows16<VarF<VAR>::F, VarF<VAR>::C>(e, lo, n0 + c0, g.N, v);
            } else if (p.lean) {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const int col = n0 + c0 + j;
                if (col < g.N)
                  lean1(e, lo + (int64_t)col * e.cs, __uint_as_float(v[j]), (e.flags & EF_BIAS) ? lean_bias(e, col) : 0.f);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const int col = n0 + c0 + j;
                if (col < g.N) epi_elem(g, rb, col, __uint_as_float(v[j]));
              }
            }
          }
        }
        continue;
      }
      // row-major output: park this warp's 32 x SC block in smem, then walk it with lanes on columns
#pragma unroll 1
      for (int pc = 0; pc < HC; pc += SC) {
        {
          // all TMEM loads of the pass in flight under one wait, then the staging stores
          uint32_t v[SC];
#pragma unroll
          for (int c0 = 0; c0 < SC; c0 += 16) {
            const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * BN + hh * HC + pc + c0);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[c0 + 0]), "=r"(v[c0 + 1]), "=r"(v[c0 + 2]), "=r"(v[c0 + 3]), "=r"(v[c0 + 4]), "=r"(v[c0 + 5]),
                  "=r"(v[c0 + 6]), "=r"(v[c0 + 7]), "=r"(v[c0 + 8]), "=r"(v[c0 + 9]), "=r"(v[c0 + 10]), "=r"(v[c0 + 11]),
                  "=r"(v[c0 + 12]), "=r"(v[c0 + 13]), "=r"(v[c0 + 14]), "=r"(v[c0 + 15])
                : "r"(taddr));
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const uint32_t dst = stage + (uint32_t)(lane * SROW * 4);
#pragma unroll
          for (int j = 0; j < SC / 4; ++j)
            sts4(dst + 16 * j, __uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]), __uint_as_float(v[4 * j + 2]),
                 __uint_as_float(v[4 * j + 3]));
        }
        if (pc + SC >= HC) {
          if (p.trace && blockIdx.x == 0 && li < 64 && warp == 2 && lane == 0) p.trace[256 + li] = clock64();
          // accumulator fully read: hand it back to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) tempty_arrive(smem_u32(tempty + ab), pair);
        }
        __syncwarp();
        const int cbase = n0 + hh * HC + pc;
        if (VAR > 0) {
          if constexpr (VAR > 0)
            lean_pass8<VarF<VAR>::F, VarF<VAR>::C, SC>(
                e, z, rbase, g.M, g.N, cbase, stage, lane,
                (BSV && e.bsum) ? smem_u32(csum) + (uint32_t)((warp - 2) * 256 * 4) : 0u);
        } else if (p.lean && p.fast) {
          constexpr int LPR = SC / 4;          // lanes per row (4 columns each)
          constexpr int RPP = 32 / LPR;        // rows per pass
          const int sub = lane / LPR, cl = lane % LPR;
          const int col = cbase + 4 * cl;
          if (col < g.N) {                     // N % 4 == 0 in lean/fast mode: the 4 columns are all valid
            float bias4[4] = {0.f, 0.f, 0.f, 0.f};
            if (e.flags & EF_BIAS) {
#pragma unroll
              for (int t = 0; t < 4; ++t) bias4[t] = lean_bias(e, col + t);
            }
            const int f = e.flags;
#pragma unroll 4
            for (int r = sub; r < 32; r += RPP) {
              const int row = rbase + r;
              if (row >= g.M) break;
              const int64_t o = lean_row(e, z, row) + col;
              const float4 a4 = lds4(stage + (uint32_t)((r * SROW + 4 * cl) * 4));
              float a[4] = {a4.x * e.alpha + bias4[0], a4.y * e.alpha + bias4[1], a4.z * e.alpha + bias4[2],
                            a4.w * e.alpha + bias4[3]};
              float t4[4];
              if (f & EF_AUX) stg4(e.aux, o, 0, a);
              if (f & EF_CROSS) {
                ldg_bf4(e.x, o, t4);
#pragma unroll
                for (int t = 0; t < 4; ++t) a[t] = t4[t] * a[t] + t4[t];
              }
              if (f & EF_RELU) {
#pragma unroll
                for (int t = 0; t < 4; ++t) a[t] = fmaxf(a[t], 0.f);
              }
              if (f & EF_MASK) {
                ldg_bf4(e.mask, o, t4);
#pragma unroll
                for (int t = 0; t < 4; ++t) a[t] = t4[t] > 0.f ? a[t] : 0.f;
              }
              if (f & EF_RESID) {
                ldg_bf4(e.resid, o, t4);
#pragma unroll
                for (int t = 0; t < 4; ++t) a[t] += t4[t];
              }
              if (f & EF_ACC) {
                ldg_c4(e.c, o, e.c_f32, t4);
#pragma unroll
                for (int t = 0; t < 4; ++t) a[t] += t4[t];
              }
              stg4(e.c, o, e.c_f32, a);
            }
          }
        } else {
          // generic path (split-K partials, irregular views)
          const float* stg = stage_all + (warp - 2) * 32 * SROW;
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
                const float acc = stg[r * SROW + lane + 32 * q];
                if (p.splits == 1) {
                  if (g.e.triu_m || g.e.dcn_bwd) epi_apply(g, z, row, col, acc);
                  else epi_elem(g, rb, col, acc);
                }
                else p.ws[((int64_t)(z * p.splits + sp) * g.M + row) * g.N + col] = acc;
              }
            }
          }
        }
        __syncwarp();
      }
      if (p.trace && blockIdx.x == 0 && li < 64 && warp == 2 && lane == 0) p.trace[320 + li] = clock64();
    }
    if constexpr (BSV) {
      if (p.dcnt && p.ep.bsum) {   // this warp's dA column sums into its row of the CTA's partial sums
#pragma unroll
        for (int j = 0; j < NPD; ++j) {
          const int col = hh * HC + 32 * j + lane;
          if (col < p.g.N) csum[(warp - 2) * 256 + col] += dsum_t[j];
        }
      }
    }
  }
  if ((p.tstore || p.lnst || p.dcnt || p.crosst || p.rst) && warp >= 2 && lane == 0) bulk_wait_all();   // TMA stores done reading smem and written
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if constexpr (BSV) {   // this CTA's partial row of the dA column sums: warps summed in a fixed order
    if (p.ep.bsum) {
      for (int col = threadIdx.x; col < p.g.N; col += blockDim.x) {
        float s_ = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) s_ += csum[w * 256 + col];
        p.ep.bsum[(int64_t)blockIdx.x * p.g.N + col] = s_;
      }
    }
  }
  if (pair) {
    cluster_sync_all();   // no CTA leaves while its peer may still touch its barriers, smem or TMEM
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
  } else {
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
  }
}

template <int BN, int STAGES, int VAR, bool PAIR>
constexpr int smem_bytes() {
  constexpr int S = eff_stages<BN, STAGES, VAR, PAIR>();
  return ring_stages<BN, S, PAIR>() * (BM * BK * 2 + (PAIR ? BN * BK : BN * BK * 2)) + epi_bytes<BN, VAR, PAIR>() +
         EpiSmem<BN>::SBIAS * 4 + (2 * ring_stages<BN, S, PAIR>() + 4) * 8 + 16 + 1024 +
         ((VarF<VAR>::F & EF_DCNB) != 0 ? 8 * 256 * 4 : 0) + (has_opbar<VAR>() ? 16 * 8 : 0);
}

template <int BN, int STAGES, int VAR>
static cudaError_t launch(const Params& p0, const CUtensorMap& ma, const CUtensorMap& mb, const OutMaps& mc,
                          cudaStream_t st) {
  constexpr int S0 = eff_stages<BN, STAGES, VAR, false>(), S1 = eff_stages<BN, STAGES, VAR, true>();
  constexpr int SMEM = smem_bytes<BN, STAGES, VAR, false>(), SMEM_P = smem_bytes<BN, STAGES, VAR, true>();
  static_assert(SMEM <= 227 * 1024 && SMEM_P <= 227 * 1024, "smem");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<BN, S0, VAR, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if constexpr (BN >= 128)
      cudaFuncSetAttribute(gemm_tc_kernel<BN, S1, VAR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_P);
    attr = true;
  }
  const int ntiles = p0.tiles_m * p0.tiles_n;
  if constexpr (wr_ok<BN, VAR>()) if (p0.wr) {   // W-resident (host: batch 1, one split, N tiles fastest, K <= 256)
    constexpr int SMEM_W = wr_smem<BN, false>(), SMEM_WP = wr_smem<BN, true>();
    static_assert(SMEM_W <= 227 * 1024 && SMEM_WP <= 227 * 1024, "smem");
    static bool wattr = false;
    if (!wattr) {
      cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES, VAR, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_W);
      cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES, VAR, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_WP);
      wattr = true;
    }
    if (p0.pair) {   // CTA pairs: a multiple of tiles_n clusters, so every cluster keeps one N tile
      static int max_cl = 0;
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = SMEM_WP; cfg.stream = st; cfg.attrs = at;
      cfg.numAttrs = pdl_enabled() ? 2 : 1;
      if (!max_cl) {
        cfg.gridDim = dim3(148);
        if (cudaOccupancyMaxActiveClusters(&max_cl, gemm_tc_kernel<BN, STAGES, VAR, true, true>, &cfg) != cudaSuccess ||
            max_cl <= 0) {
          (void)cudaGetLastError();
          max_cl = 64;
        }
      }
      const int cl = (int)std::min<int64_t>(ntiles, std::max(1, max_cl / p0.tiles_n) * p0.tiles_n);
      cfg.gridDim = dim3((unsigned)(2 * cl));
      g_last_gemm_grid = (int)cfg.gridDim.x;
      cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, STAGES, VAR, true, true>, ma, mb, mc, p0);
      if (e != cudaSuccess) return e;
      ++g_launches;
      return cudaGetLastError();
    }
    // a multiple of tiles_n CTAs: with N tiles fastest, CTA c only ever sees N tile c % tiles_n
    const int grid = (int)std::min<int64_t>(ntiles, (148 / p0.tiles_n) * p0.tiles_n);
    g_last_gemm_grid = grid;
    cudaError_t e = pdl_launch(gemm_tc_kernel<BN, STAGES, VAR, false, true>, grid, 320, SMEM_W, st, ma, mb, mc, p0);
    if (e != cudaSuccess) return e;
    ++g_launches;
    return cudaGetLastError();
  }
  const int zmax = std::max(1, (int)std::min<int64_t>(p0.g.batch, (int64_t)(1 << 30) / ((int64_t)ntiles * p0.splits)));
  for (int zb = 0; zb < p0.g.batch; zb += zmax) {
    Params p = p0;
    p.zbase = zb;
    p.nz = std::min(zmax, p0.g.batch - zb);
    const int64_t items = (int64_t)ntiles * p.nz * p.splits;
    if constexpr (BN >= 128) if (p.pair) {
      static int max_clusters = 0;
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = SMEM_P; cfg.stream = st; cfg.attrs = at;
      cfg.numAttrs = pdl_enabled() ? 2 : 1;
      if (!max_clusters) {   // SM pairs the GPC layout can co-schedule (<= 74 on 148 SMs)
        cfg.gridDim = dim3(148);
        if (cudaOccupancyMaxActiveClusters(&max_clusters, gemm_tc_kernel<BN, S1, VAR, true>, &cfg) != cudaSuccess ||
            max_clusters <= 0) {
          (void)cudaGetLastError();
          max_clusters = 64;
        }
      }
      cfg.gridDim = dim3((unsigned)(2 * std::min<int64_t>(items, max_clusters)));
      g_last_gemm_grid = (int)cfg.gridDim.x;
      cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, S1, VAR, true>, ma, mb, mc, p);
      if (e != cudaSuccess) return e;
      ++g_launches;
      continue;
    }
    {
      const int grid = (int)std::min<int64_t>(items, 148);
      g_last_gemm_grid = grid;
      cudaError_t e = pdl_launch(gemm_tc_kernel<BN, S0, VAR, false>, grid, 320, SMEM, st, ma, mb, mc, p);
      if (e != cudaSuccess) return e;
    }
    ++g_launches;
  }
  return cudaGetLastError();
}

// Launch with the epilogue variant as a template argument (one variant per kernel instantiation).
template <int BN, int STAGES>
cudaError_t launch_var(const Params& p, const CUtensorMap& ma, const CUtensorMap& mb, const OutMaps& mc,
                       cudaStream_t st, int var) {
  switch (var) {
#define LV_L(i, f, c) \
  case i: return launch<BN, STAGES, i>(p, ma, mb, mc, st);
    LEAN_VARIANTS(LV_L)
#undef LV_L
    default: return launch<BN, STAGES, 0>(p, ma, mb, mc, st);
  }
}
// defined in gemm_tc_bn{64,128,256}.cu (parallel compilation of the instantiations)
cudaError_t launch_bn64(const Params& p, const CUtensorMap& ma, const CUtensorMap& mb, const OutMaps& mc,
                        cudaStream_t st, int var);
cudaError_t launch_bn128(const Params& p, const CUtensorMap& ma, const CUtensorMap& mb, const OutMaps& mc,
                         cudaStream_t st, int var);
cudaError_t launch_bn256(const Params& p, const CUtensorMap& ma, const CUtensorMap& mb, const OutMaps& mc,
                         cudaStream_t st, int var);

}  // namespace tc
}  // namespace dhen
