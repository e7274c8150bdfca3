// attn_tc.cu — fused self-attention core for short feature-token sequences (F4 / B6 of SURVEY §8(a)):
//
//   forward   (Eq.(4)):  S = Q_h K_h^T,  P = softmax_row(S / sqrt(dh)),  O_h = P V_h
//   backward  (B6):  dV = P^T dO,  dP = dO V^T,  dS = P (dP - rowsum(P dP)) / sqrt(dh),
//                    dQ = dS K,  dK = dS^T Q
//
// One CTA owns one (sample, head) item at a time: m <= 128 tokens, dh in {64, 128}.  Q, K, V (and dO) of
// the item arrive by TMA (2-D maps over the [B*m][3d] / [B*m][d] activations; a tile's rows m..127 are
// ignored), every contraction is one chain of tcgen05.mma (M = 128, K = 16 steps) into
// TMEM, and the softmax runs on the accumulator rows straight out of TMEM (two threads per query row,
// one per 64-column half, exchanging row max / sum / D through shared memory).  P (and dS) never leave the SM: they are written to shared memory in the
// 128-B-swizzled K-major layout the next MMA reads, as the A operand (P V, dS K) or, through the same
// bytes read as an MN-major operand, as the transposed A operand (P^T dO, dS^T Q).  The backward
// recomputes S and P from Q, K (bit-identical to the forward: same MMA chain, same softmax code) instead
// of storing P, so per item the forward moves Q, K, V in and O out, the backward Q, K, V, dO in and
// dQ, dK, dV out — the attention's algorithmic bytes.
//
// Warp roles (persistent CTAs, one per SM, items strided over the grid): warp 0 = TMA producer, warp 1 =
// MMA issuer (also owns the TMEM allocation), warps 2-9 = split-row softmax / dS (warp w reads TMEM lanes
// 32 (w % 4) ..), warps 10-13 = output group (TMEM -> bf16 -> swizzled staging -> TMA store).
// Numerics follow the oracle's storage points: P and dS are rounded to bf16 (they are MMA
// operands), dS carries the 1/sqrt(dh) scale, O and dQKV are stored bf16, all accumulation is fp32.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "attn.h"
#include "gemm_tc_kernel.cuh"
#include "tuning.h"

// DHEN_RACE_PROBE (test builds only, build.py --probe N): 1 = delay injection on the current protocol,
// 2 = the same delays on round 1's dh = 64 backward protocol.  0 in every product build.
#ifndef DHEN_RACE_PROBE
#define DHEN_RACE_PROBE 0
#endif

namespace dhen {
namespace attn {

using namespace tc;

constexpr int ROWS = 128;          // MMA M / padded token count
constexpr int CHUNK = ROWS * 128;  // one 64-column (128-B) swizzled chunk of 128 rows: 16 KB

struct Params {
  int items, H, m, d;
  float scale;                 // 1 / sqrt(dh)
  __nv_bfloat16* out;          // fwd: O [B][m][d];  bwd: dQKV [B][m][3d]
};

__device__ __forceinline__ void tma_load2(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void sts16(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ uint4 lds16(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
// 32 consecutive fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// Row `row` of a 128-row, 128-B swizzled K-major operand: 16-B granule g (8 bf16) of 64-column chunk c.
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int c, int g) {
  return base + (uint32_t)(c * CHUNK + row * 128 + ((g ^ (row & 7)) << 4));
}
__device__ __forceinline__ uint32_t idesc(int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(ROWS >> 4) << 24);
}
// D (+)= A B over K = 16 * ksteps.  A / B are 128-row (or dh-row) swizzled tiles in shared memory:
//   K-major operand: k-step kk at chunk kk / 4, byte offset (kk % 4) * 32 (SBO 1024 = 8 rows)
//   MN-major operand (the transposed read of a row-major tile): k-step kk = 16 rows -> + kk * 2048,
//   the 64-wide MN chunks are CHUNK apart (LBO)
__device__ __forceinline__ void mma_chain(uint32_t d, uint32_t a, bool a_mn, uint32_t b, bool b_mn, uint32_t id,
                                          int ksteps) {
  for (int kk = 0; kk < ksteps; ++kk) {
    const uint32_t ao = a_mn ? (uint32_t)kk * 2048u : (uint32_t)((kk >> 2) * CHUNK + (kk & 3) * 32);
    const uint32_t bo = b_mn ? (uint32_t)kk * 2048u : (uint32_t)((kk >> 2) * CHUNK + (kk & 3) * 32);
    const uint64_t ad = sdesc(a + ao, a_mn ? CHUNK : 16, 1024);
    const uint64_t bd = sdesc(b + bo, b_mn ? CHUNK : 16, 1024);
    mma_f16(d, ad, bd, id, kk > 0 ? 1u : 0u);
  }
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
// Packed fp32 pairs (FFMA2 / FADD2 / FMUL2 on sm_100): each lane is an ordinary rounded fma / add / mul.
__device__ __forceinline__ uint64_t f2u(float2 a) { return *reinterpret_cast<uint64_t*>(&a); }
__device__ __forceinline__ float2 u2f(uint64_t a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(r);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
__device__ __forceinline__ float ex2(float x) {   // 2^x, MUFU.EX2 (ex2(-inf) = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// The softmax arithmetic, fixed so that every kernel that forms P (forward, and each backward recompute)
// gets bit-identical values:  columns >= m read as -inf;  mx = row max;  e_j = ex2(fma(S_j, k2, -mx k2))
// with k2 = scale log2(e);  per 64-column half, two running sums over the even and odd columns in order,
// half sum = even + odd, row sum = half 0 + half 1;  P_j = e_j * (1 / sum)  (0 for rows >= m).

// Items of this CTA (persistent CTAs, items strided over the grid).
__device__ __forceinline__ int cta_items(int items) {
  return (int)blockIdx.x < items ? (items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
}

// ------------------------------------------------------------------ backward, store group
// One CTA per SM (224 KB of shared memory), items pipelined instead of ping-ponged (two item stages of
// Q | K | V | dO | P would need 320 KB):
//   smem   Q | K  x 2 stages (the next item's Q, K arrive while this one runs), V, dO, P / dS.  The outputs
//          are staged in the bytes of the inputs that are dead by then: dV in V (read by dP), dQ and dK in
//          the item's Q and K (read by dQ / dK); each buffer is reloaded once its stores have read it.
//   TMEM   two 256-column halves, item it in half it & 1:  S [0,128) -> dV -> dQ,  dP [128,256) -> dK.
//          dQ overlays dV, so the dQ MMA waits until dV has been read out.
//   warps  0 TMA producer, 1 MMA issuer, 2-9 softmax recompute + D + dS (two threads per query row, one
//          per 64-column half; S and dP are read from TMEM once and kept in registers),
//          10-13 output group: dV, dQ, dK rows out of TMEM -> bf16 -> swizzled staging -> TMA store
//          (box 64 columns x m rows, so a ragged m never writes past its sample).
__device__ __forceinline__ void tma_store2(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(src)
               : "memory");
}
__device__ __forceinline__ void bar_sync_out() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void bar_sync_rows() { asm volatile("bar.sync 2, 256;" ::: "memory"); }
// 64 fp32 accumulator columns of this thread's TMEM lane -> bf16 -> row `row` of a 128-B swizzled
// staging chunk (the layout a SWIZZLE_128B TMA store reads)
__device__ __forceinline__ void stage_row64(uint32_t taddr, uint32_t slot, int row) {
  float v[64];
  tmem_ld32(taddr, v);
  tmem_ld32(taddr + 32, v + 32);
#pragma unroll
  for (int g = 0; g < 8; ++g)
    sts16(swz(slot, row, 0, g), pack_bf2(v[8 * g], v[8 * g + 1]), pack_bf2(v[8 * g + 2], v[8 * g + 3]),
          pack_bf2(v[8 * g + 4], v[8 * g + 5]), pack_bf2(v[8 * g + 6], v[8 * g + 7]));
}
// Row partials of the two threads that share a query row (warps w, w + 4 of the 8-warp row group),
// through xch[2][128] (shared-window address): returns (half 0's, half 1's).  The leading barrier keeps a
// partner from overwriting a value not yet read.
__device__ __forceinline__ float2 row_exchange(uint32_t xch, int hf, int row, float part) {
  bar_sync_rows();
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(xch + (uint32_t)(hf * ROWS + row) * 4), "f"(part) : "memory");
  bar_sync_rows();
  float2 r;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r.x) : "r"(xch + (uint32_t)row * 4) : "memory");
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r.y) : "r"(xch + (uint32_t)(ROWS + row) * 4) : "memory");
  return r;
}
// Split-row softmax: this thread's 64-column half (c0 = 64 hf) of its S row (TMEM, tS = the row's lane
// base) into bf16 P pairs pk[32], with softmax_row's arithmetic (above).
__device__ __forceinline__ void split_softmax(uint32_t tS, int hf, int row, int m, float scale, uint32_t xch,
                                              uint32_t* pk) {
  const int c0 = 64 * hf, L = m - c0;
  const float k2 = scale * 1.4426950408889634f;
  float v[64];
  tmem_ld32(tS + c0, v);
  tmem_ld32(tS + c0 + 32, v + 32);
  if (L < 64) {
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = j < L ? v[j] : -INFINITY;
  }
  float mx = v[0];
#pragma unroll
  for (int j = 1; j < 64; ++j) mx = fmaxf(mx, v[j]);
  const float2 xm = row_exchange(xch, hf, row, mx);
  const float off = fmaxf(xm.x, xm.y) * k2;
  const float2 kk = make_float2(k2, k2), oo = make_float2(-off, -off);
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < 64; j += 2) {
    const float2 t = fma2(make_float2(v[j], v[j + 1]), kk, oo);
    v[j] = ex2(t.x);
    v[j + 1] = ex2(t.y);
    acc = add2(acc, make_float2(v[j], v[j + 1]));
  }
  const float2 xs = row_exchange(xch, hf, row, acc.x + acc.y);
  const float inv = row < m ? 1.f / (xs.x + xs.y) : 0.f;
  const float2 ii = make_float2(inv, inv);
#pragma unroll
  for (int j = 0; j < 64; j += 2) {
    const float2 q = mul2(make_float2(v[j], v[j + 1]), ii);
    pk[j / 2] = pack_bf2(q.x, q.y);
  }
}

template <int DH>
__global__ void __launch_bounds__(448, 1) attn_bwd_ws(const __grid_constant__ CUtensorMap qkv,
                                                      const __grid_constant__ CUtensorMap dom,
                                                      const __grid_constant__ CUtensorMap dst,
                                                      const __grid_constant__ Params p) {
  pdl_release();
  constexpr int NCH = DH / 64, NB = 6 * NCH + 2;   // NB: 16-KB chunks of shared memory
  constexpr uint32_t C_S = 0, C_DP = 128, C_DV = 0, C_DK = 128, C_DQ = DH == 64 ? 64 : 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  auto sQ = [&](int s) { return sbase + (uint32_t)(s * 2 * NCH * CHUNK); };
  auto sK = [&](int s) { return sbase + (uint32_t)(s * 2 * NCH * CHUNK + NCH * CHUNK); };
  const uint32_t sV = sbase + 4 * NCH * CHUNK, sdO = sV + NCH * CHUNK, sP = sdO + NCH * CHUNK;
  uint64_t* bars = (uint64_t*)(smem + NB * CHUNK);
  auto B_ = [&](int i) { return smem_u32(bars + i); };
  // 0,1 qk_full[s]  2,3 qk_free[s] (stores read)  4 vdo_full  5 s  6 dp  7 p(4)  8 dv  9 ds(4)
  // 10 dv_drained(4)  11 dqk  12,13 tfree[half](4)  14 v_free (dV stores read)
  uint32_t* tslot = (uint32_t*)(bars + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&qkv) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&dom) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&dst) : "memory");
    for (int i = 0; i < 15; ++i)
      mbar_init(B_(i), (i == 7 || i == 9) ? 8 : (i == 10 || i == 12 || i == 13) ? 4 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  const int H = p.H, d = p.d, n = cta_items(p.items);
  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer
      for (int it = 0; it < n; ++it) {
        const int item = blockIdx.x + it * gridDim.x, b = item / H, h = item - b * H, s = it & 1;
        if (it >= 2) mbar_wait(B_(2 + s), ((it >> 1) - 1) & 1);   // item it - 2's dQ / dK stores read Q, K
        mbar_expect_tx(B_(s), 2 * NCH * CHUNK);
        for (int c = 0; c < NCH; ++c) {
          tma_load2(sQ(s) + c * CHUNK, &qkv, h * DH + 64 * c, b * p.m, B_(s));
          tma_load2(sK(s) + c * CHUNK, &qkv, d + h * DH + 64 * c, b * p.m, B_(s));
        }
        if (it >= 1) mbar_wait(B_(8), (it - 1) & 1);   // dO of item it - 1 read by dV
        mbar_expect_tx(B_(4), 2 * NCH * CHUNK);
        for (int c = 0; c < NCH; ++c) tma_load2(sdO + c * CHUNK, &dom, h * DH + 64 * c, b * p.m, B_(4));
        if (it >= 1) mbar_wait(B_(14), (it - 1) & 1);  // item it - 1's dV stores read V's bytes
        for (int c = 0; c < NCH; ++c) tma_load2(sV + c * CHUNK, &qkv, 2 * d + h * DH + 64 * c, b * p.m, B_(4));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer
      const uint32_t id_sq = idesc(ROWS, false, false), id_t = idesc(DH, true, true), id_q = idesc(DH, false, true);
      auto issueS = [&](int it) {
        const int s = it & 1;
        const uint32_t tg = tmem + (uint32_t)(s * 256);
        if (it >= 2) mbar_wait(B_(12 + s), ((it >> 1) - 1) & 1);   // half drained (item it - 2)
        mbar_wait(B_(s), (it >> 1) & 1);
        tc_after();
        mma_chain(tg + C_S, sQ(s), false, sK(s), false, id_sq, DH / 16);   // S = Q K^T
        mma_commit(B_(5));
      };
      if (n > 0) issueS(0);
      for (int it = 0; it < n; ++it) {
        const int s = it & 1;
        const uint32_t tg = tmem + (uint32_t)(s * 256), ph = it & 1;
        mbar_wait(B_(4), ph);
        tc_after();
        mma_chain(tg + C_DP, sdO, false, sV, false, id_sq, DH / 16);   // dP = dO V^T
        mma_commit(B_(6));
        mbar_wait(B_(7), ph);   // P written
        tc_after();
        mma_chain(tg + C_DV, sP, true, sdO, true, id_t, ROWS / 16);    // dV = P^T dO
        mma_commit(B_(8));
        mbar_wait(B_(9), ph);   // dS written
        if (it + 1 < n) issueS(it + 1);   // the next item's softmax input goes first
        tc_after();
        mma_chain(tg + C_DK, sP, true, sQ(s), true, id_t, ROWS / 16);  // dK = dS^T Q
        // dV of this item read out of TMEM by the output group.  For dh = 128 dQ overlays dV; for every dh the
        // wait also keeps barrier 11 (dQ / dK done) from completing for this item before the output group has
        // observed its completion for the previous one: the output group arrives on barrier 10 for item `it`
        // only after its wait on barrier 11 for item it - 1.  Without it (round 1's dh = 64 kernel) two
        // completions of barrier 11 could land while an output warp still waited on the first -- the phase
        // parity then reads "not yet" forever (the intermittent C3 hang, tests/test_gpu_attn.py).
#if DHEN_RACE_PROBE == 2
        if (DH == 128)   // probe build 2: round 1's protocol (reproduces the hang, tests/test_gpu_attn.py)
#endif
        mbar_wait(B_(10), ph);
        tc_after();
        mma_chain(tg + C_DQ, sP, false, sK(s), true, id_q, ROWS / 16); // dQ = dS K
        mma_commit(B_(11));
      }
    }
  } else if (warp < 10) {  // ---------------- softmax recompute, D, dS: two threads per query row
    // warp w and w + 4 share TMEM lanes 32 (w % 4) ..; half hf owns columns [64 hf, 64 hf + 64) of S, P,
    // dP, dS.  Row max, row sum and D = sum_j P_j dP_j are exchanged through xch[2][128].
    const int hf = (warp - 2) >> 2, q4 = warp & 3, row = q4 * 32 + lane, c0 = 64 * hf;
    const uint32_t xch = smem_u32(smem + NB * CHUNK + 256);
    for (int it = 0; it < n; ++it) {
      const uint32_t ph = it & 1;
      const uint32_t tl = tmem + (uint32_t)((it & 1) * 256) + ((uint32_t)(q4 * 32) << 16);
      uint32_t pk[32];
      float v[32];
      mbar_wait(B_(5), ph);
      tc_after();
      split_softmax(tl + C_S, hf, row, p.m, p.scale, xch, pk);
      if (it >= 1) mbar_wait(B_(11), (it - 1) & 1);   // dS of item it - 1 read by dQ / dK
#pragma unroll
      for (int g = 0; g < 8; ++g) sts16(swz(sP, row, hf, g), pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
      fence_async_smem();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(B_(7));
      mbar_wait(B_(6), ph);
      tc_after();
      float2 Dp2 = make_float2(0.f, 0.f);   // dP (fp32) is read from TMEM in 32-column pieces, twice: for D, then dS
#pragma unroll
      for (int hc = 0; hc < 2; ++hc) {
        tmem_ld32(tl + C_DP + c0 + 32 * hc, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t w = pk[16 * hc + j];
          Dp2 = fma2(make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u)),
                     make_float2(v[2 * j], v[2 * j + 1]), Dp2);
        }
      }
      const float Dp = Dp2.x + Dp2.y;
      const float2 xd = row_exchange(xch, hf, row, Dp);
      const float D = xd.x + xd.y;
      const float2 sc2 = make_float2(p.scale, p.scale), nD2 = make_float2(-D, -D);
      mbar_wait(B_(8), ph);   // dV done: P may be overwritten
      tc_after();
#pragma unroll
      for (int hc = 0; hc < 2; ++hc) {
        tmem_ld32(tl + C_DP + c0 + 32 * hc, v);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint32_t qq[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {   // dS = (scale P) (dP - D)
            const uint32_t w = pk[16 * hc + 4 * g + t];
            const float2 sp = mul2(make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u)), sc2);
            const float2 q = mul2(sp, add2(make_float2(v[8 * g + 2 * t], v[8 * g + 2 * t + 1]), nD2));
            qq[t] = pack_bf2(q.x, q.y);
          }
          sts16(swz(sP, row, hf, 4 * hc + g), qq[0], qq[1], qq[2], qq[3]);
        }
      }
      fence_async_smem();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(B_(9));
    }
  } else {                 // ---------------- output group: TMEM -> staging -> TMA store
    const int q4 = warp & 3, row = q4 * 32 + lane;
    const bool leader = warp == 10 && lane == 0;
    auto stage_chunk = [&](uint32_t taddr, uint32_t slot) { stage_row64(taddr, slot, row); };
    for (int it = 0; it < n; ++it) {
      const int item = blockIdx.x + it * gridDim.x, b = item / H, h = item - b * H, s = it & 1;
      const uint32_t ph = it & 1;
      const uint32_t tl = tmem + (uint32_t)((it & 1) * 256) + ((uint32_t)(q4 * 32) << 16);
      const int row0 = b * p.m;
      mbar_wait(B_(8), ph);   // dV done (and dP before it: V is dead)
      tc_after();
      for (int c = 0; c < NCH; ++c) stage_chunk(tl + C_DV + 64 * c, sV + c * CHUNK);
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(B_(10));
      fence_async_smem();
      bar_sync_out();
      if (leader) {
        for (int c = 0; c < NCH; ++c) tma_store2(&dst, sV + c * CHUNK, 2 * d + h * DH + 64 * c, row0);
        bulk_commit();
        bulk_wait_read<0>();
        mbar_arrive(B_(14));
      }
#if DHEN_RACE_PROBE
      // probe builds: warps 11-13 look at barrier 11 only 20 us late (the leader warp on time), the schedule
      // under which round 1's protocol lets barrier 11 complete twice unobserved
      if (warp != 10) for (int k = 0; k < 20; ++k) __nanosleep(1000);
#endif
      mbar_wait(B_(11), ph);   // dQ, dK done (Q, K of this item are dead)
      tc_after();
      for (int c = 0; c < NCH; ++c) stage_chunk(tl + C_DQ + 64 * c, sQ(s) + c * CHUNK);
      for (int c = 0; c < NCH; ++c) stage_chunk(tl + C_DK + 64 * c, sK(s) + c * CHUNK);
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(B_(12 + (it & 1)));
      fence_async_smem();
      bar_sync_out();
      if (leader) {
        for (int c = 0; c < NCH; ++c) {
          tma_store2(&dst, sQ(s) + c * CHUNK, h * DH + 64 * c, row0);
          tma_store2(&dst, sK(s) + c * CHUNK, d + h * DH + 64 * c, row0);
        }
        bulk_commit();
        bulk_wait_read<0>();
        mbar_arrive(B_(2 + s));
      }
    }
    if (leader) bulk_wait_all();
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


// ------------------------------------------------------------------ forward, store group
// Same roles as attn_bwd_ws: warps 0 TMA, 1 MMA, 2-9 split-row softmax, 10-13 O out of TMEM -> staging ->
// TMA store.  NS stages of Q | K | V; P overlays Q (and K when dh = 64) once S is done, and a stage is
// free again as soon as P V is done; O goes through its own staging buffer (dh / 64 chunks).  TMEM: two
// 128-column halves (item it in half it & 1), S [0,128) then O [0, dh) over it.
template <int DH, int NS>
__global__ void __launch_bounds__(448, 1) attn_fwd_ws(const __grid_constant__ CUtensorMap qkv,
                                                      const __grid_constant__ CUtensorMap ost,
                                                      const __grid_constant__ Params p) {
  pdl_release();
  constexpr int NCH = DH / 64, STG = 3 * NCH * CHUNK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sO = sbase + (uint32_t)(NS * STG);
  uint64_t* bars = (uint64_t*)(smem + NS * STG + NCH * CHUNK);
  auto B_ = [&](int i) { return smem_u32(bars + i); };
  // [0,NS) qk_full  [NS,2NS) v_full  [2NS,3NS) stage free (P V done)  then per half h:
  // 3NS+h s_full, 3NS+2+h p_full(8), 3NS+4+h o_full, 3NS+6+h tfree(4)
  const int GB = 3 * NS;
  uint32_t* tslot = (uint32_t*)(bars + GB + 8);
  const uint32_t xch = smem_u32(smem + NS * STG + NCH * CHUNK + 256);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&qkv) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&ost) : "memory");
    for (int i = 0; i < GB; ++i) mbar_init(B_(i), 1);
    for (int h = 0; h < 2; ++h) {
      mbar_init(B_(GB + h), 1); mbar_init(B_(GB + 2 + h), 8); mbar_init(B_(GB + 4 + h), 1); mbar_init(B_(GB + 6 + h), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  const int H = p.H, d = p.d, n = cta_items(p.items);
  auto sQ = [&](int s) { return sbase + (uint32_t)(s * STG); };
  auto sK = [&](int s) { return sbase + (uint32_t)(s * STG + NCH * CHUNK); };
  auto sV = [&](int s) { return sbase + (uint32_t)(s * STG + 2 * NCH * CHUNK); };
  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer
      for (int it = 0; it < n; ++it) {
        const int item = blockIdx.x + it * gridDim.x, b = item / H, h = item - b * H, s = it % NS;
        if (it >= NS) mbar_wait(B_(2 * NS + s), ((it / NS) - 1) & 1);   // P V of item it - NS done
        mbar_expect_tx(B_(s), 2 * NCH * CHUNK);
        for (int c = 0; c < NCH; ++c) {
          tma_load2(sQ(s) + c * CHUNK, &qkv, h * DH + 64 * c, b * p.m, B_(s));
          tma_load2(sK(s) + c * CHUNK, &qkv, d + h * DH + 64 * c, b * p.m, B_(s));
        }
        mbar_expect_tx(B_(NS + s), NCH * CHUNK);
        for (int c = 0; c < NCH; ++c) tma_load2(sV(s) + c * CHUNK, &qkv, 2 * d + h * DH + 64 * c, b * p.m, B_(NS + s));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer
      const uint32_t id_s = idesc(ROWS, false, false), id_o = idesc(DH, false, true);
      auto issueS = [&](int it) {
        const int s = it % NS, hh = it & 1;
        if (it >= 2) mbar_wait(B_(GB + 6 + hh), ((it >> 1) - 1) & 1);   // O of item it - 2 read out
        mbar_wait(B_(s), (it / NS) & 1);
        tc_after();
        mma_chain(tmem + hh * 128, sQ(s), false, sK(s), false, id_s, DH / 16);   // S = Q K^T
        mma_commit(B_(GB + hh));
      };
      if (n > 0) issueS(0);
      for (int it = 0; it < n; ++it) {
        if (it + 1 < n) issueS(it + 1);
        const int s = it % NS, hh = it & 1;
        mbar_wait(B_(GB + 2 + hh), (it >> 1) & 1);   // P written
        mbar_wait(B_(NS + s), (it / NS) & 1);        // V landed
        tc_after();
        mma_chain(tmem + hh * 128, sQ(s), false, sV(s), true, id_o, ROWS / 16);   // O = P V (P overlays Q)
        mma_commit(B_(GB + 4 + hh));
        mma_commit(B_(2 * NS + s));
      }
    }
  } else if (warp < 10) {  // ---------------- split-row softmax
    const int hf = (warp - 2) >> 2, q4 = warp & 3, row = q4 * 32 + lane;
    for (int it = 0; it < n; ++it) {
      const int s = it % NS, hh = it & 1;
      mbar_wait(B_(GB + hh), (it >> 1) & 1);
      tc_after();
      uint32_t pk[32];
      split_softmax(tmem + (uint32_t)(hh * 128) + ((uint32_t)(q4 * 32) << 16), hf, row, p.m, p.scale, xch, pk);
#pragma unroll
      for (int g = 0; g < 8; ++g) sts16(swz(sQ(s), row, hf, g), pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
      fence_async_smem();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(B_(GB + 2 + hh));
    }
  } else {                 // ---------------- output group
    const int q4 = warp & 3, row = q4 * 32 + lane;
    const bool leader = warp == 10 && lane == 0;
    for (int it = 0; it < n; ++it) {
      const int item = blockIdx.x + it * gridDim.x, b = item / H, h = item - b * H, hh = it & 1;
      mbar_wait(B_(GB + 4 + hh), (it >> 1) & 1);   // O done
      tc_after();
      if (leader) bulk_wait_read<0>();   // the previous item's O store has read the staging buffer
      bar_sync_out();
      const uint32_t tl = tmem + (uint32_t)(hh * 128) + ((uint32_t)(q4 * 32) << 16);
      for (int c = 0; c < NCH; ++c) stage_row64(tl + 64 * c, sO + c * CHUNK, row);
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(B_(GB + 6 + hh));
      fence_async_smem();
      bar_sync_out();
      if (leader) {
        for (int c = 0; c < NCH; ++c) tma_store2(&ost, sO + c * CHUNK, h * DH + 64 * c, b * p.m);
        bulk_commit();
      }
    }
    if (leader) bulk_wait_all();
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
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
// [B * m][cols] bf16 -> 2-D map, box 64 columns x 128 rows, 128-B swizzle.  An item's tile starts at row
// b * m; its rows m..127 hold the next samples' (finite) rows, or the zero fill past the tensor end, and
// the kernels never let them reach a result (columns >= m of P and dS are 0, rows >= m are not stored).
// (A 3-D [B][m][cols] map with the box taller than m, i.e. out-of-bounds rows inside the tensor, hung
// the forward on B200 — measured; the 2-D form keeps every out-of-bounds box at the tensor end.)
static bool map2(CUtensorMap* map, const void* ptr, int cols, int64_t rows) {
  EncodeFn fn = encode_fn();
  if (!fn || ((uintptr_t)ptr & 15) || (cols * 2) % 16 || rows < ROWS) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)ROWS}, es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Store map over the same [B * m][cols] tensor with box 64 columns x m rows (one sample's rows exactly).
static bool map2_store(CUtensorMap* map, const void* ptr, int cols, int64_t rows, int m) {
  EncodeFn fn = encode_fn();
  if (!fn || ((uintptr_t)ptr & 15) || (cols * 2) % 16 || m < 1 || m > ROWS) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)m}, es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool fused_ok(int dt, int B, int H, int m, int d) {
  if (!tune().attn_fused || dt != BF16 || H <= 0 || d % H) return false;
  const int dh = d / H;
  return (dh == 64 || dh == 128) && m >= 1 && m <= ROWS && (int64_t)B * m >= ROWS && (int64_t)B * H < (1ll << 31) &&
         (int64_t)B * m < (1ll << 31);
}

static int sm_count() {
  static int sms = 0;
  if (!sms) { int dev = 0; cudaGetDevice(&dev); cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev); }
  return sms;
}

// Forward: warp-specialised store-group kernel, one CTA per SM, NS item stages of Q | K | V (NS = 4 / 2 for
// dh = 64 / 128: 192 KB), split-row softmax, O through a TMA store with a box of m rows.
cudaError_t core_fwd(const void* QKV, void* O, int B, int H, int m, int d, cudaStream_t st) {
  if (!fused_ok(BF16, B, H, m, d)) return cudaErrorNotSupported;
  const int dh = d / H;
  CUtensorMap mq, ms;
  if (!map2(&mq, QKV, 3 * d, (int64_t)B * m) || !map2_store(&ms, O, d, (int64_t)B * m, m)) return cudaErrorNotSupported;
  Params p;
  p.items = B * H; p.H = H; p.m = m; p.d = d; p.scale = 1.f / sqrtf((float)dh); p.out = (__nv_bfloat16*)O;
  const int nch = dh / 64, ns = dh == 64 ? 4 : 2;
  const int smem = (ns * 3 + 1) * nch * CHUNK + 1024 + 256 + 2 * ROWS * 4;
  const int grid = std::min(p.items, sm_count());
  if (dh == 64) {
    static bool a = false;
    if (!a) { cudaFuncSetAttribute(attn_fwd_ws<64, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); a = true; }
    pdl_launch(attn_fwd_ws<64, 4>, grid, 448, smem, st, mq, ms, p);
  } else {
    static bool a = false;
    if (!a) { cudaFuncSetAttribute(attn_fwd_ws<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); a = true; }
    pdl_launch(attn_fwd_ws<128, 2>, grid, 448, smem, st, mq, ms, p);
  }
  ++g_launches;
  return cudaGetLastError();
}

// Backward: pipelined items (Q | K double-buffered), split-row softmax recompute, outputs staged in dead input
// bytes and stored by TMA.
cudaError_t core_bwd(const void* QKV, const void* dO, void* dQKV, int B, int H, int m, int d, cudaStream_t st) {
  if (!fused_ok(BF16, B, H, m, d)) return cudaErrorNotSupported;
  const int dh = d / H;
  CUtensorMap mq, mo, ms;
  if (!map2(&mq, QKV, 3 * d, (int64_t)B * m) || !map2(&mo, dO, d, (int64_t)B * m) ||
      !map2_store(&ms, dQKV, 3 * d, (int64_t)B * m, m))
    return cudaErrorNotSupported;
  Params p;
  p.items = B * H; p.H = H; p.m = m; p.d = d; p.scale = 1.f / sqrtf((float)dh); p.out = (__nv_bfloat16*)dQKV;
  const int nch = dh / 64;
  const int smem = (6 * nch + 2) * CHUNK + 1024 + 256 + 2 * ROWS * 4;   // + row exchange
  const int grid = std::min(p.items, sm_count());
  if (dh == 64) {
    static bool a = false;
    if (!a) { cudaFuncSetAttribute(attn_bwd_ws<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); a = true; }
    pdl_launch(attn_bwd_ws<64>, grid, 448, smem, st, mq, mo, ms, p);
  } else {
    static bool a = false;
    if (!a) { cudaFuncSetAttribute(attn_bwd_ws<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); a = true; }
    pdl_launch(attn_bwd_ws<128>, grid, 448, smem, st, mq, mo, ms, p);
  }
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace attn
}  // namespace dhen
