// common.cuh — shared device helpers of the DHEN sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <cstdio>

namespace dhen {

enum Dt : int { F32 = 0, BF16 = 1 };

// Programmatic dependent launch (PDL).  Every library kernel is launched with pdl_launch (the launch attribute
// lets it start while the previous kernel on the stream drains) and calls pdl_entry() before touching global
// memory: it releases its own dependents at once, then waits until its prerequisite grid has completed and its
// writes are visible (griddepcontrol.wait; a no-op for a launch without the attribute).  A dependent grid only
// launches after every CTA of its primary has triggered, so a primary's CTAs are never starved of SMs.
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_entry() {
  pdl_release();
  pdl_wait();
}
int pdl_enabled();   // env DHEN_PDL (default 0): 1 launches with programmatic stream serialization (measured: C2 neutral, C3 -2%)
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// mbarrier phase waits.  Every kernel's waits go through these.  Built with -DDHEN_WATCHDOG=1 (the
// `python -m paper_2203_11014_b200.build --watchdog` library, libdhen_wd.so) a wait that has not completed
// after DHEN_WATCHDOG_NS of wall time prints the block, thread, barrier address, expected parity, the
// mbarrier's raw state and the call site, then traps: a lost arrive or a phase mismatch becomes a reported
// launch failure instead of a silent hang.  The default build spins without a bound (no extra instructions).
#ifndef DHEN_WATCHDOG
#define DHEN_WATCHDOG 0
#endif
#ifndef DHEN_WATCHDOG_NS
#define DHEN_WATCHDOG_NS 4000000000ull
#endif
__device__ __forceinline__ uint32_t mbar_try_parity(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok;
}
__device__ __forceinline__ uint32_t mbar_try_parity_cluster(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __noinline__ inline void mbar_timeout(uint32_t a, uint32_t parity, const char* file, int line) {
  uint64_t raw;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(raw) : "r"(a) : "memory");
  uint32_t dsm;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsm));
  printf("DHEN watchdog: %s:%d block (%d,%d) of %d thread %d: mbarrier smem+0x%x parity %u not completed; raw 0x%016llx "
         "(dynamic smem %u)\n",
         file, line, blockIdx.x, blockIdx.y, gridDim.x, threadIdx.x, a, parity, (unsigned long long)raw, dsm);
  __trap();
}
template <bool CLUSTER>
__device__ __forceinline__ void mbar_wait_impl(uint32_t a, uint32_t parity, const char* file, int line) {
#if DHEN_WATCHDOG
  if (CLUSTER ? mbar_try_parity_cluster(a, parity) : mbar_try_parity(a, parity)) return;
  const uint64_t t0 = global_ns();
  for (uint32_t n = 1;; ++n) {
    if (CLUSTER ? mbar_try_parity_cluster(a, parity) : mbar_try_parity(a, parity)) return;
    if ((n & 255u) == 0u && global_ns() - t0 > DHEN_WATCHDOG_NS) mbar_timeout(a, parity, file, line);
  }
#else
  (void)file; (void)line;
  if (CLUSTER) {
    asm volatile(
        "{\n.reg .pred p;\nWAITC_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAITC_%=;\n}\n" ::"r"(a),
        "r"(parity), "r"(0x989680)
        : "memory");
  } else {
    // no suspend-time hint: try_wait blocks for a hardware-defined window and the loop re-polls, so a waiter
    // (the MMA issuer above all) resumes as soon as the phase completes
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
  }
#endif
}

__device__ __forceinline__ float ld_as_f32(const void* p, int64_t i, int dt) {
  return dt == F32 ? static_cast<const float*>(p)[i]
                   : __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}
__device__ __forceinline__ void st_from_f32(void* p, int64_t i, int dt, float v) {
  if (dt == F32) static_cast<float*>(p)[i] = v;
  else static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
}

template <typename T> __device__ __forceinline__ float tof(T v);
template <> __device__ __forceinline__ float tof<float>(float v) { return v; }
template <> __device__ __forceinline__ float tof<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T fromf(float v);
template <> __device__ __forceinline__ float fromf<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 fromf<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// A strided (optionally doubly-batched) matrix view: element (z, r, c) lives at
// ptr + (z / zdiv) * bs0 + (z % zdiv) * bs1 + R(r) + c * cs   (elements),
// R(r) = r * rs, or with a two-level row index (rdiv > 0): (r / rdiv) * rs_o + (r % rdiv) * rs.
struct View {
  void* ptr;
  int64_t rs, cs, bs0, bs1;
  int zdiv;
  int dt;
  int rdiv;
  int64_t rs_o;
  __host__ __device__ int64_t off(int64_t z, int64_t r, int64_t c) const {
    int64_t o = c * cs;
    if (zdiv == 1) o += z * bs0; else o += (z / zdiv) * bs0 + (z % zdiv) * bs1;
    if (rdiv) o += (r / rdiv) * rs_o + (r % rdiv) * rs; else o += r * rs;
    return o;
  }
};

inline View view(void* p, int dt, int64_t rs, int64_t cs, int64_t bs0 = 0, int64_t bs1 = 0, int zdiv = 1) {
  View v;
  v.ptr = p; v.rs = rs; v.cs = cs; v.bs0 = bs0; v.bs1 = bs1; v.zdiv = zdiv; v.dt = dt;
  v.rdiv = 0; v.rs_o = 0;
  return v;
}
// two-level rows: r -> (r / rdiv) * rs_o + (r % rdiv) * rs
inline View view2(void* p, int dt, int rdiv, int64_t rs_o, int64_t rs, int64_t cs) {
  View v = view(p, dt, rs, cs);
  v.rdiv = rdiv; v.rs_o = rs_o;
  return v;
}
inline View noview() { return view(nullptr, F32, 0, 0); }

}  // namespace dhen
