// common.cuh — shared device helpers of the DHEN sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace dhen {

enum Dt : int { F32 = 0, BF16 = 1 };

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
