// HBM write-bandwidth microbenchmark: is ~3.9 TB/s (memset / fill) the write ceiling of this B200, or do other store
// paths go faster?  Each method writes the same 4 GiB buffer; CUDA events around 10 launches after 3 warm-ups.
//   memset       cudaMemsetAsync
//   st.v4        grid-stride float4 stores (148 x 8 CTAs of 256 threads)
//   st.v4.cs     the same with the streaming (evict-first) hint
//   bulk S       TMA bulk stores (cp.async.bulk.global.shared::cta) of an S-byte shared buffer, one thread a CTA
//                issuing, up to 8 groups in flight; 148 x k CTAs
//   rw copy      read + write (float4 copy of 2 GiB into 2 GiB) for the mixed-traffic figure
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/write_bw tools/micro/write_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_st(float4* out, size_t n) {
  const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = v;
}
__global__ void k_stcs(float4* out, size_t n) {
  const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) __stcs(out + i, v);
}
__global__ void k_copy(const float4* __restrict__ in, float4* out, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = in[i];
}
template <int S>
__global__ void k_bulk(char* out, size_t nchunks) {
  extern __shared__ __align__(128) char sm[];
  for (int i = threadIdx.x; i < S / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm);
  int k = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * S), "r"(src), "r"(S)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (++k >= 8) asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
static double timeit(F f, size_t bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 0; }
  return bytes / (ms / 10 * 1e-3) / 1e9;
}

int main() {
  const size_t bytes = 4ull << 30;
  char* buf;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  const size_t n4 = bytes / 16;
  printf("memset        %7.0f GB/s\n", timeit([&] { cudaMemsetAsync(buf, 0, bytes); }, bytes));
  for (int bpsm : {4, 8, 16})
    printf("st.v4    x%-2d  %7.0f GB/s\n", bpsm, timeit([&] { k_st<<<148 * bpsm, 256>>>((float4*)buf, n4); }, bytes));
  for (int bpsm : {4, 8, 16})
    printf("st.v4.cs x%-2d  %7.0f GB/s\n", bpsm, timeit([&] { k_stcs<<<148 * bpsm, 256>>>((float4*)buf, n4); }, bytes));
  cudaFuncSetAttribute(k_bulk<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaFuncSetAttribute(k_bulk<65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int bpsm : {1, 2, 4})
    printf("bulk 16K x%-2d  %7.0f GB/s\n", bpsm,
           timeit([&] { k_bulk<16384><<<148 * bpsm, 128, 16384>>>(buf, bytes / 16384); }, bytes));
  for (int bpsm : {1, 2, 3})
    printf("bulk 64K x%-2d  %7.0f GB/s\n", bpsm,
           timeit([&] { k_bulk<65536><<<148 * bpsm, 128, 65536>>>(buf, bytes / 65536); }, bytes));
  const size_t h4 = n4 / 2;
  printf("copy (r+w)    %7.0f GB/s\n", timeit([&] { k_copy<<<148 * 8, 256>>>((const float4*)buf, (float4*)buf + h4, h4); }, bytes));
  return 0;
}
