// Isolated store-pattern microbenchmark: does the GEMM epilogue's store pattern itself reach HBM rates?
// grid = 148 CTAs, W warps per CTA, each warp writes 32 rows x 32 fp32 (128 B per row, 8 lanes x 16 B)
// per item, ITEMS items per CTA, rows of a [M][32] fp32 matrix (like x.kmaj_rowmajor's output).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_store(float* out, int items, int mode) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int it = 0; it < items; ++it) {
    const int tile = blockIdx.x + it * gridDim.x;          // 128-row tile
    const int rbase = tile * 128 + (warp % 4) * 32;
    if (mode == 0) {     // 8 lanes per row, 4 rows per instruction (the epilogue pattern)
      const int sub = lane / 8, cl = lane % 8;
      for (int r = sub; r < 32; r += 4) {
        float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
        *reinterpret_cast<float4*>(out + (size_t)(rbase + r) * 32 + 4 * cl) = v;
      }
    } else {             // fully contiguous: warp writes 4 KB linearly
      float4* base = reinterpret_cast<float4*>(out + (size_t)rbase * 32);
      for (int q = lane; q < 256; q += 32) base[q] = make_float4(1.f, 2.f, 3.f, 4.f);
    }
    if (nw > 4 && warp >= 4) {}  // extra warps idle
  }
}
int main() {
  const int items = 14, grid = 148;
  size_t M = (size_t)grid * items * 128;
  float* out;
  cudaMalloc(&out, M * 32 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8}) {
      for (int rep = 0; rep < 3; ++rep) k_store<<<grid, warps * 32>>>(out, items, mode);
      cudaEventRecord(a);
      for (int rep = 0; rep < 10; ++rep) k_store<<<grid, warps * 32>>>(out, items, mode);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 10;
      double bytes = (double)M * 32 * 4 * (warps == 8 ? 1 : 1);
      printf("mode %d warps %d: %.1f us  %.0f GB/s\n", mode, warps, ms * 1e3, bytes / ms / 1e6);
    }
  return 0;
}
