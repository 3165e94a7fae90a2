// L2 read-modify-write bandwidth for L2-resident working sets (design probe).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) rmw(double2* p, int64_t n, int reps) {
  for (int rep = 0; rep < reps; rep++) {
    for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256 * 4) {
      double2 v[4];
#pragma unroll
      for (int k = 0; k < 4; k++) { int64_t j = i + k * (int64_t)gridDim.x * 256; v[k] = j < n ? p[j] : make_double2(0, 0); }
#pragma unroll
      for (int k = 0; k < 4; k++) { int64_t j = i + k * (int64_t)gridDim.x * 256; if (j < n) p[j] = make_double2(v[k].x * 1.0000001, v[k].y); }
    }
  }
}
int main() {
  double2* p; cudaMalloc(&p, 1ull << 32); cudaMemset(p, 0, 1ull << 32);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int64_t mb : {8, 16, 32, 48, 64, 96, 128, 4096}) {
    int64_t n = mb * (1 << 20) / 16;
    int reps = mb >= 1024 ? 2 : 50;
    for (int occ : {2, 4, 8}) {
      rmw<<<148 * occ, 256>>>(p, n, 2);
      cudaEventRecord(a);
      rmw<<<148 * occ, 256>>>(p, n, reps);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("RMW %5lld MiB occ %d: %.3f ms  %.1f GB/s (read+write)\n", (long long)mb, occ, ms, 2.0 * n * 16 * reps / ms / 1e6);
    }
  }
  return 0;
}
