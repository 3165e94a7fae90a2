// DRAM efficiency of the access patterns of the Trotter passes (design probe, not product):
// one pass over a 16 GiB array (in place), each 64 KiB tile read and written back with
// contiguous 64 KiB blocks or with rows of R bytes strided by 64 KiB (the group-k tile
// shape: rows of 2^c amplitudes, the other tile bits 64 KiB apart).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
// tile t: contiguous -> base t*4096 amps; rows of ra amps -> row r (0..4096/ra-1) at
// (r * 4096) + (t % (4096/ra)) * ra + (t / (4096/ra)) * 4096 * (4096/ra)  [a 4096/ra x 4096 transpose block]
__device__ __forceinline__ int64_t off(int64_t t, int l, int ra) {
  if (ra == 0) return t * 4096 + l;
  const int rows = 4096 / ra;  // rows per tile
  const int64_t blk = t / rows, col = t % rows;
  const int r = l / ra, e = l % ra;
  return blk * 4096 * (int64_t)rows + (int64_t)r * 4096 + col * ra + e;
}
__global__ void __launch_bounds__(512) pass(double2* p, int64_t ntiles, int rin, int rout) {
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = p[off(t, threadIdx.x + 512 * k, rin)];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; k++) {
      double2 w = make_double2(v[k].x * 1.0000001, v[k].y);
      p[off(t, threadIdx.x + 512 * k, rout)] = w;
    }
  }
}
int main() {
  double2* p;
  const int64_t n = 1ll << 30;
  cudaMalloc(&p, n * 16);
  cudaMemset(p, 0, n * 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int64_t nt = n / 4096;
  int cfg[][2] = {{0, 0}, {8, 8}, {0, 8}, {8, 0}, {16, 16}, {32, 32}, {64, 64}, {0, 16}, {0, 32}};
  for (auto& c : cfg) {
    for (int occ : {2, 3}) {
      pass<<<148 * occ, 512>>>(p, nt, c[0], c[1]);
      cudaEventRecord(a);
      for (int r = 0; r < 3; r++) pass<<<148 * occ, 512>>>(p, nt, c[0], c[1]);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 3;
      printf("read rows %4d B  write rows %4d B (0 = contiguous 64 KiB)  occ %d: %.3f ms  %.0f GB/s  %s\n",
             c[0] * 16, c[1] * 16, occ, ms, 32.0 * n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
