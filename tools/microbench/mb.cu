// Micro-benchmarks for design decisions (not product code): fp64 FMA rate,
// HBM streaming with contiguous vs 128B/256B-row strided tiles, SHFL rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
  for (int i = 0; i < 16; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0; for (int i = 0; i < 16; i++) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void shfl_kernel(double* out, int iters) {
  int v[16]; for (int i = 0; i < 16; i++) v[i] = threadIdx.x * i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __shfl_xor_sync(0xffffffff, v[i], 1 + (i & 15)) + 1;
  }
  int s = 0; for (int i = 0; i < 16; i++) s += v[i];
  if (s == 1234567) out[0] = s;
}

// in-place RMW over tiles: tile = 2^12 amps (16B each) = rows of 2^c amps at stride
// 'stride_amps' between rows; nrows = 2^(12-c). Block handles tiles in grid-stride.
__global__ void __launch_bounds__(256) tile_rmw(double2* psi, int64_t ntiles, int c, int row_shift) {
  // tile t: low c bits of amp index inside row; rows indexed by r (12-c bits) placed at bit 'row_shift'
  // remaining tile-id bits: low part (row_shift - c bits) placed at bit c, high part above row_shift+12-c
  int rb = 12 - c;
  int lowbits = row_shift - c;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int64_t tlo = t & ((1LL << lowbits) - 1);
    int64_t thi = t >> lowbits;
    int64_t base = (tlo << c) | (thi << (row_shift + rb));
    double2 v[16];
#pragma unroll
    for (int r = 0; r < 16; r++) {
      int l = threadIdx.x + 256 * r;
      int64_t off = (l & ((1 << c) - 1)) | ((int64_t)(l >> c) << row_shift);
      v[r] = psi[base + off];
    }
#pragma unroll
    for (int r = 0; r < 16; r++) { v[r].x *= 1.0000001; v[r].y *= 0.9999999; }
#pragma unroll
    for (int r = 0; r < 16; r++) {
      int l = threadIdx.x + 256 * r;
      int64_t off = (l & ((1 << c) - 1)) | ((int64_t)(l >> c) << row_shift);
      psi[base + off] = v[r];
    }
  }
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("GPU %s SMs %d smemPerBlockOptin %zu smemPerSM %zu regsPerSM %d L2 %d clock(kHz) %d memclk %d busw %d\n", p.name,
         p.multiProcessorCount, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor,
         p.l2CacheSize, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int rep = 0; rep < 3; rep++) {
    int blocks = p.multiProcessorCount * 8, threads = 256;
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * iters * 16;
    printf("DFMA: %.3f ms  %.2f TFMA/s  = %.2f TFLOP/s\n", ms, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  }
  for (int rep = 0; rep < 2; rep++) {
    int blocks = p.multiProcessorCount * 8, threads = 256;
    cudaEventRecord(e0);
    shfl_kernel<<<blocks, threads>>>(d, 4000);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)blocks * threads / 32 * 4000 * 16;
    printf("SHFL: %.3f ms  %.3f warp-shfl/clk/SM at %d MHz\n", ms, n / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3), p.clockRate/1000);
  }
  // HBM: 2^30 amps = 16 GiB
  int64_t N = 1LL << 30;
  double2* psi; CK(cudaMalloc(&psi, N * 16));
  CK(cudaMemset(psi, 0, N * 16));
  int64_t ntiles = N >> 12;
  struct Cfg { int c, row_shift; const char* name; } cfgs[] = {
    {12, 12, "contiguous 64KiB tiles"}, {3, 12, "128B rows stride 2^12 (16 pages/tile)"},
    {3, 13, "128B rows stride 2^13 (32 pages/tile)"}, {3, 14, "128B rows stride 2^14 (64 pages/tile)"},
    {3, 15, "128B rows stride 2^15 (128 pages/tile)"}, {3, 16, "128B rows stride 2^16 (256 pages/tile)"},
    {3, 17, "128B rows stride 2^17 (512 pages/tile)"}, {3, 21, "128B rows stride 2^21 (512 pages/tile)"},
    {4, 12, "256B rows stride 2^12"}, {4, 22, "256B rows stride 2^22"}};
  for (auto& cf : cfgs) {
    for (int occ = 1; occ <= 4; occ *= 2) {
      int blocks = p.multiProcessorCount * occ;
      tile_rmw<<<blocks, 256>>>(psi, ntiles, cf.c, cf.row_shift);
      CK(cudaDeviceSynchronize());
      float best = 1e30;
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        tile_rmw<<<blocks, 256>>>(psi, ntiles, cf.c, cf.row_shift);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("RMW %-36s occ %d: %.3f ms  %.1f GB/s\n", cf.name, occ, best, 2.0 * N * 16 / best / 1e6);
    }
  }
  return 0;
}
