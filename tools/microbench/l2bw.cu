// L2 / HBM throughput probes for the L2-blocked step's design (design probe, not product).
//   RMW   : read-modify-write of an L2-resident working set (SM<->L2 traffic only)
//   COPY  : HBM stream copy src -> dst (4 GiB each)
//   TWICE : the L2-blocked step without arithmetic: per 32 MiB chunk, every
//           element is read from HBM and written back (pass A), then read and
//           written again (pass B) while it is still in L2. Grid-wide chunk
//           counters order B(c) after A(c), one chunk of lag (like qaa_superpass).
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
__global__ void __launch_bounds__(256) copyk(const double2* __restrict__ s, double2* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256 * 4) {
    double2 v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) { int64_t j = i + k * (int64_t)gridDim.x * 256; v[k] = j < n ? s[j] : make_double2(0, 0); }
#pragma unroll
    for (int k = 0; k < 4; k++) { int64_t j = i + k * (int64_t)gridDim.x * 256; if (j < n) d[j] = v[k]; }
  }
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// items: A(0), [A(1) B(0)], [A(2) B(1)], ... each item = one 64 KiB block of a chunk;
// A blocks: contiguous 64 KiB; B blocks: 512 rows of 128 B strided by 64 KiB (the
// group-k tile shape). Static round robin over the persistent grid.
__global__ void __launch_bounds__(512, 1) twice(double2* p, int nch, int tpc, unsigned* done, int evict) {
  const int64_t per = (int64_t)tpc * 4096;  // amps per chunk
  const int64_t nitems = (int64_t)(nch + 1) * tpc * 2;
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    int64_t seg = it / (2 * tpc), r = it % (2 * tpc);
    int kind, c, t;
    if (seg == 0) { if (r >= tpc) continue; kind = 0; c = 0; t = (int)r; }
    else if (r < tpc) { kind = 0; c = (int)seg; t = (int)r; if (c >= nch) continue; }
    else { kind = 1; c = (int)seg - 1; t = (int)(r - tpc); }
    double2* base = p + c * per;
    if (kind == 1) {
      if (threadIdx.x == 0) while (ld_acq(&done[c]) < (unsigned)tpc) __nanosleep(64);
      __syncthreads();
    }
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      int l = threadIdx.x + 512 * k;  // 0..4095
      int64_t off = kind == 0 ? (int64_t)t * 4096 + l : (int64_t)(l >> 3) * 4096 + t * 8 + (l & 7);
      v[k] = base[off];
    }
#pragma unroll
    for (int k = 0; k < 8; k++) {
      int l = threadIdx.x + 512 * k;
      int64_t off = kind == 0 ? (int64_t)t * 4096 + l : (int64_t)(l >> 3) * 4096 + t * 8 + (l & 7);
      double2 w = make_double2(v[k].x * 1.0000001, v[k].y);
      double2* q = base + off;
      if (evict && kind == 0)
        asm volatile("{.reg .b64 pol; createpolicy.fractional.L2::evict_last.b64 pol, 1.0; st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, pol;}" :: "l"(q), "d"(w.x), "d"(w.y) : "memory");
      else if (evict)
        asm volatile("{.reg .b64 pol; createpolicy.fractional.L2::evict_first.b64 pol, 1.0; st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, pol;}" :: "l"(q), "d"(w.x), "d"(w.y) : "memory");
      else
        *q = w;
    }
    if (kind == 0) {
      __syncthreads();
      if (threadIdx.x == 0) { __threadfence(); atomicAdd(&done[c], 1u); }
    }
  }
}
int main() {
  double2 *p, *q;
  cudaMalloc(&p, 1ull << 34);
  cudaMalloc(&q, 1ull << 32);
  cudaMemset(p, 0, 1ull << 34);
  cudaMemset(q, 0, 1ull << 32);
  unsigned* done;
  cudaMalloc(&done, 4096 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int64_t mb : {16, 32, 64, 96}) {
    int64_t n = mb * (1 << 20) / 16;
    int reps = 50;
    for (int occ : {2, 4, 8}) {
      rmw<<<148 * occ, 256>>>(p, n, 2);
      cudaEventRecord(a);
      rmw<<<148 * occ, 256>>>(p, n, reps);
      cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("RMW %5lld MiB occ %d: %.3f ms  %.1f GB/s (SM<->L2 read+write)\n", (long long)mb, occ, ms, 2.0 * n * 16 * reps / ms / 1e6);
    }
  }
  {
    int64_t n = (1ll << 32) / 16;
    for (int occ : {4, 8}) {
      copyk<<<148 * occ, 256>>>(p, q, n);
      cudaEventRecord(a);
      for (int r = 0; r < 5; r++) copyk<<<148 * occ, 256>>>(p + (r & 1) * n, q, n);
      cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("COPY 4 GiB occ %d: %.3f ms per copy  %.1f GB/s (read+write)\n", occ, ms / 5, 2.0 * n * 16 * 5 / ms / 1e6);
    }
  }
  // 16 GiB state, 2^21-amp chunks (512 of them), 512 tiles per chunk
  for (int evict : {0, 1}) {
    for (int grid : {148, 296}) for (int rep = 0; rep < 2; rep++) {
      cudaMemset(done, 0, 4096 * 4);
      cudaEventRecord(a);
      twice<<<grid, 512>>>(p, 512, 512, done, evict);
      cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("TWICE grid %d 16 GiB evict %d: %.3f ms  (2^30 amps: %.1f GB/s algorithmic 32 B/amp)  err=%s\n", grid, evict, ms,
             32.0 * (1ll << 30) / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
