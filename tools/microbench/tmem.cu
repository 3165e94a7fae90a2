// Micro-benchmark (design decision, not product code): is tensor memory a
// usable second exchange path beside shared memory for the fused Trotter pass?
// Measures per-SM throughput of tcgen05.st / tcgen05.ld (32x32b, 16x256b
// shapes) against LDS.128 / STS.128, alone and concurrently, with 16 warps per
// SM (the superpass's occupancy). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem tools/microbench/tmem.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("ERR %s line %d: %s\n", #x, __LINE__, cudaGetErrorString(e));      \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__device__ __forceinline__ void tm_alloc(uint32_t* dst, int cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tm_dealloc(uint32_t a, int cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(a), "r"(cols));
}
__device__ __forceinline__ void st32x32x16(uint32_t ta, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void ld32x32x16(uint32_t ta, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta)
      : "memory");
}
__device__ __forceinline__ void ld16x256x4(uint32_t ta, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta)
      : "memory");
}
__device__ __forceinline__ void st16x256x4(uint32_t ta, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// mode: 0 tmem st 32x32b, 1 tmem ld 32x32b, 2 tmem ld 16x256b, 3 smem LDS.128,
// 4 smem STS.128, 5 half warps LDS + half LDTM 32x32b, 6 round trip st32x32 + ld16x256 (+waits),
// 7 round trip via smem (STS + bar + LDS), 8 tmem st 16x256b
// ldbatch: loads issued before one wait (1, 2, 4)
__global__ void __launch_bounds__(512, 1) bench(int mode, int iters, int ldbatch, unsigned long long* cyc,
                                                uint32_t* sink) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tm_alloc(&taddr_s, 512);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
  uint32_t r[16], acc = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) r[i] = threadIdx.x * 16 + i;
  uint4* sv = reinterpret_cast<uint4*>(smem);
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const uint32_t col = (uint32_t)((it & 3) * 32);
    if (mode == 0 || mode == 8) {
      if (mode == 0)
        st32x32x16(tbase + col, r);
      else
        st16x256x4(tbase + col, r);
      if ((it & (ldbatch - 1)) == ldbatch - 1) wait_st();
      r[0] += 1;
    } else if (mode == 1 || mode == 2 || (mode == 5 && (warp & 4))) {
      if (mode == 2)
        ld16x256x4(tbase + col, r);
      else
        ld32x32x16(tbase + col, r);
      if ((it & (ldbatch - 1)) == ldbatch - 1) wait_ld();
#pragma unroll
      for (int i = 0; i < 16; i++) acc ^= r[i];
    } else if (mode == 3 || mode == 5) {
      // 4 LDS.128 per thread = 64 B, the same bytes as one x16 TMEM op
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const uint4 x = sv[(threadIdx.x + 512 * i + it * 32) & 8191];
        acc ^= x.x ^ x.y ^ x.z ^ x.w;
      }
    } else if (mode == 4) {
#pragma unroll
      for (int i = 0; i < 4; i++) sv[(threadIdx.x + 512 * i + it * 32) & 8191] = make_uint4(r[i], r[i + 4], it, acc);
      r[0] += 1;
    } else if (mode == 6) {
      st32x32x16(tbase + col, r);
      wait_st();
      ld16x256x4(tbase + col, r);
      wait_ld();
      r[0] ^= acc;
      acc += r[5];
    } else if (mode == 7) {
#pragma unroll
      for (int i = 0; i < 4; i++) sv[threadIdx.x + 512 * i] = make_uint4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const uint4 x = sv[(threadIdx.x ^ 37) + 512 * i];
        r[4 * i] = x.x; r[4 * i + 1] = x.y; r[4 * i + 2] = x.z; r[4 * i + 3] = x.w + 1;
      }
      __syncthreads();
    }
  }
  wait_ld();
  wait_st();
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
#pragma unroll
  for (int i = 0; i < 16; i++) acc ^= r[i];
  if (acc == 0x12345678u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) tm_dealloc(taddr_s, 512);
}

// correctness of the shape mapping: st 32x32b (thread t writes value t*64+j to
// column j of lane t), ld 16x256b; print which (lane, column) each thread got
__global__ void mapping(uint32_t* out) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tm_alloc(&taddr_s, 32);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[16];
  if (warp == 0) {
    for (int i = 0; i < 16; i++) r[i] = (uint32_t)(lane * 256 + i);
    st32x32x16(taddr_s, r);
    wait_st();
    ld16x256x4(taddr_s, r);
    wait_ld();
    for (int i = 0; i < 16; i++) out[lane * 16 + i] = r[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) tm_dealloc(taddr_s, 32);
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const int nsm = p.multiProcessorCount;
  unsigned long long* d_cyc;
  uint32_t* d_sink;
  CK(cudaMalloc(&d_cyc, nsm * 8));
  CK(cudaMalloc(&d_sink, 4096 * 4));
  CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
  mapping<<<1, 32>>>(d_sink);
  CK(cudaDeviceSynchronize());
  uint32_t h[512];
  CK(cudaMemcpy(h, d_sink, sizeof(h), cudaMemcpyDeviceToHost));
  printf("mapping st32x32b.x16 -> ld16x256b.x4: thread: (srclane,col) per reg\n");
  for (int t = 0; t < 32; t += 1) {
    printf("t%02d:", t);
    for (int i = 0; i < 16; i++) printf(" %u.%u", h[t * 16 + i] / 256, h[t * 16 + i] % 256);
    printf("\n");
  }
  const char* names[] = {"tmem st 32x32b.x16", "tmem ld 32x32b.x16", "tmem ld 16x256b.x4", "smem LDS.128 x4",
                         "smem STS.128 x4",    "8w LDS + 8w LDTM",   "rt st32x32+ld16x256", "rt smem STS+bar+LDS",
                         "tmem st 16x256b.x4"};
  const int iters = 8192;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int mode = 0; mode <= 8; mode++)
    for (int lb = 1; lb <= 4; lb *= 2) {
      if (lb > 1 && !(mode == 0 || mode == 1 || mode == 2 || mode == 5 || mode == 8)) continue;
      bench<<<nsm, 512, 131072>>>(mode, iters, lb, d_cyc, d_sink);  // warm
      CK(cudaEventRecord(e0));
      bench<<<nsm, 512, 131072>>>(mode, iters, lb, d_cyc, d_sink);
      CK(cudaEventRecord(e1));
      CK(cudaDeviceSynchronize());
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      unsigned long long hc[256];
      CK(cudaMemcpy(hc, d_cyc, nsm * 8, cudaMemcpyDeviceToHost));
      unsigned long long mx = 0;
      for (int i = 0; i < nsm; i++) mx = hc[i] > mx ? hc[i] : mx;
      // bytes moved per SM: 512 threads x 64 B per iteration (round trips: 64 B each way)
      const double bytes = 512.0 * 64.0 * iters;
      printf("%-24s batch %d: %8.1f B/clk/SM (clock64), %.3f ms, %.1f GB/s chip\n", names[mode], lb, bytes / mx, ms,
             bytes * nsm / (ms * 1e6));
    }
  return 0;
}
