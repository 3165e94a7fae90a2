// Grid-barrier cost on B200 (design probe for the single-launch small-state
// engines, not product): ITER barriers of a cooperative grid of G CTAs x 128
// threads, variants:
//   0: red.release.gpu add + ld.acquire.gpu spin (warp_evolve.cu grid_barrier)
//   1: same, spin with ld.relaxed.gpu and one fence.acq_rel.gpu after
//   2: atom.add.release.gpu, the last arriver flips a separate flag line, others
//      spin on the flag (ld.acquire) -- arrivals and polls on different lines
//   3: variant 0 + each CTA reads and writes 8 KiB of L2-resident state per round
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void bar0(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
    }
  }
  __syncthreads();
}
__device__ __forceinline__ void bar1(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    for (;;) {
      unsigned v;
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
__device__ __forceinline__ void bar2(unsigned* ctr, unsigned* flag, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    if (old == epoch * gridDim.x - 1) {
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
    } else {
      for (;;) {
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v >= epoch) break;
      }
    }
  }
  __syncthreads();
}
__global__ void k(unsigned* ctr, int iters, int variant, double2* st) {
  for (int i = 1; i <= iters; i++) {
    if (variant == 3) {
      double2* p = st + (size_t)((blockIdx.x + i) % gridDim.x) * 512;
      double2 v[4];
      for (int r = 0; r < 4; r++) v[r] = __ldcg(p + threadIdx.x + 128 * r);
      for (int r = 0; r < 4; r++) { v[r].x += 1.0; __stcg(p + threadIdx.x + 128 * r, v[r]); }
    }
    if (variant == 1) bar1(ctr, (unsigned)i * gridDim.x);
    else if (variant == 2) bar2(ctr, ctr + 32, (unsigned)i);
    else bar0(ctr, (unsigned)i * gridDim.x);
  }
}
int main() {
  unsigned* ctr;
  double2* st;
  cudaMalloc(&ctr, 4096);
  cudaMalloc(&st, 148 * 512 * sizeof(double2));
  const int iters = 2000;
  for (int G : {16, 64, 128, 148, 296}) {
    for (int variant = 0; variant < 4; variant++) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; rep++) {
        cudaMemset(ctr, 0, 4096);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        void* args[] = {&ctr, (void*)&iters, &variant, &st};
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchCooperativeKernel((void*)k, G, 128, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        if (e != cudaSuccess) { printf("G=%d variant %d: %s\n", G, variant, cudaGetErrorString(e)); break; }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("grid %3d variant %d: %.3f us per barrier\n", G, variant, best * 1e3f / iters);
    }
  }
  return 0;
}
