// DSMEM all-to-all throughput inside one thread-block cluster (design probe for a
// cluster-resident evolve, not product). Each CTA holds 4096 amplitudes (64 KiB) and
// sends block j (4096/C amplitudes) to CTA j, receiving into a second 64 KiB buffer:
//   mode 0: st.shared::cluster.v2.f64 from registers (256 threads x 16 amplitudes)
//   mode 1: cp.async.bulk.shared::cluster.shared::cta (one bulk copy per peer,
//           completion on the receiver's mbarrier)
//   mode 2: ld.shared::cluster.v2.f64 (pull) into registers, then local st.shared
// reps all-to-alls per launch, barrier.cluster between them.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}

__global__ void __launch_bounds__(256, 1) a2a(int mode, int reps, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double2* src = reinterpret_cast<double2*>(sm);
  double2* dst = src + 4096;
  uint64_t* bar = reinterpret_cast<uint64_t*>(dst + 4096);
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks(), q = (int)cl.block_rank(), t = threadIdx.x;
  const int blk = 4096 / C;  // amplitudes per peer block
  for (int i = t; i < 4096; i += 256) src[i] = make_double2(q, i);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  long long t0 = clock64();
  uint32_t ph = 0;
  for (int r = 0; r < reps; r++) {
    if (mode == 0) {
#pragma unroll
      for (int k = 0; k < 16; k++) {
        const int i = t + 256 * k;       // source index: block j = i / blk
        const int j = i / blk, o = i % blk;
        const uint32_t a = mapa(sa(dst + q * blk + o), (uint32_t)j);
        const double2 v = src[i];
        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
      }
      cl.sync();
    } else if (mode == 1) {
      if (t == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(4096u * 16u)
                     : "memory");
      cl.sync();  // every receiver armed its barrier
      if (t < C) {
        const int j = t;
        const uint32_t d = mapa(sa(dst + q * blk), (uint32_t)j);
        const uint32_t b = mapa(sa(bar), (uint32_t)j);
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
            "r"(sa(src + j * blk)), "r"((uint32_t)(blk * 16)), "r"(b)
            : "memory");
      }
      // wait for my 64 KiB to land
      asm volatile(
          "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
              sa(bar)),
          "r"(ph & 1)
          : "memory");
      ph++;
      cl.sync();  // senders done reading src before the next round
    } else {
      double2 v[16];
#pragma unroll
      for (int k = 0; k < 16; k++) {
        const int i = t + 256 * k;  // destination index: from peer j = i / blk
        const int j = i / blk, o = i % blk;
        const uint32_t a = mapa(sa(src + q * blk + o), (uint32_t)j);
        asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v[k].x), "=d"(v[k].y) : "r"(a) : "memory");
      }
#pragma unroll
      for (int k = 0; k < 16; k++) dst[t + 256 * k] = v[k];
      cl.sync();
    }
  }
  long long t1 = clock64();
  if (t == 0 && q == 0) out[blockIdx.x / C] = (double)(t1 - t0) / reps;
  // check one value
  if (t == 0 && dst[5].y != (double)((q * blk + 5) % blk + (5 / blk) * 0) && mode >= 0) {
  }
}

int main() {
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  const size_t smem = 2 * 4096 * 16 + 64;
  cudaFuncSetAttribute(a2a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(a2a, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int C : {2, 4, 8, 16}) {
    for (int mode = 0; mode < 3; mode++) {
      for (int nclusters : {1, 8}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C * nclusters);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, a2a, mode, 200, out);
        cudaError_t e2 = cudaDeviceSynchronize();
        double h = 0;
        cudaMemcpy(&h, out, sizeof(double), cudaMemcpyDeviceToHost);
        const double bytes = 4096.0 * 16 * (C - 1) / C;  // sent per CTA per all-to-all
        printf("C=%2d mode=%d clusters=%d: %.0f cycles per all-to-all, %.1f B/clk/SM out  [%s %s]\n", C, mode,
               nclusters, h, bytes / h, cudaGetErrorString(e), cudaGetErrorString(e2));
      }
    }
  }
  return 0;
}
