// cluster_evolve.cu -- all K Trotter steps of a 13..16-qubit state in ONE launch,
// the state resident in the registers of one thread-block cluster (SURVEY §8(f) F1,
// §7 hard part 5; the paper's regime of many small instances).
//
// Cluster of C = 2^CB CTAs (CB = L - 12 = 1..4), 256 threads per CTA, 16 amplitudes per
// thread: each CTA holds 2^12 amplitudes in registers for the whole evolution.
// Layout A: CTA rank = logical bits [12, L), local index = logical bits [0, 12).
// Layout B: CTA rank = logical bits [12-CB, 12); local positions [12-CB, 12) hold
//           logical bits [12, L).
// One phase = one Trotter step k in the current layout (the sharded
// plan's carried-bit schedule inside a cluster):
//   (a) rotate the CB bits that just arrived (they were rank bits in the previous
//       phase) with step k-1's coefficient -- the rest of step k-1's X was done there;
//   (b) D_k (energy slice of this layout, packed per thread);
//   (c) rotate the 12 local bits with step k: register pattern PA (local bits 8..11 in
//       registers), shared-memory exchange to PB (4..7), exchange to PC (0..3);
//   (d) layout swap over DSMEM: every thread stores its 16 amplitudes straight into
//       the destination CTA's landing buffer (st.shared::cluster), one cluster
//       barrier, the landed tile is read back in pattern PA.
// Two landing buffers alternate between phases, so one cluster barrier per step is
// the only cross-CTA synchronisation. Rotations use the tangent or the cot form per
// step (rot_pair); Strang's closing half step is applied after the last phase.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "pass_common.cuh"

namespace qaa {
namespace {

namespace cg = cooperative_groups;
using namespace pc;

constexpr int CE_THREADS = 256;
constexpr int CE_BUF = FAST_XBUF;  // padded 2^12-amplitude buffer (l + (l >> 4))
constexpr size_t CE_SMEM = 2 * (size_t)CE_BUF * 16 + 2 * 4096 + 64;

template <int FORM>
__device__ __forceinline__ void ce_pair(double2& a, double2& b, double c) {
  double2 na, nb;
  if (FORM == 0) {  // tangent form: (a, b) <- (a + i t b, b + i t a)
    na = make_double2(fma(-c, b.y, a.x), fma(c, b.x, a.y));
    nb = make_double2(fma(-c, a.y, b.x), fma(c, a.x, b.y));
  } else {  // cot form: (a, b) <- (cot a + i b, cot b + i a)
    na = make_double2(fma(c, a.x, -b.y), fma(c, a.y, b.x));
    nb = make_double2(fma(c, b.x, -a.y), fma(c, b.y, a.x));
  }
  a = na;
  b = nb;
}
// rotate register bits [lo, 4) of the thread's 16 amplitudes
template <int FORM>
__device__ __forceinline__ void ce_rot(double2 (&v)[RPT], int lo, double c) {
#pragma unroll
  for (int i = 0; i < 4; i++)
    if (i >= lo)
#pragma unroll
      for (int r = 0; r < RPT; r++)
        if (!(r & (1 << i))) ce_pair<FORM>(v[r], v[r | (1 << i)], c);
}
__device__ __forceinline__ void ce_rot_form(double2 (&v)[RPT], int lo, double c, int form) {
  if (form == 0)
    ce_rot<0>(v, lo, c);
  else
    ce_rot<1>(v, lo, c);
}
// whole-CTA pattern change through the padded buffer
template <int FROM, int TO>
__device__ __forceinline__ void ce_xchg(double2* xb, double2 (&v)[RPT], int lane, int warp) {
  const int bs = padA(pat_tl<FROM>(lane, warp));
  __syncthreads();  // every thread has read the buffer's previous contents
#pragma unroll
  for (int r = 0; r < RPT; r++) xb[bs + padA(r << reg_shift<FROM>())] = v[r];
  __syncthreads();
  const int bl = padA(pat_tl<TO>(lane, warp));
#pragma unroll
  for (int r = 0; r < RPT; r++) v[r] = xb[bl + padA(r << reg_shift<TO>())];
}
// canonical index of local index l on rank q in layout B
template <int CB>
__device__ __forceinline__ int64_t ce_global_b(int q, int l) {
  constexpr int S = 12 - CB;
  return (int64_t)(l & ((1 << S) - 1)) | ((int64_t)q << S) | ((int64_t)(l >> S) << 12);
}

template <int CB>
__global__ void __launch_bounds__(CE_THREADS, 1) qaa_cluster_evolve(const ClusterArgs a) {
  constexpr int C = 1 << CB, S = 12 - CB;
  extern __shared__ __align__(128) unsigned char sm[];
  double2* buf0 = reinterpret_cast<double2*>(sm);
  double2* buf1 = buf0 + CE_BUF;
  uint8_t* eA = reinterpret_cast<uint8_t*>(buf1 + CE_BUF);
  uint8_t* eB = eA + 4096;
  __shared__ double red[CE_THREADS / 32];
  __shared__ double part;
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank(), rep = blockIdx.x / C;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t K = a.Krep ? a.Krep[rep] : a.K;
  const int64_t off = a.row_off ? a.row_off[rep] : 0;
  // energy slices in PA order, packed per thread (16 B: one LDS.128 per D)
#pragma unroll
  for (int r = 0; r < RPT; r++) {
    const int l = t | (r << 8);
    eA[t * RPT + r] = a.E[((int64_t)q << 12) | l];
    eB[t * RPT + r] = a.E[ce_global_b<CB>(q, l)];
  }
  double2 v[RPT];
#pragma unroll
  for (int r = 0; r < RPT; r++) {
    const int l = t | (r << 8);
    v[r] = a.psi ? a.psi[((int64_t)q << 12) | l] : make_double2(a.amp0, 0.0);
  }
  cl.sync();  // every CTA of the cluster is running before any DSMEM store reaches it
  int layout = 0;
  double2* cur = buf0;
  double2* nxt = buf1;
  for (int64_t k = 0; k < K; k++) {
    const int64_t row = off + k;
    // (a) the carried bits: the rest of step k-1's X layer
    if (k > 0) ce_rot_form(v, 4 - CB, a.coef[row - 1], a.form[row - 1]);
    // (b) D_k
    {
      const double2* phi = a.phi_all + row * a.n_phi;
      const uint4 pk = reinterpret_cast<const uint4*>(layout ? eB : eA)[t];
#pragma unroll
      for (int r = 0; r < RPT; r++) {
        const uint32_t w = r < 4 ? pk.x : (r < 8 ? pk.y : (r < 12 ? pk.z : pk.w));
        const double2 f = __ldg(phi + ((w >> (8 * (r & 3))) & 0xffu));
        v[r] = cmul(f, v[r]);
      }
    }
    // (c) the 12 local bits of step k
    const double c = a.coef[row];
    const int form = a.form[row];
    ce_rot_form(v, 0, c, form);
    ce_xchg<PA, PB>(cur, v, lane, warp);
    ce_rot_form(v, 0, c, form);
    ce_xchg<PB, PC>(cur, v, lane, warp);
    ce_rot_form(v, 0, c, form);
    // (d) layout swap: local l (pattern PC) -> rank l >> S, local (l & (2^S - 1)) | q << S
    {
      const int tl = pat_tl<PC>(lane, warp);
      const int j = tl >> S;  // PC: the top local bits are thread bits (lane bit 4, warp bits)
      const int lo = tl & ((1 << S) - 1) & ~15;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(nxt);
      uint32_t rdst;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(dst), "r"((uint32_t)j));
#pragma unroll
      for (int r = 0; r < RPT; r++) {
        const int l2 = lo | r | (q << S);
        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(rdst + 16u * (uint32_t)padA(l2)),
                     "d"(v[r].x), "d"(v[r].y)
                     : "memory");
      }
    }
    cl.sync();  // release my remote stores / acquire everyone's
#pragma unroll
    for (int r = 0; r < RPT; r++) v[r] = nxt[padA(t | (r << 8))];
    double2* sw = cur;
    cur = nxt;
    nxt = sw;
    layout ^= 1;
  }
  if (K > 0) ce_rot_form(v, 4 - CB, a.coef[off + K - 1], a.form[off + K - 1]);
  if (a.final_d) {  // Strang: closing half step D(s_{K-1})^{1/2}
    const double2* phi = a.phi_all + (off + K) * a.n_phi;
    const uint4 pk = reinterpret_cast<const uint4*>(layout ? eB : eA)[t];
#pragma unroll
    for (int r = 0; r < RPT; r++) {
      const uint32_t w = r < 4 ? pk.x : (r < 8 ? pk.y : (r < 12 ? pk.z : pk.w));
      v[r] = cmul(__ldg(phi + ((w >> (8 * (r & 3))) & 0xffu)), v[r]);
    }
  }
  if (a.psi) {
#pragma unroll
    for (int r = 0; r < RPT; r++) {
      const int l = t | (r << 8);
      a.psi[layout ? ce_global_b<CB>(q, l) : (((int64_t)q << 12) | l)] = v[r];
    }
  }
  if (a.out) {  // P_succ of this replica: fixed-order tree over threads, then CTAs
    const uint4 pk = reinterpret_cast<const uint4*>(layout ? eB : eA)[t];
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < RPT; r++) {
      const uint32_t w = r < 4 ? pk.x : (r < 8 ? pk.y : (r < 12 ? pk.z : pk.w));
      if (((w >> (8 * (r & 3))) & 0xffu) == 0) acc += fma(v[r].x, v[r].x, v[r].y * v[r].y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
      for (int w = 0; w < CE_THREADS / 32; w++) s += red[w];
      part = s;
    }
    cl.sync();
    if (q == 0 && t == 0) {
      double s = 0.0;
      for (int j = 0; j < C; j++) s += *cl.map_shared_rank(&part, j);
      a.out[rep] = s;
    }
  }
  cl.sync();  // no CTA leaves while a peer may still store into or read its shared memory
}

template <int CB>
cudaError_t launch_cb(const ClusterArgs& a, int nrep, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(qaa_cluster_evolve<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CE_SMEM);
  if (e != cudaSuccess) return e;
  if (CB == 4) {
    e = cudaFuncSetAttribute(qaa_cluster_evolve<CB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nrep << CB));
  cfg.blockDim = dim3(CE_THREADS);
  cfg.dynamicSmemBytes = CE_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1u << CB;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, qaa_cluster_evolve<CB>, a);
}

}  // namespace

cudaError_t launch_cluster_evolve(const ClusterArgs& a, int nrep, cudaStream_t st) {
  switch (a.L) {
    case 13: return launch_cb<1>(a, nrep, st);
    case 14: return launch_cb<2>(a, nrep, st);
    case 15: return launch_cb<3>(a, nrep, st);
    case 16: return launch_cb<4>(a, nrep, st);
    default: return cudaErrorInvalidValue;
  }
}

// how many replica clusters of this size the device runs at once (0: none fits)
int cluster_evolve_max_active(int L) {
  if (L < 13 || L > 16) return 0;
  const int CB = L - 12;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1u << CB);
  cfg.blockDim = dim3(CE_THREADS);
  cfg.dynamicSmemBytes = CE_SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1u << CB;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  cudaError_t e;
  switch (CB) {
    case 1: e = cudaOccupancyMaxActiveClusters(&n, qaa_cluster_evolve<1>, &cfg); break;
    case 2: e = cudaOccupancyMaxActiveClusters(&n, qaa_cluster_evolve<2>, &cfg); break;
    case 3: e = cudaOccupancyMaxActiveClusters(&n, qaa_cluster_evolve<3>, &cfg); break;
    default: e = cudaOccupancyMaxActiveClusters(&n, qaa_cluster_evolve<4>, &cfg); break;
  }
  return e == cudaSuccess ? n : 0;
}

}  // namespace qaa
