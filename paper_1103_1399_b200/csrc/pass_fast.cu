// pass_fast.cu -- specialised fused Trotter pass kernels (K4).
//
// One CTA (256 threads, 8 warps) owns a 2^12-amplitude tile at a time; each
// thread holds 16 amplitudes in registers. A register "pattern" says which
// tile-local bits are register bits (rotated in-thread), lane bits (rotated
// with shuffles) and warp bits; between patterns the tile is transposed
// through shared memory (plan.hpp). Each kernel below is one fixed program:
//
//   G0_DPOST         D | PA:r8-11 | ->PC r0-3 | ->PB r4-7 | store PB
//   G0_PRE           PA:r8-11 | ->PC r0-3 | ->PB r4-7 | store PB
//   G0_PRE_D_POST    PA | ->PC | ->PB (step k) | D_{k+1} | PB | ->PC | ->PA (step k+1) | store PA
//   GK_PRE           PA:r8-11 | ->PB r4-7 + lane bit 3 | store PB
//   GK_PRE_D_POST    PA | ->PB (+lane 3) | D | PB (+lane 3) | ->PA | store PA
//
// Rotations are exp(-i beta (1 - sigma^x)) = g cos(beta) (I + i t sigma^x),
// t = tan(beta), with the scalar (g cos beta)^n folded into the step's Phi
// table: one DFMA per real component. A tile bit the group
// does not rotate gets t = 0 (exact identity).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "pass_common.cuh"

namespace qaa {
namespace {

using namespace pc;
#define FULLM QAA_FULLM

template <int FROM, int TO>
__device__ __forceinline__ void xchg(double2* xb, double2 (&v)[RPT], int lane, int warp) {
  const int bs = padA(pat_tl<FROM>(lane, warp));
#pragma unroll
  for (int r = 0; r < RPT; r++) xb[bs + padA(r << reg_shift<FROM>())] = v[r];
  __syncthreads();
  const int bl = padA(pat_tl<TO>(lane, warp));
#pragma unroll
  for (int r = 0; r < RPT; r++) v[r] = xb[bl + padA(r << reg_shift<TO>())];
  __syncthreads();
}

__device__ __forceinline__ void diag(double2 (&v)[RPT], const uint32_t (&ep)[4], const double2* phis, int lane) {
#pragma unroll
  for (int r = 0; r < RPT; r++) {
    const int e = (ep[r >> 2] >> ((r & 3) * 8)) & 0xff;
    const double2 f = phis[e * 8 + (lane & 7)];  // 8 bank-group copies: conflict-free lookup
    const double2 x = v[r];
    v[r] = make_double2(fma(f.x, x.x, -f.y * x.y), fma(f.x, x.y, f.y * x.x));
  }
}

template <int PROG>
struct ProgInfo {
  static constexpr bool has_d = PROG == FP_G0_DPOST || PROG == FP_G0_PRE_D_POST || PROG == FP_GK_PRE_D_POST;
  static constexpr int e_pat = PROG == FP_G0_DPOST ? PA : PB;
  static constexpr int store_pat = (PROG == FP_G0_PRE_D_POST || PROG == FP_GK_PRE_D_POST) ? PA : PB;
};

template <int PROG, bool LANE3>
__device__ __forceinline__ void program(const FastArgs& a, double2 (&v)[RPT], const uint32_t (&ep)[4], double2* xb,
                                        const double2* phis, int lane, int warp) {
  const double(&t0)[TILE_BITS] = a.t[0];
  const double(&t1)[TILE_BITS] = a.t[1];
  if (PROG == FP_G0_DPOST) {
    diag(v, ep, phis, lane);
    rot_regs<PA>(v, t1);
    xchg<PA, PC>(xb, v, lane, warp);
    rot_regs<PC>(v, t1);
    xchg<PC, PB>(xb, v, lane, warp);
    rot_regs<PB>(v, t1);
  } else if (PROG == FP_G0_PRE) {
    rot_regs<PA>(v, t0);
    xchg<PA, PC>(xb, v, lane, warp);
    rot_regs<PC>(v, t0);
    xchg<PC, PB>(xb, v, lane, warp);
    rot_regs<PB>(v, t0);
  } else if (PROG == FP_G0_PRE_D_POST) {
    rot_regs<PA>(v, t0);
    xchg<PA, PC>(xb, v, lane, warp);
    rot_regs<PC>(v, t0);
    xchg<PC, PB>(xb, v, lane, warp);
    rot_regs<PB>(v, t0);
    diag(v, ep, phis, lane);
    rot_regs<PB>(v, t1);
    xchg<PB, PC>(xb, v, lane, warp);
    rot_regs<PC>(v, t1);
    xchg<PC, PA>(xb, v, lane, warp);
    rot_regs<PA>(v, t1);
  } else if (PROG == FP_GK_PRE) {
    rot_regs<PA>(v, t0);
    xchg<PA, PB>(xb, v, lane, warp);
    rot_regs<PB>(v, t0);
    if (LANE3) rot_lane(v, 3, t0[3]);
  } else if (PROG == FP_GK_PRE_D_POST) {
    rot_regs<PA>(v, t0);
    xchg<PA, PB>(xb, v, lane, warp);
    rot_regs<PB>(v, t0);
    if (LANE3) rot_lane(v, 3, t0[3]);
    diag(v, ep, phis, lane);
    rot_regs<PB>(v, t1);
    if (LANE3) rot_lane(v, 3, t1[3]);
    xchg<PB, PA>(xb, v, lane, warp);
    rot_regs<PA>(v, t1);
  }
}

// CG = true: L2-only loads (data written by other SMs earlier in the same launch)
template <bool HAS_D, bool CG = false>
__device__ __forceinline__ void load(const FastArgs& a, const Off& pa, const Off& pe, int64_t T, double2 (&v)[RPT],
                                     uint32_t (&ep)[4]) {
  const int64_t base = tbase(a, T);
  const double2* src = a.psi + base;
#pragma unroll
  for (int r = 0; r < RPT; r++) v[r] = CG ? __ldcg(src + roff(pa, r)) : src[roff(pa, r)];
  if (HAS_D) {
    const uint8_t* eb = a.E + base;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      uint32_t w = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) w |= (uint32_t)eb[roff(pe, q * 4 + j)] << (8 * j);
      ep[q] = w;
    }
  }
}

__device__ __forceinline__ void store(const FastArgs& a, const Off& ps, int64_t T, const double2 (&v)[RPT]) {
  const int64_t tb = tbase(a, T);
  double2* dst = a.psi + tb;
  if (a.remote) {
    // the bit swap of the sharded layouts: the tile's top local bits (not tile
    // bits of this group) name the destination rank
    const int64_t j = tb >> a.gshift;
    dst = a.peers[j] + (tb - (j << a.gshift) + ((int64_t)a.rank << a.gshift));
  }
#pragma unroll
  for (int r = 0; r < RPT; r++) dst[roff(ps, r)] = v[r];
}

__global__ void __launch_bounds__(256) remap_kernel(const double2* src, double2* const* peers_unused, int64_t N,
                                                    int gshift, int rank, double2* p0, double2* p1, double2* p2,
                                                    double2* p3, double2* p4, double2* p5, double2* p6, double2* p7) {
  double2* peers[8] = {p0, p1, p2, p3, p4, p5, p6, p7};
  const int64_t low = ((int64_t)1 << gshift) - 1;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = x >> gshift;
    peers[j][(x & low) | ((int64_t)rank << gshift)] = src[x];
  }
  __threadfence_system();
}

template <int PROG, bool LANE3, bool PREFETCH>
__global__ void __launch_bounds__(NTHREADS, PREFETCH ? 1 : 2) qaa_pass_fast(const FastArgs a) {
  extern __shared__ double2 smem[];
  double2* xb = smem;
  double2* phis = smem + FAST_XBUF;
  using PI = ProgInfo<PROG>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (PI::has_d)
    for (int e = tid; e < a.n_phi * 8; e += NTHREADS) phis[e] = a.phi[e >> 3];
  __syncthreads();
  const Off pa = make_off<PA>(a, lane, warp);
  const Off pe = make_off<PI::e_pat>(a, lane, warp);
  const Off ps = make_off<PI::store_pat>(a, lane, warp);
  double2 va[RPT];
  uint32_t ea[4] = {0, 0, 0, 0};
  const int64_t stride = gridDim.x;
  int64_t T = blockIdx.x;
  if (!PREFETCH) {
    for (; T < a.ntiles; T += stride) {
      load<PI::has_d>(a, pa, pe, T, va, ea);
      program<PROG, LANE3>(a, va, ea, xb, phis, lane, warp);
      store(a, ps, T, va);
    }
    if (a.remote) __threadfence_system();
    return;
  }
  double2 vb[RPT];
  uint32_t eb[4] = {0, 0, 0, 0};
  if (T < a.ntiles) load<PI::has_d>(a, pa, pe, T, va, ea);
  while (T < a.ntiles) {
    int64_t Tn = T + stride;
    if (Tn < a.ntiles) load<PI::has_d>(a, pa, pe, Tn, vb, eb);
    program<PROG, LANE3>(a, va, ea, xb, phis, lane, warp);
    store(a, ps, T, va);
    T = Tn;
    if (T >= a.ntiles) break;
    Tn = T + stride;
    if (Tn < a.ntiles) load<PI::has_d>(a, pa, pe, Tn, va, ea);
    program<PROG, LANE3>(a, vb, eb, xb, phis, lane, warp);
    store(a, ps, T, vb);
    T = Tn;
  }
  if (a.remote) __threadfence_system();
}


// ============================================================================
// Persistent evolve for 13 <= L <= 21 (one launch for all K steps): the state
// (1..32 MiB) stays in L2, every pass of the plan runs over the CTA's tiles
// and ends with a grid barrier -- instead of one launch (~8 us of launch and
// ramp latency at n = 16) per pass. Cooperative launch (co-residency).
// ============================================================================
struct PersistGroup {
  int phys[TILE_BITS];
  uint32_t rot_local;
  int nseg;
  int seg_src[MAX_SEGS], seg_dst[MAX_SEGS], seg_len[MAX_SEGS];
  int64_t ntiles;
};
struct PersistArgs {
  double2* psi;
  const uint8_t* E;
  const PersistPass* passes;   // npass records (device)
  int npass;
  const double2* phi_all;      // step k's D row at phi_all + k n_phi
  int n_phi;
  const double* coef;          // tan(beta_k) per step
  PersistGroup groups[4];
  unsigned* bar;               // [2]: arrival count, generation (zeroed before launch)
};

// sense-free grid barrier: the last arriving CTA resets the count and bumps
// the generation; stores before it are released at gpu scope
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      for (;;) {
        unsigned g;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
        if (g != gen) break;
        __nanosleep(20);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

template <int PROG, bool LANE3>
__device__ __forceinline__ void persist_pass(const FastArgs& a, double2* xb, const double2* phis, int lane, int warp) {
  using PI = ProgInfo<PROG>;
  const Off pa = make_off<PA>(a, lane, warp);
  const Off pe = make_off<PI::e_pat>(a, lane, warp);
  const Off ps = make_off<PI::store_pat>(a, lane, warp);
  double2 v[RPT];
  uint32_t ep[4] = {0, 0, 0, 0};
  for (int64_t T = blockIdx.x; T < a.ntiles; T += gridDim.x) {
    load<PI::has_d, true>(a, pa, pe, T, v, ep);
    program<PROG, LANE3>(a, v, ep, xb, phis, lane, warp);
    store(a, ps, T, v);
  }
}

__global__ void __launch_bounds__(NTHREADS, 2) qaa_persist(const PersistArgs pa) {
  extern __shared__ double2 smem[];
  double2* xb = smem;
  double2* phis = smem + FAST_XBUF;
  __shared__ FastArgs fa;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int p = 0; p < pa.npass; p++) {
    const PersistPass r = pa.passes[p];
    if (tid == 0) {
      const PersistGroup& gr = pa.groups[r.group];
      fa.psi = pa.psi;
      fa.E = pa.E;
      fa.phi = r.d >= 0 ? pa.phi_all + (int64_t)r.d * pa.n_phi : nullptr;
      fa.n_phi = pa.n_phi;
      const double c0 = r.pre >= 0 ? pa.coef[r.pre] : 0.0, c1 = r.post >= 0 ? pa.coef[r.post] : 0.0;
      for (int b = 0; b < TILE_BITS; b++) {
        const bool rb = (gr.rot_local >> b) & 1;
        fa.t[0][b] = rb ? c0 : 0.0;
        fa.t[1][b] = rb ? c1 : 0.0;
        fa.phys[b] = gr.phys[b];
      }
      fa.ntiles = gr.ntiles;
      fa.nseg = gr.nseg;
      for (int s = 0; s < MAX_SEGS; s++) {
        fa.seg_src[s] = gr.seg_src[s];
        fa.seg_dst[s] = gr.seg_dst[s];
        fa.seg_len[s] = gr.seg_len[s];
      }
      fa.remote = 0;
    }
    __syncthreads();
    if (r.d >= 0)
      for (int e = tid; e < pa.n_phi * 8; e += NTHREADS) phis[e] = fa.phi[e >> 3];
    __syncthreads();
    switch (r.fp * 2 + r.lane3) {
      case FP_G0_DPOST * 2: persist_pass<FP_G0_DPOST, false>(fa, xb, phis, lane, warp); break;
      case FP_G0_PRE * 2: persist_pass<FP_G0_PRE, false>(fa, xb, phis, lane, warp); break;
      case FP_G0_PRE_D_POST * 2: persist_pass<FP_G0_PRE_D_POST, false>(fa, xb, phis, lane, warp); break;
      case FP_GK_PRE * 2: persist_pass<FP_GK_PRE, false>(fa, xb, phis, lane, warp); break;
      case FP_GK_PRE * 2 + 1: persist_pass<FP_GK_PRE, true>(fa, xb, phis, lane, warp); break;
      case FP_GK_PRE_D_POST * 2: persist_pass<FP_GK_PRE_D_POST, false>(fa, xb, phis, lane, warp); break;
      case FP_GK_PRE_D_POST * 2 + 1: persist_pass<FP_GK_PRE_D_POST, true>(fa, xb, phis, lane, warp); break;
      default: __trap();
    }
    grid_sync(pa.bar, gridDim.x);
  }
}

typedef void (*FastKernel)(const FastArgs);

template <bool PF>
FastKernel pick(int prog, bool lane3) {
  switch (prog) {
    case FP_G0_DPOST: return qaa_pass_fast<FP_G0_DPOST, false, PF>;
    case FP_G0_PRE: return qaa_pass_fast<FP_G0_PRE, false, PF>;
    case FP_G0_PRE_D_POST: return qaa_pass_fast<FP_G0_PRE_D_POST, false, PF>;
    case FP_GK_PRE: return lane3 ? qaa_pass_fast<FP_GK_PRE, true, PF> : qaa_pass_fast<FP_GK_PRE, false, PF>;
    case FP_GK_PRE_D_POST:
      return lane3 ? qaa_pass_fast<FP_GK_PRE_D_POST, true, PF> : qaa_pass_fast<FP_GK_PRE_D_POST, false, PF>;
    default: return nullptr;
  }
}

}  // namespace

// co-resident CTAs of the persistent kernel (0 on error)
int persist_max_grid(int num_sms) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qaa_persist, NTHREADS, FAST_SMEM_BYTES) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return per_sm * num_sms;
}

cudaError_t launch_persist(const PersistLaunch& L, int grid, cudaStream_t st) {
  PersistArgs a;
  memset(&a, 0, sizeof a);
  a.psi = L.psi;
  a.E = L.E;
  a.passes = L.passes;
  a.npass = L.npass;
  a.phi_all = L.phi_all;
  a.n_phi = L.n_phi;
  a.coef = L.coef;
  a.bar = L.bar;
  for (int g = 0; g < L.ngroups && g < 4; g++) {
    for (int b = 0; b < TILE_BITS; b++) a.groups[g].phys[b] = L.groups[g].phys[b];
    a.groups[g].rot_local = L.groups[g].rot_local;
    a.groups[g].nseg = L.groups[g].nseg;
    for (int s = 0; s < MAX_SEGS; s++) {
      a.groups[g].seg_src[s] = L.groups[g].seg_src[s];
      a.groups[g].seg_dst[s] = L.groups[g].seg_dst[s];
      a.groups[g].seg_len[s] = L.groups[g].seg_len[s];
    }
    a.groups[g].ntiles = L.groups[g].ntiles;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = FAST_SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, qaa_persist, a);
}

cudaError_t pass_fast_setup() {
  {
    cudaError_t e = cudaFuncSetAttribute(qaa_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FAST_SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  for (int p = 0; p < FP_COUNT; p++)
    for (int l = 0; l < 2; l++)
      for (int pf = 0; pf < 2; pf++) {
        FastKernel k = pf ? pick<true>(p, l) : pick<false>(p, l);
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FAST_SMEM_BYTES);
        if (e != cudaSuccess) return e;
      }
  return cudaSuccess;
}

cudaError_t launch_remap(const double2* src, double2* const* peers, int64_t N, int gshift, int rank, int num_sms,
                         cudaStream_t st) {
  int64_t grid = (N + 255) / 256;
  if (grid > (int64_t)num_sms * 8) grid = (int64_t)num_sms * 8;
  remap_kernel<<<(int)grid, 256, 0, st>>>(src, nullptr, N, gshift, rank, peers[0], peers[1], peers[2], peers[3],
                                          peers[4], peers[5], peers[6], peers[7]);
  return cudaGetLastError();
}

cudaError_t launch_pass_fast(const FastArgs& a, int prog, bool lane3, bool prefetch, int grid, cudaStream_t st) {
  FastKernel k = prefetch ? pick<true>(prog, lane3) : pick<false>(prog, lane3);
  if (!k) return cudaErrorInvalidValue;
  k<<<grid, NTHREADS, FAST_SMEM_BYTES, st>>>(a);
  return cudaGetLastError();
}

}  // namespace qaa
