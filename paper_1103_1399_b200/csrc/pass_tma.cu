// pass_tma.cu -- warp-specialised TMA version of the fused Trotter pass (K4).
//
// One persistent CTA per SM, 512 threads = two groups of 8 warps. Tiles are
// streamed into 3 shared-memory slots with TMA (cp.async.bulk for contiguous
// group-0 tiles, cp.async.bulk.tensor for the strided row tiles of the other
// groups) together with the tile's 4 KiB energy slice, completing on mbarriers.
// Group g takes tiles j = g, g+2, ...: it reads the landed tile into registers
// (pattern PA), runs the compiled-in register program of pass_fast.cu using
// the *same slot* as its exchange buffer (padded layout l + (l >> 4)), issues
// the TMA for tile j+3 into the slot it just freed, and stores its result with
// coalesced STG straight from registers.
// HBM reads are therefore always in flight (up to 3 tiles per SM) while the
// two consumer groups overlap their shared-memory transposes and fp64 FMAs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace qaa {
namespace {

#define FULLM 0xffffffffu
constexpr int TMA_SLOTS = 3;
constexpr int SLOT_BYTES = FAST_XBUF * 16;  // 69632: padded exchange layout
constexpr int TMA_MAX_GROUPS = 2;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
      "l"(src), "r"(bytes), "r"(sa(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, const int (&c)[5], int rank,
                                         uint64_t* bar) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  switch (rank) {
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
          "[%4];" ::"r"(sa(dst)),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(sa(bar))
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
          "%4}], [%5];" ::"r"(sa(dst)),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(sa(bar))
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
          "%4, %5}], [%6];" ::"r"(sa(dst)),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(sa(bar))
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
          "%4, %5, %6}], [%7];" ::"r"(sa(dst)),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(sa(bar))
          : "memory");
      break;
  }
}
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void group_bar(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(NTHREADS) : "memory");
}

__device__ __forceinline__ constexpr int padA(int l) { return l + (l >> 4); }

template <int P>
__device__ __forceinline__ int pat_tl(int lane, int warp) {
  if (P == PA) return lane | (warp << 5);
  if (P == PB) return (lane & 15) | ((lane >> 4) << 8) | (warp << 9);
  return (lane << 4) | (warp << 9);
}
template <int P>
__device__ __forceinline__ constexpr int reg_shift() {
  return P == PA ? 8 : (P == PB ? 4 : 0);
}

struct Off {
  int64_t thr;
  int64_t s[4];
};
template <int P>
__device__ __forceinline__ Off make_off(const TmaArgs& a, int lane, int warp) {
  Off o;
  const int tl = pat_tl<P>(lane, warp);
  int64_t t = 0;
#pragma unroll
  for (int b = 0; b < TILE_BITS; b++)
    if ((tl >> b) & 1) t += (int64_t)1 << a.phys[b];
  o.thr = t;
#pragma unroll
  for (int i = 0; i < 4; i++) o.s[i] = (int64_t)1 << a.phys[reg_shift<P>() + i];
  return o;
}
__device__ __forceinline__ int64_t roff(const Off& o, int r) {
  int64_t x = o.thr;
  if (r & 1) x += o.s[0];
  if (r & 2) x += o.s[1];
  if (r & 4) x += o.s[2];
  if (r & 8) x += o.s[3];
  return x;
}
__device__ __forceinline__ int64_t tbase(const TmaArgs& a, int64_t T) {
  int64_t b = 0;
#pragma unroll
  for (int s = 0; s < MAX_SEGS; s++)
    if (s < a.nseg) b += ((T >> a.seg_src[s]) & (((int64_t)1 << a.seg_len[s]) - 1)) << a.seg_dst[s];
  return b;
}

__device__ __forceinline__ void rot2(double2& x, double2& y, double t) {
  const double2 nx = make_double2(fma(-t, y.y, x.x), fma(t, y.x, x.y));
  const double2 ny = make_double2(fma(-t, x.y, y.x), fma(t, x.x, y.y));
  x = nx;
  y = ny;
}
template <int P>
__device__ __forceinline__ void rot_regs(double2 (&v)[RPT], const double (&t)[TILE_BITS]) {
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const double c = t[reg_shift<P>() + i];
#pragma unroll
    for (int r = 0; r < RPT; r++)
      if (!(r & (1 << i))) rot2(v[r], v[r | (1 << i)], c);
  }
}
__device__ __forceinline__ void rot_lane(double2 (&v)[RPT], int lanebit, double t) {
#pragma unroll
  for (int r = 0; r < RPT; r++) {
    const double px = __shfl_xor_sync(FULLM, v[r].x, 1 << lanebit);
    const double py = __shfl_xor_sync(FULLM, v[r].y, 1 << lanebit);
    v[r] = make_double2(fma(-t, py, v[r].x), fma(t, px, v[r].y));
  }
}
template <int FROM, int TO>
__device__ __forceinline__ void xchg(double2* xb, double2 (&v)[RPT], int lane, int warp, int g) {
  const int bs = padA(pat_tl<FROM>(lane, warp));
#pragma unroll
  for (int r = 0; r < RPT; r++) xb[bs + padA(r << reg_shift<FROM>())] = v[r];
  group_bar(g);
  const int bl = padA(pat_tl<TO>(lane, warp));
#pragma unroll
  for (int r = 0; r < RPT; r++) v[r] = xb[bl + padA(r << reg_shift<TO>())];
  group_bar(g);
}
template <int P>
__device__ __forceinline__ void diag(double2 (&v)[RPT], const uint8_t* es, const double2* phis, int lane, int warp) {
  const int tl = pat_tl<P>(lane, warp);
#pragma unroll
  for (int r = 0; r < RPT; r++) {
    const int e = es[tl | (r << reg_shift<P>())];
    const double2 f = phis[e];
    const double2 x = v[r];
    v[r] = make_double2(fma(f.x, x.x, -f.y * x.y), fma(f.x, x.y, f.y * x.x));
  }
}

template <int PROG, bool LANE3>
__device__ __forceinline__ void program(const TmaArgs& a, double2 (&v)[RPT], double2* xb, const uint8_t* es,
                                        const double2* phis, int lane, int warp, int g) {
  const double(&t0)[TILE_BITS] = a.t[0];
  const double(&t1)[TILE_BITS] = a.t[1];
  if (PROG == FP_G0_DPOST) {
    diag<PA>(v, es, phis, lane, warp);
    rot_regs<PA>(v, t1);
    xchg<PA, PC>(xb, v, lane, warp, g);
    rot_regs<PC>(v, t1);
    xchg<PC, PB>(xb, v, lane, warp, g);
    rot_regs<PB>(v, t1);
  } else if (PROG == FP_G0_PRE) {
    rot_regs<PA>(v, t0);
    xchg<PA, PC>(xb, v, lane, warp, g);
    rot_regs<PC>(v, t0);
    xchg<PC, PB>(xb, v, lane, warp, g);
    rot_regs<PB>(v, t0);
  } else if (PROG == FP_G0_PRE_D_POST) {
    rot_regs<PA>(v, t0);
    xchg<PA, PC>(xb, v, lane, warp, g);
    rot_regs<PC>(v, t0);
    xchg<PC, PB>(xb, v, lane, warp, g);
    rot_regs<PB>(v, t0);
    diag<PB>(v, es, phis, lane, warp);
    rot_regs<PB>(v, t1);
    xchg<PB, PC>(xb, v, lane, warp, g);
    rot_regs<PC>(v, t1);
    xchg<PC, PA>(xb, v, lane, warp, g);
    rot_regs<PA>(v, t1);
  } else if (PROG == FP_GK_PRE) {
    rot_regs<PA>(v, t0);
    xchg<PA, PB>(xb, v, lane, warp, g);
    rot_regs<PB>(v, t0);
    if (LANE3) rot_lane(v, 3, t0[3]);
  } else if (PROG == FP_GK_PRE_D_POST) {
    rot_regs<PA>(v, t0);
    xchg<PA, PB>(xb, v, lane, warp, g);
    rot_regs<PB>(v, t0);
    if (LANE3) rot_lane(v, 3, t0[3]);
    diag<PB>(v, es, phis, lane, warp);
    rot_regs<PB>(v, t1);
    if (LANE3) rot_lane(v, 3, t1[3]);
    xchg<PB, PA>(xb, v, lane, warp, g);
    rot_regs<PA>(v, t1);
  }
}

template <int PROG>
struct Info {
  static constexpr bool has_d = PROG == FP_G0_DPOST || PROG == FP_G0_PRE_D_POST || PROG == FP_GK_PRE_D_POST;
  static constexpr int store_pat = (PROG == FP_G0_PRE_D_POST || PROG == FP_GK_PRE_D_POST) ? PA : PB;
};

// The CTA's j-th tile. Tiles come in pairs (2m, 2m+1) that differ only in the
// lowest tile-id bit -- for the strided groups that is physical bit c, so the
// pair's two TMA loads (issued back to back, one per consumer group) fetch
// adjacent 128-byte rows: 256-byte DRAM bursts from one SM.
__device__ __forceinline__ int64_t tile_of(int64_t j) {
  return 2 * (blockIdx.x + (j >> 1) * (int64_t)gridDim.x) + (j & 1);
}

template <int PROG, int NG>
__device__ __forceinline__ void issue_tile(const CUtensorMap* tmap, const TmaArgs& a, int64_t j, double2* slots,
                                           uint8_t* eslots, uint64_t* full) {
  using I = Info<PROG>;
  const int s = (int)(j % TMA_SLOTS);
  const int64_t T = tile_of(j);
  uint64_t* fb = &full[NG * s + (int)(j % NG)];
  mbar_expect_tx(fb, TILE * 16u + (I::has_d ? (uint32_t)TILE : 0u));
  double2* dst = slots + (size_t)s * FAST_XBUF;
  if (a.contiguous) {
    bulk_g2s(dst, a.psi + tbase(a, T), TILE * 16u, fb);
  } else {
    int c[5];
#pragma unroll
    for (int d = 0; d < 5; d++) {
      const int sg = a.dim_seg[d];
      c[d] = sg < 0 ? 0 : (int)((T >> a.seg_src[sg]) & (((int64_t)1 << a.seg_len[sg]) - 1));
    }
    tma_load(dst, tmap, c, a.ndims, fb);
  }
  if (I::has_d) bulk_g2s(eslots + (size_t)s * TILE, a.Eg + T * TILE, TILE, fb);
}

template <int PROG, bool LANE3, int NG>
__global__ void __launch_bounds__(NG * NTHREADS, 1) qaa_pass_tma(const __grid_constant__ CUtensorMap tmap,
                                                                const TmaArgs a) {
  extern __shared__ __align__(128) unsigned char sm[];
  double2* slots = reinterpret_cast<double2*>(sm);
  uint8_t* eslots = sm + TMA_SLOTS * SLOT_BYTES;
  double2* phis = reinterpret_cast<double2*>(eslots + TMA_SLOTS * TILE);
  // full[NG*s + g]: slot s landed for consumer group g. Tile j uses slot j % 3
  // and group j % NG, so each (slot, group) barrier is used by every (3 NG)-th
  // tile, always by the same group, and a parity wait can never see a stale phase.
  uint64_t* full = reinterpret_cast<uint64_t*>(phis + 256);
  using I = Info<PROG>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // tiles of this CTA: pairs (2m, 2m+1), m = blockIdx.x + i gridDim.x (ntiles is even)
  const int64_t nt = 2 * ((a.ntiles / 2 - blockIdx.x + gridDim.x - 1) / gridDim.x);
  if (tid == 0) {
    for (int s = 0; s < NG * TMA_SLOTS; s++) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int64_t j = 0; j < TMA_SLOTS && j < nt; j++) issue_tile<PROG, NG>(&tmap, a, j, slots, eslots, full);
  }
  if (I::has_d)
    for (int e = tid; e < a.n_phi; e += NG * NTHREADS) phis[e] = a.phi[e];
  __syncthreads();
  // NG consumer groups of 8 warps; the group that frees a slot refills it with
  // tile j + 3 -- no producer warp, so 16 warps x 128 registers fit the
  // register file. NG = 1 keeps two slots in flight (latency-bound passes),
  // NG = 2 overlaps two groups' transposes and FMAs (compute-heavy passes).
  const int g = warp >> 3, lw = warp & 7;
  const Off ps = make_off<I::store_pat>(a, lane, lw);
  const int tlA = pat_tl<PA>(lane, lw);
  double2 v[RPT];
  for (int64_t j = g; j < nt; j += NG) {
    const int s = (int)(j % TMA_SLOTS);
    mbar_wait(&full[NG * s + g], (uint32_t)((j / (NG * TMA_SLOTS)) & 1));
    double2* xb = slots + (size_t)s * FAST_XBUF;
    const uint8_t* es = eslots + (size_t)s * TILE;
#pragma unroll
    for (int r = 0; r < RPT; r++) v[r] = xb[tlA | (r << 8)];  // landed layout: tile-local order
    group_bar(g);
    program<PROG, LANE3>(a, v, xb, es, phis, lane, lw, g);
    // release the slot: order this group's generic smem accesses before the
    // async-proxy (TMA) write that refills it
    fence_async_shared();
    group_bar(g);
    if ((tid & (NTHREADS - 1)) == 0 && j + TMA_SLOTS < nt)
      issue_tile<PROG, NG>(&tmap, a, j + TMA_SLOTS, slots, eslots, full);
    const int64_t T = tile_of(j);
    double2* dst = a.psi + tbase(a, T);
#pragma unroll
    for (int r = 0; r < RPT; r++) dst[roff(ps, r)] = v[r];
  }
}

typedef void (*TmaKernel)(const CUtensorMap, const TmaArgs);

template <int NG>
TmaKernel pick_ng(int prog, bool lane3) {
  switch (prog) {
    case FP_G0_DPOST: return qaa_pass_tma<FP_G0_DPOST, false, NG>;
    case FP_G0_PRE: return qaa_pass_tma<FP_G0_PRE, false, NG>;
    case FP_G0_PRE_D_POST: return qaa_pass_tma<FP_G0_PRE_D_POST, false, NG>;
    case FP_GK_PRE: return lane3 ? qaa_pass_tma<FP_GK_PRE, true, NG> : qaa_pass_tma<FP_GK_PRE, false, NG>;
    case FP_GK_PRE_D_POST:
      return lane3 ? qaa_pass_tma<FP_GK_PRE_D_POST, true, NG> : qaa_pass_tma<FP_GK_PRE_D_POST, false, NG>;
    default: return nullptr;
  }
}
TmaKernel pick(int prog, bool lane3, int ng) { return ng == 1 ? pick_ng<1>(prog, lane3) : pick_ng<2>(prog, lane3); }

}  // namespace

constexpr size_t TMA_SMEM_BYTES =
    (size_t)TMA_SLOTS * SLOT_BYTES + (size_t)TMA_SLOTS * TILE + 256 * 16 + TMA_MAX_GROUPS * TMA_SLOTS * 8;

cudaError_t pass_tma_setup() {
  for (int p = 0; p < FP_COUNT; p++)
    for (int l = 0; l < 2; l++)
      for (int ng = 1; ng <= 2; ng++) {
        cudaError_t e =
            cudaFuncSetAttribute(pick(p, l, ng), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TMA_SMEM_BYTES);
        if (e != cudaSuccess) return e;
      }
  return cudaSuccess;
}

cudaError_t launch_pass_tma(const CUtensorMap* map, const TmaArgs& a, int prog, bool lane3, int ngroups, int grid,
                            cudaStream_t st) {
  TmaKernel k = pick(prog, lane3, ngroups);
  if (!k) return cudaErrorInvalidValue;
  k<<<grid, ngroups * NTHREADS, TMA_SMEM_BYTES, st>>>(*map, a);
  return cudaGetLastError();
}

}  // namespace qaa
