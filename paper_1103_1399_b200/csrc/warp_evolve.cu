// warp_evolve.cu -- all K Trotter steps of a 13..21-qubit state in ONE cooperative
// launch with WARP-sized tiles (SURVEY §7 hard part 5; the
// paper's regime of small instances; VERDICT r01 "persistent evolve for 13 <= n <= 21").
//
// The state (1..32 MiB) stays in L2. A pass of the cyclic step-spanning plan
// (plan.cpp build_pass_schedule, step_spanning 1: K(P-1)+1 passes) runs over tiles
// of 2^9 amplitudes, ONE WARP per tile (16 amplitudes per lane), so a tile's
// program needs no block barrier and is short; passes are separated by a grid
// barrier. Tile groups (WarpGeo): group 0 = physical bits 0..8; group g >= 1 =
// bits {0, 1} (64-byte rows, not rotated) + the next <= 7 bits, filled up with
// more low bits (not rotated) when fewer remain. L = 16: 2 groups, one pass per
// step; 17 <= L <= 23: 3 groups, two passes per step.
// Per tile: load in pattern PL (lane = tile bits 0..4, registers = 5..8; coalesced),
// rotate 5..8, warp-local shared-memory exchange to PX (registers = 0..3, lane =
// 4..8), rotate 0..3 and tile bit 4 (lane bit 0, shuffle), D with the group's
// energy slice packed in PX order (one 16-byte load per lane), the post rotations
// in reverse order, exchange back to PL, store.
// State loads bypass L1 (ld.global.cg): other SMs wrote the data in the previous pass.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "pass_common.cuh"

namespace qaa {
namespace {

using namespace pc;

constexpr int WE_WARPS = 8;
constexpr int WE_BUF = 512 + 32;  // per-warp exchange buffer (amplitudes), padded l + (l >> 4)

template <int FORM>
__device__ __forceinline__ void we_pair(double2& a, double2& b, double c) {
  double2 na, nb;
  if (FORM == 0) {
    na = make_double2(fma(-c, b.y, a.x), fma(c, b.x, a.y));
    nb = make_double2(fma(-c, a.y, b.x), fma(c, a.x, b.y));
  } else {
    na = make_double2(fma(c, a.x, -b.y), fma(c, a.y, b.x));
    nb = make_double2(fma(c, b.x, -a.y), fma(c, b.y, a.x));
  }
  a = na;
  b = nb;
}
// rotate the register bits i (0..3) selected by mask
template <int FORM>
__device__ __forceinline__ void we_regs(double2 (&v)[16], uint32_t mask, double c) {
#pragma unroll
  for (int i = 0; i < 4; i++)
    if ((mask >> i) & 1)
#pragma unroll
      for (int r = 0; r < 16; r++)
        if (!(r & (1 << i))) we_pair<FORM>(v[r], v[r | (1 << i)], c);
}
// rotate lane bit 0: each lane updates its own element from its partner's,
// own' = own + i c partner (tangent) or c own + i partner (cot) -- the same
// formula on both sides of the pair
template <int FORM>
__device__ __forceinline__ void we_lane0(double2 (&v)[16], double c) {
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const double px = __shfl_xor_sync(0xffffffffu, v[r].x, 1);
    const double py = __shfl_xor_sync(0xffffffffu, v[r].y, 1);
    v[r] = FORM == 0 ? make_double2(fma(-c, py, v[r].x), fma(c, px, v[r].y))
                     : make_double2(fma(c, v[r].x, -py), fma(c, v[r].y, px));
  }
}
__device__ __forceinline__ void we_rot(double2 (&v)[16], uint32_t rot, double c, int form, bool pl) {
  if (pl) {
    if (form == 0) we_regs<0>(v, (rot >> 5) & 15, c);
    else we_regs<1>(v, (rot >> 5) & 15, c);
  } else {
    if (form == 0) {
      we_regs<0>(v, rot & 15, c);
      if ((rot >> 4) & 1) we_lane0<0>(v, c);
    } else {
      we_regs<1>(v, rot & 15, c);
      if ((rot >> 4) & 1) we_lane0<1>(v, c);
    }
  }
}
// PL (l = lane | r << 5) <-> PX (l = r | lane << 4) through the warp's padded buffer
template <bool TO_PX>
__device__ __forceinline__ void we_xchg(double2* xb, double2 (&v)[16], int lane) {
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int l = TO_PX ? (lane | (r << 5)) : (r | (lane << 4));
    xb[l + (l >> 4)] = v[r];
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int l = TO_PX ? (r | (lane << 4)) : (lane | (r << 5));
    v[r] = xb[l + (l >> 4)];
  }
}
__device__ __forceinline__ double2 ldcg2(const double2* p) {
  double2 v;
  asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target, int poll_ns = 0) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      if (poll_ns) __nanosleep(poll_ns);  // many teams polling: keep the L2 slices free
    }
  }
  __syncthreads();
}

// One pass of the plan over the tiles T = wid, wid + nwarps, ... < ntiles of the
// state psi (the tile program of the header comment).
__device__ __forceinline__ void we_pass(const WarpGeo& g, const WarpPass& ps, double2* psi, const uint8_t* Eg,
                                        const double2* phi_all, int n_phi, int64_t wid, int64_t nwarps,
                                        int64_t ntiles, int lane, double2* xb) {
  // per-thread offsets of the load/store pattern PL: lane part + 4 register strides
  int64_t thrL = 0, sL[4];
#pragma unroll
  for (int b = 0; b < 5; b++)
    if ((lane >> b) & 1) thrL += (int64_t)1 << g.phys[b];
#pragma unroll
  for (int i = 0; i < 4; i++) sL[i] = (int64_t)1 << g.phys[5 + i];
  const bool pre = ps.flags & WP_PRE, d = ps.flags & WP_D, post = ps.flags & WP_POST;
  const int fpre = (ps.flags >> 3) & 1, fpost = (ps.flags >> 4) & 1;
  const double2* phi = phi_all + ps.d * n_phi;
  const uint32_t rot = g.rot;
  for (int64_t T = wid; T < ntiles; T += nwarps) {
    // tile base: the tile-id bits scattered to the group's free physical bits
    int64_t base = 0;
    for (int i = 0; i < g.nfree; i++)
      if ((T >> i) & 1) base += (int64_t)1 << g.free_bits[i];
    double2 v[16];
    const double2* src = psi + base + thrL;
#pragma unroll
    for (int r = 0; r < 16; r++) {
      int64_t o = 0;
#pragma unroll
      for (int i = 0; i < 4; i++)
        if ((r >> i) & 1) o += sL[i];
      v[r] = ldcg2(src + o);
    }
    uint4 pk = make_uint4(0, 0, 0, 0);
    if (d) pk = __ldg(reinterpret_cast<const uint4*>(Eg + (T << 9) + (lane << 4)));
    if (pre) we_rot(v, rot, ps.cpre, fpre, true);
    we_xchg<true>(xb, v, lane);
    double2 f[16];
    if (d) {  // the D factors: loads issued before the PX rotations that precede their use
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const uint32_t w = r < 4 ? pk.x : (r < 8 ? pk.y : (r < 12 ? pk.z : pk.w));
        f[r] = __ldg(phi + ((w >> (8 * (r & 3))) & 0xffu));
      }
    }
    if (pre) we_rot(v, rot, ps.cpre, fpre, false);
    if (d) {
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = cmul(f[r], v[r]);
    }
    if (post) we_rot(v, rot, ps.cpost, fpost, false);
    we_xchg<false>(xb, v, lane);
    if (post) we_rot(v, rot, ps.cpost, fpost, true);
    double2* dst = psi + base + thrL;
#pragma unroll
    for (int r = 0; r < 16; r++) {
      int64_t o = 0;
#pragma unroll
      for (int i = 0; i < 4; i++)
        if ((r >> i) & 1) o += sL[i];
      __stcg(dst + o, v[r]);
    }
  }
}

__global__ void __launch_bounds__(WE_WARPS * 32, 1) qaa_warp_evolve(const WarpEvolveArgs a) {
  const int nw = blockDim.x >> 5;  // warps per CTA (<= WE_WARPS)
  extern __shared__ __align__(16) double2 xbuf[];  // WE_WARPS x WE_BUF
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* xb = xbuf + warp * WE_BUF;
  const int64_t ntiles = (int64_t)1 << (a.L - 9);
  const int64_t nwarps = (int64_t)gridDim.x * nw;
  const int64_t wid = (int64_t)warp * gridDim.x + blockIdx.x;  // consecutive tiles on different SMs
  // pass records carry their coefficients (host-packed): one 32-byte load per pass,
  // the next one issued before the grid barrier so its latency hides behind it
  WarpPass nx = a.plan[0];
  for (int64_t p = 0; p < a.npass; p++) {
    const WarpPass ps = nx;
    if (p + 1 < a.npass) nx = a.plan[p + 1];
    we_pass(a.geo[ps.group], ps, a.psi, a.Eg[ps.group], a.phi_all, a.n_phi, wid, nwarps, ntiles, lane, xb);
    if (p + 1 < a.npass) grid_barrier(a.bar, (unsigned)(p + 1) * gridDim.x);
  }
}

// ---------------------------------------------------------------------------
// Quad-warp tiles (QAA_OPT_WARPTILE 3): the same tiles, tile groups, pass records
// and grid barriers as qaa_warp_evolve, but each 2^9-amplitude tile is processed
// by FOUR warps (one 128-thread CTA, 4 amplitudes per lane), so the tile's fp64
// work and shuffles are spread over the SM's four sub-partitions instead of one:
// the per-pass critical path (one tile per SM at L = 16) is about a quarter as
// long. Patterns (w = warp of the quad, r = register):
//   P1 (load / store, coalesced): l = lane | r << 5 | w << 7
//   P2 (D):                       l = lane | w << 5 | r << 7
// The lane bits (tile bits 0..4) are rotated with shuffles in either pattern; a
// P1 <-> P2 exchange through shared memory (every warp access is 32 consecutive
// amplitudes: conflict-free, no padding) swaps bits 5,6 <-> 7,8 between the
// registers and the warps. Energies come from the same per-group table as the
// warp-tile kernel (tile-local order): 4 coalesced byte loads per thread.
constexpr int QW_THREADS = 128;

template <int FORM>
__device__ __forceinline__ void qw_lane(double2 (&v)[4], int j, double c) {
#pragma unroll
  for (int r = 0; r < 4; r++) {
    const double px = __shfl_xor_sync(0xffffffffu, v[r].x, 1 << j);
    const double py = __shfl_xor_sync(0xffffffffu, v[r].y, 1 << j);
    v[r] = FORM == 0 ? make_double2(fma(-c, py, v[r].x), fma(c, px, v[r].y))
                     : make_double2(fma(c, v[r].x, -py), fma(c, v[r].y, px));
  }
}
// rotate the register bits (mask bit i = register bit i) and, if lanes, the
// lane bits selected by rot bits 0..4
template <int FORM>
__device__ __forceinline__ void qw_rot_t(double2 (&v)[4], uint32_t regmask, uint32_t lanemask, double c) {
#pragma unroll
  for (int i = 0; i < 2; i++)
    if ((regmask >> i) & 1)
#pragma unroll
      for (int r = 0; r < 4; r++)
        if (!(r & (1 << i))) we_pair<FORM>(v[r], v[r | (1 << i)], c);
#pragma unroll
  for (int j = 0; j < 5; j++)
    if ((lanemask >> j) & 1) qw_lane<FORM>(v, j, c);
}
__device__ __forceinline__ void qw_rot(double2 (&v)[4], uint32_t regmask, uint32_t lanemask, double c, int form) {
  if (form == 0) qw_rot_t<0>(v, regmask, lanemask, c);
  else qw_rot_t<1>(v, regmask, lanemask, c);
}
// Two buffers (P1 -> P2 in xb, P2 -> P1 in xb + 512): a thread's last read of one
// buffer precedes its arrival at the other buffer's barrier, so each exchange
// needs only the barrier between its stores and its loads.
template <bool TO_P2>
__device__ __forceinline__ void qw_xchg(double2* xb, double2 (&v)[4], int lane, int w) {
  if (!TO_P2) xb += 512;
#pragma unroll
  for (int r = 0; r < 4; r++) xb[TO_P2 ? (lane | (r << 5) | (w << 7)) : (lane | (w << 5) | (r << 7))] = v[r];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; r++) v[r] = xb[TO_P2 ? (lane | (w << 5) | (r << 7)) : (lane | (r << 5) | (w << 7))];
}

// one pass of the plan over tiles T = t0, t0 + tstep, ... < ntiles (the quad's
// tile program of the comment above)
__device__ __forceinline__ void qw_pass(const WarpGeo& g, const WarpPass& ps, double2* psi, const uint8_t* Eg,
                                        const double2* phi_all, int n_phi, int64_t t0, int64_t tstep,
                                        int64_t ntiles, int lane, int w, double2* xb, bool have_f0 = false,
                                        const double2* f0 = nullptr) {
  const bool pre = ps.flags & WP_PRE, d = ps.flags & WP_D, post = ps.flags & WP_POST;
  const int fpre = (ps.flags >> 3) & 1, fpost = (ps.flags >> 4) & 1;
  const double2* phi = phi_all + ps.d * n_phi;
  const uint32_t rot = g.rot;
  const uint32_t lm = rot & 31u, r1 = (rot >> 5) & 3u, r2 = (rot >> 7) & 3u;
  // P1 offsets: lane part + warp part; register strides (tile bits 5, 6)
  int64_t thr = 0;
#pragma unroll
  for (int b = 0; b < 5; b++)
    if ((lane >> b) & 1) thr += (int64_t)1 << g.phys[b];
#pragma unroll
  for (int b = 0; b < 2; b++)
    if ((w >> b) & 1) thr += (int64_t)1 << g.phys[7 + b];
  const int64_t s5 = (int64_t)1 << g.phys[5], s6 = (int64_t)1 << g.phys[6];
  for (int64_t T = t0; T < ntiles; T += tstep) {
    int64_t base = 0;
    for (int i = 0; i < g.nfree; i++)
      if ((T >> i) & 1) base += (int64_t)1 << g.free_bits[i];
    const double2* src = psi + base + thr;
    double2 v[4];
    v[0] = ldcg2(src);
    v[1] = ldcg2(src + s5);
    v[2] = ldcg2(src + s6);
    v[3] = ldcg2(src + s5 + s6);
    // D factors: looked up as soon as the energies land, so the (per-pass, L1-cold)
    // phi row load overlaps the pre rotations and the first exchange
    double2 f[4];
    if (d && have_f0 && T == t0) {  // prefetched before the grid barrier (qaa_quad_evolve)
#pragma unroll
      for (int r = 0; r < 4; r++) f[r] = f0[r];
    } else if (d) {
      const uint8_t* et = Eg + (T << 9) + lane + (w << 5);
#pragma unroll
      for (int r = 0; r < 4; r++) f[r] = __ldg(phi + __ldg(et + (r << 7)));
    }
    if (pre) qw_rot(v, r1, lm, ps.cpre, fpre);
    qw_xchg<true>(xb, v, lane, w);
    if (pre) qw_rot(v, r2, 0u, ps.cpre, fpre);
    if (d) {
#pragma unroll
      for (int r = 0; r < 4; r++) v[r] = cmul(f[r], v[r]);
    }
    if (post) qw_rot(v, r2, lm, ps.cpost, fpost);
    qw_xchg<false>(xb, v, lane, w);
    if (post) qw_rot(v, r1, 0u, ps.cpost, fpost);
    double2* dst = psi + base + thr;
    __stcg(dst, v[0]);
    __stcg(dst + s5, v[1]);
    __stcg(dst + s6, v[2]);
    __stcg(dst + s5 + s6, v[3]);
  }
}

__global__ void __launch_bounds__(QW_THREADS) qaa_quad_evolve(const WarpEvolveArgs a) {
  __shared__ __align__(16) double2 xb[1024];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t ntiles = (int64_t)1 << (a.L - 9);
  WarpPass nx = a.plan[0];
  double2 fn[4];  // the next pass's D factors for this CTA's first tile
  bool fn_ok = false;
  for (int64_t p = 0; p < a.npass; p++) {
    const WarpPass ps = nx;
    if (p + 1 < a.npass) nx = a.plan[p + 1];
    qw_pass(a.geo[ps.group], ps, a.psi, a.Eg[ps.group], a.phi_all, a.n_phi, blockIdx.x, gridDim.x, ntiles, lane,
            w, xb, fn_ok, fn);
    if (p + 1 < a.npass) {
      // the energies and phi rows do not depend on the state: look the next pass's
      // factors up now, so their two dependent loads land while the barrier waits
      fn_ok = (nx.flags & WP_D) && (int64_t)blockIdx.x < ntiles;
      if (fn_ok) {
        const uint8_t* et = a.Eg[nx.group] + ((int64_t)blockIdx.x << 9) + lane + (w << 5);
        const double2* phn = a.phi_all + nx.d * a.n_phi;
#pragma unroll
        for (int r = 0; r < 4; r++) fn[r] = __ldg(phn + __ldg(et + (r << 7)));
      }
      grid_barrier(a.bar, (unsigned)(p + 1) * gridDim.x);
    }
  }
}

// F1 sweep on quad-warp tiles: teams of `team` 128-thread CTAs (several per SM),
// team j evolves replicas j, j + nteams, ... (longest first) from the uniform
// state in its own buffer, a team barrier between passes, and leaves P_succ in
// out[] (fixed-order reduction: lanes, warps, then CTAs in id order).
__global__ void __launch_bounds__(QW_THREADS) qaa_quad_sweep(const WarpSweepArgs a) {
  __shared__ __align__(16) double2 xb[1024];
  __shared__ double red[4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int team = a.team, nteams = gridDim.x / team;
  const int j = blockIdx.x / team, lc = blockIdx.x % team;
  if (j >= nteams) return;
  const int64_t ntiles = (int64_t)1 << (a.L - 9);
  double2* psi = a.scratch + ((int64_t)j << a.L);
  double* part = a.partial + (int64_t)j * team;
  unsigned* ctr = a.bar + 32 * j;
  unsigned epoch = 0;
  const int64_t N = (int64_t)1 << a.L;
  for (int rep = j; rep < a.nrep; rep += nteams) {
    for (int64_t i = (int64_t)lc * QW_THREADS + threadIdx.x; i < N; i += (int64_t)team * QW_THREADS)
      __stcg(psi + i, make_double2(a.amp0, 0.0));
    grid_barrier(ctr, ++epoch * (unsigned)team, a.poll_ns);
    const WarpPass* plan = a.plan + a.plan_off[rep];
    const int64_t np = a.plan_len[rep];
    for (int64_t p = 0; p < np; p++) {
      const WarpPass ps = plan[p];
      qw_pass(a.geo[ps.group], ps, psi, a.Eg[ps.group], a.phi_all, a.n_phi, lc, team, ntiles, lane, w, xb);
      grid_barrier(ctr, ++epoch * (unsigned)team, a.poll_ns);
    }
    // P_succ over this CTA's group-0 tiles (group 0: tile bit b = physical bit b)
    double acc = 0.0;
    const WarpGeo& g0 = a.geo[0];
    for (int64_t T = lc; T < ntiles; T += team) {
      int64_t base = 0;
      for (int i = 0; i < g0.nfree; i++)
        if ((T >> i) & 1) base += (int64_t)1 << g0.free_bits[i];
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const int l = threadIdx.x + QW_THREADS * r;
        if (__ldg(a.Eg[0] + (T << 9) + l) == 0) {
          const double2 v = ldcg2(psi + base + l);
          acc += fma(v.x, v.x, v.y * v.y);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[w] = acc;
    __syncthreads();
    if (threadIdx.x == 0) part[lc] = ((red[0] + red[1]) + red[2]) + red[3];
    grid_barrier(ctr, ++epoch * (unsigned)team, a.poll_ns);
    if (lc == 0 && threadIdx.x == 0) {
      double sum = 0.0;
      for (int c = 0; c < team; c++) sum += __ldcg(part + c);  // other SMs wrote them: bypass L1
      a.out[rep] = sum;
    }
    grid_barrier(ctr, ++epoch * (unsigned)team, a.poll_ns);  // part[] and psi are reused by the next replica
  }
}

// F1 sweep on warp tiles: the grid is split into teams of `team` CTAs; team j
// evolves replicas j, j + nteams, ... (longest first, host order) from the
// uniform state in its own state buffer, with a team-wide barrier (its own
// monotone counter) between passes, and leaves P_succ = sum_{E = 0} |psi|^2 of
// each replica in out[] (fixed-order reduction: lanes, then warps in id order).
__global__ void __launch_bounds__(WE_WARPS * 32, 1) qaa_warp_sweep(const WarpSweepArgs a) {
  const int nw = blockDim.x >> 5;
  extern __shared__ __align__(16) double2 xbuf[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* xb = xbuf + warp * WE_BUF;
  const int team = a.team, nteams = gridDim.x / team;
  const int j = blockIdx.x / team, lc = blockIdx.x % team;
  if (j >= nteams) return;
  const int64_t ntiles = (int64_t)1 << (a.L - 9);
  const int64_t nwarps = (int64_t)team * nw;
  const int64_t wid = (int64_t)warp * team + lc;
  double2* psi = a.scratch + ((int64_t)j << a.L);
  double* part = a.partial + (int64_t)j * nwarps;  // per warp of the team
  unsigned* ctr = a.bar + 32 * j;                    // one 128-byte line per team
  unsigned epoch = 0;
  const int64_t N = (int64_t)1 << a.L;
  for (int rep = j; rep < a.nrep; rep += nteams) {
    // uniform start, every team warp on its slice
    for (int64_t i = (wid << 5) + lane; i < N; i += nwarps << 5) __stcg(psi + i, make_double2(a.amp0, 0.0));
    grid_barrier(ctr, ++epoch * (unsigned)team);
    const WarpPass* plan = a.plan + a.plan_off[rep];
    const int64_t np = a.plan_len[rep];
    for (int64_t p = 0; p < np; p++) {
      const WarpPass ps = plan[p];
      we_pass(a.geo[ps.group], ps, psi, a.Eg[ps.group], a.phi_all, a.n_phi, wid, nwarps, ntiles, lane, xb);
      grid_barrier(ctr, ++epoch * (unsigned)team);
    }
    // P_succ: this warp's tiles of group 0 (PX order matches Eg[0])
    double acc = 0.0;
    const WarpGeo& g0 = a.geo[0];
    for (int64_t T = wid; T < ntiles; T += nwarps) {
      int64_t base = 0;
      for (int i = 0; i < g0.nfree; i++)
        if ((T >> i) & 1) base += (int64_t)1 << g0.free_bits[i];
      const uint4 pk = __ldg(reinterpret_cast<const uint4*>(a.Eg[0] + (T << 9) + (lane << 4)));
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const uint32_t w = r < 4 ? pk.x : (r < 8 ? pk.y : (r < 12 ? pk.z : pk.w));
        if (((w >> (8 * (r & 3))) & 0xffu) == 0) {
          const int l = r | (lane << 4);  // group 0: tile bit b = physical bit b
          const double2 v = ldcg2(psi + base + l);
          acc += fma(v.x, v.x, v.y * v.y);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) part[wid] = acc;
    grid_barrier(ctr, ++epoch * (unsigned)team);
    if (lc == 0 && threadIdx.x == 0) {
      double sum = 0.0;
      for (int64_t w = 0; w < nwarps; w++) sum += __ldcg(part + w);  // other SMs wrote them: bypass L1
      a.out[rep] = sum;
    }
    grid_barrier(ctr, ++epoch * (unsigned)team);  // part[] and psi are reused by the next replica
  }
}

// Eg[T * 512 + lane * 16 + r] = E[base(T) + tile-local index (r | lane << 4) scattered]
__global__ void warp_energy_kernel(const uint8_t* E, uint8_t* Eg, WarpGeo g, int L) {
  const int64_t n = (int64_t)1 << L;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t T = i >> 9;
    const int l = (int)(i & 511);  // = lane * 16 + r, the PX local index r | lane << 4
    int64_t x = 0;
    for (int j = 0; j < g.nfree; j++)
      if ((T >> j) & 1) x += (int64_t)1 << g.free_bits[j];
    for (int b = 0; b < 9; b++)
      if ((l >> b) & 1) x += (int64_t)1 << g.phys[b];
    Eg[i] = E[x];
  }
}

}  // namespace

cudaError_t launch_warp_energy(const uint8_t* E, uint8_t* Eg, const WarpGeo& g, int L, int num_sms, cudaStream_t st) {
  warp_energy_kernel<<<num_sms * 4, 256, 0, st>>>(E, Eg, g, L);
  return cudaGetLastError();
}

cudaError_t launch_warp_evolve(const WarpEvolveArgs& a, int grid, int warps, cudaStream_t st) {
  if (warps < 1 || warps > WE_WARPS) return cudaErrorInvalidValue;
  const int smem = warps * WE_BUF * (int)sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(qaa_warp_evolve, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(warps * 32);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, qaa_warp_evolve, a);
}

cudaError_t launch_quad_evolve(const WarpEvolveArgs& a, int grid, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(QW_THREADS);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, qaa_quad_evolve, a);
}
cudaError_t launch_quad_sweep(const WarpSweepArgs& a, int grid, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(QW_THREADS);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, qaa_quad_sweep, a);
}
int quad_sweep_max_active() {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, qaa_quad_sweep, QW_THREADS, 0) != cudaSuccess) return 0;
  return nb;
}
int quad_evolve_max_active() {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, qaa_quad_evolve, QW_THREADS, 0) != cudaSuccess) return 0;
  return nb;
}

cudaError_t launch_warp_sweep(const WarpSweepArgs& a, int grid, cudaStream_t st) {
  const int smem = WE_WARPS * WE_BUF * (int)sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(qaa_warp_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(WE_WARPS * 32);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, qaa_warp_sweep, a);
}

}  // namespace qaa
