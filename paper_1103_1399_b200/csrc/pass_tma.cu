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

#include "pass_common.cuh"

namespace qaa {
namespace {

using namespace pc;
#define FULLM QAA_FULLM
// Cross-warp exchange through the padded layout. The leading barrier is the
// write-after-read guard (every warp of the group has finished reading the
// buffer: the landed tile or the previous exchange), placed after the caller's
// rotations so warp skew overlaps FMAs; the second orders the STS before the LDS.
// Swap register bit 3 with lane bit 3 (PB <-> PB3: PB3 holds tile bit 3 in
// register bit 3 and tile bit 7 in lane bit 3). Half the amplitudes move, one
// 64-bit shuffle pair each: 32 SHFL per thread, half the cost of rotating lane
// bit 3 in place (every amplitude needs its partner).
__device__ __forceinline__ void swap_r3_l3(double2 (&v)[RPT], int lane) {
  const bool hi = (lane >> 3) & 1;
#pragma unroll
  for (int r = 0; r < 8; r++) {
    const double2 x = hi ? v[r] : v[r | 8];
    const double2 y = make_double2(__shfl_xor_sync(FULLM, x.x, 8), __shfl_xor_sync(FULLM, x.y, 8));
    if (hi)
      v[r] = y;
    else
      v[r | 8] = y;
  }
}
// rotate the four register bits of PB3: register bits 0..2 = tile bits 4..6, 3 = tile bit 3
__device__ __forceinline__ void rot_regs_pb3(double2 (&v)[RPT], const double (&t)[TILE_BITS]) {
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const double c = i < 3 ? t[4 + i] : t[3];
#pragma unroll
    for (int r = 0; r < RPT; r++)
      if (!(r & (1 << i))) rot2(v[r], v[r | (1 << i)], c);
  }
}
template <int FROM, int TO>
__device__ __forceinline__ void xchg(double2* xb, double2 (&v)[RPT], int lane, int warp, int g) {
  const int bs = padA(pat_tl<FROM>(lane, warp));
  group_bar(g);
#pragma unroll
  for (int r = 0; r < RPT; r++) xb[bs + padA(r << reg_shift<FROM>())] = v[r];
  group_bar(g);
  const int bl = padA(pat_tl<TO>(lane, warp));
#pragma unroll
  for (int r = 0; r < RPT; r++) v[r] = xb[bl + padA(r << reg_shift<TO>())];
}
// Split-phase write-after-read guard (the L2-blocked step, SuperArgs.v2): every
// thread of the group arrives on the group's WAR mbarrier (count 256, release
// semantics: its reads of the buffer are performed first) right after its last
// read of the buffer, and waits on it only right before its next write into the
// buffer -- the rotations in between no longer wait for the slowest warp.
struct War {
  uint64_t* bar;
  uint32_t ph;
};
template <bool SPLIT>
__device__ __forceinline__ void war_arrive(War& w) {
  if (SPLIT) mbar_arrive_notx(w.bar);
}
template <int FROM, int TO, bool SPLIT>
__device__ __forceinline__ void xchg_s(double2* xb, double2 (&v)[RPT], int lane, int warp, int g, War& w) {
  if (!SPLIT) {
    xchg<FROM, TO>(xb, v, lane, warp, g);
    return;
  }
  const int bs = padA(pat_tl<FROM>(lane, warp));
  mbar_wait(w.bar, w.ph & 1);
  w.ph++;
#pragma unroll
  for (int r = 0; r < RPT; r++) xb[bs + padA(r << reg_shift<FROM>())] = v[r];
  group_bar(g);
  const int bl = padA(pat_tl<TO>(lane, warp));
#pragma unroll
  for (int r = 0; r < RPT; r++) v[r] = xb[bl + padA(r << reg_shift<TO>())];
}
// Warp-local exchange PB -> PC, in place in the landed (unpadded) tile. Both
// patterns hold warp bits 9..11, so a warp only ever touches its own 512
// amplitudes: no group barrier. Position of local index l: l ^ ((l >> 4) & 7)
// (bits 4..6 XORed into the 16-byte bank group): a quarter-warp of PB varies
// bits 0..2, one of PC bits 4..6 -- 8 distinct bank groups either way.
__device__ __forceinline__ int swz(int l) { return l ^ ((l >> 4) & 7); }
__device__ __forceinline__ void xchg_local_pb_pc(double2* xb, double2 (&v)[RPT], int lane, int warp) {
  const int tb = pat_tl<PB>(lane, warp), tc = pat_tl<PC>(lane, warp);
  __syncwarp();  // every lane's landed read of these positions is done
#pragma unroll
  for (int r = 0; r < RPT; r++) xb[swz(tb | (r << 4))] = v[r];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < RPT; r++) v[r] = xb[swz(tc | r)];
}
// D: PACKED = the group-k energy slice in PB thread-major order (16 bytes per
// thread, one conflict-free LDS.128); otherwise tile-local order, one byte per amplitude
template <int P, bool PACKED>
__device__ __forceinline__ void diag(double2 (&v)[RPT], const uint8_t* es, const double2* phis, int lane, int warp) {
  const int tl = pat_tl<P>(lane, warp);
  uint4 pk = make_uint4(0, 0, 0, 0);
  if (PACKED) pk = reinterpret_cast<const uint4*>(es)[lane + 32 * warp];
#pragma unroll
  for (int r = 0; r < RPT; r++) {
    const uint32_t w = r < 4 ? pk.x : (r < 8 ? pk.y : (r < 12 ? pk.z : pk.w));
    const int e = PACKED ? (int)((w >> (8 * (r & 3))) & 0xffu) : es[tl | (r << reg_shift<P>())];
    // Phi is stored 8x interleaved (entry e of copy c at 8e + c): the 8 lanes of
    // a quarter-warp read copies lane & 7, i.e. 8 distinct 16-byte bank groups,
    // whatever their energies -- a conflict-free 128-bit lookup
    const double2 f = phis[e * PHI_COPIES + (lane & (PHI_COPIES - 1))];
    const double2 x = v[r];
    v[r] = make_double2(fma(f.x, x.x, -f.y * x.y), fma(f.x, x.y, f.y * x.x));
  }
}

// EARLY: the final PA rotation stops after its first register bit (which reads
// every register, so the last exchange's loads have landed); the caller releases
// the slot and then applies bits 1..3 (program_tail) -- the slot's refill starts
// that much earlier
template <int PROG, bool LANE3, bool SPLIT = false, int DIAG = 0, bool EARLY = false>
__device__ __forceinline__ void program(const TmaArgs& a, double2 (&v)[RPT], double2* xb, const uint8_t* es,
                                        const double2* phis, int lane, int warp, int g, War& w) {
  static_assert(!SPLIT || PROG == FP_G0_PRE || PROG == FP_GK_PRE || PROG == FP_GK_PRE_D_POST,
                "split-phase WAR guard: L2-blocked step programs only");
  const double(&t0)[TILE_BITS] = a.t[0];
  const double(&t1)[TILE_BITS] = a.t[1];
  if (PROG == FP_G0_DPOST) {
    diag<PA, false>(v, es, phis, lane, warp);
    rot_regs<PA>(v, t1);
    xchg<PA, PC>(xb, v, lane, warp, g);
    rot_regs<PC>(v, t1);
    xchg<PC, PB>(xb, v, lane, warp, g);
    rot_regs<PB>(v, t1);
  } else if (PROG == FP_G0_PRE) {
    // landed read in PB; PB -> PC warp-local; one cross-warp exchange to PA
    if (!(DIAG & 1)) rot_regs<PB>(v, t0);
    if (!(DIAG & 2)) xchg_local_pb_pc(xb, v, lane, warp);
    if (!(DIAG & 2)) war_arrive<SPLIT>(w);
    if (!(DIAG & 1)) rot_regs<PC>(v, t0);
    if (!(DIAG & 2)) xchg_s<PC, PA, SPLIT>(xb, v, lane, warp, g, w);
    if (!(DIAG & 1)) rot_regs_range<PA, 0, EARLY ? 1 : 4>(v, t0);
  } else if (PROG == FP_G0_PRE_D_POST) {
    rot_regs<PA>(v, t0);
    xchg<PA, PC>(xb, v, lane, warp, g);
    rot_regs<PC>(v, t0);
    xchg<PC, PB>(xb, v, lane, warp, g);
    rot_regs<PB>(v, t0);
    diag<PB, false>(v, es, phis, lane, warp);
    rot_regs<PB>(v, t1);
    xchg<PB, PC>(xb, v, lane, warp, g);
    rot_regs<PC>(v, t1);
    xchg<PC, PA>(xb, v, lane, warp, g);
    rot_regs<PA>(v, t1);
  } else if (PROG == FP_GK_PRE) {
    if (!(DIAG & 2)) war_arrive<SPLIT>(w);
    if (!(DIAG & 1)) rot_regs<PA>(v, t0);
    if (!(DIAG & 2)) xchg_s<PA, PB, SPLIT>(xb, v, lane, warp, g, w);
    if (!(DIAG & 1)) rot_regs<PB>(v, t0);
    if (LANE3) rot_lane(v, 3, t0[3]);
  } else if (PROG == FP_GK_PRE_D_POST) {
    if (!(DIAG & 2)) war_arrive<SPLIT>(w);
    if (!(DIAG & 1)) rot_regs<PA>(v, t0);
    if (!(DIAG & 2)) xchg_s<PA, PB, SPLIT>(xb, v, lane, warp, g, w);
    if (!(DIAG & 2)) war_arrive<SPLIT>(w);
    if (!(DIAG & 1)) rot_regs<PB>(v, t0);
    if (LANE3) {
      // tile bit 3 through a register: PB -> PB3, D in PB3 (the packed energy
      // slice follows PB3), post rotations of bits 3..6, PB3 -> PB, bit 7
      if (!(DIAG & 1)) swap_r3_l3(v, lane);
      if (!(DIAG & 1)) rot_regbit<3>(v, t0[3]);
      if (!(DIAG & 4)) diag<PB, true>(v, es, phis, lane, warp);
      if (!(DIAG & 1)) rot_regs_pb3(v, t1);
      if (!(DIAG & 1)) swap_r3_l3(v, lane);
      if (!(DIAG & 1)) rot_regbit<3>(v, t1[7]);
    } else {
      if (!(DIAG & 4)) diag<PB, true>(v, es, phis, lane, warp);
      if (!(DIAG & 1)) rot_regs<PB>(v, t1);
    }
    if (!(DIAG & 2)) xchg_s<PB, PA, SPLIT>(xb, v, lane, warp, g, w);
    if (!(DIAG & 1)) rot_regs_range<PA, 0, EARLY ? 1 : 4>(v, t1);
  }
}
// the rest of an EARLY program's final PA rotation
template <int PROG>
__device__ __forceinline__ void program_tail(const TmaArgs& a, double2 (&v)[RPT]) {
  static_assert(PROG == FP_G0_PRE || PROG == FP_GK_PRE_D_POST, "EARLY: L2-blocked step programs only");
  rot_regs_range<PA, 1, 4>(v, PROG == FP_G0_PRE ? a.t[0] : a.t[1]);
}

template <int PROG>
struct Info {
  static constexpr bool has_d = PROG == FP_G0_DPOST || PROG == FP_G0_PRE_D_POST || PROG == FP_GK_PRE_D_POST;
  static constexpr int store_pat = (PROG == FP_G0_PRE_D_POST || PROG == FP_GK_PRE_D_POST || PROG == FP_G0_PRE) ? PA : PB;
  // pattern of the read from the landed tile (both are conflict-free on the
  // unpadded layout: a quarter-warp reads 8 consecutive amplitudes)
  static constexpr int load_pat = PROG == FP_G0_PRE ? PB : PA;
};

template <int P>
__device__ __forceinline__ void load_landed(double2 (&v)[RPT], const double2* xb, int lane, int warp) {
  const int tl = pat_tl<P>(lane, warp);
#pragma unroll
  for (int r = 0; r < RPT; r++) v[r] = xb[tl | (r << reg_shift<P>())];
}

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
  uint64_t* full = reinterpret_cast<uint64_t*>(phis + TMA_MAX_PHI * PHI_COPIES);
  unsigned* cnt = slot_counters(sm);
  using I = Info<PROG>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < TMA_SLOTS) cnt[tid] = 0;
  // tiles of this CTA: pairs (2m, 2m+1), m = blockIdx.x + i gridDim.x (ntiles is even)
  const int64_t nt = 2 * ((a.ntiles / 2 - blockIdx.x + gridDim.x - 1) / gridDim.x);
  if (tid == 0) {
    for (int s = 0; s < NG * TMA_SLOTS; s++) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int64_t j = 0; j < TMA_SLOTS && j < nt; j++) issue_tile<PROG, NG>(&tmap, a, j, slots, eslots, full);
  }
  if (I::has_d)
    for (int e = tid; e < a.n_phi * PHI_COPIES; e += NG * NTHREADS) phis[e] = a.phi[e / PHI_COPIES];
  __syncthreads();
  // NG consumer groups of 8 warps; the group that frees a slot refills it with
  // tile j + 3 -- no producer warp, so 16 warps x 128 registers fit the
  // register file. NG = 1 keeps two slots in flight (latency-bound passes),
  // NG = 2 overlaps two groups' transposes and FMAs (compute-heavy passes).
  const int g = warp >> 3, lw = warp & 7;
  const Off ps = make_off<I::store_pat>(a, lane, lw);
  double2 v[RPT];
  for (int64_t j = g; j < nt; j += NG) {
    const int s = (int)(j % TMA_SLOTS);
    mbar_wait(&full[NG * s + g], (uint32_t)((j / period<NG>()) & 1));
    double2* xb = slots + (size_t)s * FAST_XBUF;
    const uint8_t* es = eslots + (size_t)s * TILE;
    load_landed<I::load_pat>(v, xb, lane, lw);  // landed layout: tile-local order
    // no barrier: the first shared-memory write of every program is warp-local
    // in place or an exchange with a leading barrier
    War w{nullptr, 0};
    program<PROG, LANE3>(a, v, xb, es, phis, lane, lw, g, w);
    // release the slot (the program's final rotations consumed every value this
    // warp read from it); the last warp of the group refills it
    __syncwarp();
    if (lane == 0 && last_warp_out(&cnt[s]) && j + TMA_SLOTS < nt)
      issue_tile<PROG, NG>(&tmap, a, j + TMA_SLOTS, slots, eslots, full);
    const int64_t T = tile_of(j);
    double2* dst = a.psi + tbase(a, T);
#pragma unroll
    for (int r = 0; r < RPT; r++) dst[roff(ps, r)] = v[r];
  }
}

// ============================================================================
// L2-blocked Trotter step ("super-pass"): group 0 (rotate step j) and then
// group k (rotate step j, D_{j+1}, rotate step j+1) over the same L2-resident
// chunk -- exactly the pass pair [G0 pre j][Gk pre j, D_{j+1}, post j+1] of the
// schedule-mode-2 plan, fused into one HBM round trip.
// A chunk fixes every physical bit outside (group 0 u group k) tile bits, so
// its 2^tpc_bits group-0 tiles and 2^tpc_bits group-k tiles cover the same
// 2^(12+tpc_bits) amplitudes (32 MiB at n = 30). Group-0 tiles come from HBM
// as contiguous 64 KiB bulk copies and are written back into L2; the group-k
// tiles of the chunk (128-byte strided rows) then hit L2, and their dirty
// lines leave L2 as write-backs.
//
// Work is one sequence: A(0), then for c = 0..nch-1: [A(c+1)] B(c), where
// A(c) = the group-0 tiles of chunk c and B(c) = its group-k tiles, dealt
// round robin (tile J of CTA b = item b + J gridDim.x; optionally through a
// global atomic counter). B(c) needs every A(c) tile stored (done[c] ==
// 2^tpc_bits); the one-segment lag keeps two chunks live in L2. The issuing
// thread never waits: an unmet dependency marks the slot "deferred", and the
// owning group -- whose own later items all come later in the sequence, so hold
// nothing chunk c needs -- waits and loads it itself. A group's items are taken
// in sequence order (item J is fetched when J-3 is freed, and J-3, J-1 belong
// to the same group), so its first END is its last item. Without D (BD = false)
// the group-k sub-pass is a plain rotate, optionally storing into the peers'
// next shard buffers (the sharded plan's layout swap).
// ============================================================================
// BD: the group-k sub-pass is rotate/D/rotate (single GPU); otherwise a plain
// rotate whose tiles may be stored straight into the peers' next shard buffers
// (a.remote: the layout swap of the sharded plan)
// V2 (SuperArgs.v2, default): split-phase write-after-read guards on a per-group
// mbarrier (xchg_s) and a DEFERRED per-warp publish of the group-0 tiles: a warp
// does not wait for its group after its stores; it remembers the chunk and adds
// its 1/8 of the tile to done[c] (red.release) at its next tile's first exchange,
// when its stores have drained -- or before any wait on a chunk and at the end,
// so a chunk's count can never wait on a warp that waits for it.
template <bool LANE3, int NG, bool BD, bool V2, int DIAG = 0, bool REV = false, bool EARLY = false>
__global__ void __launch_bounds__(NG * NTHREADS, 1) qaa_superpass(const __grid_constant__ CUtensorMap kmap,
                                                                 const SuperArgs a) {
  static_assert(!EARLY || (BD && V2 && !REV && DIAG == 0), "EARLY slot release: default step only");
  constexpr int BPROG = BD ? FP_GK_PRE_D_POST : FP_GK_PRE;
  extern __shared__ __align__(128) unsigned char sm[];
  double2* slots = reinterpret_cast<double2*>(sm);
  uint8_t* eslots = sm + TMA_SLOTS * SLOT_BYTES;
  double2* phis = reinterpret_cast<double2*>(eslots + TMA_SLOTS * TILE);
  uint64_t* full = reinterpret_cast<uint64_t*>(phis + TMA_MAX_PHI * PHI_COPIES);
  uint64_t* late = full + NG * TMA_SLOTS;  // per group: deferred group-k loads
  SlotMeta* meta = reinterpret_cast<SlotMeta*>(late + NG);
  unsigned* cnt = slot_counters(sm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < TMA_SLOTS) cnt[tid] = 0;
  // hints: data read once more in this launch (group-0 output) stays, the rest
  // (the loaded tiles, group-k output, energy slices) is marked evict-first
  const uint64_t pol_dead = a.hints ? policy_evict_first() : policy_evict_normal();
  const uint64_t pol_keep = a.hints == 2 ? policy_evict_last() : policy_evict_normal();
  if (tid == 0) {
    for (int s = 0; s < NG * TMA_SLOTS; s++) mbar_init(&full[s], 1);
    for (int g = 0; g < NG; g++) mbar_init(&late[g], 1);
    if (V2)
      for (int g = 0; g < NG; g++) mbar_init(&slot_consumed(sm)[g], NTHREADS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int64_t J = 0; J < TMA_SLOTS; J++) super_issue<NG, BD, REV>(&kmap, a, J, slots, eslots, full, meta, pol_dead);
  }
  if (BD)
    for (int e = tid; e < a.gk.n_phi * PHI_COPIES; e += NG * NTHREADS) phis[e] = a.gk.phi[e / PHI_COPIES];
  __syncthreads();
  const int g = warp >> 3, lw = warp & 7, gtid = tid & (NTHREADS - 1);
  const Off psk = make_off<Info<BPROG>::store_pat>(a.gk, lane, lw);
  const Off ps0 = make_off<Info<FP_G0_PRE>::store_pat>(a.g0, lane, lw);
  uint32_t late_phase = 0;
  double2 v[RPT];
  War war{V2 ? &slot_consumed(sm)[g] : nullptr, 0};
  int pend = -1;        // V2: chunk of this warp's unpublished group-0 tiles
  unsigned pcnt = 0;    // ... and how many (all of chunk pend)
  const unsigned chunk_done = 1u << (a.tpc_bits + a.done_shift);
  // one gpu-scope release per publish: its fence waits for ALL of the warp's
  // earlier stores, so batching pub_batch tiles of a chunk into one release cuts
  // the fence stalls (at the price of completing a chunk up to a tile later)
  auto publish = [&]() {
    if (V2 && pend >= 0) {
      __syncwarp();
      if (lane == 0) red_release_add(&a.done[pend], pcnt);
      pend = -1;
      pcnt = 0;
    }
  };
  for (int64_t J = g;; J += NG) {
    const int s = (int)(J % TMA_SLOTS);
    // never block with an unpublished tile: the landed tile may wait on a load
    // whose issuer waits for this chunk (the refill order is not J order)
    // (warp-uniform decision: publish() contains a __syncwarp)
    if (V2 && pend >= 0 && __any_sync(FULLM, !mbar_test(&full[NG * s + g], (uint32_t)((J / period<NG>()) & 1))))
      publish();
    mbar_wait_bounded(&full[NG * s + g], (uint32_t)((J / period<NG>()) & 1));
    const SlotMeta m = meta[s];
    if (m.kind == SK_END) {
      publish();
      // tile J+3 belongs to the other group and is only ever issued by the
      // finisher of J: pass the end marker on before leaving
      group_bar(g);
      if (gtid == 0) super_issue<NG, BD, REV>(&kmap, a, J + TMA_SLOTS, slots, eslots, full, meta, pol_dead);
      break;
    }
    double2* xb = slots + (size_t)s * FAST_XBUF;
    uint8_t* es = eslots + (size_t)s * TILE;
    if (m.kind == SK_B_DEFERRED) {
      publish();
      if (DIAG & 8) __trap();  // super_issue never defers in this variant
      const long long dt0 = a.dbg ? clock64() : 0;
      if (gtid == 0) {
        unsigned long long t0 = 0;
        for (uint32_t it = 0; ld_acquire(&a.done[m.c]) < chunk_done; it++) {
          __nanosleep(32);
          wait_bound(it, t0);
        }
        fence_async_global();
        if (REV) {
          mbar_expect_tx(&late[g], TILE * 16u);
          bulk_g2s_hint(xb, a.g0.psi + tbase(a.g0, m.T), TILE * 16u, &late[g], pol_dead);
        } else {
          load_gk<BD>(&kmap, a, m.T, xb, es, &late[g], pol_dead);
        }
      }
      mbar_wait_bounded(&late[g], late_phase & 1);
      late_phase++;
      if (a.dbg && gtid == 0) atomicAdd(&a.dbg[7], (unsigned long long)(clock64() - dt0));
    } else if (m.kind == SK_A_DEFERRED) {
      // split roles: the group-0 side ran ahead; wait until the group-k side has
      // issued chunk c - L (a throttle on the L2 live set, not a data dependency)
      if (gtid == 0) {
        const int L = 1 + (a.lag > 1 ? a.lag : 1);
        unsigned long long t0 = 0;
        for (uint32_t it = 0;; it++) {
          unsigned nb;
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(nb) : "l"(&a.doneB[m.c - L]) : "memory");
          if (nb >= (1u << a.tpc_bits)) break;
          __nanosleep(64);
          wait_bound(it, t0);
        }
        mbar_expect_tx(&late[g], TILE * 16u);
        bulk_g2s_hint(xb, a.g0.psi + tbase(a.g0, m.T), TILE * 16u, &late[g], pol_dead);
      }
      mbar_wait_bounded(&late[g], late_phase & 1);
      late_phase++;
    }
    const bool isb = m.kind != SK_A && m.kind != SK_A_DEFERRED;
    const bool gkt = REV ? !isb : isb;  // a group-k tile (rotate/D/rotate)
    if (gkt) {
      load_landed<Info<BPROG>::load_pat>(v, xb, lane, lw);
      if (a.tm_flags & 1) publish();
      program<BPROG, LANE3, V2, DIAG, EARLY>(a.gk, v, xb, es, phis, lane, lw, g, war);
    } else {
      load_landed<Info<FP_G0_PRE>::load_pat>(v, xb, lane, lw);
      if (a.tm_flags & 1) publish();
      program<FP_G0_PRE, false, V2, DIAG, EARLY>(a.g0, v, xb, nullptr, phis, lane, lw, g, war);
    }
    auto tail = [&]() {
      if (EARLY) {
        if (gkt) program_tail<FP_GK_PRE_D_POST>(a.gk, v);
        else program_tail<FP_G0_PRE>(a.g0, v);
      }
    };
    // the previous group-0 tiles' stores have drained by now; keep batching while
    // this tile is a group-0 tile of the same chunk
    if (!(pcnt < (unsigned)a.pub_batch && !gkt && !REV && m.c == pend)) publish();
    // group-k tile stored by ONE TMA tensor store from the slot (tm_flags 4, v2):
    // write-after-read guard, tile-local STS, proxy fence, group barrier; the
    // storing thread refills the slot once the store has read it
    const bool tstore = !REV && V2 && BD && isb && (a.tm_flags & 4) && !a.gk.contiguous && !(DIAG & 32);
    if (tstore) {
      tail();
      war_arrive<true>(war);  // the final rotations consumed every value read from the slot
      mbar_wait(war.bar, war.ph & 1);
      war.ph++;
      const int tl = pat_tl<PA>(lane, lw);
#pragma unroll
      for (int r = 0; r < RPT; r++) xb[tl | (r << reg_shift<PA>())] = v[r];
      fence_async_shared();
      group_bar(g);
      if (gtid == 0) {
        int cc[5];
#pragma unroll
        for (int d = 0; d < 5; d++) {
          const int sg = a.gk.dim_seg[d];
          cc[d] = sg < 0 ? 0 : (int)((m.T >> a.gk.seg_src[sg]) & ((1u << a.gk.seg_len[sg]) - 1));
        }
        tma_store_hint(&kmap, cc, a.gk.ndims, xb, pol_dead);
        bulk_commit();
        bulk_wait_read0();
        super_issue<NG, BD, REV>(&kmap, a, J + TMA_SLOTS, slots, eslots, full, meta, pol_dead);
      }
      continue;
    }
    __syncwarp();
    if (lane == 0 && last_warp_out(&cnt[s])) super_issue<NG, BD, REV>(&kmap, a, J + TMA_SLOTS, slots, eslots, full, meta, pol_dead);
    tail();
    if (REV) {
      // group-k tiles (A items) keep their output in L2 for the group-0 sub-pass;
      // group-0 tiles (B items) are the step's final, contiguous HBM write-back
      if (gkt) {
        double2* dst = a.gk.psi + tbase(a.gk, m.T);
#pragma unroll
        for (int r = 0; r < RPT; r++) st_hint(dst + roff(psk, r), v[r], pol_keep);
        pend = m.c;
        pcnt++;
      } else {
        double2* dst = a.g0.psi + tbase(a.g0, m.T);
#pragma unroll
        for (int r = 0; r < RPT; r++) st_hint(dst + roff(ps0, r), v[r], pol_dead);
      }
      continue;
    }
    if (isb) {
      const int64_t tb = tbase(a.gk, m.T);
      if (!BD && a.remote) {
        // the bit swap of the sharded layouts: the tile's top local bits (not
        // tile bits of this group) name the destination rank (pass_fast.cu store)
        const int64_t j = tb >> a.gshift;
        double2* dst = a.peers[j] + (tb - (j << a.gshift) + ((int64_t)a.rank << a.gshift));
#pragma unroll
        for (int r = 0; r < RPT; r++) dst[roff(psk, r)] = v[r];
      } else if (!(DIAG & 32)) {
        double2* dst = a.gk.psi + tb;
#pragma unroll
        for (int r = 0; r < RPT; r++) st_hint(dst + roff(psk, r), v[r], pol_dead);
      }
    } else {
      double2* dst = a.g0.psi + tbase(a.g0, m.T);
      if (!(DIAG & 64)) {
#pragma unroll
        for (int r = 0; r < RPT; r++) st_hint(dst + roff(ps0, r), v[r], pol_keep);
      }
      if (V2) {
        pend = m.c;  // published one tile later (publish() above)
        pcnt++;
        if (a.tm_flags & 2) publish();
      } else {
        // publish: the group's stores of this group-0 tile happen before the
        // barrier; one gpu-scope release add makes them visible to the
        // acquiring issuer of chunk c's group-k tiles (the grid-sync pattern).
        group_bar(g);
        if (gtid == 0) red_release_add(&a.done[m.c], 1u);
      }
    }
  }
  if (!BD && a.remote) __threadfence_system();
  if (V2 && BD && (a.tm_flags & 4) && gtid == 0) bulk_wait0();  // every tensor store has landed
}


// ============================================================================
// L2-blocked step with a PRODUCER WARP (QAA_OPT_SUPER bit 14): warp 16 alone
// decides what each slot holds and issues its loads; the 16 consumer warps only
// wait for landed tiles, so a chunk dependency never stalls them (with the
// consumer-issued schedule above, 70-80 % of the group-k tiles were found
// deferred and their groups waited on the chunk, then on the load).
// Each CTA owns the group-0 tiles (A) and group-k tiles (B) b, b + grid, ... of
// a launch (chunk order); the producer takes its next B tile when that chunk is
// complete, else its next A tile as long as A stays within one chunk of B (two
// chunks live in L2), else the B tile, waiting for its chunk itself. A filled
// slot never waits on anything but its own load, and every A tile is issued
// before any wait on its chunk, so every chunk completes: no deadlock.
// ============================================================================
constexpr int PW_THREADS = 2 * NTHREADS + 32;

template <bool BD>
__device__ __forceinline__ void pw_issue_b(const CUtensorMap* kmap, const SuperArgs& a, unsigned t, int s,
                                           uint64_t* fb, double2* slots, uint8_t* eslots, SlotMeta* meta,
                                           uint64_t pol) {
  const uint32_t c = t >> a.tpc_bits, i = t & ((1u << a.tpc_bits) - 1);
  const uint32_t T = pdep32(i, a.k_imask) | pdep32(c, a.k_cmask);
  const unsigned target = 1u << a.tpc_bits;
  const long long t0 = (a.tm_flags & 8) ? clock64() : 0;
  unsigned long long tw = 0;
  for (uint32_t it = 0; ld_acquire(&a.done[c]) < target; it++) {
    __nanosleep(64);
    wait_bound(it, tw);
  }
  if (a.tm_flags & 8) atomicAdd(&a.dbg[2], (unsigned long long)(clock64() - t0));
  fence_async_global();  // generic-proxy stores of chunk c -> this async-proxy read
  meta[s] = SlotMeta{SK_B, (int)c, T, 0};
  load_gk<BD>(kmap, a, T, slots + (size_t)s * FAST_XBUF, eslots + (size_t)s * TILE, fb, pol);
}
__device__ __forceinline__ void pw_issue_a(const SuperArgs& a, unsigned t, int s, uint64_t* fb, double2* slots,
                                           SlotMeta* meta, uint64_t pol) {
  const uint32_t c = t >> a.tpc_bits, i = t & ((1u << a.tpc_bits) - 1);
  const uint32_t T = pdep32(i, a.z_imask) | pdep32(c, a.z_cmask);
  meta[s] = SlotMeta{SK_A, (int)c, T, 0};
  mbar_expect_tx(fb, TILE * 16u);
  bulk_g2s_hint(slots + (size_t)s * FAST_XBUF, a.g0.psi + tbase(a.g0, T), TILE * 16u, fb, pol);
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <bool BD>
__device__ void pw_producer(const CUtensorMap* kmap, const SuperArgs& a, double2* slots, uint8_t* eslots,
                            uint64_t* full, uint64_t* empty, SlotMeta* meta, uint64_t pol) {
  // this CTA's own tiles of each kind, round robin, chunk order; the choice
  // between them is made BEFORE waiting for the slot, so the global readiness
  // load overlaps the consumers' work on it
  const unsigned n = (unsigned)a.nchunks << a.tpc_bits;
  const unsigned target = 1u << a.tpc_bits;
  unsigned tA = blockIdx.x, tB = blockIdx.x;
  int ends = 0;
  for (int J = 0; ends < 2; J++) {
    const int s = J % TMA_SLOTS;
    int kind = SK_END;
    if (tB < n) {
      const unsigned cb = tB >> a.tpc_bits;
      if (ld_acquire(&a.done[cb]) >= target) kind = SK_B;
      else if (tA < n && (tA >> a.tpc_bits) <= cb + 1) kind = SK_A;
      else kind = SK_B;  // wait for the chunk at issue time
      if ((a.tm_flags & 8) && kind == SK_B && ld_acquire(&a.done[cb]) < target) atomicAdd(&a.dbg[3], 1ull);
    } else if (tA < n) {
      kind = SK_A;
    }
    if (J >= TMA_SLOTS) {
      const long long t0 = (a.tm_flags & 8) ? clock64() : 0;
      mbar_wait_sleep(&empty[s], (uint32_t)(((J - TMA_SLOTS) / TMA_SLOTS) & 1));
      if (a.tm_flags & 8) atomicAdd(&a.dbg[4], (unsigned long long)(clock64() - t0));
      fence_async_shared();  // the consumers' generic reads of the slot -> the async-proxy refill
    }
    uint64_t* fb = &full[2 * s + (J & 1)];
    if (kind == SK_B) {
      pw_issue_b<BD>(kmap, a, tB, s, fb, slots, eslots, meta, pol);
      tB += gridDim.x;
    } else if (kind == SK_A) {
      pw_issue_a(a, tA, s, fb, slots, meta, pol);
      tA += gridDim.x;
    } else {
      meta[s] = SlotMeta{SK_END, 0, 0, 0};
      mbar_arrive_notx(fb);
      ends++;
    }
  }
}

template <bool LANE3, bool BD>
__global__ void __launch_bounds__(PW_THREADS, 1) qaa_superpass_pw(const __grid_constant__ CUtensorMap kmap,
                                                                 const SuperArgs a) {
  constexpr int NG = 2;
  constexpr int BPROG = BD ? FP_GK_PRE_D_POST : FP_GK_PRE;
  extern __shared__ __align__(128) unsigned char sm[];
  double2* slots = reinterpret_cast<double2*>(sm);
  uint8_t* eslots = sm + TMA_SLOTS * SLOT_BYTES;
  double2* phis = reinterpret_cast<double2*>(eslots + TMA_SLOTS * TILE);
  uint64_t* full = reinterpret_cast<uint64_t*>(phis + TMA_MAX_PHI * PHI_COPIES);
  SlotMeta* meta = reinterpret_cast<SlotMeta*>(full + NG * TMA_SLOTS + NG);
  uint64_t* empty = slot_consumed(sm);  // per slot: its 8 consumer warps are done with it
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t pol_dead = a.hints ? policy_evict_first() : policy_evict_normal();
  const uint64_t pol_keep = a.hints == 2 ? policy_evict_last() : policy_evict_normal();
  if (tid == 0) {
    for (int s = 0; s < NG * TMA_SLOTS; s++) mbar_init(&full[s], 1);
    for (int s = 0; s < TMA_SLOTS; s++) mbar_init(&empty[s], NTHREADS / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (BD)
    for (int e = tid; e < a.gk.n_phi * PHI_COPIES; e += PW_THREADS) phis[e] = a.gk.phi[e / PHI_COPIES];
  __syncthreads();
  if (warp == 2 * (NTHREADS / 32)) {
    if (lane == 0) pw_producer<BD>(&kmap, a, slots, eslots, full, empty, meta, pol_dead);
    return;
  }
  const int g = warp >> 3, lw = warp & 7, gtid = tid & (NTHREADS - 1);
  double2 v[RPT];
  War war{nullptr, 0};
  for (int J = g;; J += NG) {
    const int s = J % TMA_SLOTS;
    const long long t0 = (a.tm_flags & 8) ? clock64() : 0;
    mbar_wait_sleep(&full[NG * s + g], (uint32_t)((J / period<NG>()) & 1));
    if ((a.tm_flags & 8) && lane == 0) {
      atomicAdd(&a.dbg[0], (unsigned long long)(clock64() - t0));
      atomicAdd(&a.dbg[1], 1ull);
    }
    const SlotMeta m = meta[s];
    if (m.kind == SK_END) break;
    double2* xb = slots + (size_t)s * FAST_XBUF;
    uint8_t* es = eslots + (size_t)s * TILE;
    const bool isb = m.kind != SK_A;
    if (isb) {
      load_landed<Info<BPROG>::load_pat>(v, xb, lane, lw);
      program<BPROG, LANE3>(a.gk, v, xb, es, phis, lane, lw, g, war);
    } else {
      load_landed<Info<FP_G0_PRE>::load_pat>(v, xb, lane, lw);
      program<FP_G0_PRE, false>(a.g0, v, xb, nullptr, phis, lane, lw, g, war);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_notx(&empty[s]);
    if (isb) {
      const Off psk = make_off<Info<BPROG>::store_pat>(a.gk, lane, lw);
      const int64_t tb = tbase(a.gk, m.T);
      if (!BD && a.remote) {
        const int64_t j = tb >> a.gshift;
        double2* dst = a.peers[j] + (tb - (j << a.gshift) + ((int64_t)a.rank << a.gshift));
#pragma unroll
        for (int r = 0; r < RPT; r++) dst[roff(psk, r)] = v[r];
      } else {
        double2* dst = a.gk.psi + tb;
#pragma unroll
        for (int r = 0; r < RPT; r++) st_hint(dst + roff(psk, r), v[r], pol_dead);
      }
    } else {
      const Off ps0 = make_off<Info<FP_G0_PRE>::store_pat>(a.g0, lane, lw);
      double2* dst = a.g0.psi + tbase(a.g0, m.T);
#pragma unroll
      for (int r = 0; r < RPT; r++) st_hint(dst + roff(ps0, r), v[r], pol_keep);
      group_bar(g);
      if (gtid == 0) red_release_add(&a.done[m.c], 1u);
    }
  }
  if (!BD && a.remote) __threadfence_system();
}

typedef void (*PwKernel)(const CUtensorMap, const SuperArgs);
PwKernel pick_pw(bool lane3, bool bd) {
  return bd ? (lane3 ? qaa_superpass_pw<true, true> : qaa_superpass_pw<false, true>)
            : (lane3 ? qaa_superpass_pw<true, false> : qaa_superpass_pw<false, false>);
}

typedef void (*SuperKernel)(const CUtensorMap, const SuperArgs);
template <bool BD, bool V2>
SuperKernel pick_super_bd(bool lane3, int ng) {
  if (ng == 1) return lane3 ? qaa_superpass<true, 1, BD, V2> : qaa_superpass<false, 1, BD, V2>;
  return lane3 ? qaa_superpass<true, 2, BD, V2> : qaa_superpass<false, 2, BD, V2>;
}
// diagnostic variants (QAA_OPT_DIAG, bench configuration only; results are wrong
// by design): 1 = no rotations, 2 = no shared-memory exchanges, 4 = no D,
// 8 = group-k tiles ignore the chunk dependency (super_issue), with 7: 16 = no
// group-k tile loads, 32 = no group-k stores, 64 = no group-0 stores
SuperKernel pick_super_diag(int diag) {
  switch (diag) {
    case 1: return qaa_superpass<true, 2, true, true, 1>;
    case 2: return qaa_superpass<true, 2, true, true, 2>;
    case 3: return qaa_superpass<true, 2, true, true, 3>;
    case 4: return qaa_superpass<true, 2, true, true, 4>;
    case 7: return qaa_superpass<true, 2, true, true, 7>;
    case 8: return qaa_superpass<true, 2, true, true, 8>;
    case 15: return qaa_superpass<true, 2, true, true, 15>;
    case 23: return qaa_superpass<true, 2, true, true, 23>;
    case 39: return qaa_superpass<true, 2, true, true, 39>;
    case 71: return qaa_superpass<true, 2, true, true, 71>;
    default: return nullptr;
  }
}
SuperKernel pick_super_rev(bool lane3) {
  return lane3 ? qaa_superpass<true, 2, true, true, 0, true> : qaa_superpass<false, 2, true, true, 0, true>;
}
SuperKernel pick_super_early(bool lane3) {
  return lane3 ? qaa_superpass<true, 2, true, true, 0, false, true> : qaa_superpass<false, 2, true, true, 0, false, true>;
}
SuperKernel pick_super(bool lane3, int ng, bool bd, bool v2) {
  if (v2) return bd ? pick_super_bd<true, true>(lane3, ng) : pick_super_bd<false, true>(lane3, ng);
  return bd ? pick_super_bd<true, false>(lane3, ng) : pick_super_bd<false, false>(lane3, ng);
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



cudaError_t launch_superpass(const CUtensorMap* kmap, const SuperArgs& a, bool lane3, int ngroups, bool bd, int grid,
                             cudaStream_t st) {
  SuperKernel k = pick_super(lane3, ngroups, bd, a.v2 != 0);  // shared-memory attribute set in pass_tma_setup
  if (a.rev) {  // reversed pair: [group k rotate/D/rotate][group 0 rotate] (v2, two groups, with D)
    if (!bd || !a.v2 || ngroups != 2) return cudaErrorInvalidValue;
    k = pick_super_rev(lane3);
  }
  if (a.early && bd && a.v2 && ngroups == 2 && !a.rev && !a.diag) k = pick_super_early(lane3);
  if (a.diag && bd) {  // the D-less closing pair keeps the real kernel
    if (!lane3 || ngroups != 2 || !a.v2 || !pick_super_diag(a.diag)) return cudaErrorInvalidValue;
    k = pick_super_diag(a.diag);
  }
  // cooperative launch: the chunk dependencies spin across CTAs, so every CTA
  // must be co-resident -- the launch fails instead of deadlocking
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)(ngroups * NTHREADS));
  cfg.dynamicSmemBytes = TMA_SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, *kmap, a);
}

cudaError_t launch_superpass_pw(const CUtensorMap* kmap, const SuperArgs& a, bool lane3, bool bd, int grid,
                                cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)PW_THREADS);
  cfg.dynamicSmemBytes = TMA_SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, pick_pw(lane3, bd), *kmap, a);
}

cudaError_t pass_tma_setup() {
  for (int l = 0; l < 2; l++)
    for (int bd = 0; bd < 2; bd++) {
      cudaError_t e = cudaFuncSetAttribute(pick_pw(l, bd), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)TMA_SMEM_BYTES);
      if (e != cudaSuccess) return e;
    }
  for (int l = 0; l < 2; l++)
    for (int ng = 1; ng <= 2; ng++)
      for (int bd = 0; bd < 2; bd++)
        for (int v2 = 0; v2 < 2; v2++) {
          cudaError_t e = cudaFuncSetAttribute(pick_super(l, ng, bd, v2), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)TMA_SMEM_BYTES);
          if (e != cudaSuccess) return e;
        }
  for (int l = 0; l < 2; l++) {
    cudaError_t e = cudaFuncSetAttribute(pick_super_rev(l), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)TMA_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(pick_super_early(l), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TMA_SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  for (int d = 1; d < 128; d++)
    if (pick_super_diag(d)) {
      cudaError_t e = cudaFuncSetAttribute(pick_super_diag(d), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)TMA_SMEM_BYTES);
      if (e != cudaSuccess) return e;
    }
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
