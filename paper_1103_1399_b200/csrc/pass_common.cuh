// pass_common.cuh -- device helpers shared by the fused Trotter pass kernels
// (pass_fast.cu, pass_tma.cu, pass_tmem.cu): mbarrier / TMA / L2-policy PTX
// wrappers, the tangent-form rotation, tile addressing, and the work queue of
// the L2-blocked Trotter step.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace qaa {
namespace pc {

#define QAA_FULLM 0xffffffffu

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_notx(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
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
// one non-blocking probe of the phase
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(sa(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait bounds are in TIME (%globaltimer, checked every 4096 polls), not poll
// counts, so slow tool runs (compute-sanitizer racecheck serialises warps) do not
// trip them: a wait longer than WAIT_LIMIT_NS is a lost arrival -> trap (launch
// error) instead of a hang.
constexpr unsigned long long WAIT_LIMIT_NS = 60ull * 1000000000ull;
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// call with the poll count; traps once the wait started >= WAIT_LIMIT_NS ago
__device__ __forceinline__ void wait_bound(uint32_t it, unsigned long long& t0) {
  if ((it & 4095u) != 4095u) return;
  const unsigned long long now = globaltimer_ns();
  if (t0 == 0) t0 = now;
  else if (now - t0 > WAIT_LIMIT_NS) __trap();
}
// bounded wait: a lost arrival becomes a trap (launch error) instead of a hang
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* b, uint32_t parity) {
  unsigned long long t0 = 0;
  for (uint32_t it = 0;; it++) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(sa(b)), "r"(parity)
        : "memory");
    if (ok) return;
    wait_bound(it, t0);
  }
}

// waiting threads suspend in the barrier (suspend-time hint, ns) instead of
// spinning: the other consumer group keeps the issue slots
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  for (uint32_t it = 0;; it++) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(sa(b)), "r"(parity), "r"(1000000u)
        : "memory");
    if (ok) return;
    if (it > 8192u) __trap();
  }
}

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
      "l"(src), "r"(bytes), "r"(sa(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(sa(dst)),
      "l"(src), "r"(bytes), "r"(sa(bar)), "l"(pol)
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
__device__ __forceinline__ void tma_load_hint(void* dst, const CUtensorMap* map, const int (&c)[5], int rank,
                                              uint64_t* bar, uint64_t pol) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  switch (rank) {
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
          "[%1, {%2, %3}], [%4], %5;" ::"r"(sa(dst)),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(sa(bar)), "l"(pol)
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
          "[%1, {%2, %3, %4}], [%5], %6;" ::"r"(sa(dst)),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(sa(bar)), "l"(pol)
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
          "[%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(sa(dst)),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(sa(bar)), "l"(pol)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
          "[%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(sa(dst)),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(sa(bar)), "l"(pol)
          : "memory");
      break;
  }
}

// TMA tensor store of a tile from shared memory (bulk group of the issuing thread)
__device__ __forceinline__ void tma_store_hint(const CUtensorMap* map, const int (&c)[5], int rank, const void* src,
                                               uint64_t pol) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  switch (rank) {
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(m),
          "r"(c[0]), "r"(c[1]), "r"(sa(src)), "l"(pol)
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;" ::"l"(
              m),
          "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(sa(src)), "l"(pol)
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3, %4}], [%5], %6;" ::"l"(
              m),
          "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(sa(src)), "l"(pol)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3, %4, %5}], [%6], "
          "%7;" ::"l"(m),
          "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(sa(src)), "l"(pol)
          : "memory");
      break;
  }
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// L2 eviction-priority hints (createpolicy + .L2::cache_hint), used by the
// L2-blocked step to keep the chunk data that is read again and stream out the rest
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// named barrier over `count` threads
__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ------------------------------------------------------------------ arithmetic
// (x, y) <- (x + i t y, y + i t x): the tangent form of exp(-i beta (1 - sigma^x))
// up to the scalar g cos(beta) folded into the step's Phi table
__device__ __forceinline__ void rot2(double2& x, double2& y, double t) {
  const double2 nx = make_double2(fma(-t, y.y, x.x), fma(t, y.x, x.y));
  const double2 ny = make_double2(fma(-t, x.y, y.x), fma(t, x.x, y.y));
  x = nx;
  y = ny;
}
// rotate register bit I of a thread's 16 amplitudes with coefficient c
template <int I>
__device__ __forceinline__ void rot_regbit(double2 (&v)[RPT], double c) {
#pragma unroll
  for (int r = 0; r < RPT; r++)
    if (!(r & (1 << I))) rot2(v[r], v[r | (1 << I)], c);
}
// psi <- Phi[e] psi
__device__ __forceinline__ double2 cmul(double2 f, double2 x) {
  return make_double2(fma(f.x, x.x, -f.y * x.y), fma(f.x, x.y, f.y * x.x));
}

// ------------------------------------------------------------------ tile addressing
// base offset of tile T: the tile-id bit segments scattered to their physical positions
template <class A>
__device__ __forceinline__ int64_t tbase(const A& a, int64_t T) {
  int64_t b = 0;
#pragma unroll
  for (int s = 0; s < MAX_SEGS; s++)
    if (s < a.nseg) b += ((T >> a.seg_src[s]) & (((int64_t)1 << a.seg_len[s]) - 1)) << a.seg_dst[s];
  return b;
}
// per-thread global offsets of a register pattern: thread part + one stride per register bit
struct Off {
  int64_t thr;
  int64_t s[4];
};
__device__ __forceinline__ int64_t roff(const Off& o, int r) {
  int64_t x = o.thr;
  if (r & 1) x += o.s[0];
  if (r & 2) x += o.s[1];
  if (r & 4) x += o.s[2];
  if (r & 8) x += o.s[3];
  return x;
}
// tile-local index tl (thread part) and the 4 register bits' tile-local positions
template <class A>
__device__ __forceinline__ Off make_off_tl(const A& a, int tl, const int (&rbits)[4]) {
  Off o;
  int64_t t = 0;
#pragma unroll
  for (int b = 0; b < TILE_BITS; b++)
    if ((tl >> b) & 1) t += (int64_t)1 << a.phys[b];
  o.thr = t;
#pragma unroll
  for (int i = 0; i < 4; i++) o.s[i] = (int64_t)1 << a.phys[rbits[i]];
  return o;
}
__device__ __forceinline__ uint32_t pdep32(uint32_t x, uint32_t mask) {
  uint32_t r = 0;
  for (uint32_t m = mask; m; m &= m - 1) {
    if (x & 1u) r |= m & (~m + 1u);
    x >>= 1;
  }
  return r;
}

// ------------------------------------------------------------------ PA/PB/PC register patterns (plan.hpp)
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
template <int P, class A>
__device__ __forceinline__ Off make_off(const A& a, int lane, int warp) {
  const int rb[4] = {reg_shift<P>(), reg_shift<P>() + 1, reg_shift<P>() + 2, reg_shift<P>() + 3};
  return make_off_tl(a, pat_tl<P>(lane, warp), rb);
}
// rotate the 4 register bits of pattern P with per-tile-bit coefficients t[.]
// register bits I0 <= i < I1 of pattern P only (rot_regs = 0..4)
template <int P, int I0, int I1>
__device__ __forceinline__ void rot_regs_range(double2 (&v)[RPT], const double (&t)[TILE_BITS]) {
#pragma unroll
  for (int i = I0; i < I1; i++) {
    const double c = t[reg_shift<P>() + i];
#pragma unroll
    for (int r = 0; r < RPT; r++)
      if (!(r & (1 << i))) rot2(v[r], v[r | (1 << i)], c);
  }
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
// rotate a lane bit: every amplitude needs its partner lane's value
__device__ __forceinline__ void rot_lane(double2 (&v)[RPT], int lanebit, double t) {
#pragma unroll
  for (int r = 0; r < RPT; r++) {
    const double px = __shfl_xor_sync(QAA_FULLM, v[r].x, 1 << lanebit);
    const double py = __shfl_xor_sync(QAA_FULLM, v[r].y, 1 << lanebit);
    v[r] = make_double2(fma(-t, py, v[r].x), fma(t, px, v[r].y));
  }
}

// ------------------------------------------------------------------ TMA pass / L2-blocked step infrastructure
constexpr int TMA_SLOTS = 3;
constexpr int SLOT_BYTES = FAST_XBUF * 16;  // 69632: padded exchange layout
constexpr int TMA_MAX_GROUPS = 2;
constexpr int PHI_COPIES = 8;  // bank-group copies of the D table (diag below)
// dynamic shared memory: 3 slots (padded exchange layout), 3 energy slices, the
// D table copies, mbarriers (full, late), slot metadata, slot counters (last 32 B)
constexpr size_t TMA_SMEM_BYTES = (size_t)TMA_SLOTS * SLOT_BYTES + (size_t)TMA_SLOTS * TILE +
                                   (size_t)TMA_MAX_PHI * PHI_COPIES * 16 + TMA_MAX_GROUPS * TMA_SLOTS * 8 +
                                   TMA_MAX_GROUPS * 8 + TMA_SLOTS * 16 + 128 + 32;
// pass_tmem.cu: per (slot, group) "landed data consumed" mbarriers, then per-slot
// late-load mbarriers and late-load counters, just below the slot counters
__device__ __forceinline__ uint64_t* slot_consumed(unsigned char* sm) {
  return reinterpret_cast<uint64_t*>(sm + TMA_SMEM_BYTES - 32 - 128);
}
__device__ __forceinline__ uint64_t* slot_late(unsigned char* sm) { return slot_consumed(sm) + 2 * TMA_SLOTS; }
__device__ __forceinline__ unsigned* slot_late_count(unsigned char* sm) {
  return reinterpret_cast<unsigned*>(slot_late(sm) + TMA_SLOTS);
}
__device__ __forceinline__ unsigned* slot_counters(unsigned char* sm) {
  return reinterpret_cast<unsigned*>(sm + TMA_SMEM_BYTES - 32);
}

// tile j uses slot j % 3 and consumer group j % NG: each (slot, group)
// barrier sees one phase per lcm(3, NG) tiles
template <int NG>
__device__ __forceinline__ constexpr int period() {
  return NG % TMA_SLOTS == 0 ? NG : NG * TMA_SLOTS;
}
__device__ __forceinline__ void group_bar(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(NTHREADS) : "memory");
}

// "Last warp out refills": each warp, once its values of slot s are consumed,
// bumps the slot's counter (acq_rel at CTA scope); the 8th warp of the group
// resets it and refills the slot -- no group barrier before the refill.
__device__ __forceinline__ bool last_warp_out(unsigned* cnt) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(sa(cnt)) : "memory");
  if (old != (NTHREADS / 32) - 1) return false;
  *cnt = 0;
  fence_async_shared();  // generic-proxy accesses of the slot before the async-proxy refill
  return true;
}
enum SuperKind : int { SK_END = 0, SK_A = 1, SK_B = 2, SK_B_DEFERRED = 3, SK_B_ISSUING = 4, SK_B_LATE = 5, SK_A_DEFERRED = 6 };

// queue position q -> (kind, chunk, intra index); false past the end
// Sequence with a lag of L = max(1, a.lag) chunks: A(0) .. A(L-1), then for
// u = 0, 1, ...: [A(u + L)] B(u) -- B(u) follows the group-0 tiles of L later chunks,
// so L + 1 chunks are live in L2 (L = 1: 64 MiB at n = 30).
__device__ __forceinline__ bool decode_item(const SuperArgs& a, unsigned long long q, int* kind, int64_t* c,
                                            uint32_t* i) {
  const unsigned long long tpc = 1ull << a.tpc_bits;
  const unsigned long long nch = (unsigned long long)a.nchunks;
  unsigned long long L = a.lag > 1 ? (unsigned long long)a.lag : 1ull;
  if (L > nch) L = nch;
  if (q >= 2 * nch * tpc) return false;
  if (q < L * tpc) {
    *kind = SK_A;
    *c = (int64_t)(q / tpc);
    *i = (uint32_t)(q % tpc);
    return true;
  }
  const unsigned long long r0 = q - L * tpc, F = nch - L;  // F segments of 2 tpc items
  if (r0 < F * 2 * tpc) {
    const unsigned long long u = r0 / (2 * tpc), r = r0 % (2 * tpc);
    if (r < tpc) {
      *kind = SK_A;
      *c = (int64_t)(u + L);
      *i = (uint32_t)r;
    } else {
      *kind = SK_B;
      *c = (int64_t)u;
      *i = (uint32_t)(r - tpc);
    }
    return true;
  }
  const unsigned long long r1 = r0 - F * 2 * tpc;
  *kind = SK_B;
  *c = (int64_t)(F + r1 / tpc);
  *i = (uint32_t)(r1 % tpc);
  return true;
}

struct SlotMeta {
  int kind;
  int c;
  uint32_t T;
  int pad;
};

// group-k tile T (tensor-map rows) and, with D, its energy slice, completing on bar
template <bool BD>
__device__ __forceinline__ void load_gk(const CUtensorMap* kmap, const SuperArgs& a, uint32_t T, double2* dst,
                                       uint8_t* edst, uint64_t* bar, uint64_t pol) {
  mbar_expect_tx(bar, TILE * 16u + (BD ? (uint32_t)TILE : 0u));
  if (a.gk.contiguous) {
    bulk_g2s_hint(dst, a.gk.psi + tbase(a.gk, T), TILE * 16u, bar, pol);
  } else {
    int cc[5];
#pragma unroll
    for (int d = 0; d < 5; d++) {
      const int sg = a.gk.dim_seg[d];
      cc[d] = sg < 0 ? 0 : (int)((T >> a.gk.seg_src[sg]) & ((1u << a.gk.seg_len[sg]) - 1));
    }
    tma_load_hint(dst, kmap, cc, a.gk.ndims, bar, pol);
  }
  if (BD) bulk_g2s_hint(edst, a.gk.Eg + (int64_t)T * TILE, TILE, bar, pol);
}

// fetch the next work item for slot J % 3 (tile J of this CTA) and start its load
// REV (reversed pair, SuperArgs-compatible): the first sub-pass (A items) runs the
// group-k tiles -- strided rows from HBM, with D -- and the second (B items) the
// group-0 tiles, contiguous from L2, so the step's HBM write-back is contiguous.
template <int NG, bool BD, bool REV = false>
__device__ void super_issue(const CUtensorMap* kmap, const SuperArgs& a, int64_t J, double2* slots, uint8_t* eslots,
                            uint64_t* full, SlotMeta* meta, uint64_t pol_dead) {
  const int s = (int)(J % TMA_SLOTS);
  uint64_t* fb = &full[NG * s + (int)(J % NG)];
  int kind;
  int64_t c;
  uint32_t i;
  // queue position: a.queue != nullptr -> dynamic (global atomic counter);
  // otherwise static round robin, tile J of CTA b = item b + J * gridDim.x
  if (a.split_a > 0) {
    // split roles: this CTA's J-th tile of its own kind, in chunk order
    const bool isA = (int)blockIdx.x < a.split_a;
    const unsigned long long nrole = isA ? (unsigned)a.split_a : gridDim.x - (unsigned)a.split_a;
    const unsigned long long q = (isA ? blockIdx.x : blockIdx.x - (unsigned)a.split_a) + (unsigned long long)J * nrole;
    if (q >= ((unsigned long long)a.nchunks << a.tpc_bits)) {
      meta[s] = SlotMeta{SK_END, 0, 0, 0};
      mbar_arrive_notx(fb);
      return;
    }
    kind = isA ? SK_A : SK_B;
    c = (int64_t)(q >> a.tpc_bits);
    i = (uint32_t)(q & ((1ull << a.tpc_bits) - 1));
    const int L = 1 + (a.lag > 1 ? a.lag : 1);
    if (isA && c >= L) {
      unsigned nb;
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(nb) : "l"(&a.doneB[c - L]) : "memory");
      if (nb < (1u << a.tpc_bits)) {  // the group-k side is behind: wait at processing time
        const uint32_t T = pdep32(i, a.z_imask) | pdep32((uint32_t)c, a.z_cmask);
        meta[s] = SlotMeta{SK_A_DEFERRED, (int)c, T, 0};
        mbar_arrive_notx(fb);
        return;
      }
    }
    if (!isA) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(&a.doneB[c]) : "memory");
  } else {
    const unsigned long long qpos =
        a.queue ? atomicAdd(a.queue, 1ull) : (unsigned long long)blockIdx.x + (unsigned long long)J * gridDim.x;
    if (!decode_item(a, qpos, &kind, &c, &i)) {
      meta[s] = SlotMeta{SK_END, 0, 0, 0};
      mbar_arrive_notx(fb);
      return;
    }
  }
  if (kind == SK_A) {
    if (REV) {
      const uint32_t T = pdep32(i, a.k_imask) | pdep32((uint32_t)c, a.k_cmask);
      meta[s] = SlotMeta{SK_A, (int)c, T, 0};
      load_gk<BD>(kmap, a, T, slots + (size_t)s * FAST_XBUF, eslots + (size_t)s * TILE, fb, pol_dead);
      return;
    }
    const uint32_t T = pdep32(i, a.z_imask) | pdep32((uint32_t)c, a.z_cmask);
    meta[s] = SlotMeta{SK_A, (int)c, T, 0};
    mbar_expect_tx(fb, TILE * 16u);
    bulk_g2s_hint(slots + (size_t)s * FAST_XBUF, a.g0.psi + tbase(a.g0, T), TILE * 16u, fb, pol_dead);
    return;
  }
  const uint32_t T = REV ? (pdep32(i, a.z_imask) | pdep32((uint32_t)c, a.z_cmask))
                         : (pdep32(i, a.k_imask) | pdep32((uint32_t)c, a.k_cmask));
  if ((a.diag & 8) || ld_acquire(&a.done[c]) >= (1u << (a.tpc_bits + a.done_shift))) {
    fence_async_global();  // generic-proxy stores of chunk c -> this async-proxy read
    meta[s] = SlotMeta{SK_B, (int)c, T, 0};
    if (a.diag & 16) {  // timing diagnostic: the group-k tile "lands" without a load
      mbar_arrive_notx(fb);
    } else if (REV) {
      mbar_expect_tx(fb, TILE * 16u);
      bulk_g2s_hint(slots + (size_t)s * FAST_XBUF, a.g0.psi + tbase(a.g0, T), TILE * 16u, fb, pol_dead);
    } else {
      load_gk<BD>(kmap, a, T, slots + (size_t)s * FAST_XBUF, eslots + (size_t)s * TILE, fb, pol_dead);
    }
  } else {
    meta[s] = SlotMeta{SK_B_DEFERRED, (int)c, T, 0};
    if (a.dbg) atomicAdd(&a.dbg[5], 1ull);  // diagnostics (tm_flags 8): deferred group-k tiles
    mbar_arrive_notx(fb);
  }
  if (a.dbg) atomicAdd(&a.dbg[6], 1ull);  // group-k tiles issued
}

}  // namespace pc
}  // namespace qaa
