// pass_tmem.cu -- the L2-blocked Trotter step with tensor-memory exchanges
// (DESIGN.md §4 "Tensor-memory exchanges").
//
// Same work sequence, slots and chunk dependencies as pass_tma.cu's
// qaa_superpass: per chunk, the group-0 tiles (rotate step j) then the group-k
// tiles (rotate step j, D_{j+1}, rotate step j+1). What changes is how a tile's
// register patterns are changed. qaa_superpass moves every pattern change
// through shared memory (2 transposes per group-0 tile, 2 + a register/lane
// shuffle swap per group-k tile): ~2 LSU wavefronts per amplitude and step,
// the unit that bounds it. Here most changes go through TENSOR MEMORY
// (tcgen05.st / tcgen05.ld, a separate datapath: measured 173 B/clk/SM
// write, 140-157 B/clk/SM read, a round trip 2.3x the rate of an smem
// exchange; tools/microbench/tmem.cu):
//
//   T1  (one warp)   st 32x32b + ld 16x256b: register bits 0,1 <-> lane bits 3,4
//                    (lanes 0..2 shift up to 2..4);
//   T1^-1            st 16x256b + ld 32x32b.
//
// Both are warp-local: no barrier, each warp only touches its own 64 TMEM
// columns. A warp can only reach its own 32 TMEM lanes (warp id mod 4), so the
// tile bits held in warp bits never move through TMEM: each tile takes ONE
// shared-memory exchange for them (which also gives the store its coalesced
// 128-byte rows). Per amplitude and step: 9 LSU units of 16 B (qaa_superpass:
// 14) and 6 TMEM round trips. Patterns (tile-local bits of register bits
// r0..r3 | lane bits l0..l4 | warp bit 2 | quadrant warp bits):
//
//   group 0 (12 bits rotated once):
//     G1 r(8,9,10,11) l(0,1,2,3,4) w5 q(6,7)   landed (contiguous 64 KiB)
//     --smem-->  G2 r(0,5,6,7) l(8,3,4,1,2) w9 q(10,11)
//     --T1-->    G3 r(1,2,6,7) l(0,5,8,3,4)
//     --T1-->    G4 r(3,4,6,7) l(1,2,0,5,8)   store
//   group k (row bits 0..2 sit in the warp bits and are never rotated; 3..11
//   are rotated before and after D):
//     K1 r(6,7,8,9) l(3,4,5,10,11) w0 q(1,2)   landed (128B-swizzled tensor map)
//     --T1-->    K2 r(10,11,8,9) l(6,7,3,4,5)
//     --T1-->    K3 r(4,5,8,9) l(10,11,6,7,3)
//     --T1-->    K4 r(7,3,8,9) l(4,5,10,11,6)   D here (packed energy slice)
//     --T1^-1--> K3, --smem--> K5 r(6,10,11,7) l(0,1,2,3,4) w5 q(8,9)   store
//   (without D: K1 -> K2 -> K3 -> K4 --smem--> K5)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "pass_common.cuh"

namespace qaa {
namespace {
using namespace pc;

// ------------------------------------------------------------------ patterns
struct PatDef {
  int r[4];
  int l[5];
  int w2;
  int q[2];
};
constexpr PatDef t1(const PatDef& p) {
  return PatDef{{p.l[3], p.l[4], p.r[2], p.r[3]}, {p.r[0], p.r[1], p.l[0], p.l[1], p.l[2]}, p.w2, {p.q[0], p.q[1]}};
}
constexpr bool same(const PatDef& a, const PatDef& b) {
  for (int i = 0; i < 4; i++)
    if (a.r[i] != b.r[i]) return false;
  for (int i = 0; i < 5; i++)
    if (a.l[i] != b.l[i]) return false;
  return a.w2 == b.w2 && a.q[0] == b.q[0] && a.q[1] == b.q[1];
}
constexpr bool complete(const PatDef& p) {  // a bijection of the 12 tile bits
  unsigned m = 0;
  for (int i = 0; i < 4; i++) m |= 1u << p.r[i];
  for (int i = 0; i < 5; i++) m |= 1u << p.l[i];
  m |= 1u << p.w2;
  m |= 1u << p.q[0];
  m |= 1u << p.q[1];
  return m == 0xFFFu;
}
constexpr PatDef G1{{8, 9, 10, 11}, {0, 1, 2, 3, 4}, 5, {6, 7}};
constexpr PatDef G2{{0, 5, 6, 7}, {8, 3, 4, 1, 2}, 9, {10, 11}};
constexpr PatDef G3 = t1(G2);
constexpr PatDef G4 = t1(G3);
constexpr PatDef K1{{6, 7, 8, 9}, {3, 4, 5, 10, 11}, 0, {1, 2}};
constexpr PatDef K2 = t1(K1);
constexpr PatDef K3 = t1(K2);
constexpr PatDef K4 = t1(K3);
constexpr PatDef K5{{6, 10, 11, 7}, {0, 1, 2, 3, 4}, 5, {8, 9}};
static_assert(complete(G1) && complete(G2) && complete(G3) && complete(G4), "group-0 patterns");
static_assert(complete(K1) && complete(K2) && complete(K3) && complete(K4) && complete(K5), "group-k patterns");
static_assert(same(G3, PatDef{{1, 2, 6, 7}, {0, 5, 8, 3, 4}, 9, {10, 11}}), "G3");
static_assert(same(G4, PatDef{{3, 4, 6, 7}, {1, 2, 0, 5, 8}, 9, {10, 11}}), "G4");
static_assert(same(K2, PatDef{{10, 11, 8, 9}, {6, 7, 3, 4, 5}, 0, {1, 2}}), "K2");
static_assert(same(K3, PatDef{{4, 5, 8, 9}, {10, 11, 6, 7, 3}, 0, {1, 2}}), "K3");
static_assert(same(K4, PatDef{{7, 3, 8, 9}, {4, 5, 10, 11, 6}, 0, {1, 2}}), "K4");
// every tile bit rotated exactly once: group 0 G1 {8..11} + G2 {0,5,6,7} + G3 new
// {1,2} + G4 new {3,4}; group k pre K1 {6,7,8,9} + K2 new {10,11} + K3 new {4,5} +
// K4 new {3}, post K4 {7,3,8,9} + K3 new {4,5} + K5 new {6,10,11}

enum : int { PG1, PG2, PG3, PG4, PK1, PK2, PK3, PK4, PK5 };
__device__ __forceinline__ constexpr PatDef pat(int id) {
  return id == PG1 ? G1 : id == PG2 ? G2 : id == PG3 ? G3 : id == PG4 ? G4 : id == PK1 ? K1 : id == PK2 ? K2 : id == PK3 ? K3 : id == PK4 ? K4 : K5;
}
// tile-local index of the thread's register-0 amplitude; lw = warp in the group
template <int ID>
__device__ __forceinline__ int tl_of(int lane, int lw) {
  constexpr PatDef p = pat(ID);
  int t = 0;
#pragma unroll
  for (int i = 0; i < 5; i++) t |= ((lane >> i) & 1) << p.l[i];
  t |= (lw & 1) << p.q[0];
  t |= ((lw >> 1) & 1) << p.q[1];
  t |= ((lw >> 2) & 1) << p.w2;
  return t;
}
template <int ID>
__device__ __forceinline__ constexpr int roff_l(int r) {
  constexpr PatDef p = pat(ID);
  return ((r & 1) << p.r[0]) | (((r >> 1) & 1) << p.r[1]) | (((r >> 2) & 1) << p.r[2]) | (((r >> 3) & 1) << p.r[3]);
}
// rotate register bit I of pattern ID with that tile bit's coefficient
template <int ID, int I>
__device__ __forceinline__ void rot(double2 (&v)[RPT], const double (&t)[TILE_BITS]) {
  constexpr PatDef p = pat(ID);
  rot_regbit<I>(v, t[p.r[I]]);
}
template <int ID, class A>
__device__ __forceinline__ Off pat_off(const A& a, int lane, int lw) {
  constexpr PatDef p = pat(ID);
  const int rb[4] = {p.r[0], p.r[1], p.r[2], p.r[3]};
  return make_off_tl(a, tl_of<ID>(lane, lw), rb);
}

// ------------------------------------------------------------------ shared-memory layouts
// landed group-k tile (128-byte-swizzled tensor map): 16-byte chunk c of row r at r*8 + (c ^ (r & 7))
__device__ __forceinline__ int swz128(int l) { return l ^ ((l >> 3) & 7); }
// exchange layouts: XOR the three low bits with the reader's quarter-warp lane
// bits so both the writing and the reading pattern touch 8 distinct 16-byte
// bank groups per quarter warp (conflict-free 128-bit accesses)
template <int B0, int B1, int B2>
__device__ __forceinline__ int xswz(int l) {
  return l ^ (((l >> B0) & 1) | (((l >> B1) & 1) << 1) | (((l >> B2) & 1) << 2));
}
// G1 -> G2: writer quarter lanes = bits 0,1,2; reader = 8,3,4
__device__ __forceinline__ int sw_g12(int l) { return xswz<8, 3, 4>(l); }
// K3 -> K5: writer = 10,11,6; reader = 0,1,2
__device__ __forceinline__ int sw_k35(int l) { return xswz<10, 11, 6>(l); }
// K4 -> K5: writer = 4,5,10; reader = 0,1,2
__device__ __forceinline__ int sw_k45(int l) { return xswz<4, 5, 10>(l); }

template <int ID, int SW>
__device__ __forceinline__ int lay(int l) {
  return SW == 0 ? l : SW == 1 ? swz128(l) : SW == 2 ? sw_g12(l) : SW == 3 ? sw_k35(l) : sw_k45(l);
}
template <int ID, int SW>
__device__ __forceinline__ void lds_pat(double2 (&v)[RPT], const double2* xb, int lane, int lw) {
  const int tl = tl_of<ID>(lane, lw);
#pragma unroll
  for (int r = 0; r < RPT; r++) v[r] = xb[lay<ID, SW>(tl | roff_l<ID>(r))];
}
template <int ID, int SW>
__device__ __forceinline__ void sts_pat(const double2 (&v)[RPT], double2* xb, int lane, int lw) {
  const int tl = tl_of<ID>(lane, lw);
#pragma unroll
  for (int r = 0; r < RPT; r++) xb[lay<ID, SW>(tl | roff_l<ID>(r))] = v[r];
}
// in-place exchange in the landed slot. Write-after-read: every warp of the
// group arrived on `consumed` right after its landed read (long done for a
// group-k tile), so this wait rarely blocks -- unlike a group barrier it does not
// wait for the slowest warp's progress. Then STS, the read-after-write group
// barrier, LDS.
template <int FROM, int TO, int SW>
__device__ __forceinline__ void smem_xchg(double2 (&v)[RPT], double2* xb, int lane, int lw, int g, uint64_t* consumed,
                                          uint32_t parity) {
  mbar_wait_sleep(consumed, parity);
  sts_pat<FROM, SW>(v, xb, lane, lw);
  group_bar(g);
  lds_pat<TO, SW>(v, xb, lane, lw);
}

// ------------------------------------------------------------------ tensor memory
__device__ __forceinline__ uint32_t lo32(double d) { return (uint32_t)__double2loint(d); }
__device__ __forceinline__ uint32_t hi32(double d) { return (uint32_t)__double2hiint(d); }
__device__ __forceinline__ double mkd(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }

// four 32x32b.x16 stores: block B (amplitudes 4B..4B+3) to columns col + 16 B:
// [re(4B+m) lo,hi for m = 0..3 | im(4B+m) lo,hi], then wait for completion
__device__ __forceinline__ void tm_st_32x32(uint32_t col, const double2 (&v)[RPT]) {
#define QAA_BLK(B)                                                                                                    \
  "r"(lo32(v[4 * B].x)), "r"(hi32(v[4 * B].x)), "r"(lo32(v[4 * B + 1].x)), "r"(hi32(v[4 * B + 1].x)), "r"(lo32(v[4 * B + 2].x)),              \
      "r"(hi32(v[4 * B + 2].x)), "r"(lo32(v[4 * B + 3].x)), "r"(hi32(v[4 * B + 3].x)), "r"(lo32(v[4 * B].y)), "r"(hi32(v[4 * B].y)),          \
      "r"(lo32(v[4 * B + 1].y)), "r"(hi32(v[4 * B + 1].y)), "r"(lo32(v[4 * B + 2].y)), "r"(hi32(v[4 * B + 2].y)), "r"(lo32(v[4 * B + 3].y)), \
      "r"(hi32(v[4 * B + 3].y))
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19};\n"
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%1], {%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35};\n"
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%2], {%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51};\n"
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%3], {%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64,%65,%66,%67};\n"
      "tcgen05.wait::st.sync.aligned;\n" ::"r"(col),
      "r"(col + 16), "r"(col + 32), "r"(col + 48), QAA_BLK(0), QAA_BLK(1), QAA_BLK(2), QAA_BLK(3)
      : "memory");
#undef QAA_BLK
}
// four 32x32b.x16 loads (the inverse of tm_st_32x32), waited on before the
// registers are used
__device__ __forceinline__ void tm_ld_32x32(uint32_t col, double2 (&v)[RPT]) {
  uint32_t x[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%64];\n"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%65];\n"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47}, [%66];\n"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%67];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]), "=r"(x[8]),
        "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15]), "=r"(x[16]),
        "=r"(x[17]), "=r"(x[18]), "=r"(x[19]), "=r"(x[20]), "=r"(x[21]), "=r"(x[22]), "=r"(x[23]), "=r"(x[24]),
        "=r"(x[25]), "=r"(x[26]), "=r"(x[27]), "=r"(x[28]), "=r"(x[29]), "=r"(x[30]), "=r"(x[31]), "=r"(x[32]),
        "=r"(x[33]), "=r"(x[34]), "=r"(x[35]), "=r"(x[36]), "=r"(x[37]), "=r"(x[38]), "=r"(x[39]), "=r"(x[40]),
        "=r"(x[41]), "=r"(x[42]), "=r"(x[43]), "=r"(x[44]), "=r"(x[45]), "=r"(x[46]), "=r"(x[47]), "=r"(x[48]),
        "=r"(x[49]), "=r"(x[50]), "=r"(x[51]), "=r"(x[52]), "=r"(x[53]), "=r"(x[54]), "=r"(x[55]), "=r"(x[56]),
        "=r"(x[57]), "=r"(x[58]), "=r"(x[59]), "=r"(x[60]), "=r"(x[61]), "=r"(x[62]), "=r"(x[63])
      : "r"(col), "r"(col + 16), "r"(col + 32), "r"(col + 48)
      : "memory");
#pragma unroll
  for (int B = 0; B < 4; B++)
#pragma unroll
    for (int m = 0; m < 4; m++)
      v[4 * B + m] = make_double2(mkd(x[16 * B + 2 * m], x[16 * B + 2 * m + 1]),
                                  mkd(x[16 * B + 8 + 2 * m], x[16 * B + 8 + 2 * m + 1]));
}
// four 16x256b.x4 loads at addresses a0..a3 (lane base and column of each),
// giving reader amplitudes q = 0..3: per load, (a, B0') -> v[J(q, a, B0')]
// with re at regs 8 B0' + 2a (+1), im at 8 B0' + 4 + 2a (+1)
template <int J0, int J1, int J2, int J3>
__device__ __forceinline__ void tm_ld_16x256(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                             double2 (&v)[RPT]) {
  uint32_t x[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%64];\n"
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%65];\n"
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47}, [%66];\n"
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%67];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]), "=r"(x[8]),
        "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15]), "=r"(x[16]),
        "=r"(x[17]), "=r"(x[18]), "=r"(x[19]), "=r"(x[20]), "=r"(x[21]), "=r"(x[22]), "=r"(x[23]), "=r"(x[24]),
        "=r"(x[25]), "=r"(x[26]), "=r"(x[27]), "=r"(x[28]), "=r"(x[29]), "=r"(x[30]), "=r"(x[31]), "=r"(x[32]),
        "=r"(x[33]), "=r"(x[34]), "=r"(x[35]), "=r"(x[36]), "=r"(x[37]), "=r"(x[38]), "=r"(x[39]), "=r"(x[40]),
        "=r"(x[41]), "=r"(x[42]), "=r"(x[43]), "=r"(x[44]), "=r"(x[45]), "=r"(x[46]), "=r"(x[47]), "=r"(x[48]),
        "=r"(x[49]), "=r"(x[50]), "=r"(x[51]), "=r"(x[52]), "=r"(x[53]), "=r"(x[54]), "=r"(x[55]), "=r"(x[56]),
        "=r"(x[57]), "=r"(x[58]), "=r"(x[59]), "=r"(x[60]), "=r"(x[61]), "=r"(x[62]), "=r"(x[63])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3)
      : "memory");
  constexpr int J[4] = {J0, J1, J2, J3};
#pragma unroll
  for (int q = 0; q < 4; q++)
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
      for (int b0 = 0; b0 < 2; b0++) {
        const int j = J[q] | a | (b0 << 2);
        const uint32_t* y = x + 16 * q;
        v[j] = make_double2(mkd(y[8 * b0 + 2 * a], y[8 * b0 + 2 * a + 1]), mkd(y[8 * b0 + 4 + 2 * a], y[8 * b0 + 5 + 2 * a]));
      }
}
// the inverse: four 16x256b.x4 stores of v[J(q, a, B0')] to a0..a3, then wait
template <int J0, int J1, int J2, int J3>
__device__ __forceinline__ void tm_st_16x256(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                             const double2 (&v)[RPT]) {
#define QAA_Q(JQ)                                                                                                   \
  "r"(lo32(v[JQ | 0].x)), "r"(hi32(v[JQ | 0].x)), "r"(lo32(v[JQ | 1].x)), "r"(hi32(v[JQ | 1].x)), "r"(lo32(v[JQ | 0].y)), "r"(hi32(v[JQ | 0].y)), \
      "r"(lo32(v[JQ | 1].y)), "r"(hi32(v[JQ | 1].y)), "r"(lo32(v[JQ | 4].x)), "r"(hi32(v[JQ | 4].x)), "r"(lo32(v[JQ | 5].x)),                \
      "r"(hi32(v[JQ | 5].x)), "r"(lo32(v[JQ | 4].y)), "r"(hi32(v[JQ | 4].y)), "r"(lo32(v[JQ | 5].y)), "r"(hi32(v[JQ | 5].y))
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19};\n"
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%1], {%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35};\n"
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%2], {%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51};\n"
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%3], {%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64,%65,%66,%67};\n"
      "tcgen05.wait::st.sync.aligned;\n" ::"r"(a0),
      "r"(a1), "r"(a2), "r"(a3), QAA_Q(J0), QAA_Q(J1), QAA_Q(J2), QAA_Q(J3)
      : "memory");
#undef QAA_Q
}
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// TMEM address of (lane, column): lane in bits 31..16
__device__ __forceinline__ uint32_t tma_(uint32_t base, int lane, int col) {
  return base + ((uint32_t)lane << 16) + (uint32_t)col;
}
// Per consumer group g: columns [128 g, 128 g + 128); each warp of a quadrant
// pair owns 64 of them (its 16 amplitudes as four 16-column blocks). Only the
// warp itself touches them, in program order (each ld is waited on before the
// next st), so one buffer per warp suffices.
//
// T1: reader register j' = a | h << 1 | B0' << 2 | p << 3 (a: lane + 8, h: lane + 16,
// p: block pair)
__device__ __forceinline__ void tm_t1(double2 (&v)[RPT], uint32_t tb, int g, int lw) {
  const int q = 32 * (lw & 3);
  const int c = 128 * g + 64 * (lw >> 2);
  tm_st_32x32(tma_(tb, q, c), v);
  // (p, h) = (0,0), (0,1), (1,0), (1,1) -> J = h << 1 | p << 3
  tm_ld_16x256<0, 2, 8, 10>(tma_(tb, q, c), tma_(tb, q + 16, c), tma_(tb, q, c + 32), tma_(tb, q + 16, c + 32), v);
}
// T1^-1: the T1 reader layout back to the writer's
__device__ __forceinline__ void tm_t1_inv(double2 (&v)[RPT], uint32_t tb, int g, int lw) {
  const int q = 32 * (lw & 3);
  const int c = 128 * g + 64 * (lw >> 2);
  tm_st_16x256<0, 2, 8, 10>(tma_(tb, q, c), tma_(tb, q + 16, c), tma_(tb, q, c + 32), tma_(tb, q + 16, c + 32), v);
  tm_ld_32x32(tma_(tb, q, c), v);
}

// D in pattern K4 from the packed energy slice: thread t = lane + 32 lw holds
// its 16 energies (register order) at bytes 16 t .. 16 t + 15
__device__ __forceinline__ void diag_packed(double2 (&v)[RPT], const uint8_t* es, const double2* phis, int lane,
                                            int lw) {
  const uint4 pk = reinterpret_cast<const uint4*>(es)[lane + 32 * lw];
#pragma unroll
  for (int r = 0; r < RPT; r++) {
    const uint32_t w = r < 4 ? pk.x : (r < 8 ? pk.y : (r < 12 ? pk.z : pk.w));
    const int e = (int)((w >> (8 * (r & 3))) & 0xffu);
    // Phi stored 8x interleaved: the 8 lanes of a quarter warp read 8 distinct bank groups
    v[r] = cmul(phis[e * PHI_COPIES + (lane & (PHI_COPIES - 1))], v[r]);
  }
}

// ------------------------------------------------------------------ per-tile programs
// group 0: rotate all 12 tile bits with t[0]; leaves v in G4
template <class F, class P>
__device__ __forceinline__ void prog_g0(double2 (&v)[RPT], const double (&t)[TILE_BITS], double2* xb, uint32_t tb,
                                        int lane, int lw, int g, uint64_t* consumed, uint32_t parity, int flags,
                                        F&& release, P&& publish) {
  lds_pat<PG1, 0>(v, xb, lane, lw);
  __syncwarp();
  if (lane == 0) mbar_arrive_notx(consumed);
  rot<PG1, 0>(v, t);
  rot<PG1, 1>(v, t);
  rot<PG1, 2>(v, t);
  rot<PG1, 3>(v, t);
  publish();  // the previous group-0 tile's stores have drained meanwhile
  smem_xchg<PG1, PG2, 2>(v, xb, lane, lw, g, consumed, parity);
  // the slot is consumed: the last warp out refills it while the TMEM steps run
  if (!(flags & 1)) release();
  rot<PG2, 0>(v, t);
  rot<PG2, 1>(v, t);
  rot<PG2, 2>(v, t);
  rot<PG2, 3>(v, t);
  tm_t1(v, tb, g, lw);
  rot<PG3, 0>(v, t);
  rot<PG3, 1>(v, t);
  tm_t1(v, tb, g, lw);
  rot<PG4, 0>(v, t);
  rot<PG4, 1>(v, t);
  if (flags & 1) release();
}
// group k: BD = rotate t0, D, rotate t1 (K1 ... K5); else rotate t0 (K1 ... K4 -> K5)
template <bool BD, class F, class P>
__device__ __forceinline__ void prog_gk(double2 (&v)[RPT], const double (&t0)[TILE_BITS],
                                        const double (&t1)[TILE_BITS], double2* xb, const uint8_t* es,
                                        const double2* phis, uint32_t tb, int lane, int lw, int g, uint64_t* consumed,
                                        uint32_t parity, F&& release, P&& publish) {
  lds_pat<PK1, 1>(v, xb, lane, lw);
  __syncwarp();
  if (lane == 0) mbar_arrive_notx(consumed);
  rot<PK1, 0>(v, t0);
  rot<PK1, 1>(v, t0);
  rot<PK1, 2>(v, t0);
  rot<PK1, 3>(v, t0);
  publish();
  tm_t1(v, tb, g, lw);
  rot<PK2, 0>(v, t0);
  rot<PK2, 1>(v, t0);
  tm_t1(v, tb, g, lw);
  rot<PK3, 0>(v, t0);
  rot<PK3, 1>(v, t0);
  tm_t1(v, tb, g, lw);
  rot<PK4, 1>(v, t0);
  if (BD) {
    diag_packed(v, es, phis, lane, lw);
    rot<PK4, 0>(v, t1);
    rot<PK4, 1>(v, t1);
    rot<PK4, 2>(v, t1);
    rot<PK4, 3>(v, t1);
    tm_t1_inv(v, tb, g, lw);
    rot<PK3, 0>(v, t1);
    rot<PK3, 1>(v, t1);
    smem_xchg<PK3, PK5, 3>(v, xb, lane, lw, g, consumed, parity);
  } else {
    smem_xchg<PK4, PK5, 4>(v, xb, lane, lw, g, consumed, parity);
  }
  release();
  if (BD) {
    rot<PK5, 0>(v, t1);
    rot<PK5, 1>(v, t1);
    rot<PK5, 2>(v, t1);
  }
}


// ------------------------------------------------------------------ work items with early late loads
// A group-k tile whose chunk is not complete when its slot is refilled is
// DEFERRED: its energy slice is fetched right away (on the slot's full barrier),
// the state tile later. Any thread that frees a slot retries the deferred
// slots and, once done[c] is complete, claims one (CAS DEFERRED -> ISSUING) and
// starts its state load on the slot's own late barrier -- the load latency then
// overlaps the owning group's current tile instead of being waited out.
__device__ __forceinline__ int ld_kind(const SlotMeta* m) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(sa(&m->kind)) : "memory");
  return v;
}
__device__ __forceinline__ void st_kind(SlotMeta* m, int k) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(sa(&m->kind)), "r"(k) : "memory");
}
__device__ __forceinline__ unsigned done_target(const SuperArgs& a) { return 1u << (a.tpc_bits + 3); }

// the state part of a group-k tile (its energy slice was fetched at issue time)
__device__ __forceinline__ void load_gk_state(const CUtensorMap* kmap, const SuperArgs& a, uint32_t T, double2* dst,
                                              uint64_t* bar, uint64_t pol) {
  mbar_expect_tx(bar, TILE * 16u);
  int cc[5];
#pragma unroll
  for (int d = 0; d < 5; d++) {
    const int sg = a.gk.dim_seg[d];
    cc[d] = sg < 0 ? 0 : (int)((T >> a.gk.seg_src[sg]) & ((1u << a.gk.seg_len[sg]) - 1));
  }
  tma_load_hint(dst, kmap, cc, a.gk.ndims, bar, pol);
}
// issuer of a claimed slot (kind == ISSUING, chunk complete): record the late
// phase parity, start the state load, publish LATE
__device__ __forceinline__ void issue_late(const CUtensorMap* kmap, const SuperArgs& a, int s, double2* slots,
                                           SlotMeta* meta, uint64_t* late, unsigned* late_cnt, uint64_t pol) {
  meta[s].pad = (int)(late_cnt[s]++ & 1u);
  fence_async_global();  // generic-proxy stores of the chunk -> this async-proxy read
  load_gk_state(kmap, a, meta[s].T, slots + (size_t)s * FAST_XBUF, &late[s], pol);
  st_kind(&meta[s], SK_B_LATE);
}
// non-blocking: start the late loads of deferred slots whose chunk is complete
__device__ __forceinline__ void retry_deferred(const CUtensorMap* kmap, const SuperArgs& a, double2* slots,
                                               SlotMeta* meta, uint64_t* late, unsigned* late_cnt, uint64_t pol) {
#pragma unroll
  for (int s = 0; s < TMA_SLOTS; s++) {
    if (ld_kind(&meta[s]) != SK_B_DEFERRED) continue;
    if (ld_acquire(&a.done[meta[s].c]) < done_target(a)) continue;
    if (atomicCAS(&meta[s].kind, SK_B_DEFERRED, SK_B_ISSUING) != SK_B_DEFERRED) continue;
    issue_late(kmap, a, s, slots, meta, late, late_cnt, pol);
  }
}
template <int NG, bool BD>
__device__ void super_issue_tm(const CUtensorMap* kmap, const SuperArgs& a, int64_t J, double2* slots,
                               uint8_t* eslots, uint64_t* full, SlotMeta* meta, uint64_t pol_dead) {
  const int s = (int)(J % TMA_SLOTS);
  uint64_t* fb = &full[NG * s + (int)(J % NG)];
  int kind;
  int64_t c;
  uint32_t i;
  const unsigned long long qpos =
      a.queue ? atomicAdd(a.queue, 1ull) : (unsigned long long)blockIdx.x + (unsigned long long)J * gridDim.x;
  if (!decode_item(a, qpos, &kind, &c, &i)) {
    st_kind(&meta[s], SK_END);
    mbar_arrive_notx(fb);
    return;
  }
  if (kind == SK_A) {
    const uint32_t T = pdep32(i, a.z_imask) | pdep32((uint32_t)c, a.z_cmask);
    meta[s].c = (int)c;
    meta[s].T = T;
    st_kind(&meta[s], SK_A);
    mbar_expect_tx(fb, TILE * 16u);
    bulk_g2s_hint(slots + (size_t)s * FAST_XBUF, a.g0.psi + tbase(a.g0, T), TILE * 16u, fb, pol_dead);
    return;
  }
  const uint32_t T = pdep32(i, a.k_imask) | pdep32((uint32_t)c, a.k_cmask);
  meta[s].c = (int)c;
  meta[s].T = T;
  if (ld_acquire(&a.done[c]) >= done_target(a)) {
    fence_async_global();
    st_kind(&meta[s], SK_B);
    load_gk<BD>(kmap, a, T, slots + (size_t)s * FAST_XBUF, eslots + (size_t)s * TILE, fb, pol_dead);
  } else {
    st_kind(&meta[s], SK_B_DEFERRED);
    if (BD) {  // the energy slice does not depend on the chunk: fetch it now
      mbar_expect_tx(fb, TILE);
      bulk_g2s_hint(eslots + (size_t)s * TILE, a.gk.Eg + (int64_t)T * TILE, TILE, fb, pol_dead);
    } else {
      mbar_arrive_notx(fb);
    }
  }
}

// ------------------------------------------------------------------ the kernel
template <int NG, bool BD>
__global__ void __launch_bounds__(NG * NTHREADS, 1) qaa_superpass_tm(const __grid_constant__ CUtensorMap kmap,
                                                                    const SuperArgs a) {
  extern __shared__ __align__(1024) unsigned char sm[];
  double2* slots = reinterpret_cast<double2*>(sm);
  uint8_t* eslots = sm + TMA_SLOTS * SLOT_BYTES;
  double2* phis = reinterpret_cast<double2*>(eslots + TMA_SLOTS * TILE);
  uint64_t* full = reinterpret_cast<uint64_t*>(phis + TMA_MAX_PHI * PHI_COPIES);
  uint64_t* late = full + NG * TMA_SLOTS;
  SlotMeta* meta = reinterpret_cast<SlotMeta*>(late + NG);
  unsigned* cnt = slot_counters(sm);
  uint64_t* cons = slot_consumed(sm);
  uint64_t* slate = slot_late(sm);
  unsigned* late_cnt = slot_late_count(sm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the swizzled group-k landing needs 1024-byte aligned slots
  if (tid == 0 && (sa(sm) & 1023u)) __trap();
  if (tid < TMA_SLOTS) cnt[tid] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(sa(&cnt[4])) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  const uint64_t pol_dead = a.hints ? policy_evict_first() : policy_evict_normal();
  const uint64_t pol_keep = a.hints == 2 ? policy_evict_last() : policy_evict_normal();
  if (tid == 0) {
    for (int s = 0; s < NG * TMA_SLOTS; s++) mbar_init(&full[s], 1);
    for (int g = 0; g < NG; g++) mbar_init(&late[g], 1);
    for (int s = 0; s < NG * TMA_SLOTS; s++) mbar_init(&cons[s], NTHREADS / 32);
    for (int s = 0; s < TMA_SLOTS; s++) {
      mbar_init(&slate[s], 1);
      late_cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int J = 0; J < TMA_SLOTS; J++) super_issue_tm<NG, BD>(&kmap, a, J, slots, eslots, full, meta, pol_dead);
  }
  if (BD)
    for (int e = tid; e < a.gk.n_phi * PHI_COPIES; e += NG * NTHREADS) phis[e] = a.gk.phi[e / PHI_COPIES];
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tb = cnt[4];
  const int g = warp >> 3, lw = warp & 7, gtid = tid & (NTHREADS - 1);
  double2 v[RPT];
  // Publishing a group-0 tile (done[c] += 1 per warp, with release semantics) is
  // deferred into the next tile's program, after its first rotations: by then the
  // stores have drained and the release fence costs nothing. Before anything
  // that can wait on done[] (a deferred group-k tile, the end) it is flushed.
  int pend_c = -1;
  auto publish = [&]() {
    if (pend_c >= 0) {
      __syncwarp();
      if (lane == 0) red_release_add(&a.done[pend_c], 1u);
      pend_c = -1;
    }
  };
  for (int J = g;; J += NG) {
    const int s = J % TMA_SLOTS;
    const long long t_full0 = (a.tm_flags & 8) ? clock64() : 0;
    if (a.tm_flags & 4)
      mbar_wait_bounded(&full[NG * s + g], (uint32_t)((J / period<NG>()) & 1));
    else
      mbar_wait_sleep(&full[NG * s + g], (uint32_t)((J / period<NG>()) & 1));
    const SlotMeta m = meta[s];
    if ((a.tm_flags & 8) && lane == 0) {
      atomicAdd(&a.dbg[0], (unsigned long long)(clock64() - t_full0));
      atomicAdd(&a.dbg[1], 1ull);
      if (m.kind >= SK_B_DEFERRED) atomicAdd(&a.dbg[2], 1ull);
      if (m.kind == SK_B_LATE) atomicAdd(&a.dbg[7], 1ull);
    }
    if (m.kind == SK_END || m.kind >= SK_B_DEFERRED) publish();
    if (m.kind == SK_END) {
      group_bar(g);
      if (gtid == 0) super_issue_tm<NG, BD>(&kmap, a, J + TMA_SLOTS, slots, eslots, full, meta, pol_dead);
      break;
    }
    double2* xb = slots + (size_t)s * FAST_XBUF;
    uint8_t* es = eslots + (size_t)s * TILE;
    if (m.kind >= SK_B_DEFERRED) {  // deferred, possibly already claimed and issued early
      const long long t_late0 = (a.tm_flags & 8) ? clock64() : 0;
      if (gtid == 0 && atomicCAS(&meta[s].kind, SK_B_DEFERRED, SK_B_ISSUING) == SK_B_DEFERRED) {
        // nobody started it early: wait for the chunk here
        for (uint32_t it = 0; ld_acquire(&a.done[m.c]) < done_target(a); it++) {
          __nanosleep(32);
          if (it > (1u << 26)) __trap();
        }
        if (a.tm_flags & 8) atomicAdd(&a.dbg[6], (unsigned long long)(clock64() - t_late0));
        issue_late(&kmap, a, s, slots, meta, slate, late_cnt, pol_dead);
      }
      for (uint32_t it = 0; ld_kind(&meta[s]) != SK_B_LATE; it++) {
        __nanosleep(32);
        if (it > (1u << 26)) __trap();
      }
      if (a.tm_flags & 4)
        mbar_wait_bounded(&slate[s], (uint32_t)meta[s].pad);
      else
        mbar_wait_sleep(&slate[s], (uint32_t)meta[s].pad);
      if ((a.tm_flags & 8) && lane == 0) atomicAdd(&a.dbg[3], (unsigned long long)(clock64() - t_late0));
    }
    const bool isb = m.kind != SK_A;
    // "last warp out refills" the slot with tile J + 3 once the program has
    // consumed it (after its shared-memory exchange)
    auto release = [&]() {
      __syncwarp();
      if (lane == 0 && last_warp_out(&cnt[s])) {
        super_issue_tm<NG, BD>(&kmap, a, J + TMA_SLOTS, slots, eslots, full, meta, pol_dead);
        if (!(a.tm_flags & 16)) retry_deferred(&kmap, a, slots, meta, slate, late_cnt, pol_dead);
      }
    };
    uint64_t* consumed = &cons[NG * s + g];
    const uint32_t parity = (uint32_t)((J / period<NG>()) & 1);
    const long long t_prog0 = (a.tm_flags & 8) ? clock64() : 0;
    if (isb)
      prog_gk<BD>(v, a.gk.t[0], a.gk.t[1], xb, es, phis, tb, lane, lw, g, consumed, parity, release, publish);
    else
      prog_g0(v, a.g0.t[0], xb, tb, lane, lw, g, consumed, parity, a.tm_flags, release, publish);
    if ((a.tm_flags & 8) && lane == 0) atomicAdd(&a.dbg[isb ? 5 : 4], (unsigned long long)(clock64() - t_prog0));
    if (isb) {
      const Off psk = pat_off<PK5>(a.gk, lane, lw);  // recomputed per tile: frees 10 registers
      const int64_t tbs = tbase(a.gk, m.T);
      if (!BD && a.remote) {
        const int64_t j = tbs >> a.gshift;
        double2* dst = a.peers[j] + (tbs - (j << a.gshift) + ((int64_t)a.rank << a.gshift));
#pragma unroll
        for (int r = 0; r < RPT; r++) dst[roff(psk, r)] = v[r];
      } else {
        double2* dst = a.gk.psi + tbs;
#pragma unroll
        for (int r = 0; r < RPT; r++) st_hint(dst + roff(psk, r), v[r], pol_dead);
      }
    } else {
      const Off ps0 = pat_off<PG4>(a.g0, lane, lw);
      double2* dst = a.g0.psi + tbase(a.g0, m.T);
#pragma unroll
      for (int r = 0; r < RPT; r++) st_hint(dst + roff(ps0, r), v[r], pol_keep);
      // published per warp (done_shift = 3: eight arrivals per tile), no group
      // barrier: a slow warp does not hold the other seven
      pend_c = m.c;
      if (a.tm_flags & 2) publish();
    }
  }
  publish();
  if (!BD && a.remote) __threadfence_system();
  tm_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb) : "memory");
}

typedef void (*TmKernel)(const CUtensorMap, const SuperArgs);
TmKernel pick_tm(int ng, bool bd) {
  if (ng == 1) return bd ? qaa_superpass_tm<1, true> : qaa_superpass_tm<1, false>;
  return bd ? qaa_superpass_tm<2, true> : qaa_superpass_tm<2, false>;
}

}  // namespace

// host: byte position of tile-local index l in the packed energy slice of
// pattern K4 (thread t = lane + 32 lw holds register r at byte 16 t + r)
void superpass_tm_energy_positions(uint16_t* pos) {
  for (int l = 0; l < TILE; l++) {
    int r = 0, lane = 0, lw = 0;
    for (int i = 0; i < 4; i++) r |= ((l >> K4.r[i]) & 1) << i;
    for (int i = 0; i < 5; i++) lane |= ((l >> K4.l[i]) & 1) << i;
    lw = ((l >> K4.q[0]) & 1) | (((l >> K4.q[1]) & 1) << 1) | (((l >> K4.w2) & 1) << 2);
    pos[l] = (uint16_t)(16 * (lane + 32 * lw) + r);
  }
}

cudaError_t superpass_tm_setup() {
  for (int ng = 1; ng <= 2; ng++)
    for (int bd = 0; bd < 2; bd++) {
      cudaError_t e =
          cudaFuncSetAttribute(pick_tm(ng, bd), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TMA_SMEM_BYTES);
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}

// cooperative launch: the chunk dependencies spin across CTAs, so every CTA of
// the grid must be co-resident (the launch fails instead of deadlocking)
cudaError_t launch_superpass_tm(const CUtensorMap* kmap, const SuperArgs& a, int ngroups, bool bd, int grid,
                                cudaStream_t st) {
  TmKernel k = pick_tm(ngroups, bd);
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

}  // namespace qaa
