// plan.hpp -- host-side pass planner for the fused Trotter passes (SURVEY §8
// A6/A7, K4/H2). Pure C++ (no CUDA); shared by the library and the host-only
// qaa_plan_describe() entry point that the CPU tests call.
//
// Geometry: the local state of 2^L amplitudes is processed in
// tiles of 2^TILE_BITS amplitudes. A tile is the set of indices obtained by
// fixing every physical bit outside a group's 12 "tile bits". Every tile keeps
// the low `row_bits` physical bits (contiguous runs of 2^c amplitudes, i.e.
// 128/256/512-byte rows) so HBM accesses stay coalesced; the remaining tile
// bits are the qubits that group rotates. Group 0 tiles are the contiguous
// bits 0..11 and rotate all twelve; each later group rotates a chunk of the
// higher bits (padded with unrotated low bits when the chunk is short).
//
// Step spanning: the X layer of one step is a product of
// commuting single-qubit factors, so a step only needs every group once
// between D_k and D_{k+1}. Cycling the groups and placing D_{k+1} inside the
// pass that finishes step k (X_k^g, D_{k+1}, X_{k+1}^g on the same tile)
// gives P-1 HBM passes per step for P groups instead of P.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace qaa {

constexpr int TILE_BITS = 12;
constexpr int TILE = 1 << TILE_BITS;
constexpr int NTHREADS = 256;  // 8 warps x 32 lanes, 16 amplitudes per thread
constexpr int RPT = 16;        // register amplitudes per thread
constexpr int MAX_OPS = 32;
constexpr int MAX_SEGS = 8;

// Register patterns: which tile-local bits live in the 4 register bits, the 5
// lane bits and the 3 warp bits of a thread's 16 amplitudes.
//   PA: regs {8,9,10,11} lanes {0,1,2,3,4} warps {5,6,7}   (load pattern)
//   PB: regs {4,5,6,7}   lanes {0,1,2,3,8} warps {9,10,11}
//   PC: regs {0,1,2,3}   lanes {4,5,6,7,8} warps {9,10,11}
// PA and PB keep local bits 0..2 in the lanes, so they are store-coalesced.
enum Pattern : int { PA = 0, PB = 1, PC = 2, NPAT = 3 };

int pattern_reg_local(int pat, int i);   // local bit of register bit i (0..3)
int pattern_lane_local(int pat, int i);  // local bit of lane bit i (0..4)
int pattern_warp_local(int pat, int i);  // local bit of warp bit i (0..2)
bool pattern_storable(int pat);

enum OpKind : uint8_t { OP_ROT_REG = 1, OP_ROT_LANE = 2, OP_XCHG = 3, OP_DIAG = 4 };

struct Op {
  uint8_t kind;
  uint8_t arg;   // register bit (0..3), lane bit (0..4) or target pattern
  uint8_t slot;  // coefficient slot: 0 = pre step, 1 = post step
  uint8_t pad;
};

struct Program {
  Op ops[MAX_OPS];
  int nops = 0;
  int e_pattern = -1;   // pattern in which D is applied (-1: no D)
  int final_pattern = PA;
  int n_exch = 0, n_shfl = 0;
};

struct Group {
  int phys[TILE_BITS];      // tile-local bit -> physical bit
  uint32_t rot_local = 0;   // tile-local bits this group rotates
  uint64_t rot_phys = 0;    // physical qubits this group rotates
  int nseg = 0;             // tile id bits -> physical bits, as runs
  int seg_src[MAX_SEGS], seg_dst[MAX_SEGS], seg_len[MAX_SEGS];
  int64_t ntiles = 0;
};

struct Geometry {
  int L = 0;          // local qubits
  int row_bits = 3;
  std::vector<Group> groups;
};

// One HBM pass: on `group`, rotate for step pre_step (if >= 0), then apply
// D_{d_step} (if >= 0), then rotate for step post_step (if >= 0).
struct PassPlan {
  int group;
  int64_t pre_step, d_step, post_step;
};

// Builds the groups for L >= TILE_BITS + 1 local qubits. Returns false with a
// message if row_bits is unsupported.
bool build_geometry(int L, int row_bits, Geometry* g, std::string* err);

// Pass schedule for K steps (step_spanning: see header comment).
// step_spanning: 0 = one D per step in the first (group-0) pass, P passes per
// step; 1 = cyclic spanning, P-1 passes per step, D visits every group;
// 2 = spanning with D only on groups >= 1 (group 0 always a plain pass; falls
// back to 1 when P < 3).
void build_pass_schedule(int ngroups, int64_t K, int step_spanning, std::vector<PassPlan>* out);

// ---------------------------------------------------------------- sharded plan
// World W = 2^g ranks hold the state on its top g qubits.
// Layout A: rank r = logical bits [L, n); local bit p = logical p.
// Layout B: rank r = logical bits [L-g, L); local bits [L-g, L) hold logical
// [L, n) (the previous rank field). Going A <-> B is one all-to-all of
// contiguous chunks (the bit swap), done by the last pass of every phase
// storing its tiles straight into the peers' next buffers.
// Step k runs as one phase in layout k % 2:
//   [top group: rotate the g carried bits for step k-1, D_k, rotate all of
//    its bits for step k], then groups 1..P-3, 0 and P-2 rotate for step k,
//    the last (P-2) storing remotely (layout flips).
// After the last phase the carried bits get their step K-1 rotation and, if
// the state is in layout B, a plain remap returns it to layout A.
enum ShardKind : int { SK_PASS = 0, SK_REMAP = 1 };
struct ShardPass {
  int kind;
  int group;
  int64_t pre_step;
  uint32_t pre_local;   // tile-local bits rotated for pre_step
  int64_t d_step;
  int64_t post_step;
  uint32_t post_local;  // tile-local bits rotated for post_step
  int remote;           // tiles go to the peers' next buffers (A <-> B)
  int layout;           // layout of the state this pass reads (0 = A, 1 = B)
};
bool build_shard_schedule(const Geometry& geo, int gbits, int64_t K, std::vector<ShardPass>* out, std::string* err);

// Register-pattern program for one pass: rotate pre_local (slot 0), apply D
// (if has_d), rotate post_local (slot 1); minimises exchanges + shuffles.
bool build_program(uint32_t pre_local, bool has_d, uint32_t post_local, Program* prog);

}  // namespace qaa
