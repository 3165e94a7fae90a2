// kernels.cuh -- device-side entry points of libqaa (launch wrappers). The
// C-ABI units api_*.cu are the only callers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "plan.hpp"

namespace qaa {

// Arguments of one fused Trotter pass (K4). Passed by value
// (lives in the kernel's constant parameter bank).
struct PassArgs {
  double2* psi;            // local state, canonical/physical layout
  const uint8_t* E;        // energy table, same indexing as psi
  const double2* phi;      // D row: Phi[e] for e = 0..n_phi-1 (nullptr: no D)
  int n_phi;
  int e_pattern;           // register pattern in which D is applied (-1: none)
  int final_pattern;
  int nops;
  double coef[2];          // rotation coefficient per slot (t = tan beta, or cot beta)
  int form[2];             // 0: tangent form (psi0 + i t psi1); 1: cot form (u psi0 + i psi1)
  int64_t ntiles;
  int phys[TILE_BITS];
  int nseg;
  int seg_src[MAX_SEGS], seg_dst[MAX_SEGS], seg_len[MAX_SEGS];
  Op ops[MAX_OPS];
};

constexpr size_t PASS_SMEM_BYTES = sizeof(double2) * TILE + sizeof(double2) * 256;

// Generic (interpreted) pass: any register program, tangent or cot form per
// slot. Used only when a pass needs the cot form (|tan beta| > 1e4) or an
// uncommon program; the specialised kernels below handle the common passes.
cudaError_t launch_pass(const PassArgs& a, int grid, cudaStream_t st);
cudaError_t pass_kernel_setup();  // opt-in shared memory size

// Specialised fused passes (pass_fast.cu): the register program is compiled
// in, rotations are tangent form with a per-tile-bit coefficient (0 = the
// bit is not rotated by this group, an exact identity), shared-memory
// exchanges use the additive padded layout l + (l >> 4).
enum FastProg : int {
  FP_G0_DPOST = 0,       // group 0: D, then rotate all 12 tile bits      (first pass)
  FP_G0_PRE = 1,         // group 0: rotate all 12 tile bits
  FP_G0_PRE_D_POST = 2,  // group 0: rotate (step k), D_{k+1}, rotate (step k+1)
  FP_GK_PRE = 3,         // group k>0: rotate tile bits 3..11
  FP_GK_PRE_D_POST = 4,  // group k>0: rotate, D, rotate
  FP_COUNT = 5
};
struct FastArgs {
  double2* psi;
  const uint8_t* E;
  const double2* phi;
  int n_phi;
  double t[2][TILE_BITS];  // [slot][tile-local bit]: tan beta, or 0 if not rotated
  int64_t ntiles;
  int phys[TILE_BITS];
  int nseg;
  int seg_src[MAX_SEGS], seg_dst[MAX_SEGS], seg_len[MAX_SEGS];
  // sharded remap: when remote != 0 the tile at local index x
  // is stored into peers[j] at (x mod 2^gshift) | (rank << gshift), j = x >> gshift
  int remote;
  int gshift;
  int rank;
  double2* peers[8];
};
// plain remap for the sharded layout swap: every local amplitude x goes to
// peers[x >> gshift] at (x mod 2^gshift) | (rank << gshift)
cudaError_t launch_remap(const double2* src, double2* const* peers, int64_t N, int gshift, int rank, int num_sms,
                         cudaStream_t st);
constexpr int FAST_XBUF = TILE + TILE / 16;  // padded exchange buffer (amplitudes)
constexpr size_t FAST_SMEM_BYTES = sizeof(double2) * (FAST_XBUF + 256 * 8);  // + 8 copies of the D table
cudaError_t pass_fast_setup();

// Persistent evolve (pass_fast.cu qaa_persist) for 13 <= L <= 21: all passes of
// the plan in one cooperative launch, a grid barrier between passes.
struct PersistPass {
  int fp, lane3, group;
  int pre, d, post;  // step indices, -1 = absent
};
struct PersistLaunch {
  double2* psi;
  const uint8_t* E;
  const PersistPass* passes;  // device array
  int npass;
  const double2* phi_all;
  int n_phi;
  const double* coef;
  int ngroups;
  const Group* groups;        // host, copied by value into the launch
  unsigned* bar;              // device [2], zeroed
};
int persist_max_grid(int num_sms);
cudaError_t launch_persist(const PersistLaunch& L, int grid, cudaStream_t st);
cudaError_t launch_pass_fast(const FastArgs& a, int prog, bool lane3, bool prefetch, int grid, cudaStream_t st);

// Warp-specialised TMA pass (pass_tma.cu): same programs as FastArgs, tiles
// streamed into shared memory by a producer warp (bulk copy for contiguous
// tiles, tensor-map copy for strided ones), energies from a per-group
// permuted table Eg (tile T's 4096 bytes contiguous at Eg + 4096 T).
struct TmaArgs {
  double2* psi;
  const uint8_t* Eg;
  const double2* phi;
  int n_phi;
  double t[2][TILE_BITS];
  int64_t ntiles;
  int phys[TILE_BITS];
  int nseg;
  int seg_src[MAX_SEGS], seg_dst[MAX_SEGS], seg_len[MAX_SEGS];
  int contiguous;   // 1: tile is 64 KiB contiguous at psi + tbase(T)
  int ndims;        // tensor-map rank (2..5) otherwise
  int dim_seg[5];   // per dim: -1 = tile dim (coordinate 0), else the tile-id segment giving the coordinate
};
// the TMA kernels keep 8 bank-group copies of the D table in shared memory:
// they need E_max + 1 <= TMA_MAX_PHI (else the host uses the register kernels)
constexpr int TMA_MAX_PHI = 64;
cudaError_t pass_tma_setup();
// L2-blocked Trotter step (pass_tma.cu qaa_superpass): group 0 rotate, then
// group k rotate/D/rotate, over the same L2-resident chunk; see the comment there.
struct SuperArgs {
  TmaArgs gk;          // group k: t[0] = step j, t[1] = step j+1; phi/n_phi = D_{j+1}; Eg = its energy slices
  TmaArgs g0;          // group 0 (contiguous tiles): t[0] = step j
  int64_t nchunks;
  int tpc_bits;        // tiles per chunk per sub-pass = 2^tpc_bits
  uint32_t k_imask, k_cmask;  // group-k tile id = pdep(i, k_imask) | pdep(c, k_cmask)
  uint32_t z_imask, z_cmask;  // group-0 tile id
  int hints;           // L2 eviction hints: 0 none, 1 evict-first for dead data, 2 + evict-last for group-0 output
  // sharded plan (kernel variant without D): group-k tiles go to the peers' next
  // shard buffers, tile at local index x -> peers[x >> gshift] at
  // (x mod 2^gshift) | (rank << gshift) (the layout bit swap)
  int remote;
  int gshift;
  int rank;
  double2* peers[8];
  unsigned* done;      // [nchunks] group-0 tiles stored per chunk (zeroed before launch)
  int lag;             // chunks between A(c) and B(c) in the work sequence (0 = 1)
  // split roles (split_a > 0): CTAs [0, split_a) run only group-0 tiles, the rest
  // only group-k tiles, each in chunk order; B(c) waits for done[c], A(c) for
  // doneB[c - lag - 1] == 2^tpc_bits (all B(c - lag - 1) issued: bounds the L2 live set)
  int split_a;
  unsigned* doneB;     // [nchunks] group-k tiles issued per chunk (zeroed before launch)
  unsigned* qab;       // producer-warp variant: [0] next group-0 tile, [1] next group-k tile (zeroed)
  int done_shift;      // done[c] counts 2^done_shift arrivals per tile (3: one per warp: pass_tmem.cu, v2)
  int v2;              // qaa_superpass: split-phase WAR guards + deferred per-warp publish (default 1)
  int pub_batch;       // v2: group-0 tiles of one chunk a warp publishes with ONE release (default 1)
  int early;           // v2 with D: release a slot before the final 3 register-bit rotations (EARLY)
  int diag;            // QAA_OPT_DIAG: diagnostic kernel variant (work removed; wrong results by design)
  int rev;             // reversed pair: A items = group-k rotate/D/rotate tiles, B items = group-0 tiles
  int tm_flags;        // pass_tmem.cu A/B switches: 1 = group-0 slot released at the tile's end,
                       // 2 = publish right after the stores, 4 = spin (no suspend hint) in waits,
                       // 8 = count waits into dbg (diagnostics), 16 = no early retry of deferred loads
  unsigned long long* dbg;  // [8] diagnostics counters (tm_flags & 8)
  unsigned long long* queue;  // global work counter (zeroed before launch)
};
cudaError_t launch_superpass(const CUtensorMap* kmap, const SuperArgs& a, bool lane3, int ngroups, bool bd, int grid,
                             cudaStream_t st);
// the same step with a producer warp (pass_tma.cu qaa_superpass_pw): two consumer
// groups + one warp that claims tiles dynamically and issues every load
cudaError_t launch_superpass_pw(const CUtensorMap* kmap, const SuperArgs& a, bool lane3, bool bd, int grid,
                                cudaStream_t st);
cudaError_t launch_pass_tma(const CUtensorMap* map, const TmaArgs& a, int prog, bool lane3, int ngroups, int grid,
                            cudaStream_t st);
// gather a group's energy layout: Eg[T*4096 + pack(l)] = E[tbase(T) + off(l)], pack =
// the thread-major order of register pattern PB (16 bytes per thread, one LDS.128)
// pos != nullptr: byte position pos[l] of tile-local index l instead (pass_tmem.cu pattern K3)
cudaError_t launch_permute_energy(const uint8_t* E, uint8_t* Eg, const int (&phys)[TILE_BITS], int nseg,
                                  const int* seg_src, const int* seg_dst, const int* seg_len, int64_t ntiles,
                                  int pb3, int num_sms, cudaStream_t st, const uint16_t* pos = nullptr);
// L2-blocked Trotter step with tensor-memory pattern changes (pass_tmem.cu):
// same SuperArgs; kmap = the group-k map with the 128-byte swizzle, gk.Eg = the
// K3-packed energy slices (bd). Cooperative launch (co-residency guaranteed).
cudaError_t superpass_tm_setup();
void superpass_tm_energy_positions(uint16_t* pos);  // host: TILE entries
cudaError_t launch_superpass_tm(const CUtensorMap* kmap, const SuperArgs& a, int ngroups, bool bd, int grid,
                                cudaStream_t st);

// Sharded phase barrier on the device (api_shard.cu shard_barrier): add 1 to
// every rank's IPC-mapped arrival counter, wait for the own one to reach target.
cudaError_t launch_shard_barrier(unsigned* const* peer_flags, unsigned* my_flag, int world, unsigned target,
                                 cudaStream_t st);

// Whole-evolution kernel for L <= 12 local qubits: one CTA keeps the state in
// shared memory for all K steps (SURVEY §7 hard part 5; latency-bound sizes).
struct ResidentArgs {
  double2* psi;
  const uint8_t* E;
  int L;
  int64_t K;
  const double2* phi_all;   // K rows of n_phi entries
  int n_phi;
  const double* coef;       // K coefficients
  const int32_t* form;      // K forms
  int final_d;              // 1: apply row K of phi_all after the last X (Strang closing half step)
};
cudaError_t launch_resident(const ResidentArgs& a, cudaStream_t st);
// 13 <= L <= 16: all K steps in one launch, the state in the registers of one
// thread-block cluster of 2^(L-12) CTAs per replica (cluster_evolve.cu)
struct ClusterArgs {
  double2* psi;             // single evolve: canonical state in/out; nullptr: replicas start uniform
  const uint8_t* E;
  int L;
  double amp0;              // 2^{-n/2} (replicas)
  int64_t K;                // steps (single evolve)
  const int64_t* Krep;      // per replica steps (sweep) or nullptr
  const int64_t* row_off;   // per replica first row of phi_all/coef/form, or nullptr
  const double2* phi_all;   // rows of n_phi entries
  int n_phi;
  const double* coef;
  const int32_t* form;
  int final_d;              // Strang: apply row off+K after the last X
  double* out;              // per replica P_succ, or nullptr
};
cudaError_t launch_cluster_evolve(const ClusterArgs& a, int nrep, cudaStream_t st);
int cluster_evolve_max_active(int L);
// 13 <= L <= 21: all passes of the cyclic plan in one cooperative launch, one
// warp per 2^9-amplitude tile, grid barrier between passes (warp_evolve.cu)
struct WarpGeo {
  int phys[9];          // tile bit b -> physical bit
  uint32_t rot;         // tile bits rotated by this group
  int nfree;            // L - 9
  int free_bits[32];    // tile-id bit i -> physical bit
};
struct WarpPass {
  int group;
  int flags;       // WP_PRE | WP_D | WP_POST, bit 3 / bit 4: pre / post in the cot form
  int64_t d;       // row of phi_all for D
  double cpre, cpost;  // rotation coefficients (tan or cot of beta) of the pre / post steps
};
enum { WP_PRE = 1, WP_D = 2, WP_POST = 4 };
struct WarpEvolveArgs {
  double2* psi;
  int L;
  WarpGeo geo[4];
  const uint8_t* Eg[4];   // per group: tile T's energies at Eg + 512 T, PX order (lane * 16 + r)
  const WarpPass* plan;
  int64_t npass;
  const double2* phi_all;
  int n_phi;
  const double* coef;
  const int32_t* form;
  unsigned* bar;          // grid barrier arrivals (zeroed before launch)
};
// F1 sweep on warp tiles: teams of `team` CTAs, one replica at a time per team
struct WarpSweepArgs {
  int L;
  double amp0;             // 2^{-n/2}
  WarpGeo geo[4];
  const uint8_t* Eg[4];
  const WarpPass* plan;    // all replicas' pass records
  const int64_t* plan_off; // [nrep] first record of replica r
  const int64_t* plan_len; // [nrep]
  int nrep;
  const double2* phi_all;
  int n_phi;
  int team;                // CTAs per team (grid = nteams * team)
  double2* scratch;        // nteams states of 2^L amplitudes
  double* partial;         // nteams * team * 8 per-warp partial sums
  unsigned* bar;           // nteams barrier counters, 128 bytes apart (zeroed)
  double* out;             // [nrep] P_succ
  int poll_ns;             // quad sweep: __nanosleep between team-barrier polls (0 = spin)
};
cudaError_t launch_warp_sweep(const WarpSweepArgs& a, int grid, cudaStream_t st);
cudaError_t launch_warp_energy(const uint8_t* E, uint8_t* Eg, const WarpGeo& g, int L, int num_sms, cudaStream_t st);
cudaError_t launch_warp_evolve(const WarpEvolveArgs& a, int grid, int warps, cudaStream_t st);
// the same plan with four warps per tile (QAA_OPT_WARPTILE 3; grid <= SMs x quad_evolve_max_active())
cudaError_t launch_quad_evolve(const WarpEvolveArgs& a, int grid, cudaStream_t st);
int quad_evolve_max_active();
// F1 sweep on teams of quad-warp CTAs (WarpSweepArgs.team CTAs per replica, partial: nteams * team doubles)
cudaError_t launch_quad_sweep(const WarpSweepArgs& a, int grid, cudaStream_t st);
int quad_sweep_max_active();
// 10 <= L <= 12: register-phase variant (2-3x faster than the per-qubit loop)
cudaError_t launch_resident_phases(const ResidentArgs& a, cudaStream_t st);

// Lanczos spectrum of H(s) (F3, spectrum.cu).
struct LanczosArgs {
  int n;
  int num_sms;
  const uint8_t* E;
  double wb, wp;          // weights of H_B and H_P at s
  int kmax, nev;
  double2* basis;         // (kmax + 1) * 2^n vectors
  double* scratch;        // >= 8 * num_sms doubles
  const double2* state;   // for the ground-state overlap (may be null)
};
cudaError_t lanczos_spectrum(const LanczosArgs& p, cudaStream_t st, double* evals, double* overlap, int* iters);

// Batched small-n sweep (F1): nrep independent evolutions of the uniform
// state, one CTA each, replica r with K[r] steps whose table rows start at
// row_off[r]; out[r] = P_succ.
struct SweepArgs {
  const uint8_t* E;
  int L;
  double amp0;              // 2^{-n/2}
  const int64_t* K;
  const int64_t* row_off;
  const double2* phi_all;
  int n_phi;
  const double* coef;
  const int32_t* form;
  int final_d;
  double* out;
};
cudaError_t launch_sweep(const SweepArgs& a, int nrep, cudaStream_t st);
// 13 <= L <= 16: one thread-block cluster of 2^(L-13) CTAs per replica
cudaError_t launch_sweep_cluster(const SweepArgs& a, int nrep, cudaStream_t st);

// Energy table (K1; the paper's kernel):
// E[x] = sum_c [(xg & M_c) == V_c], xg = x_offset + x, also folding
// max(E) and the zero count into the given device counters.
cudaError_t launch_energy_table(uint8_t* E, int64_t N, uint64_t x_offset, const uint64_t* MV, int m,
                                unsigned* d_max, unsigned long long* d_zeros, int num_sms, cudaStream_t st,
                                int lowbits = 63, int hishift = 0, bool force_w64 = false);
// Z compaction (A3): writes x_offset + x for every E[x] == 0 (order unspecified).
cudaError_t launch_compact_zeros(const uint8_t* E, int64_t N, uint64_t x_offset, uint64_t* Z,
                                 unsigned long long* d_count, int num_sms, cudaStream_t st);

// Initial states (K3).
cudaError_t launch_fill(double2* psi, int64_t N, double re, double im, int num_sms, cudaStream_t st);
cudaError_t launch_set_one(double2* psi, int64_t idx, cudaStream_t st);

// Reductions (K5). Deterministic: fixed grid, fixed trees.
// basic: partial[b*3 + {0,1,2}] = {sum |psi|^2, sum E|psi|^2, sum_{E=0} |psi|^2}
constexpr int RED_BLOCKS_PER_SM = 2;
cudaError_t launch_obs_basic(const double2* psi, const uint8_t* E, int64_t N, double* partial, int grid,
                             cudaStream_t st);
// sigma^x pair sums for the tile bits of one group geometry (k <= 12 tile bits):
// partial[b*12 + j] = sum over pairs of tile-local bit j of Re(conj(psi0) psi1).
struct SigmaArgs {
  const double2* psi;
  int k;                    // tile bits (12, or L when L <= 12)
  uint32_t mask;            // tile-local bits to evaluate
  int phys[TILE_BITS];
  int nseg;
  int seg_src[MAX_SEGS], seg_dst[MAX_SEGS], seg_len[MAX_SEGS];
  int64_t ntiles;
};
cudaError_t launch_obs_sigma(const SigmaArgs& a, double* partial, int grid, cudaStream_t st);
// <sigma^x> of the rank qubits of a sharded state (layout A): partial[b*3 + t] =
// this rank's part of sum_x Re(conj(psi[x]) psi[x ^ 2^(L+t)]), the partner being
// the same local index on rank r ^ 2^t, read over NVLink through its IPC mapping.
struct PeerDotArgs {
  const double2* peer[3];  // rank r ^ 2^t's current shard buffer, t < g
  int g;                   // rank qubits (1..3)
};
cudaError_t launch_obs_peer_dot(const double2* psi, const PeerDotArgs& a, int64_t N, double* partial, int grid,
                                cudaStream_t st);
// sum of |psi[Z[i]]|^2 over a sorted list (1 block).
cudaError_t launch_gather_success(const double2* psi, const uint64_t* Z, int64_t nz, uint64_t x_offset,
                                  double* out, cudaStream_t st);
// out[j] = sum_b partial[b*stride + j] for j < nvals, fixed order (1 block).
cudaError_t launch_reduce_partials(const double* partial, int nblocks, int stride, int nvals, double* out,
                                   cudaStream_t st);

}  // namespace qaa
