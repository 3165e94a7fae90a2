/*
 * qaa.h -- C-ABI of libqaa: B200-native first-order Trotter evolution of the
 * quantum adiabatic algorithm for 3-SAT (Diaz-Pier, Venegas-Andraca,
 * Gomez-Munoz, arXiv 1103.1399).
 *
 * Citations: "P:n" is line n of the paper's text; "R<k>" is reading
 * k in DESIGN.md (where the paper is silent or garbled); "SURVEY §8" is the
 * hot-path scope table.
 *
 * What is computed (Eq. 1 at P:69-72):
 *   H(s) = (1 - s) H_B + s H_P,  H_B = sum_j (1 - sigma^x_j)/2   (R1, R2)
 *   H_P  = diag(E),  E(x) = number of clauses all of whose literals are false
 *          under assignment x (constant 1, duplicates counted, R4/R5)
 *   psi_0 = 2^{-n/2} sum_x |x>
 *   K first-order Trotter steps of length dt = T/K; step k uses s_k (midpoint
 *   (k+1/2)/K unless a schedule is given, R8) and applies
 *   exp(-i dt s_k H_P) first, then exp(-i dt (1 - s_k) H_B)      (R7)
 *
 * Conventions (R-conventions): basis index x, bit j-1 of x is
 * variable x_j (x_1 least significant), bit value 1 = true. Amplitudes are
 * complex128 stored interleaved (re, im), i.e. torch.complex128 /
 * cuDoubleComplex layout. hbar = 1; all reported values are raw (no
 * renormalisation, R12).
 *
 * Error model: every call returns a qaa_status; nothing aborts, exits or
 * throws across the ABI. qaa_last_error(ctx) names the offending argument.
 * USAGE, INPUT and CAP leave the context usable. A CUDA or NCCL failure
 * poisons the context: every later call except qaa_destroy returns
 * QAA_E_STATE. A context is used by one host thread at a time.
 *
 * Asynchrony: init and evolve are enqueued on the context's stream and return
 * without a host synchronisation; the reductions (success_prob, energy,
 * norm2, sigma_x) and copies synchronise the stream before returning.
 */
#ifndef QAA_H
#define QAA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QAA_OK = 0,
  QAA_E_USAGE = 1, /* bad argument value or call order the caller controls */
  QAA_E_INPUT = 2, /* malformed instance (literal 0 or |literal| > n)       */
  QAA_E_CAP = 3,   /* problem exceeds a capacity (device memory, m > 255)   */
  QAA_E_STATE = 4, /* call out of order (e.g. evolve before init), or the
                      context is poisoned by an earlier CUDA/NCCL error      */
  QAA_E_CUDA = 5,  /* CUDA runtime error (poisons the context)              */
  QAA_E_NCCL = 6   /* a host collective (qaa_comm callback) failed; poisons
                      the context. The name is historical: the sharded path
                      uses CUDA IPC peer stores, not NCCL                    */
} qaa_status;

typedef struct qaa_ctx qaa_ctx;

/* Host-side collectives the library needs when world > 1: the bootstrap of the
 * CUDA-IPC peer pointers at load, the scalar reductions of the observables, and
 * the per-phase barrier only when QAA_OPT_SHARD_SYNC = 1 (by default the phase
 * barrier runs on the device, through IPC-mapped arrival counters).
 * The caller implements them over its process group (the Python binding uses
 * torch.distributed). Both return 0 on success; any other value makes the
 * library call fail with QAA_E_NCCL (and poisons the context).
 *  barrier     returns after every rank has entered it.
 *  allgather   recv[r*bytes .. (r+1)*bytes) = rank r's `send` (bytes each). */
typedef struct {
  void* user;
  int (*barrier)(void* user);
  int (*allgather)(void* user, const void* send, void* recv, size_t bytes);
} qaa_comm;

/* Creation parameters. All pointers are borrowed: the caller keeps
 * ownership and must keep them valid for the life of the context.
 *  device        CUDA device ordinal.
 *  stream        cudaStream_t to enqueue on; NULL = the library creates one.
 *  rank, world   this process's rank and the number of ranks (world = 1, or
 *                a power of two up to 8 when the state is sharded over GPUs
 *                on its top log2(world) qubits).
 *  nccl_id       reserved, must be NULL (the global-qubit exchange is the
 *                library's own CUDA-IPC peer-store pass, not NCCL).
 *  state         optional caller-owned device buffer for the local state
 *                (>= 16 * 2^L bytes, 256-byte aligned); NULL = library-owned.
 *                Must be NULL when world > 1 (the library owns the two
 *                IPC-shared shard buffers the layout swap alternates between).
 *  state_bytes   its size in bytes.
 *  comm          host collectives (required when world > 1, else ignored);
 *                copied, the function pointers must stay valid.
 * Sharding: rank r holds canonical indices [r 2^L, (r+1) 2^L),
 * L = n - log2(world). Every rank must run on a GPU that can reach the
 * others' memory through CUDA IPC (one node; NVLink/NVSwitch, or the same GPU). */
typedef struct {
  int device;
  void* stream;
  int rank;
  int world;
  const void* nccl_id;
  void* state;
  size_t state_bytes;
  const qaa_comm* comm;
} qaa_config;

/* Create a context. Errors: USAGE (NULL pointers, world not in {1,2,4,8},
 * rank out of range, world > 1 without comm or with a caller state buffer),
 * CUDA (device/stream setup). */
qaa_status qaa_create(const qaa_config* cfg, qaa_ctx** out);

/* Release every library-owned resource. Safe on a poisoned context and on NULL. */
void qaa_destroy(qaa_ctx* ctx);

/* Human-readable description of the last error on this context (never NULL). */
const char* qaa_last_error(const qaa_ctx* ctx);

/* Load a 3-SAT instance: n variables, m clauses, lits = 3*m
 * DIMACS-signed literals +-(1..n), clause c = lits[3c..3c+2] (copied; the
 * caller keeps ownership). Builds the energy table E (uint8 per basis state,
 * SURVEY §8 A2) and the solution set Z = {x : E(x) = 0} (A3) on the
 * device; resets the state to "uninitialised". Tautological clauses never
 * count; duplicates count with multiplicity (R5). m = 0 is allowed (E = 0).
 * Errors: USAGE (n < 1, m < 0, lits == NULL with m > 0, n - log2(world) < 1),
 * INPUT (a literal 0 or |l| > n), CAP (m > 255, or the local state plus
 * tables do not fit in device memory or a caller-owned state buffer).
 * Synchronises the stream. Collective when world > 1. */
qaa_status qaa_load_instance(qaa_ctx* ctx, int n, int m, const int32_t* lits);

/* psi <- 2^{-n/2} for every x. Errors: STATE (no instance). */
qaa_status qaa_init_uniform(qaa_ctx* ctx);

/* Test hook: psi <- |x> (basis state, x < 2^n). Errors: STATE, USAGE. */
qaa_status qaa_init_basis(qaa_ctx* ctx, uint64_t x);

/* Apply `steps` first-order Trotter steps of total time T:
 * dt = T/steps, s_k = schedule[k] if schedule != NULL (host array of `steps`
 * doubles in [0, 1]) else (k + 0.5)/steps. T = 0 is the identity.
 * Coefficients are computed on the host in binary64 (R11). Enqueued on the
 * stream; returns without a host sync (also when sharded: the per-phase
 * barrier runs on the device unless QAA_OPT_SHARD_SYNC = 1). The state is left
 * in canonical layout.
 * Errors: STATE (no init), USAGE (T < 0 or not finite, steps < 1, a schedule
 * value outside [0, 1]). Collective when world > 1 (identical arguments). */
qaa_status qaa_evolve(qaa_ctx* ctx, double T, int64_t steps, const double* schedule);

/* *out = sum_{x in Z} |psi[x]|^2 (raw; 0 for an UNSAT instance).
 * Deterministic (fixed reduction tree). Synchronises; same value on all ranks. */
qaa_status qaa_success_prob(qaa_ctx* ctx, double* out);

/* *out = <psi|H(s)|psi> (raw) = (1-s) sum_j (||psi||^2 - <sigma^x_j>)/2 + s sum_x E(x)|psi[x]|^2.
 * Errors: USAGE (s outside [0, 1]). Synchronises. Collective. */
qaa_status qaa_energy(qaa_ctx* ctx, double s, double* out);

/* *out = ||psi||^2 (raw). Synchronises. Collective. */
qaa_status qaa_norm2(qaa_ctx* ctx, double* out);

/* out[j] = <psi|sigma^x_{j}|psi> for qubit j = 0..n-1 (variable x_{j+1}); `out`
 * holds n doubles. Synchronises. Collective. */
qaa_status qaa_sigma_x(qaa_ctx* ctx, double* out);

/* Batched small-n sweep (the paper's regime of many small
 * instances): evolve `nrep` independent copies of the uniform state
 * of the loaded instance, replica r for total time T[r] in K[r] steps of the
 * midpoint schedule (splitting order of QAA_OPT_ORDER), all in ONE launch with
 * the state resident in shared memory (no HBM traffic): one CTA per replica for
 * n <= 13, one thread-block cluster of 2^(n-13) CTAs (2^13 amplitudes each,
 * cluster qubits exchanged through distributed shared memory) for 14 <= n <= 16;
 * out[r] = P_succ of replica r (host array of nrep doubles). The context's own
 * state is not touched. Synchronises.
 * Errors: USAGE (world > 1, n > 16, nrep < 1, NULL arrays, T[r] < 0 or not
 * finite, K[r] < 1), STATE (no instance). */
qaa_status qaa_sweep(qaa_ctx* ctx, int nrep, const double* T, const int64_t* K, double* out);

/* Low spectrum of H(s) (the adiabatic-theorem diagnostic of
 * P:66-67): Lanczos with full re-orthogonalisation on the matrix-free
 * H(s) psi (same weights as evolve, incl. the driving term), from a fixed
 * pseudo-random start vector, at most kmax iterations (stops early on an
 * invariant subspace). evals[0..nev-1] = the nev smallest Ritz values (gap =
 * evals[1] - evals[0]); if overlap != NULL, *overlap = |<g(s)|psi>|^2 /
 * <psi|psi> with g(s) the ground Ritz vector and psi the current state; *iters
 * (optional) = iterations used. Stores kmax+1 vectors of 2^n amplitudes.
 * Synchronises. Errors: USAGE (s outside [0,1], kmax not in 2..512, nev not in
 * 1..kmax), CAP (world > 1, n > 24, basis does not fit), STATE. */
qaa_status qaa_spectrum(qaa_ctx* ctx, double s, int kmax, int nev, double* evals, double* overlap, int* iters);

/* Driving term (the paper's unspecified "driving Hamiltonian",
 * P:193, R3): from the next evolve/energy/sweep on, H(s) = (1-s) H_B + s H_P +
 * s(1-s) (gx H_B + gz H_P), i.e. the step weights become (1-s) + gx s(1-s) for
 * H_B and s + gz s(1-s) for H_P (energy(s) reports this H(s)). gx = gz = 0
 * (default) is Eq. 1 exactly. Errors: USAGE (not finite). */
qaa_status qaa_set_driver(qaa_ctx* ctx, double gx, double gz);

/* Energy-table enumerator as a workload (the paper's own GPU
 * kernel): recompute the loaded instance's local table
 * E(x) `reps` times (after one warm-up) and return the average device time per
 * table in *ms (CUDA events on the context's stream). The table is rewritten
 * with identical values. Synchronises. Errors: USAGE, STATE (no instance). */
qaa_status qaa_time_energy_table(qaa_ctx* ctx, int reps, double* ms);

/* *out = |Z|, the number of satisfying assignments (all ranks). */
qaa_status qaa_num_solutions(qaa_ctx* ctx, uint64_t* out);

/* *out = max_x E(x) over the whole instance. */
qaa_status qaa_max_energy(qaa_ctx* ctx, uint32_t* out);

/* Copy amplitudes [first, first+count) of the canonical global index space
 * to host memory dst (2*count doubles, caller-owned). Each rank copies the
 * part it owns and leaves the rest of dst untouched. Synchronises.
 * Errors: USAGE (range outside [0, 2^n)), STATE (no instance). */
qaa_status qaa_copy_state(qaa_ctx* ctx, uint64_t first, uint64_t count, double* dst_host);

/* Overwrite amplitudes [first, first+count) from host memory (2*count doubles).
 * Marks the state initialised. Synchronises. Test and checkpoint hook. */
qaa_status qaa_set_state(qaa_ctx* ctx, uint64_t first, uint64_t count, const double* src_host);

/* Copy energy-table entries E(x), x in [first, first+count), to host (uint8).
 * Each rank copies the part it owns. Synchronises. */
qaa_status qaa_copy_energy_table(qaa_ctx* ctx, uint64_t first, uint64_t count, uint8_t* dst_host);

/* Device pointer of the local state (2^L complex128), for zero-copy wrapping. */
qaa_status qaa_state_ptr(qaa_ctx* ctx, void** out, uint64_t* amps);

/* ---------------------------------------------------------------- tuning / stats */

/* Options (take effect at the next load/evolve):
 *  QAA_OPT_ROW_BITS      c in {3, 4, 5}: log2 of the contiguous amplitude run
 *                        every tile keeps (128/256/512-byte rows). Default 3.
 *  QAA_OPT_PROFILE       1 = record a CUDA event pair around every pass kernel
 *                        launch of evolve (read back with qaa_get_stats).
 *  QAA_OPT_STEP_SPANNING 2 (default) = step spanning with D only on the strided
 *                        groups (group 0 is a plain contiguous pass every step);
 *                        1 = cyclic step spanning (D visits every group); both merge
 *                        the last tile group of step k with the first of step k+1
 *                        around D_{k+1}: P-1 passes per step;
 *                        0 = one D per step in the first pass only (P passes/step).
 *  QAA_OPT_CTAS_PER_SM   register-kernel variant: 1 = one CTA per SM with register
 *                        double-buffered prefetch, 2 = two CTAs per SM, no prefetch.
 *  QAA_OPT_KERNEL        2 (default) = auto: the register-prefetch kernel up to 19 local
 *                        qubits (latency-bound passes), the TMA kernels above;
 *                        1 = always the TMA pass kernels (mbarrier ring of 3 shared-memory
 *                        slots, 1-2 consumer groups; the L2-blocked step needs them);
 *                        0 = always the register-prefetch pass kernel.
 *  QAA_OPT_TMA_GROUPS    consumer groups (8 warps each) per TMA CTA: 0 = auto (1 for
 *                        passes without D: two tiles in flight; 2 for D passes: two
 *                        groups overlap their transposes and FMAs), or force 1 / 2.
 *  QAA_OPT_SUPER         bit 0 (default 1): L2-blocked Trotter steps when the plan has three
 *                        tile groups (22 <= n <= 30 on one GPU) and schedule mode 2: each pass
 *                        pair [group 0 rotate][group k rotate, D, rotate] runs as ONE launch
 *                        over 32 MiB chunks resident in L2, one HBM round trip per step
 *                        (K + 1 launches for K steps: the closing plain pair fuses too); bit 1: one consumer group per CTA
 *                        (default two); bits 2-3: L2 eviction hints (0 = evict-last for the
 *                        group-0 output read back by the group-k sub-pass and evict-first
 *                        for dead data; 1 = no hints; 2 = evict-first only); bit 4: use it
 *                        even below 256 chunks (n < 28), where the two-pass plan is faster
 *                        and is chosen otherwise; bit 5: hand out the tiles through a
 *                        global atomic work queue instead of the static round robin
 *                        (measured 2-4 % slower); bit 6: the tensor-memory variant
 *                        (pass_tmem.cu: register-pattern changes through tcgen05.st/ld
 *                        instead of shared memory; measured 3-10 % slower);
 *                        bits 7-10 and 13: its A/B switches and diagnostics counters
 *                        (SuperArgs.tm_flags; with the default kernel bit 7 = publish a
 *                        group-0 tile after the next landed read, bit 8 = right after its
 *                        stores, bit 9 = store each group-k tile with one TMA tensor store
 *                        from shared memory -- bitwise equal, measured 2 % slower); bits 11-12: chunk lag - 1 (default lag 1: two chunks
 *                        live in L2; 2-3 measured slower); bit 14: producer-warp variant;
 *                        bit 15: the round-1 synchronisation (a group barrier before every
 *                        exchange write and before each group-0 tile's publish) instead of
 *                        the default split-phase write-after-read mbarriers and deferred
 *                        per-warp publish (measured 2-5 % slower). Values 0..65535.
 *  QAA_OPT_SUPER_GRID    CTAs of an L2-blocked launch (0 = one per SM, default; else 1..SMs):
 *                        a tuning hook -- a chunk's 2^tpc tiles are dealt round robin, so a
 *                        grid dividing them evenly balances the per-chunk work.
 *  QAA_OPT_SUPER_SPLIT   split roles in the L2-blocked launch: this many CTAs run only the
 *                        group-0 tiles (from HBM), the others only the group-k tiles, each
 *                        side in chunk order (0 = one interleaved sequence, default).
 *  QAA_OPT_SHARD_SYNC    sharded phase barrier: 0 (default) = on the device (every rank adds
 *                        1 to every rank's CUDA-IPC-mapped arrival counter after its peer
 *                        stores, then waits for its own to reach epoch * world), so a
 *                        sharded qaa_evolve is enqueued without a host sync; 1 = stream
 *                        sync + the caller's qaa_comm barrier per phase (the round-1 plan).
 *  QAA_OPT_PERSIST       1: for 13 <= n - log2(world) <= 21 on one GPU with the automatic
 *                        kernel choice, all K steps run as ONE cooperative launch of the
 *                        persistent pass kernel (state L2-resident, a grid barrier between
 *                        passes) instead of one launch per pass. 0 (default): per-pass
 *                        launches -- measured faster (7.4 vs 8.9 us/step at n = 13..18:
 *                        a pass is bound by one CTA's tile program, not by the launch).
 *  QAA_OPT_CLUSTER       1 (default): for 13 <= n <= 16 on one GPU with the automatic kernel
 *                        choice, all K steps run as ONE launch with the state resident in the
 *                        registers of a thread-block cluster of 2^(n-12) CTAs (cluster bits
 *                        swapped with local bits over DSMEM once per step); 0: per-pass
 *                        kernels through HBM/L2.
 *  QAA_OPT_WARPTILE      1 (default): for 13 <= n <= 16 on one GPU with the automatic kernel
 *                        choice, all passes of the cyclic step-spanning plan run as ONE
 *                        cooperative launch over 2^9-amplitude tiles (state in L2), a grid
 *                        barrier between passes, FOUR warps per tile (one 128-thread CTA,
 *                        4 amplitudes per lane: the tile's work spread over the SM's four
 *                        sub-partitions); takes precedence over QAA_OPT_CLUSTER (measured
 *                        3.2-3.5 us per step at n = 13..16, vs 4.3-5.0 with one warp per
 *                        tile and 5.4-8.3 cluster-resident). 2: ONE warp per tile (16
 *                        amplitudes per lane), also for 17 <= n <= 21 (there slower than the
 *                        per-pass kernels; a test hook), and qaa_sweep on teams of warp-tile
 *                        CTAs (n <= 21; at n = 13..16 no faster than the default
 *                        cluster-resident sweep). 3: four warps per tile, 13 <= n <= 21
 *                        (test hook above 16), and qaa_sweep on teams of quad-warp CTAs
 *                        (n <= 21; test hook: not reliably faster than the clusters). 0: off.
 *  QAA_OPT_WARP_GRID     tuning hook for the warp-tile launch: ctas * 16 + warps per CTA
 *                        (1..8); 0 (default) = automatic.
 *  QAA_OPT_SUPER_REV     1: the L2-blocked step with its two sub-passes in the other order
 *                        (three tile groups): [group k: rotate, D, rotate] tiles first (strided
 *                        rows from HBM, output kept in L2), then [group 0: rotate] (contiguous
 *                        from L2, the step's only HBM write-back contiguous). 0 (default).
 *  QAA_OPT_DIAG          timing diagnostics ONLY (results are wrong by design): the
 *                        L2-blocked step at the bench configuration with work removed --
 *                        1 = no rotations, 2 = no shared-memory exchanges, 4 = no D,
 *                        8 = group-k tiles ignore the chunk dependency; sums 3, 7, 15.
 *                        Other configurations return QAA_E_CUDA at evolve. Default 0.
 *  QAA_OPT_ENERGY_W64    test hook: 1 = the 64-bit energy-table kernel even when every
 *                        assignment fits 32 bits (default 0: 32-bit kernel for n <= 32).
 *  QAA_OPT_SUPER_PUB     L2-blocked step: batch + 16 * early. batch = group-0 tiles of one
 *                        chunk a warp publishes with ONE gpu-scope release (1..8, default 1;
 *                        each release's fence waits for all of the warp's earlier stores);
 *                        early = 1: a tile's shared-memory slot is released before the last
 *                        three register-bit rotations of its program (refill starts earlier).
 *  QAA_OPT_SWEEP_TUNE    tuning hook for the quad-warp team sweep: poll_ns * 16 + log2(tiles
 *                        per CTA) + 1 (poll_ns = __nanosleep between team-barrier polls,
 *                        <= 4095; low 4 bits 0 = automatic tiles per CTA). Default 0.
 *  QAA_OPT_ORDER         1 (default) = first-order Lie-Trotter, D then X (R7);
 *                        2 = second-order Strang splitting, D^{1/2} X D^{1/2} per step, at
 *                        the same HBM cost (the half D's of adjacent steps are merged, the
 *                        closing half step rides on the last pass). Single GPU. */
enum {
  QAA_OPT_ROW_BITS = 1,
  QAA_OPT_PROFILE = 2,
  QAA_OPT_STEP_SPANNING = 3,
  QAA_OPT_CTAS_PER_SM = 4,
  QAA_OPT_KERNEL = 5,
  QAA_OPT_TMA_GROUPS = 6,
  QAA_OPT_SUPER = 7,
  QAA_OPT_ORDER = 8,
  QAA_OPT_ENERGY_W64 = 9,
  QAA_OPT_SUPER_GRID = 10,
  QAA_OPT_SUPER_SPLIT = 11,
  QAA_OPT_SHARD_SYNC = 12,
  QAA_OPT_PERSIST = 13,
  QAA_OPT_DIAG = 14,
  QAA_OPT_CLUSTER = 16,
  QAA_OPT_WARPTILE = 17,
  QAA_OPT_WARP_GRID = 18,
  QAA_OPT_SUPER_REV = 19,
  QAA_OPT_SWEEP_TUNE = 20,
  QAA_OPT_SUPER_PUB = 21
};
qaa_status qaa_set_option(qaa_ctx* ctx, int key, int64_t value);

typedef struct {
  int64_t evolve_calls;      /* since the last reset */
  int64_t trotter_steps;     /* total Trotter steps applied */
  int64_t pass_launches;     /* pass-kernel launches (HBM passes over the state) */
  int64_t other_launches;    /* every other kernel launched by evolve */
  int64_t passes_per_step_num, passes_per_step_den; /* steady-state ratio of the plan */
  double pass_kernel_ms;     /* sum of event-timed pass-kernel durations (QAA_OPT_PROFILE) */
  int64_t pass_kernels_timed;
  int64_t bytes_per_pass;    /* algorithmic bytes one pass launch moves: 32 B/amp (+1 B/amp E for D passes, averaged) */
  int64_t amps_local;
  int n, n_local, groups, tile_bits, row_bits;
  int64_t kernel_launches_total; /* every kernel this context launched since reset */
  int64_t super_launches;    /* of pass_launches: L2-blocked launches (QAA_OPT_SUPER) */
  double super_kernel_ms;    /* of pass_kernel_ms: their event-timed durations */
  int64_t super_kernels_timed;
  int64_t tm_launches;       /* of super_launches: tensor-memory exchange variant (pass_tmem.cu) */
  int64_t persist_launches;  /* of pass_launches: persistent whole-evolve launches (QAA_OPT_PERSIST) */
  int64_t pw_launches;       /* of super_launches: producer-warp variant (QAA_OPT_SUPER bit 14) */
  uint64_t tm_diag[8];       /* diagnostics (QAA_OPT_SUPER bit 10), summed over warps' lane 0 since the
                                context's first such launch: [0] cycles in slot-landed waits, [1] items,
                                [2] deferred group-k items, [3] cycles in deferred waits, [4] / [5]
                                cycles in group-0 / group-k tile programs; zeros otherwise */
  int64_t cluster_launches;  /* of pass_launches: cluster-resident whole-evolve launches (QAA_OPT_CLUSTER) */
  int64_t warp_launches;     /* of pass_launches: warp-tile whole-evolve launches (QAA_OPT_WARPTILE) */
} qaa_stats;
qaa_status qaa_get_stats(qaa_ctx* ctx, qaa_stats* out);
qaa_status qaa_reset_stats(qaa_ctx* ctx);

/* ------------------------------------------------------------- host-only planner */

/* Pure host function (no device needed): describe the pass plan evolve uses
 * for n_local local qubits, row bits c and K steps. Writes up to `cap`
 * records of QAA_PLAN_RECORD int32 each:
 *   {group, pre_step, d_step, post_step, pre_lo, pre_hi, post_lo, post_hi,
 *    n_exchanges, n_shuffles}
 * where steps are -1 when absent and (lo, hi) are the low/high 32 bits of the
 * mask of physical qubits rotated for pre_step / post_step. *count = number of
 * passes (may exceed cap). For n_local <= 12 (resident kernel) every step is
 * one record {0, -1, k, k, mask, 0, mask, 0, 0, 0}... with pre_mask 0.
 * Used by the CPU tests of the schedule logic. */
#define QAA_PLAN_RECORD 10
qaa_status qaa_plan_describe(int n_local, int row_bits, int step_spanning, int64_t K,
                             int32_t* records, int64_t cap, int64_t* count);

/* Pure host function: the sharded pass plan for n qubits over `world` ranks
 * (plan.hpp ShardPass). Records of QAA_SHARD_RECORD int32:
 *   {kind (0 pass, 1 plain remap), group, pre_step, d_step, post_step,
 *    remote (1: the pass stores into the peers' other buffer = layout swap),
 *    layout (0 = A, 1 = B, of the state the pass reads),
 *    pre_mask, post_mask (physical local qubits rotated for pre/post step), 0}
 * Errors: USAGE (bad sizes), CAP (n too small to shard over `world`). */
#define QAA_SHARD_RECORD 10
qaa_status qaa_plan_describe_sharded(int n, int world, int row_bits, int64_t K, int32_t* records, int64_t cap,
                                     int64_t* count);

/* Library version string. */
const char* qaa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QAA_H */
