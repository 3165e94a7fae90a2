// api_internal.hpp -- state and helpers shared by the C-ABI translation units
// (api_*.cu) of libqaa: the opaque context, error helpers, and the internal
// functions one unit calls in another. Not part of the public ABI (include/qaa.h).
#pragma once
#include <nvtx3/nvToolsExt.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/qaa.h"
#include "kernels.cuh"
#include "plan.hpp"

using namespace qaa;

namespace {
constexpr int64_t ZLIST_CAP = 1 << 16;  // keep Z as a sorted list up to this size
constexpr int RESIDENT_MAX_L = TILE_BITS;
constexpr int SWEEP_MAX_L = 16;
constexpr int PERSIST_MAX_L = 21;
// The L2-blocked step pays from 256 chunks up (n >= 28 on one GPU, measured):
// below that the strided groups have padded 256-byte rows, the two-pass plan
// streams at the copy peak and the chunk pipeline is too short (n = 24: 0.44
// vs 0.19 ms/step).
constexpr int64_t SUPER_MIN_CHUNKS = 256;  // qaa_sweep: one CTA up to 12, one cluster of <= 8 CTAs up to 16

struct ClauseRecHost {
  uint64_t mhi, vhi;
  uint32_t spread[4];
};
static_assert(sizeof(ClauseRecHost) == 32, "clause record layout");
}  // namespace

// NVTX ranges around the C-ABI calls and the kernel launches of an evolve (header-only
// NVTX v3: free when no tool is attached; visible in nsys / ncu --nvtx)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define QAA_NVTX(name) NvtxRange qaa_nvtx_range_(name)

constexpr int WARP_MIN_L = 13, WARP_MAX_L = 21;  // warp_evolve.cu range (QAA_OPT_WARPTILE 2)
constexpr int WARP_AUTO_MAX_L = 16;               // default range: faster than the per-pass kernels up to here
int warp_group_count(int L);
struct qaa_ctx;
qaa_status ensure_warp_tables(qaa_ctx* ctx);  // warp-tile geometry + per-group energy tables

struct qaa_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int rank = 0, world = 1, gbits = 0;
  int num_sms = 148;
  // state
  double2* state = nullptr;
  bool own_state = false;
  size_t state_cap_bytes = 0;
  // instance
  int n = 0, L = 0, m = 0;
  bool loaded = false, initialized = false, poisoned = false;
  uint8_t* E = nullptr;
  size_t E_cap = 0;
  uint64_t* Z = nullptr;
  size_t Z_cap = 0;
  int64_t nz_local = 0;
  uint64_t nz_total = 0;
  bool z_listed = false;
  unsigned emax = 0;
  Geometry geom;
  // coefficient tables
  void* d_coef = nullptr;
  size_t d_coef_cap = 0;
  void* h_coef = nullptr;
  size_t h_coef_cap = 0;
  cudaEvent_t coef_done = nullptr;
  bool coef_pending = false;
  // reductions
  double* d_part = nullptr;
  size_t d_part_cap = 0;
  double* d_out = nullptr;   // 64 doubles
  double* h_out = nullptr;   // pinned, 64 doubles
  unsigned* d_counters = nullptr;  // [0] = max (unsigned), [2..3] = zero count (u64)
  // options
  int row_bits = 3;
  int profile = 0;
  int step_spanning = 2;  // plan.hpp build_pass_schedule modes
  int order = 1;  // 1: Lie-Trotter (D then X, R7); 2: Strang (half D, X, half D; NEXT F4)
  double drv_x = 0.0, drv_z = 0.0;  // driving term s(1-s)(g_x H_B + g_z H_P) (NEXT F4, R3)
  int ctas_per_sm = 1;
  int kernel_mode = 2;  // 1: TMA pass kernels, 0: register-prefetch pass, 2: auto (register up to L = 19)
  int tma_groups = 0;   // consumer groups per TMA CTA: 0 = auto (1 without D, 2 with D)
  int super_mode = 1;   // L2-blocked D passes (qaa_superpass) when the plan has 3 tile groups
  int super_groups = 2;
  int super_hints = 2;
  int super_force = 0;
  int energy_w64 = 0;  // test hook: 64-bit energy-table kernel even when x fits 32 bits
  bool shard_super_ok = false;  // sharded plan: fused [group 0][group P-2 + layout swap] launches
  SuperArgs shard_super;
  CUtensorMap shard_kmap[2];    // group P-2 over shard buffer 0 / 1
  bool shard_top_ok = false;    // sharded top-group D passes on the TMA kernel
  CUtensorMap shard_top_map[2]; // top group over shard buffer 0 / 1
  TmaArgs shard_top;            // its geometry
  uint8_t* shard_top_eg[2] = {nullptr, nullptr};  // its permuted energies, layout A / B
  size_t shard_top_eg_cap = 0;
  int super_dynamic = 0;
  int super_tm = 0;             // tensor-memory exchanges in the L2-blocked step (pass_tmem.cu)
  int super_tm_flags = 0;
  int super_lag = 1;
  int super_pw = 0;  // producer-warp L2-blocked step
  int diag = 0;      // QAA_OPT_DIAG (timing diagnostics only)
  int cluster_evolve = 1;  // QAA_OPT_CLUSTER: 13 <= L <= 16 in one cluster-resident launch
  int warptile = 1;        // QAA_OPT_WARPTILE: 13 <= L <= 21 in one warp-tile cooperative launch
  int warp_grid = 0;       // QAA_OPT_WARP_GRID: ctas * 16 + warps (0 = automatic)
  int super_pub = 1;       // QAA_OPT_SUPER_PUB: group-0 tiles per release in the L2-blocked step
  int sweep_tune = 0;      // QAA_OPT_SWEEP_TUNE: poll_ns * 16 + log2(tiles per CTA) + 1 (0 = automatic)
  bool wt_built = false;   // Ewt / wgeo match the loaded instance
  int wt_groups = 0;
  WarpGeo wgeo[4];
  uint8_t* Ewt[4] = {nullptr, nullptr, nullptr, nullptr};
  void* d_wsweep = nullptr;  // warp-tile sweep: plans, offsets, team states, partials, barriers
  size_t d_wsweep_cap = 0;
  int super_v2 = 1;
  int super_rev = 0;  // QAA_OPT_SUPER_REV: reversed pairs [group k rotate/D/rotate][group 0 rotate]  // split-phase WAR guards + deferred publish (QAA_OPT_SUPER bit 15 clears it)
  int super_grid = 0;  // 0: one CTA per SM
  int super_split = 0;
  int persist = 0;  // persistent evolve for 13 <= L <= 21 (opt-in: measured slower)
  void* d_persist = nullptr;  // its barrier words and pass records
  size_t d_persist_cap = 0;  // split roles: CTAs running group-0 tiles only (0 = interleaved sequence)
  unsigned long long* d_tm_diag = nullptr;  // pass_tmem.cu diagnostics counters (QAA_OPT_SUPER bit 10)
  bool tm_built = false;        // build_tm ran for the current geometry (lazily, on first use)
  int tm_ok[4] = {0, 0, 0, 0};  // per paired group: swizzled map (+ K4-packed energies) ready
  CUtensorMap tmaps_sw[4];
  TmaArgs tm_geo[4];             // its tensor-map dims (ndims, dim_seg) for the load coordinates
  uint8_t* Eg_tm[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t Eg_tm_cap[4] = {0, 0, 0, 0};
  uint16_t* d_pos_tm = nullptr;  // byte position of each tile-local index in a K3-packed slice
  SuperArgs super_static[4];
  bool super_ok[4] = {false, false, false, false};
  void* clause_recs = nullptr;  // device clause records (A1) of the loaded instance
  size_t clause_recs_cap = 0;
  int n_recs = 0;
  void* d_super = nullptr;  // done[] counters + queue
  size_t d_super_cap = 0;
  // TMA state per tile group (built at load)
  std::vector<uint8_t*> Eg;  // per-group permuted energies (Eg[0] = E)
  std::vector<size_t> Eg_cap;
  std::vector<CUtensorMap> tmaps;
  std::vector<TmaArgs> tma_static;
  std::vector<int> tma_ok;
  // programs
  std::map<std::tuple<int, int, int, int>, Program> progs;
  // sharded state (world > 1): two IPC-shared shard buffers, layout A/B tables
  qaa_comm comm;
  bool has_comm = false;
  double2* bufs[2] = {nullptr, nullptr};
  size_t buf_cap = 0;
  int cur = 0;                       // buffer holding the current state
  double2* peers[2][8] = {{nullptr}};  // peers[b][r]: rank r's buffer b (own rank: local pointer)
  bool peer_open[2][8] = {{false}};
  unsigned* sync_buf = nullptr;      // own arrival counter of the device-side phase barrier (IPC-exported)
  unsigned* peer_sync[8] = {nullptr};  // every rank's counter (own rank: local pointer)
  bool peer_sync_open[8] = {false};
  unsigned sync_epoch = 0;           // barriers issued so far (identical on every rank)
  int shard_sync = 0;                // 0: device-side barrier (async evolve), 1: host barrier + stream sync
  uint8_t* E_B = nullptr;            // energies in layout B
  size_t E_B_cap = 0;
  // stats
  qaa_stats stats;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
  std::vector<char> ev_super;  // ev_pool[i] timed an L2-blocked (qaa_superpass) launch
  size_t ev_used = 0;
  std::string err;
};

inline qaa_status fail(qaa_ctx* c, qaa_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) {
    c->err = buf;
    if (st == QAA_E_CUDA || st == QAA_E_NCCL) c->poisoned = true;
  }
  return st;
}

#define CUDA_TRY(call)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(ctx, QAA_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                      \
  } while (0)

// CUDA_TRY for helpers that report through a status out-parameter and return true
#define CUDA_TRY_ST(call)                                                                          \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      *st = fail(ctx, QAA_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                 __LINE__);                                                                        \
      return true;                                                                                 \
    }                                                                                              \
  } while (0)

#define CHECK_CTX()                                                             \
  do {                                                                          \
    if (!ctx) return QAA_E_USAGE;                                               \
    if (ctx->poisoned) return fail(ctx, QAA_E_STATE, "context poisoned: %s", ctx->err.c_str()); \
    cudaSetDevice(ctx->device);                                                 \
  } while (0)

inline qaa_status ensure_buffer(qaa_ctx* ctx, void** p, size_t* cap, size_t bytes) {
  if (*cap >= bytes && *p) return QAA_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return fail(ctx, QAA_E_CAP, "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
  }
  *cap = bytes;
  return QAA_OK;
}

inline qaa_status ensure_host(qaa_ctx* ctx, void** p, size_t* cap, size_t bytes) {
  if (*cap >= bytes && *p) return QAA_OK;
  if (*p) cudaFreeHost(*p);
  *p = nullptr;
  *cap = 0;
  CUDA_TRY(cudaMallocHost(p, bytes));
  *cap = bytes;
  return QAA_OK;
}

// H1: per-step coefficients (host, binary64 libm; R11).
struct StepCoef {
  double coef;
  int form;
};

// Weights of H_B and H_P at s: Eq. 1 gives (1 - s, s); the optional driving
// term s(1-s)(g_x H_B + g_z H_P) (NEXT F4, R3) adds s(1-s) g to each. With
// g = 0 both are bit-identical to 1 - s and s.
inline double weight_b(const qaa_ctx* c, double s) { return (1.0 - s) + c->drv_x * s * (1.0 - s); }
inline double weight_p(const qaa_ctx* c, double s) { return s + c->drv_z * s * (1.0 - s); }

// Pass-kernel choice. Auto: the register-prefetch kernel while the state is
// small enough for a pass to be latency-bound (L <= 19: a few dozen tiles, the
// LDG path has the shorter tile latency, measured 30 % faster at n = 13..19),
// the TMA kernels above (n = 23..27: 20-30 % faster; the L2-blocked step from 28).
constexpr int AUTO_REGISTER_MAX_L = 19;
inline bool use_tma(const qaa_ctx* ctx) {
  return ctx->kernel_mode == 1 || (ctx->kernel_mode == 2 && ctx->L > AUTO_REGISTER_MAX_L);
}


// ------------------------------------------------------------------ cross-unit internals
// api_tma.cu: tensor maps, permuted energy tables, L2-blocked chunk plans
qaa_status build_tma(qaa_ctx* ctx);
void build_shard_super(qaa_ctx* ctx);
qaa_status build_shard_top(qaa_ctx* ctx);
qaa_status build_tm(qaa_ctx* ctx);
// api_shard.cu: host collectives through the caller's qaa_comm, shard buffers, sharded evolve
qaa_status comm_barrier(qaa_ctx* ctx);
qaa_status comm_allgather(qaa_ctx* ctx, const void* send, void* recv, size_t bytes);
qaa_status comm_sum(qaa_ctx* ctx, double* v, int n);
qaa_status setup_shard_buffers(qaa_ctx* ctx, size_t bytes);
qaa_status shard_remap(qaa_ctx* ctx);
qaa_status shard_barrier(qaa_ctx* ctx);
qaa_status evolve_sharded(qaa_ctx* ctx, int64_t K, const std::vector<StepCoef>& sc, const double2* dphi, int n_phi);
// api_evolve.cu: coefficient rows (H1), profiling events, plan choice
void build_step(double T, int64_t K, double wb, double theta, int n, int n_phi, double2* phi_row, StepCoef* sc);
qaa_status ensure_events(qaa_ctx* ctx, size_t need);
bool super_usable(qaa_ctx* ctx);
// api_observe.cu: reduction scratch
qaa_status ensure_part(qaa_ctx* ctx, size_t doubles);
