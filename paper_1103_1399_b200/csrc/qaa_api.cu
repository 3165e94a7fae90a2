// qaa_api.cu -- the C-ABI of libqaa (include/qaa.h): context, validation,
// host coefficient builder (H1), pass planning (H2, plan.cpp) and launches.
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
  uint8_t* E_B = nullptr;            // energies in layout B
  size_t E_B_cap = 0;
  // stats
  qaa_stats stats;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
  std::vector<char> ev_super;  // ev_pool[i] timed an L2-blocked (qaa_superpass) launch
  size_t ev_used = 0;
  std::string err;
};

static qaa_status fail(qaa_ctx* c, qaa_status st, const char* fmt, ...) {
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

#define CHECK_CTX()                                                             \
  do {                                                                          \
    if (!ctx) return QAA_E_USAGE;                                               \
    if (ctx->poisoned) return fail(ctx, QAA_E_STATE, "context poisoned: %s", ctx->err.c_str()); \
    cudaSetDevice(ctx->device);                                                 \
  } while (0)

static qaa_status ensure_buffer(qaa_ctx* ctx, void** p, size_t* cap, size_t bytes) {
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

static qaa_status ensure_host(qaa_ctx* ctx, void** p, size_t* cap, size_t bytes) {
  if (*cap >= bytes && *p) return QAA_OK;
  if (*p) cudaFreeHost(*p);
  *p = nullptr;
  *cap = 0;
  CUDA_TRY(cudaMallocHost(p, bytes));
  *cap = bytes;
  return QAA_OK;
}

extern "C" {

const char* qaa_version(void) { return "qaa-b200 0.1 (sm_100a)"; }

qaa_status qaa_create(const qaa_config* cfg, qaa_ctx** out) {
  if (!cfg || !out) return QAA_E_USAGE;
  *out = nullptr;
  if (cfg->world != 1 && cfg->world != 2 && cfg->world != 4 && cfg->world != 8) return QAA_E_USAGE;
  if (cfg->rank < 0 || cfg->rank >= cfg->world) return QAA_E_USAGE;
  qaa_ctx* ctx = new (std::nothrow) qaa_ctx();
  if (!ctx) return QAA_E_CAP;
  *out = ctx;
  memset(&ctx->stats, 0, sizeof ctx->stats);
  ctx->device = cfg->device;
  ctx->rank = cfg->rank;
  ctx->world = cfg->world;
  ctx->gbits = cfg->world == 1 ? 0 : (cfg->world == 2 ? 1 : (cfg->world == 4 ? 2 : 3));
  if (ctx->world > 1) {
    if (!cfg->comm || !cfg->comm->barrier || !cfg->comm->allgather)
      return fail(ctx, QAA_E_USAGE, "world > 1 needs comm callbacks (barrier, allgather)");
    if (cfg->state) return fail(ctx, QAA_E_USAGE, "world > 1: the library owns the shard buffers (state must be NULL)");
    if (cfg->nccl_id) return fail(ctx, QAA_E_USAGE, "nccl_id is reserved and must be NULL");
    ctx->comm = *cfg->comm;
    ctx->has_comm = true;
  }
  CUDA_TRY(cudaSetDevice(cfg->device));
  CUDA_TRY(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cfg->device));
  if (cfg->stream) {
    ctx->stream = (cudaStream_t)cfg->stream;
  } else {
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  if (cfg->state) {
    if (((uintptr_t)cfg->state) % 256 != 0) return fail(ctx, QAA_E_USAGE, "state buffer must be 256-byte aligned");
    ctx->state = (double2*)cfg->state;
    ctx->state_cap_bytes = cfg->state_bytes;
    ctx->own_state = false;
  }
  CUDA_TRY(cudaMalloc(&ctx->d_out, 64 * sizeof(double)));
  CUDA_TRY(cudaMallocHost(&ctx->h_out, 64 * sizeof(double)));
  CUDA_TRY(cudaMalloc(&ctx->d_counters, 16));
  CUDA_TRY(cudaEventCreateWithFlags(&ctx->coef_done, cudaEventDisableTiming));
  CUDA_TRY(pass_kernel_setup());
  CUDA_TRY(pass_fast_setup());
  CUDA_TRY(pass_tma_setup());
  return QAA_OK;
}

void qaa_destroy(qaa_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->own_state && ctx->state) cudaFree(ctx->state);
  if (ctx->E) cudaFree(ctx->E);
  if (ctx->Z) cudaFree(ctx->Z);
  if (ctx->d_coef) cudaFree(ctx->d_coef);
  if (ctx->h_coef) cudaFreeHost(ctx->h_coef);
  if (ctx->d_part) cudaFree(ctx->d_part);
  if (ctx->d_out) cudaFree(ctx->d_out);
  if (ctx->h_out) cudaFreeHost(ctx->h_out);
  if (ctx->d_counters) cudaFree(ctx->d_counters);
  if (ctx->d_super) cudaFree(ctx->d_super);
  if (ctx->clause_recs) cudaFree(ctx->clause_recs);
  for (size_t g = 1; g < ctx->Eg.size(); g++)
    if (ctx->Eg[g]) cudaFree(ctx->Eg[g]);
  for (int b = 0; b < 2; b++) {
    for (int r = 0; r < 8; r++)
      if (ctx->peer_open[b][r]) cudaIpcCloseMemHandle(ctx->peers[b][r]);
    if (ctx->bufs[b]) cudaFree(ctx->bufs[b]);
  }
  if (ctx->E_B) cudaFree(ctx->E_B);
  for (int b = 0; b < 2; b++)
    if (ctx->shard_top_eg[b]) cudaFree(ctx->shard_top_eg[b]);
  if (ctx->coef_done) cudaEventDestroy(ctx->coef_done);
  for (auto& p : ctx->ev_pool) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  cudaGetLastError();
  delete ctx;
}

const char* qaa_last_error(const qaa_ctx* ctx) {
  if (!ctx) return "null context";
  return ctx->err.c_str();
}

qaa_status qaa_set_option(qaa_ctx* ctx, int key, int64_t value) {
  if (!ctx) return QAA_E_USAGE;
  switch (key) {
    case QAA_OPT_ROW_BITS:
      if (value < 1 || value > 5) return fail(ctx, QAA_E_USAGE, "row_bits must be in 1..5, got %lld", (long long)value);
      ctx->row_bits = (int)value;
      ctx->progs.clear();
      if (ctx->loaded && ctx->L > RESIDENT_MAX_L) {
        std::string e;
        if (!build_geometry(ctx->L, ctx->row_bits, &ctx->geom, &e)) return fail(ctx, QAA_E_USAGE, "%s", e.c_str());
      }
      return QAA_OK;
    case QAA_OPT_PROFILE:
      ctx->profile = value != 0;
      return QAA_OK;
    case QAA_OPT_STEP_SPANNING:
      if (value < 0 || value > 2) return fail(ctx, QAA_E_USAGE, "step_spanning must be 0, 1 or 2");
      ctx->step_spanning = (int)value;
      return QAA_OK;
    case QAA_OPT_ENERGY_W64:
      if (value < 0 || value > 1) return fail(ctx, QAA_E_USAGE, "energy_w64 must be 0 or 1");
      ctx->energy_w64 = (int)value;
      return QAA_OK;
    case QAA_OPT_ORDER:
      if (value != 1 && value != 2) return fail(ctx, QAA_E_USAGE, "splitting order must be 1 or 2");
      ctx->order = (int)value;
      return QAA_OK;
    case QAA_OPT_SUPER:
      if (value < 0 || value > 63) return fail(ctx, QAA_E_USAGE, "super option must be in 0..63");
      // bit 0: L2-blocked Trotter steps; bit 1: one consumer group per CTA (default two);
      // bits 2-3: L2 eviction hints (0 = evict-last for the group-0 output that the
      // group-k sub-pass reads back + evict-first for dead data; 1 = none; 2 = evict-first only)
      ctx->super_mode = (int)(value & 1);
      ctx->super_groups = (value & 2) ? 1 : 2;
      ctx->super_force = (value & 16) ? 1 : 0;  // also below SUPER_MIN_CHUNKS (tests)
      ctx->super_dynamic = (value & 32) ? 1 : 0;  // dynamic work queue instead of static round robin
      ctx->super_hints = ((value >> 2) & 3) == 1 ? 0 : (((value >> 2) & 3) == 2 ? 1 : 2);
      return QAA_OK;
    case QAA_OPT_TMA_GROUPS:
      if (value < 0 || value > 2) return fail(ctx, QAA_E_USAGE, "tma groups must be 0 (auto), 1 or 2");
      ctx->tma_groups = (int)value;
      return QAA_OK;
    case QAA_OPT_KERNEL:
      if (value < 0 || value > 2) return fail(ctx, QAA_E_USAGE, "kernel mode must be 0, 1 or 2 (auto)");
      ctx->kernel_mode = (int)value;
      return QAA_OK;
    case QAA_OPT_CTAS_PER_SM:
      if (value < 1 || value > 4) return fail(ctx, QAA_E_USAGE, "ctas_per_sm must be in 1..4");
      ctx->ctas_per_sm = (int)value;
      return QAA_OK;
    default:
      return fail(ctx, QAA_E_USAGE, "unknown option key %d", key);
  }
}

// Per-group TMA descriptors and permuted energy tables (pass_tma.cu).
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    cudaGetLastError();
  }
  return fn;
}

// Tile-group geometry for the TMA kernels: t (contiguous flag, tensor-map
// dims -> tile-id segments) and, for strided groups, the <= 5-D tensor map of
// 128-byte rows over the state at `base`. Returns false if not expressible.
static bool encode_group(qaa_ctx* ctx, const Group& gr, void* base, CUtensorMap* mapp, TmaArgs* tp) {
  const int L = ctx->L;
  auto enc = tensor_map_encoder();
  TmaArgs& t = *tp;
  CUtensorMap& map = *mapp;
  memset(&t, 0, sizeof t);
  memset(&map, 0, sizeof map);
  bool ok = true;
  bool in_tile[64] = {false};
  for (int b = 0; b < TILE_BITS; b++) in_tile[gr.phys[b]] = true;
  bool contiguous = true;
  for (int b = 0; b < TILE_BITS; b++) contiguous = contiguous && gr.phys[b] == b;
  t.contiguous = contiguous ? 1 : 0;
  if (!contiguous) {
    // dims: runs of tile bits (split to box-size limits) and gap runs (box 1)
    cuuint64_t gdim[5], gstride[5];
    cuuint32_t box[5], estr[5];
    int nd = 0, gap_index = 0;
    for (int p = 0; p < L && ok;) {
      int q = p;
      while (q + 1 < L && in_tile[q + 1] == in_tile[p]) q++;
      int bits = q - p + 1;
      if (in_tile[p]) {
        int start = p;
        while (bits > 0 && ok) {
          const int lim = nd == 0 ? 7 : 8;
          const int take = bits < lim ? bits : lim;
          if (nd >= 5) { ok = false; break; }
          gdim[nd] = (cuuint64_t)1 << (take + (nd == 0 ? 1 : 0));
          box[nd] = (cuuint32_t)gdim[nd];
          gstride[nd] = (cuuint64_t)16 << start;
          t.dim_seg[nd] = -1;
          nd++;
          start += take;
          bits -= take;
        }
      } else {
        if (nd >= 5 || nd == 0) { ok = false; break; }
        gdim[nd] = (cuuint64_t)1 << bits;
        box[nd] = 1;
        gstride[nd] = (cuuint64_t)16 << p;
        t.dim_seg[nd] = gap_index++;
        nd++;
      }
      p = q + 1;
    }
    if (ok && enc) {
      for (int d = 0; d < nd; d++) estr[d] = 1;
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)nd, base, gdim, gstride + 1,
                       box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      ok = r == CUDA_SUCCESS;
    } else {
      ok = false;
    }
    t.ndims = nd;
  }
  return ok;
}

// Chunk geometry of the L2-blocked pair (group 0, group k): a chunk fixes every
// physical bit outside both groups' tile bits; false if the two sub-passes do
// not have the same number of tiles per chunk or k rotates a row bit.
static bool make_super_args(qaa_ctx* ctx, int k, const TmaArgs& t0, const TmaArgs& tk, SuperArgs* out) {
  const int L = ctx->L;
  const Group& g0 = ctx->geom.groups[0];
  const Group& gk = ctx->geom.groups[(size_t)k];
  if (gk.rot_local & ~0xFF8u) return false;
  bool in0[64] = {false}, ink[64] = {false};
  for (int b = 0; b < TILE_BITS; b++) {
    in0[g0.phys[b]] = true;
    ink[gk.phys[b]] = true;
  }
  SuperArgs sa;
  memset(&sa, 0, sizeof sa);
  // group-k tile-id bits = its non-tile bits in ascending physical order
  int bit = 0;
  for (int p = 0; p < L; p++) {
    if (ink[p]) continue;
    if (in0[p]) sa.k_imask |= 1u << bit;
    else sa.k_cmask |= 1u << bit;
    bit++;
  }
  bit = 0;
  for (int p = 0; p < L; p++) {
    if (in0[p]) continue;
    if (ink[p]) sa.z_imask |= 1u << bit;
    else sa.z_cmask |= 1u << bit;
    bit++;
  }
  const int ik = __builtin_popcount(sa.k_imask), iz = __builtin_popcount(sa.z_imask);
  const int cb = __builtin_popcount(sa.k_cmask);
  if (ik != iz || cb != __builtin_popcount(sa.z_cmask)) return false;
  sa.tpc_bits = ik;
  sa.nchunks = (int64_t)1 << cb;
  sa.gk = tk;
  sa.g0 = t0;
  *out = sa;
  return true;
}

// Sharded plan with three local tile groups: the pass pair [group 0 rotate]
// [group 1 rotate + layout-swap stores] of every phase runs as one L2-blocked
// launch (pass_tma.cu qaa_superpass without D, remote group-k stores). Needs
// group 1's tensor map over both shard buffers.
// Sharded top group (rotate carried bits, D, rotate all) on the TMA kernel:
// its tensor map over both shard buffers and its energy slices permuted from
// the layout-A and layout-B tables. Falls back to the register kernel if a map
// cannot be encoded or the tables do not fit.
static qaa_status build_shard_top(qaa_ctx* ctx) {
  ctx->shard_top_ok = false;
  const int P = (int)ctx->geom.groups.size();
  if (P < 2 || !ctx->bufs[0] || !ctx->bufs[1] || !ctx->E_B) return QAA_OK;
  const Group& gt = ctx->geom.groups[(size_t)P - 1];
  if (gt.rot_local & ~0xFF8u) return QAA_OK;
  TmaArgs tb[2];
  for (int b = 0; b < 2; b++)
    if (!encode_group(ctx, gt, ctx->bufs[b], &ctx->shard_top_map[b], &tb[b]) || tb[b].contiguous) return QAA_OK;
  const size_t N = (size_t)1 << ctx->L;
  if (ctx->shard_top_eg_cap < N) {
    for (int b = 0; b < 2; b++) {
      if (ctx->shard_top_eg[b]) cudaFree(ctx->shard_top_eg[b]);
      ctx->shard_top_eg[b] = nullptr;
    }
    ctx->shard_top_eg_cap = 0;
    for (int b = 0; b < 2; b++)
      if (cudaMalloc(&ctx->shard_top_eg[b], N) != cudaSuccess) {
        cudaGetLastError();
        return QAA_OK;  // register-kernel fallback
      }
    ctx->shard_top_eg_cap = N;
  }
  for (int b = 0; b < 2; b++) {
    CUDA_TRY(launch_permute_energy(b ? ctx->E_B : ctx->E, ctx->shard_top_eg[b], gt.phys, gt.nseg, gt.seg_src,
                                   gt.seg_dst, gt.seg_len, gt.ntiles, (gt.rot_local >> 3) & 1, ctx->num_sms,
                                   ctx->stream));
    ctx->stats.kernel_launches_total++;
  }
  ctx->shard_top = tb[0];
  ctx->shard_top_ok = true;
  return QAA_OK;
}

static void build_shard_super(qaa_ctx* ctx) {
  ctx->shard_super_ok = false;
  const int P = (int)ctx->geom.groups.size();
  if (P < 3 || !ctx->bufs[0] || !ctx->bufs[1]) return;
  const int k = P - 2;  // the remote (layout-swap) group, right after group 0 in every phase
  TmaArgs t0, tkb[2];
  CUtensorMap m0;
  if (!encode_group(ctx, ctx->geom.groups[0], ctx->bufs[0], &m0, &t0) || !t0.contiguous) return;
  for (int b = 0; b < 2; b++)
    if (!encode_group(ctx, ctx->geom.groups[(size_t)k], ctx->bufs[b], &ctx->shard_kmap[b], &tkb[b])) return;
  if (!make_super_args(ctx, k, t0, tkb[0], &ctx->shard_super)) return;
  ctx->shard_super_ok = true;
}

static qaa_status build_tma(qaa_ctx* ctx) {
  // the permuted tables of the previous load are reused when big enough (a
  // 1 GiB cudaFree/cudaMalloc pair per load costs more than the permutation)
  std::vector<uint8_t*> old_eg = ctx->Eg;
  std::vector<size_t> old_cap = ctx->Eg_cap;
  auto release_old = [&]() {
    for (size_t g = 1; g < old_eg.size(); g++)
      if (old_eg[g]) cudaFree(old_eg[g]);
  };
  ctx->Eg.clear();
  ctx->Eg_cap.clear();
  ctx->tmaps.clear();
  ctx->tma_static.clear();
  ctx->tma_ok.clear();
  if (ctx->L <= RESIDENT_MAX_L) {
    release_old();
    return QAA_OK;
  }
  const int L = ctx->L;
  const size_t N = (size_t)1 << L;
  for (size_t gi = 0; gi < ctx->geom.groups.size(); gi++) {
    const Group& gr = ctx->geom.groups[gi];
    TmaArgs t;
    CUtensorMap map;
    bool ok = encode_group(ctx, gr, (void*)ctx->state, &map, &t);
    // permuted energies
    uint8_t* eg = nullptr;
    if (gi == 0) {
      eg = ctx->E;
    } else if (ok) {
      cudaError_t e = cudaSuccess;
      if (gi < old_eg.size() && old_eg[gi] && old_cap[gi] >= N) {
        eg = old_eg[gi];
        old_eg[gi] = nullptr;  // taken over
      } else {
        e = cudaMalloc(&eg, N);
      }
      if (e != cudaSuccess) {
        cudaGetLastError();
        eg = nullptr;
        ok = false;  // not enough memory for the permuted table: register kernel fallback
      } else {
        CUDA_TRY(launch_permute_energy(ctx->E, eg, gr.phys, gr.nseg, gr.seg_src, gr.seg_dst, gr.seg_len, gr.ntiles,
                                       (gr.rot_local >> 3) & 1, ctx->num_sms, ctx->stream));
        ctx->stats.kernel_launches_total++;
      }
    }
    t.Eg = eg;
    ctx->Eg.push_back(eg);
    ctx->Eg_cap.push_back(gi == 0 || !eg ? 0 : N);
    ctx->tmaps.push_back(map);
    ctx->tma_static.push_back(t);
    ctx->tma_ok.push_back(ok ? 1 : 0);
  }
  release_old();
  // L2-blocked D passes pair group 0 with group k (k = 1, 2) on chunks that fix
  // every physical bit outside their tile bits (pass_tma.cu qaa_superpass)
  for (int k = 0; k < 4; k++) ctx->super_ok[k] = false;
  const int P = (int)ctx->geom.groups.size();
  if ((P == 3 || P == 4) && ctx->tma_ok[0])
    for (int k = 1; k < P; k++)
      if (ctx->tma_ok[(size_t)k] &&
          make_super_args(ctx, k, ctx->tma_static[0], ctx->tma_static[(size_t)k], &ctx->super_static[k]))
        ctx->super_ok[k] = true;
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return QAA_OK;
}

// ------------------------------------------------------------------ sharding helpers
static qaa_status comm_barrier(qaa_ctx* ctx) {
  if (ctx->comm.barrier(ctx->comm.user) != 0) return fail(ctx, QAA_E_NCCL, "comm barrier failed");
  return QAA_OK;
}
static qaa_status comm_allgather(qaa_ctx* ctx, const void* send, void* recv, size_t bytes) {
  if (ctx->comm.allgather(ctx->comm.user, send, recv, bytes) != 0) return fail(ctx, QAA_E_NCCL, "comm allgather failed");
  return QAA_OK;
}
// sum of `n` doubles over ranks, added in rank order (deterministic)
static qaa_status comm_sum(qaa_ctx* ctx, double* v, int n) {
  if (ctx->world == 1) return QAA_OK;
  std::vector<double> all((size_t)n * ctx->world);
  qaa_status st = comm_allgather(ctx, v, all.data(), sizeof(double) * (size_t)n);
  if (st) return st;
  for (int j = 0; j < n; j++) {
    double s = 0.0;
    for (int r = 0; r < ctx->world; r++) s += all[(size_t)r * n + j];
    v[j] = s;
  }
  return QAA_OK;
}

// Two shard buffers per rank, exported with CUDA IPC; every rank maps every
// other rank's buffers so the layout-swap pass can store into them directly
// (NVLink/NVSwitch peer stores across GPUs, plain stores on one GPU).
static qaa_status setup_shard_buffers(qaa_ctx* ctx, size_t bytes) {
  if (ctx->buf_cap >= bytes && ctx->bufs[0]) {
    ctx->state = ctx->bufs[ctx->cur = 0];
    return QAA_OK;
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  for (int b = 0; b < 2; b++) {
    for (int r = 0; r < 8; r++) {
      if (ctx->peer_open[b][r]) cudaIpcCloseMemHandle(ctx->peers[b][r]);
      ctx->peer_open[b][r] = false;
      ctx->peers[b][r] = nullptr;
    }
    if (ctx->bufs[b]) cudaFree(ctx->bufs[b]);
    ctx->bufs[b] = nullptr;
  }
  ctx->buf_cap = 0;
  for (int b = 0; b < 2; b++) {
    cudaError_t e = cudaMalloc(&ctx->bufs[b], bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, QAA_E_CAP, "shard buffers of 2 x %zu bytes do not fit on the device", bytes);
    }
  }
  ctx->buf_cap = bytes;
  cudaIpcMemHandle_t mine[2];
  for (int b = 0; b < 2; b++) CUDA_TRY(cudaIpcGetMemHandle(&mine[b], ctx->bufs[b]));
  std::vector<cudaIpcMemHandle_t> all(2 * (size_t)ctx->world);
  qaa_status st = comm_allgather(ctx, mine, all.data(), sizeof mine);
  if (st) return st;
  for (int r = 0; r < ctx->world; r++)
    for (int b = 0; b < 2; b++) {
      if (r == ctx->rank) {
        ctx->peers[b][r] = ctx->bufs[b];
        continue;
      }
      void* p = nullptr;
      CUDA_TRY(cudaIpcOpenMemHandle(&p, all[2 * (size_t)r + b], cudaIpcMemLazyEnablePeerAccess));
      ctx->peers[b][r] = (double2*)p;
      ctx->peer_open[b][r] = true;
    }
  st = comm_barrier(ctx);
  if (st) return st;
  ctx->cur = 0;
  ctx->state = ctx->bufs[0];
  ctx->own_state = false;
  ctx->state_cap_bytes = bytes;
  return QAA_OK;
}

// one layout swap (A <-> B) of the whole sharded state: stores, barrier, flip
static qaa_status shard_remap(qaa_ctx* ctx) {
  CUDA_TRY(launch_remap(ctx->bufs[ctx->cur], ctx->peers[ctx->cur ^ 1], (int64_t)1 << ctx->L, ctx->L - ctx->gbits,
                        ctx->rank, ctx->num_sms, ctx->stream));
  ctx->stats.kernel_launches_total++;
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  qaa_status st = comm_barrier(ctx);
  if (st) return st;
  ctx->cur ^= 1;
  ctx->state = ctx->bufs[ctx->cur];
  return QAA_OK;
}

qaa_status qaa_load_instance(qaa_ctx* ctx, int n, int m, const int32_t* lits) {
  CHECK_CTX();
  if (n < 1 || n > 40) return fail(ctx, QAA_E_USAGE, "n must be in 1..40, got %d", n);
  if (m < 0) return fail(ctx, QAA_E_USAGE, "m must be >= 0, got %d", m);
  if (m > 0 && !lits) return fail(ctx, QAA_E_USAGE, "lits is NULL with m = %d", m);
  const int L = n - ctx->gbits;
  if (L < 1) return fail(ctx, QAA_E_USAGE, "n = %d too small for world = %d", n, ctx->world);
  for (int i = 0; i < 3 * m; i++)
    if (lits[i] == 0 || lits[i] > n || lits[i] < -n)
      return fail(ctx, QAA_E_INPUT, "literal %d of clause %d is %d, outside +-(1..%d)", i % 3, i / 3, lits[i], n);
  if (m > 255) return fail(ctx, QAA_E_CAP, "m = %d exceeds 255 (uint8 energy table)", m);
  // encode clauses (A1): violated iff (x & M) == V; drop tautologies.
  std::vector<ClauseRecHost> recs;
  for (int c = 0; c < m; c++) {
    uint64_t M = 0, V = 0;
    bool taut = false;
    for (int j = 0; j < 3; j++) {
      const int l = lits[3 * c + j];
      const uint64_t bit = 1ull << ((l > 0 ? l : -l) - 1);
      const uint64_t want = l > 0 ? 0 : bit;  // value of x_|l| that makes the literal false
      if ((M & bit) && ((V & bit) != want)) taut = true;
      M |= bit;
      V |= want;
    }
    if (taut) continue;
    ClauseRecHost r;
    r.mhi = M & ~15ull;
    r.vhi = V & ~15ull;
    memset(r.spread, 0, sizeof r.spread);
    for (int i = 0; i < 16; i++)
      if (((uint64_t)i & M & 15ull) == (V & 15ull)) r.spread[i >> 2] |= 1u << (8 * (i & 3));
    recs.push_back(r);
  }
  const int64_t N = (int64_t)1 << L;
  const size_t state_bytes = (size_t)N * sizeof(double2);
  // capacity
  if (ctx->world > 1) {
    Geometry gtest;
    std::string e;
    std::vector<ShardPass> sp;
    if (L <= RESIDENT_MAX_L || !build_geometry(L, ctx->row_bits, &gtest, &e) ||
        !build_shard_schedule(gtest, ctx->gbits, 1, &sp, &e))
      return fail(ctx, QAA_E_CAP, "n = %d cannot be sharded over %d ranks: %s", n, ctx->world,
                  e.empty() ? "n - log2(world) must be >= 13" : e.c_str());
    qaa_status st = setup_shard_buffers(ctx, state_bytes);
    if (st) return st;
  } else if (!ctx->own_state && ctx->state) {
    if (ctx->state_cap_bytes < state_bytes)
      return fail(ctx, QAA_E_CAP, "caller state buffer holds %zu bytes, need %zu for n = %d", ctx->state_cap_bytes,
                  state_bytes, n);
  } else {
    if (ctx->state_cap_bytes < state_bytes) {
      if (ctx->state) cudaFree(ctx->state);
      ctx->state = nullptr;
      ctx->state_cap_bytes = 0;
      void* p = nullptr;
      qaa_status st = ensure_buffer(ctx, &p, &ctx->state_cap_bytes, state_bytes);
      if (st) return fail(ctx, QAA_E_CAP, "state of %zu bytes (n = %d) does not fit on the device", state_bytes, n);
      ctx->state = (double2*)p;
      ctx->own_state = true;
    }
  }
  {
    void* p = ctx->E;
    qaa_status st = ensure_buffer(ctx, &p, &ctx->E_cap, std::max<size_t>((size_t)N, 16));
    ctx->E = (uint8_t*)p;
    if (st) return st;
  }
  ctx->loaded = false;
  ctx->initialized = false;
  ctx->n = n;
  ctx->L = L;
  ctx->m = m;
  if (L > RESIDENT_MAX_L) {
    std::string e;
    if (!build_geometry(L, ctx->row_bits, &ctx->geom, &e)) return fail(ctx, QAA_E_USAGE, "%s", e.c_str());
  } else {
    ctx->geom = Geometry();
  }
  ctx->progs.clear();
  // clause records to device (kept for qaa_time_energy_table)
  const size_t rec_bytes = std::max<size_t>(recs.size(), 1) * sizeof(ClauseRecHost);
  {
    qaa_status st = ensure_buffer(ctx, &ctx->clause_recs, &ctx->clause_recs_cap, rec_bytes);
    if (st) return st;
  }
  if (ctx->coef_pending) CUDA_TRY(cudaEventSynchronize(ctx->coef_done));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (!recs.empty())
    CUDA_TRY(cudaMemcpyAsync(ctx->clause_recs, recs.data(), rec_bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->n_recs = (int)recs.size();
  CUDA_TRY(cudaMemsetAsync(ctx->d_counters, 0, 16, ctx->stream));
  const uint64_t x_offset = (uint64_t)ctx->rank << L;
  CUDA_TRY(launch_energy_table(ctx->E, N, x_offset, (const uint64_t*)ctx->clause_recs, (int)recs.size(), ctx->d_counters,
                               (unsigned long long*)(ctx->d_counters + 2), ctx->num_sms, ctx->stream, 63, 0,
                               ctx->energy_w64 != 0));
  ctx->stats.kernel_launches_total++;
  unsigned hc[4];
  CUDA_TRY(cudaMemcpyAsync(hc, ctx->d_counters, 16, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  ctx->emax = hc[0];
  uint64_t zeros;
  memcpy(&zeros, &hc[2], 8);
  ctx->nz_local = (int64_t)zeros;
  ctx->nz_total = zeros;
  ctx->z_listed = false;
  if (ctx->world > 1) {
    // layout-B energies: local p -> x = (p mod 2^(L-g)) | r 2^(L-g) | (p >> (L-g)) 2^L
    void* p = ctx->E_B;
    qaa_status st = ensure_buffer(ctx, &p, &ctx->E_B_cap, (size_t)N);
    ctx->E_B = (uint8_t*)p;
    if (st) return st;
    CUDA_TRY(launch_energy_table(ctx->E_B, N, (uint64_t)ctx->rank << (L - ctx->gbits), (const uint64_t*)ctx->clause_recs,
                                 (int)recs.size(), ctx->d_counters, (unsigned long long*)(ctx->d_counters + 2),
                                 ctx->num_sms, ctx->stream, L - ctx->gbits, L, ctx->energy_w64 != 0));
    ctx->stats.kernel_launches_total++;
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    // global |Z| and max E over ranks
    uint64_t mine[2] = {zeros, (uint64_t)ctx->emax};
    std::vector<uint64_t> all(2 * (size_t)ctx->world);
    qaa_status st2 = comm_allgather(ctx, mine, all.data(), sizeof mine);
    if (st2) return st2;
    ctx->nz_total = 0;
    ctx->emax = 0;
    for (int r = 0; r < ctx->world; r++) {
      ctx->nz_total += all[2 * (size_t)r];
      ctx->emax = std::max<unsigned>(ctx->emax, (unsigned)all[2 * (size_t)r + 1]);
    }
  }
  if (ctx->nz_local > 0 && ctx->nz_local <= ZLIST_CAP) {
    void* p = ctx->Z;
    qaa_status st = ensure_buffer(ctx, &p, &ctx->Z_cap, (size_t)ctx->nz_local * 8);
    ctx->Z = (uint64_t*)p;
    if (st) return st;
    CUDA_TRY(cudaMemsetAsync(ctx->d_counters, 0, 16, ctx->stream));
    CUDA_TRY(launch_compact_zeros(ctx->E, N, x_offset, ctx->Z, (unsigned long long*)(ctx->d_counters + 2),
                                  ctx->num_sms, ctx->stream));
    ctx->stats.kernel_launches_total++;
    std::vector<uint64_t> hz((size_t)ctx->nz_local);
    CUDA_TRY(cudaMemcpyAsync(hz.data(), ctx->Z, hz.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    std::sort(hz.begin(), hz.end());  // fixed order => deterministic gather sum
    CUDA_TRY(cudaMemcpyAsync(ctx->Z, hz.data(), hz.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    ctx->z_listed = true;
  }
  if (ctx->world == 1) {
    qaa_status st = build_tma(ctx);
    if (st) return st;
  } else {
    build_shard_super(ctx);
    qaa_status st = build_shard_top(ctx);
    if (st) return st;
  }
  ctx->loaded = true;
  return QAA_OK;
}

qaa_status qaa_init_uniform(qaa_ctx* ctx) {
  CHECK_CTX();
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "init_uniform before load_instance");
  const double a = 1.0 / std::sqrt(std::ldexp(1.0, ctx->n));
  CUDA_TRY(launch_fill(ctx->state, (int64_t)1 << ctx->L, a, 0.0, ctx->num_sms, ctx->stream));
  ctx->stats.kernel_launches_total++;
  ctx->initialized = true;
  return QAA_OK;
}

qaa_status qaa_init_basis(qaa_ctx* ctx, uint64_t x) {
  CHECK_CTX();
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "init_basis before load_instance");
  if (ctx->n < 64 && x >= (1ull << ctx->n)) return fail(ctx, QAA_E_USAGE, "basis index %llu >= 2^n", (unsigned long long)x);
  CUDA_TRY(launch_fill(ctx->state, (int64_t)1 << ctx->L, 0.0, 0.0, ctx->num_sms, ctx->stream));
  ctx->stats.kernel_launches_total++;
  if ((int)(x >> ctx->L) == ctx->rank) {
    CUDA_TRY(launch_set_one(ctx->state, (int64_t)(x & ((1ull << ctx->L) - 1)), ctx->stream));
    ctx->stats.kernel_launches_total++;
  }
  ctx->initialized = true;
  return QAA_OK;
}

// H1: per-step coefficients (host, binary64 libm; R11).
namespace {
struct StepCoef {
  double coef;
  int form;
};
}  // namespace

// Weights of H_B and H_P at s: Eq. 1 gives (1 - s, s); the optional driving
// term s(1-s)(g_x H_B + g_z H_P) (NEXT F4, R3) adds s(1-s) g to each. With
// g = 0 both are bit-identical to 1 - s and s.
static double weight_b(const qaa_ctx* c, double s) { return (1.0 - s) + c->drv_x * s * (1.0 - s); }
static double weight_p(const qaa_ctx* c, double s) { return s + c->drv_z * s * (1.0 - s); }

// One row of the coefficient table: the X coefficient of a step whose H_B
// weight is wb (tan or cot of beta = dt wb / 2) and Phi[e] = e^{-i theta e} *
// (X normalisation)^n. theta is dt wP(s) for Lie-Trotter; Strang passes the
// merged half steps (R7, §4).
static void build_step(double T, int64_t K, double wb, double theta, int n, int n_phi, double2* phi_row,
                       StepCoef* sc) {
  const double dt = T / (double)K;
  const double beta = 0.5 * dt * wb;  // X: exp(-i beta (1 - sigma^x)) per qubit
  const double cb = std::cos(beta), sb = std::sin(beta);
  double mag;
  // tangent form (I + i t sigma^x), t = tan beta, whenever |t| <= 1e4: it is a
  // scaled unitary, so rounding stays relative to |psi| for any such t; only
  // beta within ~1e-4 of pi/2 (mod pi) switches to the cot form.
  if (std::fabs(sb) <= 1e4 * std::fabs(cb)) {
    sc->form = 0;
    sc->coef = sb / cb;  // tan beta
    mag = cb;
  } else {
    sc->form = 1;
    sc->coef = cb / sb;  // cot beta
    mag = sb;
  }
  const double scale = std::pow(mag, (double)n);  // |(g cos b)^n| (or sin)
  const double nb = (double)n * beta;             // arg of g^n = -n beta
  for (int e = 0; e < n_phi; e++) {
    const double ang = theta * (double)e + nb;
    phi_row[e] = make_double2(scale * std::cos(ang), -scale * std::sin(ang));
  }
}

static qaa_status ensure_events(qaa_ctx* ctx, size_t need) {
  while (ctx->ev_pool.size() < need) {
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreate(&a));
    CUDA_TRY(cudaEventCreate(&b));
    ctx->ev_pool.push_back({a, b});
  }
  return QAA_OK;
}

// Sharded evolve (plan.hpp ShardPass): every phase ends with a
// pass whose tiles are stored straight into the peers' other shard buffer
// (the bit swap of the top local and the rank qubits), then one host barrier.
// Pass-kernel choice. Auto: the register-prefetch kernel while the state is
// small enough for a pass to be latency-bound (L <= 19: a few dozen tiles, the
// LDG path has the shorter tile latency, measured 30 % faster at n = 13..19),
// the TMA kernels above (n = 23..27: 20-30 % faster; the L2-blocked step from 28).
constexpr int AUTO_REGISTER_MAX_L = 19;
static bool use_tma(const qaa_ctx* ctx) {
  return ctx->kernel_mode == 1 || (ctx->kernel_mode == 2 && ctx->L > AUTO_REGISTER_MAX_L);
}

static qaa_status evolve_sharded(qaa_ctx* ctx, int64_t K, const std::vector<StepCoef>& sc, const double2* dphi,
                                 int n_phi) {
  for (int64_t k = 0; k < K; k++)
    if (sc[(size_t)k].form != 0)
      return fail(ctx, QAA_E_USAGE, "sharded evolve needs |tan(dt(1-s)/2)| <= 1e4 (step %lld)", (long long)k);
  std::vector<ShardPass> plan;
  std::string e;
  if (!build_shard_schedule(ctx->geom, ctx->gbits, K, &plan, &e)) return fail(ctx, QAA_E_CAP, "%s", e.c_str());
  if (ctx->profile) {
    qaa_status st = ensure_events(ctx, ctx->ev_used + plan.size());
    if (st) return st;
  }
  const int P = (int)ctx->geom.groups.size();
  FastArgs fa;
  memset(&fa, 0, sizeof fa);
  fa.n_phi = n_phi;
  fa.gshift = ctx->L - ctx->gbits;
  fa.rank = ctx->rank;
  const bool fuse = ctx->shard_super_ok && ctx->super_mode && use_tma(ctx) &&
                    (ctx->super_force || ctx->shard_super.nchunks >= SUPER_MIN_CHUNKS);
  for (size_t pi = 0; pi < plan.size(); pi++) {
    const ShardPass& sp = plan[pi];
    if (sp.kind == SK_REMAP) {
      qaa_status st = shard_remap(ctx);
      if (st) return st;
      continue;
    }
    if (fuse && pi + 1 < plan.size()) {
      // [group 0: rotate][group 1: rotate + layout-swap stores] -> one L2-blocked launch
      const ShardPass& sn = plan[pi + 1];
      if (sp.kind == SK_PASS && sp.group == 0 && sp.pre_step >= 0 && sp.d_step < 0 && sp.post_step < 0 &&
          !sp.remote && sn.kind == SK_PASS && sn.group == P - 2 && sn.pre_step >= 0 && sn.d_step < 0 &&
          sn.post_step < 0 && sn.remote && sn.layout == sp.layout) {
        SuperArgs a = ctx->shard_super;
        const Group& g0 = ctx->geom.groups[0];
        const Group& g1 = ctx->geom.groups[(size_t)(P - 2)];
        a.g0.psi = ctx->bufs[ctx->cur];
        a.gk.psi = ctx->bufs[ctx->cur];
        a.gk.phi = nullptr;
        a.gk.n_phi = n_phi;
        for (int b = 0; b < TILE_BITS; b++) {
          a.g0.t[0][b] = ((sp.pre_local >> b) & 1) ? sc[(size_t)sp.pre_step].coef : 0.0;
          a.g0.t[1][b] = 0.0;
          a.g0.phys[b] = g0.phys[b];
          a.gk.t[0][b] = ((sn.pre_local >> b) & 1) ? sc[(size_t)sn.pre_step].coef : 0.0;
          a.gk.t[1][b] = 0.0;
          a.gk.phys[b] = g1.phys[b];
        }
        a.g0.ntiles = g0.ntiles;
        a.gk.ntiles = g1.ntiles;
        a.g0.nseg = g0.nseg;
        a.gk.nseg = g1.nseg;
        for (int q = 0; q < MAX_SEGS; q++) {
          a.g0.seg_src[q] = g0.seg_src[q];
          a.g0.seg_dst[q] = g0.seg_dst[q];
          a.g0.seg_len[q] = g0.seg_len[q];
          a.gk.seg_src[q] = g1.seg_src[q];
          a.gk.seg_dst[q] = g1.seg_dst[q];
          a.gk.seg_len[q] = g1.seg_len[q];
        }
        a.hints = ctx->super_hints;
        a.remote = 1;
        a.gshift = ctx->L - ctx->gbits;
        a.rank = ctx->rank;
        for (int r = 0; r < 8; r++) a.peers[r] = ctx->peers[ctx->cur ^ 1][r];
        const size_t need = (size_t)a.nchunks * sizeof(unsigned) + 256;
        if (ctx->d_super_cap < need) {
          CUDA_TRY(cudaStreamSynchronize(ctx->stream));
          qaa_status st = ensure_buffer(ctx, &ctx->d_super, &ctx->d_super_cap, need);
          if (st) return st;
        }
        a.queue = ctx->super_dynamic ? (unsigned long long*)ctx->d_super : nullptr;
        a.done = (unsigned*)((char*)ctx->d_super + 256);
        CUDA_TRY(cudaMemsetAsync(ctx->d_super, 0, need, ctx->stream));
        if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].first, ctx->stream));
        CUDA_TRY(launch_superpass(&ctx->shard_kmap[ctx->cur], a, (g1.rot_local >> 3) & 1, ctx->super_groups, false,
                                  ctx->num_sms, ctx->stream));
        if (ctx->profile) {
          CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].second, ctx->stream));
          if (ctx->ev_super.size() < ctx->ev_pool.size()) ctx->ev_super.resize(ctx->ev_pool.size(), 0);
          ctx->ev_super[ctx->ev_used] = 1;
          ctx->ev_used++;
        }
        ctx->stats.pass_launches++;
        ctx->stats.super_launches++;
        ctx->stats.kernel_launches_total++;
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        qaa_status st = comm_barrier(ctx);
        if (st) return st;
        ctx->cur ^= 1;
        ctx->state = ctx->bufs[ctx->cur];
        pi++;
        continue;
      }
    }
    const Group& gr = ctx->geom.groups[(size_t)sp.group];
    const bool d = sp.d_step >= 0;
    int fp;
    if (sp.group == 0)
      fp = FP_G0_PRE;  // group 0 never carries D in the sharded plan
    else
      fp = d ? FP_GK_PRE_D_POST : FP_GK_PRE;
    if (sp.group == 0 && (d || sp.post_step >= 0)) return fail(ctx, QAA_E_USAGE, "internal: unexpected shard pass");
    if (sp.group > 0 && (gr.rot_local & ~0xFF8u)) return fail(ctx, QAA_E_USAGE, "sharded plan needs row_bits >= 3");
    if (d && sp.group == P - 1 && !sp.remote && ctx->shard_top_ok && use_tma(ctx) &&
        n_phi <= TMA_MAX_PHI) {
      // top group: carried bits of step k-1, D_k, all its bits of step k -- TMA kernel
      TmaArgs ta = ctx->shard_top;
      ta.psi = ctx->bufs[ctx->cur];
      ta.Eg = ctx->shard_top_eg[sp.layout];
      ta.phi = dphi + (size_t)sp.d_step * n_phi;
      ta.n_phi = n_phi;
      for (int b = 0; b < TILE_BITS; b++) {
        ta.t[0][b] = (sp.pre_step >= 0 && ((sp.pre_local >> b) & 1)) ? sc[(size_t)sp.pre_step].coef : 0.0;
        ta.t[1][b] = (sp.post_step >= 0 && ((sp.post_local >> b) & 1)) ? sc[(size_t)sp.post_step].coef : 0.0;
        ta.phys[b] = gr.phys[b];
      }
      ta.ntiles = gr.ntiles;
      ta.nseg = gr.nseg;
      for (int q = 0; q < MAX_SEGS; q++) {
        ta.seg_src[q] = gr.seg_src[q];
        ta.seg_dst[q] = gr.seg_dst[q];
        ta.seg_len[q] = gr.seg_len[q];
      }
      const int tgrid = (int)std::min<int64_t>(gr.ntiles / 2, ctx->num_sms);
      if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].first, ctx->stream));
      CUDA_TRY(launch_pass_tma(&ctx->shard_top_map[ctx->cur], ta, FP_GK_PRE_D_POST, (gr.rot_local >> 3) & 1,
                               ctx->tma_groups ? ctx->tma_groups : 2, tgrid, ctx->stream));
      if (ctx->profile) {
        CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].second, ctx->stream));
        ctx->ev_used++;
      }
      ctx->stats.pass_launches++;
      ctx->stats.kernel_launches_total++;
      continue;
    }
    fa.psi = ctx->bufs[ctx->cur];
    fa.E = sp.layout ? ctx->E_B : ctx->E;
    fa.phi = d ? dphi + (size_t)sp.d_step * n_phi : nullptr;
    for (int b = 0; b < TILE_BITS; b++) {
      fa.t[0][b] = (sp.pre_step >= 0 && ((sp.pre_local >> b) & 1)) ? sc[(size_t)sp.pre_step].coef : 0.0;
      fa.t[1][b] = (sp.post_step >= 0 && ((sp.post_local >> b) & 1)) ? sc[(size_t)sp.post_step].coef : 0.0;
      fa.phys[b] = gr.phys[b];
    }
    fa.ntiles = gr.ntiles;
    fa.nseg = gr.nseg;
    for (int s = 0; s < gr.nseg; s++) {
      fa.seg_src[s] = gr.seg_src[s];
      fa.seg_dst[s] = gr.seg_dst[s];
      fa.seg_len[s] = gr.seg_len[s];
    }
    fa.remote = sp.remote;
    for (int r = 0; r < 8; r++) fa.peers[r] = ctx->peers[ctx->cur ^ 1][r];
    const int grid = (int)std::min<int64_t>(gr.ntiles, ctx->num_sms);
    const bool lane3 = ((sp.pre_local | sp.post_local | gr.rot_local) >> 3) & 1;
    if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].first, ctx->stream));
    CUDA_TRY(launch_pass_fast(fa, fp, lane3, true, grid, ctx->stream));
    if (ctx->profile) {
      CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].second, ctx->stream));
      ctx->ev_used++;
    }
    ctx->stats.pass_launches++;
    ctx->stats.kernel_launches_total++;
    if (sp.remote) {
      CUDA_TRY(cudaStreamSynchronize(ctx->stream));
      qaa_status st = comm_barrier(ctx);
      if (st) return st;
      ctx->cur ^= 1;
      ctx->state = ctx->bufs[ctx->cur];
    }
  }
  (void)P;
  return QAA_OK;
}

// L2-blocked Trotter steps (pass_tma.cu qaa_superpass). The schedule-mode-2
// plan with 3 tile groups is, after its first pass, a sequence of pass pairs
//   [group 0: rotate step j] [group k: rotate step j, D_{j+1}, rotate step j+1]
// (k alternating 1, 2); each pair becomes ONE launch over L2-resident chunks,
// so every Trotter step but the first and last is one HBM round trip.
// Three tile groups (n <= 30 on one GPU): every pass pair [group 0][group k
// rotate/D/rotate] fuses. Four groups (n = 31..33): per step [group 0] [group b]
// [group a rotate/D/rotate]; the plain pair [group 0][group b] fuses (the
// kernel variant without D), so a step is two HBM round trips instead of three.
static bool super_usable(qaa_ctx* ctx) {
  const size_t P = ctx->geom.groups.size();
  if (!(ctx->super_mode && ctx->world == 1 && use_tma(ctx) && (P == 3 || P == 4) &&
        (int)ctx->emax + 1 <= TMA_MAX_PHI))
    return false;
  for (size_t k = 1; k < P; k++)
    if (!ctx->super_ok[k] || (!ctx->super_force && ctx->super_static[k].nchunks < SUPER_MIN_CHUNKS)) return false;
  return true;
}

static qaa_status launch_super_pair(qaa_ctx* ctx, int k, double t_g0, double t_pre, double t_post,
                                    const double2* phi, int n_phi) {
  int64_t nch = 0;
  for (size_t g = 1; g < ctx->geom.groups.size() && g < 4; g++) nch = std::max(nch, ctx->super_static[g].nchunks);
  const size_t need = (size_t)nch * sizeof(unsigned) + 256;
  if (ctx->d_super_cap < need) {
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    qaa_status st = ensure_buffer(ctx, &ctx->d_super, &ctx->d_super_cap, need);
    if (st) return st;
  }
  SuperArgs a = ctx->super_static[k];
  const Group& gk = ctx->geom.groups[(size_t)k];
  const Group& g0 = ctx->geom.groups[0];
  a.gk.psi = ctx->state;
  a.g0.psi = ctx->state;
  a.gk.phi = phi;
  a.gk.n_phi = n_phi;
  for (int b = 0; b < TILE_BITS; b++) {
    const bool rk = (gk.rot_local >> b) & 1;
    a.gk.t[0][b] = rk ? t_pre : 0.0;
    a.gk.t[1][b] = rk ? t_post : 0.0;
    a.gk.phys[b] = gk.phys[b];
    a.g0.t[0][b] = ((g0.rot_local >> b) & 1) ? t_g0 : 0.0;
    a.g0.t[1][b] = 0.0;
    a.g0.phys[b] = g0.phys[b];
  }
  a.gk.ntiles = gk.ntiles;
  a.g0.ntiles = g0.ntiles;
  a.gk.nseg = gk.nseg;
  a.g0.nseg = g0.nseg;
  for (int s = 0; s < MAX_SEGS; s++) {
    a.gk.seg_src[s] = gk.seg_src[s];
    a.gk.seg_dst[s] = gk.seg_dst[s];
    a.gk.seg_len[s] = gk.seg_len[s];
    a.g0.seg_src[s] = g0.seg_src[s];
    a.g0.seg_dst[s] = g0.seg_dst[s];
    a.g0.seg_len[s] = g0.seg_len[s];
  }
  a.hints = ctx->super_hints;
  a.queue = ctx->super_dynamic ? (unsigned long long*)ctx->d_super : nullptr;
  a.done = (unsigned*)((char*)ctx->d_super + 256);
  CUDA_TRY(cudaMemsetAsync(ctx->d_super, 0, 256 + (size_t)a.nchunks * sizeof(unsigned), ctx->stream));
  // phi == nullptr: the plain pair of a four-group plan (kernel variant without D)
  return launch_superpass(&ctx->tmaps[(size_t)k], a, (gk.rot_local >> 3) & 1, ctx->super_groups, phi != nullptr,
                          ctx->num_sms, ctx->stream) == cudaSuccess
             ? QAA_OK
             : fail(ctx, QAA_E_CUDA, "superpass launch failed");
}

static const Program* get_program(qaa_ctx* ctx, int g, bool pre, bool d, bool post) {
  auto key = std::make_tuple(g, (int)pre, (int)d, (int)post);
  auto it = ctx->progs.find(key);
  if (it != ctx->progs.end()) return &it->second;
  const Group& gr = ctx->geom.groups[g];
  Program p;
  if (!build_program(pre ? gr.rot_local : 0u, d, post ? gr.rot_local : 0u, &p)) return nullptr;
  return &(ctx->progs[key] = p);
}

qaa_status qaa_evolve(qaa_ctx* ctx, double T, int64_t K, const double* schedule) {
  CHECK_CTX();
  if (!ctx->loaded || !ctx->initialized) return fail(ctx, QAA_E_STATE, "evolve before load_instance/init");
  if (!(T >= 0.0) || !std::isfinite(T)) return fail(ctx, QAA_E_USAGE, "T must be finite and >= 0, got %g", T);
  if (K < 1) return fail(ctx, QAA_E_USAGE, "steps must be >= 1, got %lld", (long long)K);
  if (schedule)
    for (int64_t k = 0; k < K; k++)
      if (!(schedule[k] >= 0.0 && schedule[k] <= 1.0))
        return fail(ctx, QAA_E_USAGE, "schedule[%lld] = %g outside [0, 1]", (long long)k, schedule[k]);
  const int n_phi = (int)ctx->emax + 1;
  if (ctx->order == 2 && ctx->world > 1)
    return fail(ctx, QAA_E_USAGE, "second-order (Strang) splitting is single-GPU in this build");
  const size_t phi_bytes = (size_t)(ctx->order == 2 ? K + 1 : K) * n_phi * sizeof(double2);
  const size_t coef_bytes = (size_t)K * sizeof(double);
  const size_t form_bytes = (size_t)K * sizeof(int32_t);
  const size_t total = phi_bytes + coef_bytes + form_bytes + 256;
  // staging buffer may still be feeding a previous async copy
  if (ctx->coef_pending) {
    CUDA_TRY(cudaEventSynchronize(ctx->coef_done));
    ctx->coef_pending = false;
  }
  {
    qaa_status st = ensure_host(ctx, &ctx->h_coef, &ctx->h_coef_cap, total);
    if (st) return st;
  }
  double2* hphi = (double2*)ctx->h_coef;
  double* hcoef = (double*)((char*)ctx->h_coef + phi_bytes);
  int32_t* hform = (int32_t*)((char*)ctx->h_coef + phi_bytes + coef_bytes);
  std::vector<StepCoef> sc((size_t)K);
  const double dtK = T / (double)K;
  for (int64_t k = 0; k < K; k++) {
    const double s = schedule ? schedule[k] : ((double)k + 0.5) / (double)K;  // R8 midpoint
    double theta = dtK * weight_p(ctx, s);
    if (ctx->order == 2) {  // Strang: D(s_{k-1})^{1/2} D(s_k)^{1/2} merged before X_k
      const double sp = k == 0 ? 0.0 : (schedule ? schedule[k - 1] : ((double)k - 0.5) / (double)K);
      theta = 0.5 * dtK * (weight_p(ctx, sp) + weight_p(ctx, s));
    }
    build_step(T, K, weight_b(ctx, s), theta, ctx->n, n_phi, hphi + (size_t)k * n_phi, &sc[(size_t)k]);
    hcoef[k] = sc[(size_t)k].coef;
    hform[k] = sc[(size_t)k].form;
  }
  if (ctx->order == 2) {  // closing half step D(s_{K-1})^{1/2}, no X after it
    const double sl = schedule ? schedule[K - 1] : ((double)K - 0.5) / (double)K;
    const double theta = 0.5 * dtK * weight_p(ctx, sl);
    for (int e = 0; e < n_phi; e++)
      hphi[(size_t)K * n_phi + e] = make_double2(std::cos(theta * (double)e), -std::sin(theta * (double)e));
  }
  // the device table is read by kernels still queued from a previous evolve:
  // growing it must not free memory under them
  if (ctx->d_coef_cap < total) CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  {
    qaa_status st = ensure_buffer(ctx, &ctx->d_coef, &ctx->d_coef_cap, total);
    if (st) return st;
  }
  CUDA_TRY(cudaMemcpyAsync(ctx->d_coef, ctx->h_coef, total - 256, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(cudaEventRecord(ctx->coef_done, ctx->stream));
  ctx->coef_pending = true;
  const double2* dphi = (const double2*)ctx->d_coef;
  const double* dcoef = (const double*)((char*)ctx->d_coef + phi_bytes);
  const int32_t* dform = (const int32_t*)((char*)ctx->d_coef + phi_bytes + coef_bytes);

  ctx->stats.evolve_calls++;
  ctx->stats.trotter_steps += K;
  if (ctx->world > 1) return evolve_sharded(ctx, K, sc, dphi, n_phi);
  if (ctx->L <= RESIDENT_MAX_L) {
    ResidentArgs ra;
    ra.psi = ctx->state;
    ra.E = ctx->E;
    ra.L = ctx->L;
    ra.K = K;
    ra.phi_all = dphi;
    ra.n_phi = n_phi;
    ra.coef = dcoef;
    ra.form = dform;
    ra.final_d = ctx->order == 2 ? 1 : 0;
    size_t ev = ctx->ev_used;
    if (ctx->profile) {
      qaa_status st = ensure_events(ctx, ev + 1);
      if (st) return st;
      CUDA_TRY(cudaEventRecord(ctx->ev_pool[ev].first, ctx->stream));
    }
    if (ctx->L >= 10)
      CUDA_TRY(launch_resident_phases(ra, ctx->stream));
    else
      CUDA_TRY(launch_resident(ra, ctx->stream));
    if (ctx->profile) {
      CUDA_TRY(cudaEventRecord(ctx->ev_pool[ev].second, ctx->stream));
      ctx->ev_used = ev + 1;
    }
    ctx->stats.pass_launches++;
    ctx->stats.kernel_launches_total++;
    return QAA_OK;
  }
  std::vector<PassPlan> plan;
  build_pass_schedule((int)ctx->geom.groups.size(), K, ctx->step_spanning, &plan);
  // Strang: the closing half step D_K follows the pass that completes X_{K-1}
  // (its program becomes rotate + D; it runs on the generic kernel)
  if (ctx->order == 2) plan.back().d_step = K;
  const int max_grid = ctx->num_sms * ctx->ctas_per_sm;
  if (ctx->profile) {
    qaa_status st = ensure_events(ctx, ctx->ev_used + plan.size());
    if (st) return st;
  }
  PassArgs a;
  memset(&a, 0, sizeof a);
  a.psi = ctx->state;
  a.E = ctx->E;
  a.n_phi = n_phi;
  FastArgs fa;
  memset(&fa, 0, sizeof fa);
  fa.psi = ctx->state;
  fa.E = ctx->E;
  fa.n_phi = n_phi;
  const bool prefetch = ctx->ctas_per_sm == 1;
  const int fast_grid_cap = ctx->num_sms * (prefetch ? 1 : 2);
  const bool sup = super_usable(ctx) && ctx->step_spanning == 2 && ctx->order == 1;
  for (size_t pi = 0; pi < plan.size(); pi++) {
    const PassPlan& pp = plan[pi];
    if (sup && pi + 1 < plan.size()) {
      // [group 0: pre j] [group k: pre j, D_{j+1}, post j+1] -> one L2-blocked launch
      const PassPlan& pn = plan[pi + 1];
      const bool with_d = pn.d_step >= 0 && pn.post_step >= 0;
      // plain pair: every step of a four-group plan, and the closing pair of a call
      const bool plain = pn.d_step < 0 && pn.post_step < 0;
      if (pp.group == 0 && pp.pre_step >= 0 && pp.d_step < 0 && pp.post_step < 0 && pn.group >= 1 &&
          pn.pre_step == pp.pre_step && (with_d || plain) && ctx->super_ok[(size_t)pn.group] &&
          sc[(size_t)pp.pre_step].form == 0 && (!with_d || sc[(size_t)pn.post_step].form == 0)) {
        if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].first, ctx->stream));
        qaa_status st = launch_super_pair(ctx, pn.group, sc[(size_t)pp.pre_step].coef, sc[(size_t)pn.pre_step].coef,
                                          with_d ? sc[(size_t)pn.post_step].coef : 0.0,
                                          with_d ? dphi + (size_t)pn.d_step * n_phi : nullptr, n_phi);
        if (st) return st;
        if (ctx->profile) {
          CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].second, ctx->stream));
          if (ctx->ev_super.size() < ctx->ev_pool.size()) ctx->ev_super.resize(ctx->ev_pool.size(), 0);
          ctx->ev_super[ctx->ev_used] = 1;
          ctx->ev_used++;
        }
        ctx->stats.pass_launches++;
        ctx->stats.super_launches++;
        ctx->stats.kernel_launches_total++;
        pi++;
        continue;
      }
    }
    const Group& gr = ctx->geom.groups[pp.group];
    const bool pre = pp.pre_step >= 0, d = pp.d_step >= 0, post = pp.post_step >= 0;
    int fp = -1;
    if (pp.group == 0) {
      if (!pre && d && post) fp = FP_G0_DPOST;
      else if (pre && !d && !post) fp = FP_G0_PRE;
      else if (pre && d && post) fp = FP_G0_PRE_D_POST;
    } else if ((gr.rot_local & ~0xFF8u) == 0) {
      if (pre && !d && !post) fp = FP_GK_PRE;
      else if (d && post) fp = FP_GK_PRE_D_POST;  // without pre: its t0 row is all zeros
    }
    if ((pre && sc[(size_t)pp.pre_step].form != 0) || (post && sc[(size_t)pp.post_step].form != 0)) fp = -1;
    if (fp >= 0 && use_tma(ctx) && ctx->tma_ok[(size_t)pp.group] && n_phi <= TMA_MAX_PHI) {
      TmaArgs ta = ctx->tma_static[(size_t)pp.group];
      ta.psi = ctx->state;
      ta.phi = d ? dphi + (size_t)pp.d_step * n_phi : nullptr;
      ta.n_phi = n_phi;
      for (int b = 0; b < TILE_BITS; b++) {
        const bool rb = (gr.rot_local >> b) & 1;
        ta.t[0][b] = (pre && rb) ? sc[(size_t)pp.pre_step].coef : 0.0;
        ta.t[1][b] = (post && rb) ? sc[(size_t)pp.post_step].coef : 0.0;
        ta.phys[b] = gr.phys[b];
      }
      ta.ntiles = gr.ntiles;
      ta.nseg = gr.nseg;
      for (int s = 0; s < gr.nseg; s++) {
        ta.seg_src[s] = gr.seg_src[s];
        ta.seg_dst[s] = gr.seg_dst[s];
        ta.seg_len[s] = gr.seg_len[s];
      }
      const int grid = (int)std::min<int64_t>(gr.ntiles / 2, ctx->num_sms);
      if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].first, ctx->stream));
      // auto: one consumer group for the contiguous group-0 rotate pass (two tiles
      // in flight), two elsewhere (measured, profiles/r01_*)
      const int ng = ctx->tma_groups ? ctx->tma_groups : ((fp == FP_G0_PRE) ? 1 : 2);
      CUDA_TRY(launch_pass_tma(&ctx->tmaps[(size_t)pp.group], ta, fp, (gr.rot_local >> 3) & 1, ng, grid, ctx->stream));
      if (ctx->profile) {
        CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].second, ctx->stream));
        ctx->ev_used++;
      }
      ctx->stats.pass_launches++;
      ctx->stats.kernel_launches_total++;
      continue;
    }
    if (fp >= 0) {
      fa.phi = d ? dphi + (size_t)pp.d_step * n_phi : nullptr;
      for (int b = 0; b < TILE_BITS; b++) {
        const bool rb = (gr.rot_local >> b) & 1;
        fa.t[0][b] = (pre && rb) ? sc[(size_t)pp.pre_step].coef : 0.0;
        fa.t[1][b] = (post && rb) ? sc[(size_t)pp.post_step].coef : 0.0;
        fa.phys[b] = gr.phys[b];
      }
      fa.ntiles = gr.ntiles;
      fa.nseg = gr.nseg;
      for (int s = 0; s < gr.nseg; s++) {
        fa.seg_src[s] = gr.seg_src[s];
        fa.seg_dst[s] = gr.seg_dst[s];
        fa.seg_len[s] = gr.seg_len[s];
      }
      const int grid = (int)std::min<int64_t>(gr.ntiles, fast_grid_cap);
      if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].first, ctx->stream));
      CUDA_TRY(launch_pass_fast(fa, fp, (gr.rot_local >> 3) & 1, prefetch, grid, ctx->stream));
      if (ctx->profile) {
        CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].second, ctx->stream));
        ctx->ev_used++;
      }
      ctx->stats.pass_launches++;
      ctx->stats.kernel_launches_total++;
      continue;
    }
    const Program* prog = get_program(ctx, pp.group, pp.pre_step >= 0, pp.d_step >= 0, pp.post_step >= 0);
    if (!prog) return fail(ctx, QAA_E_USAGE, "no register program for group %d", pp.group);
    a.phi = pp.d_step >= 0 ? dphi + (size_t)pp.d_step * n_phi : nullptr;
    a.e_pattern = prog->e_pattern;
    a.final_pattern = prog->final_pattern;
    a.nops = prog->nops;
    for (int i = 0; i < prog->nops; i++) a.ops[i] = prog->ops[i];
    if (pp.pre_step >= 0) {
      a.coef[0] = sc[(size_t)pp.pre_step].coef;
      a.form[0] = sc[(size_t)pp.pre_step].form;
    }
    if (pp.post_step >= 0) {
      a.coef[1] = sc[(size_t)pp.post_step].coef;
      a.form[1] = sc[(size_t)pp.post_step].form;
    }
    a.ntiles = gr.ntiles;
    for (int b = 0; b < TILE_BITS; b++) a.phys[b] = gr.phys[b];
    a.nseg = gr.nseg;
    for (int s = 0; s < gr.nseg; s++) {
      a.seg_src[s] = gr.seg_src[s];
      a.seg_dst[s] = gr.seg_dst[s];
      a.seg_len[s] = gr.seg_len[s];
    }
    const int grid = (int)std::min<int64_t>(gr.ntiles, max_grid);
    if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].first, ctx->stream));
    CUDA_TRY(launch_pass(a, grid, ctx->stream));
    if (ctx->profile) {
      CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].second, ctx->stream));
      ctx->ev_used++;
    }
    ctx->stats.pass_launches++;
    ctx->stats.kernel_launches_total++;
  }
  return QAA_OK;
}

// ------------------------------------------------------------------ observables
static qaa_status ensure_part(qaa_ctx* ctx, size_t doubles) {
  void* p = ctx->d_part;
  qaa_status st = ensure_buffer(ctx, &p, &ctx->d_part_cap, doubles * sizeof(double));
  ctx->d_part = (double*)p;
  return st;
}

// basic[0..2] = {norm2, <H_P>, sum_{E=0}|psi|^2}
static qaa_status obs_basic(qaa_ctx* ctx, double* basic) {
  const int64_t N = (int64_t)1 << ctx->L;
  int grid = ctx->num_sms * RED_BLOCKS_PER_SM;
  if ((int64_t)grid * 256 > N) grid = (int)std::max<int64_t>(1, (N + 255) / 256);
  qaa_status st = ensure_part(ctx, (size_t)grid * 3);
  if (st) return st;
  CUDA_TRY(launch_obs_basic(ctx->state, ctx->E, N, ctx->d_part, grid, ctx->stream));
  CUDA_TRY(launch_reduce_partials(ctx->d_part, grid, 3, 3, ctx->d_out, ctx->stream));
  ctx->stats.kernel_launches_total += 2;
  CUDA_TRY(cudaMemcpyAsync(ctx->h_out, ctx->d_out, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  for (int j = 0; j < 3; j++) basic[j] = ctx->h_out[j];
  return comm_sum(ctx, basic, 3);
}

// sx[phys + phys_offset] = local pair sums of sigma^x on the rotated bits of
// every group (only_top: the top group's bits >= L - g, after a swap to layout B)
static qaa_status obs_sigma_local(qaa_ctx* ctx, double* sx, bool only_top);

// sx[j] = <sigma^x_j> for all n qubits (collective when sharded: the global
// qubits are measured in layout B, between two layout swaps)
static qaa_status obs_sigma(qaa_ctx* ctx, double* sx) {
  for (int j = 0; j < ctx->n; j++) sx[j] = 0.0;
  qaa_status st = obs_sigma_local(ctx, sx, false);
  if (st) return st;
  if (ctx->world > 1) {
    st = shard_remap(ctx);
    if (st) return st;
    st = obs_sigma_local(ctx, sx, true);
    if (st) return st;
    st = shard_remap(ctx);
    if (st) return st;
    st = comm_sum(ctx, sx, ctx->n);
    if (st) return st;
  }
  return QAA_OK;
}

static qaa_status obs_sigma_local(qaa_ctx* ctx, double* sx, bool only_top) {
  std::vector<SigmaArgs> jobs;
  if (ctx->L <= RESIDENT_MAX_L) {
    SigmaArgs a;
    memset(&a, 0, sizeof a);
    a.psi = ctx->state;
    a.k = ctx->L;
    a.mask = (1u << ctx->L) - 1;
    for (int b = 0; b < TILE_BITS; b++) a.phys[b] = b < ctx->L ? b : 0;
    a.nseg = 0;
    a.ntiles = 1;
    jobs.push_back(a);
  } else {
    for (size_t gi = 0; gi < ctx->geom.groups.size(); gi++) {
      const Group& g = ctx->geom.groups[gi];
      if (only_top && gi + 1 != ctx->geom.groups.size()) continue;
      SigmaArgs a;
      memset(&a, 0, sizeof a);
      a.psi = ctx->state;
      a.k = TILE_BITS;
      a.mask = g.rot_local;
      if (only_top) {
        a.mask = 0;
        for (int b = 0; b < TILE_BITS; b++)
          if (g.phys[b] >= ctx->L - ctx->gbits) a.mask |= 1u << b;
      }
      for (int b = 0; b < TILE_BITS; b++) a.phys[b] = g.phys[b];
      a.nseg = g.nseg;
      for (int s = 0; s < g.nseg; s++) {
        a.seg_src[s] = g.seg_src[s];
        a.seg_dst[s] = g.seg_dst[s];
        a.seg_len[s] = g.seg_len[s];
      }
      a.ntiles = g.ntiles;
      jobs.push_back(a);
    }
  }
  for (const SigmaArgs& a : jobs) {
    const int grid = (int)std::min<int64_t>(a.ntiles, (int64_t)ctx->num_sms * 2);
    qaa_status st = ensure_part(ctx, (size_t)grid * TILE_BITS);
    if (st) return st;
    CUDA_TRY(launch_obs_sigma(a, ctx->d_part, grid, ctx->stream));
    CUDA_TRY(launch_reduce_partials(ctx->d_part, grid, TILE_BITS, TILE_BITS, ctx->d_out, ctx->stream));
    ctx->stats.kernel_launches_total += 2;
    CUDA_TRY(cudaMemcpyAsync(ctx->h_out, ctx->d_out, TILE_BITS * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    // layout B keeps the rank qubits of layout A (logical L..n-1) at local L-g..L-1
    const int off = only_top ? ctx->gbits : 0;
    for (int j = 0; j < a.k; j++)
      if (a.mask >> j & 1) sx[a.phys[j] + off] = 2.0 * ctx->h_out[j];
  }
  return QAA_OK;
}

qaa_status qaa_success_prob(qaa_ctx* ctx, double* out) {
  CHECK_CTX();
  if (!out) return fail(ctx, QAA_E_USAGE, "out is NULL");
  if (!ctx->loaded || !ctx->initialized) return fail(ctx, QAA_E_STATE, "success_prob before init");
  if (ctx->nz_total == 0) {
    *out = 0.0;
    return QAA_OK;
  }
  if (ctx->nz_total > (uint64_t)ZLIST_CAP) {  // same decision on every rank (collectives must match)
    double b[3];
    qaa_status st = obs_basic(ctx, b);  // collective
    if (st) return st;
    *out = b[2];
    return QAA_OK;
  }
  double v = 0.0;
  if (ctx->nz_local > 0) {
    CUDA_TRY(launch_gather_success(ctx->state, ctx->Z, ctx->nz_local, (uint64_t)ctx->rank << ctx->L, ctx->d_out,
                                   ctx->stream));
    ctx->stats.kernel_launches_total++;
    CUDA_TRY(cudaMemcpyAsync(ctx->h_out, ctx->d_out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    v = ctx->h_out[0];
  }
  qaa_status st = comm_sum(ctx, &v, 1);
  if (st) return st;
  *out = v;
  return QAA_OK;
}

qaa_status qaa_norm2(qaa_ctx* ctx, double* out) {
  CHECK_CTX();
  if (!out) return fail(ctx, QAA_E_USAGE, "out is NULL");
  if (!ctx->loaded || !ctx->initialized) return fail(ctx, QAA_E_STATE, "norm2 before init");
  double b[3];
  qaa_status st = obs_basic(ctx, b);
  if (st) return st;
  *out = b[0];
  return QAA_OK;
}

qaa_status qaa_sigma_x(qaa_ctx* ctx, double* out) {
  CHECK_CTX();
  if (!out) return fail(ctx, QAA_E_USAGE, "out is NULL");
  if (!ctx->loaded || !ctx->initialized) return fail(ctx, QAA_E_STATE, "sigma_x before init");
  return obs_sigma(ctx, out);
}

qaa_status qaa_energy(qaa_ctx* ctx, double s, double* out) {
  CHECK_CTX();
  if (!out) return fail(ctx, QAA_E_USAGE, "out is NULL");
  if (!(s >= 0.0 && s <= 1.0)) return fail(ctx, QAA_E_USAGE, "s = %g outside [0, 1]", s);
  if (!ctx->loaded || !ctx->initialized) return fail(ctx, QAA_E_STATE, "energy before init");
  double b[3];
  qaa_status st = obs_basic(ctx, b);
  if (st) return st;
  std::vector<double> sx((size_t)ctx->n, 0.0);
  st = obs_sigma(ctx, sx.data());
  if (st) return st;
  double hb = 0.0;
  for (int j = 0; j < ctx->n; j++) hb += 0.5 * (b[0] - sx[(size_t)j]);
  *out = weight_b(ctx, s) * hb + weight_p(ctx, s) * b[1];
  return QAA_OK;
}

qaa_status qaa_num_solutions(qaa_ctx* ctx, uint64_t* out) {
  CHECK_CTX();
  if (!out) return fail(ctx, QAA_E_USAGE, "out is NULL");
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "num_solutions before load_instance");
  *out = ctx->nz_total;
  return QAA_OK;
}

qaa_status qaa_max_energy(qaa_ctx* ctx, uint32_t* out) {
  CHECK_CTX();
  if (!out) return fail(ctx, QAA_E_USAGE, "out is NULL");
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "max_energy before load_instance");
  *out = ctx->emax;
  return QAA_OK;
}

static bool local_range(qaa_ctx* ctx, uint64_t first, uint64_t count, uint64_t* lo, uint64_t* hi) {
  const uint64_t own_lo = (uint64_t)ctx->rank << ctx->L, own_hi = own_lo + (1ull << ctx->L);
  *lo = std::max(first, own_lo);
  *hi = std::min(first + count, own_hi);
  return *lo < *hi;
}

qaa_status qaa_copy_state(qaa_ctx* ctx, uint64_t first, uint64_t count, double* dst) {
  CHECK_CTX();
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "copy_state before load_instance");
  if (count && !dst) return fail(ctx, QAA_E_USAGE, "dst is NULL");
  if (first + count > (1ull << ctx->n) || first + count < first)
    return fail(ctx, QAA_E_USAGE, "range [%llu, +%llu) outside [0, 2^%d)", (unsigned long long)first,
                (unsigned long long)count, ctx->n);
  uint64_t lo, hi;
  if (local_range(ctx, first, count, &lo, &hi)) {
    const uint64_t off = lo - ((uint64_t)ctx->rank << ctx->L);
    CUDA_TRY(cudaMemcpyAsync(dst + 2 * (lo - first), ctx->state + off, (hi - lo) * sizeof(double2),
                             cudaMemcpyDeviceToHost, ctx->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return QAA_OK;
}

qaa_status qaa_set_state(qaa_ctx* ctx, uint64_t first, uint64_t count, const double* src) {
  CHECK_CTX();
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "set_state before load_instance");
  if (count && !src) return fail(ctx, QAA_E_USAGE, "src is NULL");
  if (first + count > (1ull << ctx->n) || first + count < first)
    return fail(ctx, QAA_E_USAGE, "range outside [0, 2^%d)", ctx->n);
  uint64_t lo, hi;
  if (local_range(ctx, first, count, &lo, &hi)) {
    const uint64_t off = lo - ((uint64_t)ctx->rank << ctx->L);
    CUDA_TRY(cudaMemcpyAsync(ctx->state + off, src + 2 * (lo - first), (hi - lo) * sizeof(double2),
                             cudaMemcpyHostToDevice, ctx->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  ctx->initialized = true;
  return QAA_OK;
}

qaa_status qaa_copy_energy_table(qaa_ctx* ctx, uint64_t first, uint64_t count, uint8_t* dst) {
  CHECK_CTX();
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "copy_energy_table before load_instance");
  if (count && !dst) return fail(ctx, QAA_E_USAGE, "dst is NULL");
  if (first + count > (1ull << ctx->n) || first + count < first)
    return fail(ctx, QAA_E_USAGE, "range outside [0, 2^%d)", ctx->n);
  uint64_t lo, hi;
  if (local_range(ctx, first, count, &lo, &hi)) {
    const uint64_t off = lo - ((uint64_t)ctx->rank << ctx->L);
    CUDA_TRY(cudaMemcpyAsync(dst + (lo - first), ctx->E + off, hi - lo, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return QAA_OK;
}

qaa_status qaa_state_ptr(qaa_ctx* ctx, void** out, uint64_t* amps) {
  CHECK_CTX();
  if (!out || !amps) return fail(ctx, QAA_E_USAGE, "NULL output");
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "state_ptr before load_instance");
  *out = ctx->state;
  *amps = 1ull << ctx->L;
  return QAA_OK;
}

qaa_status qaa_spectrum(qaa_ctx* ctx, double s, int kmax, int nev, double* evals, double* overlap, int* iters) {
  CHECK_CTX();
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "spectrum before load_instance");
  if (!(s >= 0.0 && s <= 1.0)) return fail(ctx, QAA_E_USAGE, "s = %g outside [0, 1]", s);
  if (kmax < 2 || kmax > 512 || nev < 1 || nev > kmax || !evals)
    return fail(ctx, QAA_E_USAGE, "need 2 <= kmax <= 512, 1 <= nev <= kmax, evals != NULL");
  if (ctx->world != 1 || ctx->L > 24) return fail(ctx, QAA_E_CAP, "spectrum: single GPU, n <= 24");
  if (overlap && !ctx->initialized) return fail(ctx, QAA_E_STATE, "overlap needs an initialised state");
  const size_t vec = ((size_t)1 << ctx->L) * sizeof(double2);
  void* basis = nullptr;
  cudaError_t e = cudaMalloc(&basis, vec * (size_t)(kmax + 1));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, QAA_E_CAP, "Lanczos basis of %d vectors does not fit", kmax + 1);
  }
  qaa_status st = ensure_part(ctx, (size_t)ctx->num_sms * 8 + 16);
  if (st) {
    cudaFree(basis);
    return st;
  }
  LanczosArgs p;
  p.n = ctx->L;
  p.num_sms = ctx->num_sms;
  p.E = ctx->E;
  p.wb = weight_b(ctx, s);
  p.wp = weight_p(ctx, s);
  p.kmax = kmax;
  p.nev = nev;
  p.basis = (double2*)basis;
  p.scratch = ctx->d_part;
  p.state = overlap ? ctx->state : nullptr;
  int it = 0;
  e = lanczos_spectrum(p, ctx->stream, evals, overlap, &it);
  cudaFree(basis);
  if (e != cudaSuccess) return fail(ctx, QAA_E_CUDA, "Lanczos failed: %s", cudaGetErrorString(e));
  ctx->stats.kernel_launches_total += 4 * (int64_t)it * (it + 1);
  if (iters) *iters = it;
  return QAA_OK;
}

qaa_status qaa_set_driver(qaa_ctx* ctx, double gx, double gz) {
  if (!ctx) return QAA_E_USAGE;
  if (!std::isfinite(gx) || !std::isfinite(gz)) return fail(ctx, QAA_E_USAGE, "driver weights must be finite");
  ctx->drv_x = gx;
  ctx->drv_z = gz;
  return QAA_OK;
}

qaa_status qaa_time_energy_table(qaa_ctx* ctx, int reps, double* ms) {
  CHECK_CTX();
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "time_energy_table before load_instance");
  if (reps < 1 || !ms) return fail(ctx, QAA_E_USAGE, "reps must be >= 1 and ms non-NULL");
  if (!ctx->clause_recs) return fail(ctx, QAA_E_STATE, "no clause records");
  const int64_t N = (int64_t)1 << ctx->L;
  cudaEvent_t a, b;
  CUDA_TRY(cudaEventCreate(&a));
  CUDA_TRY(cudaEventCreate(&b));
  // warm-up, then `reps` timed launches recomputing E in place (same values)
  CUDA_TRY(launch_energy_table(ctx->E, N, (uint64_t)ctx->rank << ctx->L, (const uint64_t*)ctx->clause_recs,
                               ctx->n_recs, ctx->d_counters, (unsigned long long*)(ctx->d_counters + 2), ctx->num_sms,
                               ctx->stream, 63, 0, ctx->energy_w64 != 0));
  CUDA_TRY(cudaEventRecord(a, ctx->stream));
  for (int r = 0; r < reps; r++)
    CUDA_TRY(launch_energy_table(ctx->E, N, (uint64_t)ctx->rank << ctx->L, (const uint64_t*)ctx->clause_recs,
                                 ctx->n_recs, ctx->d_counters, (unsigned long long*)(ctx->d_counters + 2),
                                 ctx->num_sms, ctx->stream, 63, 0, ctx->energy_w64 != 0));
  CUDA_TRY(cudaEventRecord(b, ctx->stream));
  CUDA_TRY(cudaEventSynchronize(b));
  float t = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&t, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  ctx->stats.kernel_launches_total += reps + 1;
  *ms = (double)t / reps;
  return QAA_OK;
}

qaa_status qaa_sweep(qaa_ctx* ctx, int nrep, const double* T, const int64_t* K, double* out) {
  CHECK_CTX();
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "sweep before load_instance");
  if (ctx->world != 1 || ctx->L > SWEEP_MAX_L)
    return fail(ctx, QAA_E_USAGE, "sweep needs world = 1 and n <= %d (state resident in one CTA or cluster)",
                SWEEP_MAX_L);
  if (nrep < 1 || !T || !K || !out) return fail(ctx, QAA_E_USAGE, "sweep needs nrep >= 1 and non-NULL arrays");
  int64_t rows = 0;
  for (int r = 0; r < nrep; r++) {
    if (!(T[r] >= 0.0) || !std::isfinite(T[r])) return fail(ctx, QAA_E_USAGE, "T[%d] = %g invalid", r, T[r]);
    if (K[r] < 1) return fail(ctx, QAA_E_USAGE, "K[%d] = %lld < 1", r, (long long)K[r]);
    rows += K[r] + (ctx->order == 2 ? 1 : 0);
  }
  const int n_phi = (int)ctx->emax + 1;
  const size_t phi_bytes = (size_t)rows * n_phi * sizeof(double2);
  const size_t tail = (size_t)rows * (sizeof(double) + sizeof(int32_t)) + (size_t)nrep * 2 * sizeof(int64_t);
  const size_t total = phi_bytes + tail + (size_t)nrep * sizeof(double) + 512;
  if (ctx->coef_pending) {
    CUDA_TRY(cudaEventSynchronize(ctx->coef_done));
    ctx->coef_pending = false;
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  qaa_status st = ensure_host(ctx, &ctx->h_coef, &ctx->h_coef_cap, total);
  if (st) return st;
  st = ensure_buffer(ctx, &ctx->d_coef, &ctx->d_coef_cap, total);
  if (st) return st;
  char* hb = (char*)ctx->h_coef;
  double2* hphi = (double2*)hb;
  double* hcoef = (double*)(hb + phi_bytes);
  int32_t* hform = (int32_t*)(hcoef + rows);
  int64_t* hK = (int64_t*)(((uintptr_t)(hform + rows) + 15) & ~(uintptr_t)15);
  int64_t* hoff = hK + nrep;
  int64_t row = 0;
  for (int r = 0; r < nrep; r++) {
    hK[r] = K[r];
    hoff[r] = row;
    const double dt = T[r] / (double)K[r];
    for (int64_t k = 0; k < K[r]; k++) {
      const double s = ((double)k + 0.5) / (double)K[r];
      double theta = dt * weight_p(ctx, s);
      if (ctx->order == 2)
        theta = 0.5 * dt * (weight_p(ctx, k == 0 ? 0.0 : ((double)k - 0.5) / (double)K[r]) + weight_p(ctx, s));
      StepCoef c;
      build_step(T[r], K[r], weight_b(ctx, s), theta, ctx->n, n_phi, hphi + (size_t)(row + k) * n_phi, &c);
      hcoef[row + k] = c.coef;
      hform[row + k] = c.form;
    }
    row += K[r];
    if (ctx->order == 2) {
      const double theta = 0.5 * dt * weight_p(ctx, ((double)K[r] - 0.5) / (double)K[r]);
      for (int e = 0; e < n_phi; e++)
        hphi[(size_t)row * n_phi + e] = make_double2(std::cos(theta * (double)e), -std::sin(theta * (double)e));
      hcoef[row] = 0.0;
      hform[row] = 0;
      row++;
    }
  }
  const size_t used = (size_t)((char*)(hoff + nrep) - hb);
  CUDA_TRY(cudaMemcpyAsync(ctx->d_coef, ctx->h_coef, used, cudaMemcpyHostToDevice, ctx->stream));
  char* db = (char*)ctx->d_coef;
  SweepArgs a;
  a.E = ctx->E;
  a.L = ctx->L;
  a.amp0 = 1.0 / std::sqrt(std::ldexp(1.0, ctx->n));
  a.phi_all = (const double2*)db;
  a.n_phi = n_phi;
  a.coef = (const double*)(db + phi_bytes);
  a.form = (const int32_t*)(db + ((char*)hform - hb));
  a.K = (const int64_t*)(db + ((char*)hK - hb));
  a.row_off = (const int64_t*)(db + ((char*)hoff - hb));
  a.final_d = ctx->order == 2 ? 1 : 0;
  double* dout = (double*)(db + ((used + 15) & ~(size_t)15));
  a.out = dout;
  if (ctx->L >= 10)  // register phases, one CTA (n <= 13) or one cluster (n = 14..16) per replica
    CUDA_TRY(launch_sweep_cluster(a, nrep, ctx->stream));
  else
    CUDA_TRY(launch_sweep(a, nrep, ctx->stream));
  ctx->stats.kernel_launches_total++;
  CUDA_TRY(cudaMemcpyAsync(out, dout, (size_t)nrep * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return QAA_OK;
}

qaa_status qaa_get_stats(qaa_ctx* ctx, qaa_stats* out) {
  CHECK_CTX();
  if (!out) return fail(ctx, QAA_E_USAGE, "out is NULL");
  if (ctx->ev_used) {
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    for (size_t i = 0; i < ctx->ev_used; i++) {
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, ctx->ev_pool[i].first, ctx->ev_pool[i].second));
      ctx->stats.pass_kernel_ms += ms;
      ctx->stats.pass_kernels_timed++;
      if (i < ctx->ev_super.size() && ctx->ev_super[i]) {
        ctx->stats.super_kernel_ms += ms;
        ctx->stats.super_kernels_timed++;
        ctx->ev_super[i] = 0;
      }
    }
    ctx->ev_used = 0;
  }
  qaa_stats s = ctx->stats;
  s.n = ctx->n;
  s.n_local = ctx->L;
  s.amps_local = ctx->loaded ? ((int64_t)1 << ctx->L) : 0;
  s.groups = ctx->L > RESIDENT_MAX_L ? (int)ctx->geom.groups.size() : 1;
  s.tile_bits = ctx->L > RESIDENT_MAX_L ? TILE_BITS : ctx->L;
  s.row_bits = ctx->row_bits;
  const int P = s.groups;
  s.passes_per_step_num = (ctx->step_spanning && P > 1) ? P - 1 : P;
  if (ctx->L > RESIDENT_MAX_L && super_usable(ctx) && ctx->step_spanning == 2) s.passes_per_step_num = P - 2;
  if (ctx->world > 1) s.passes_per_step_num = P;  // sharded: one phase of P passes per step (§7)
  s.passes_per_step_den = 1;
  s.bytes_per_pass = s.amps_local * 32;
  *out = s;
  return QAA_OK;
}

qaa_status qaa_reset_stats(qaa_ctx* ctx) {
  CHECK_CTX();
  if (ctx->ev_used) CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  ctx->ev_used = 0;
  memset(&ctx->stats, 0, sizeof ctx->stats);
  return QAA_OK;
}

qaa_status qaa_plan_describe(int n_local, int row_bits, int step_spanning, int64_t K, int32_t* rec, int64_t cap,
                             int64_t* count) {
  if (!count || n_local < 1 || n_local > 40 || K < 1 || (cap > 0 && !rec)) return QAA_E_USAGE;
  if (n_local <= RESIDENT_MAX_L) {
    const uint64_t mask = (n_local >= 64) ? ~0ull : ((1ull << n_local) - 1);
    for (int64_t k = 0; k < K && k < cap; k++) {
      int32_t* r = rec + k * QAA_PLAN_RECORD;
      r[0] = 0;
      r[1] = -1;
      r[2] = (int32_t)k;
      r[3] = (int32_t)k;
      r[4] = 0;
      r[5] = 0;
      r[6] = (int32_t)(mask & 0xffffffffu);
      r[7] = (int32_t)(mask >> 32);
      r[8] = 0;
      r[9] = 0;
    }
    *count = K;
    return QAA_OK;
  }
  Geometry g;
  std::string e;
  if (!build_geometry(n_local, row_bits, &g, &e)) return QAA_E_USAGE;
  std::vector<PassPlan> plan;
  build_pass_schedule((int)g.groups.size(), K, step_spanning, &plan);
  *count = (int64_t)plan.size();
  for (int64_t i = 0; i < (int64_t)plan.size() && i < cap; i++) {
    const PassPlan& pp = plan[(size_t)i];
    const Group& gr = g.groups[pp.group];
    Program prog;
    if (!build_program(pp.pre_step >= 0 ? gr.rot_local : 0u, pp.d_step >= 0, pp.post_step >= 0 ? gr.rot_local : 0u,
                       &prog))
      return QAA_E_USAGE;
    const uint64_t pre = pp.pre_step >= 0 ? gr.rot_phys : 0, post = pp.post_step >= 0 ? gr.rot_phys : 0;
    int32_t* r = rec + i * QAA_PLAN_RECORD;
    r[0] = pp.group;
    r[1] = (int32_t)pp.pre_step;
    r[2] = (int32_t)pp.d_step;
    r[3] = (int32_t)pp.post_step;
    r[4] = (int32_t)(pre & 0xffffffffu);
    r[5] = (int32_t)(pre >> 32);
    r[6] = (int32_t)(post & 0xffffffffu);
    r[7] = (int32_t)(post >> 32);
    r[8] = prog.n_exch;
    r[9] = prog.n_shfl;
  }
  return QAA_OK;
}

}  // extern "C"

extern "C" qaa_status qaa_plan_describe_sharded(int n, int world, int row_bits, int64_t K, int32_t* rec, int64_t cap,
                                                int64_t* count) {
  if (!count || K < 1 || (cap > 0 && !rec)) return QAA_E_USAGE;
  if (world != 2 && world != 4 && world != 8) return QAA_E_USAGE;
  const int g = world == 2 ? 1 : (world == 4 ? 2 : 3);
  const int L = n - g;
  if (n < 1 || n > 40 || L <= RESIDENT_MAX_L) return QAA_E_CAP;
  Geometry geo;
  std::string e;
  if (!build_geometry(L, row_bits, &geo, &e)) return QAA_E_USAGE;
  std::vector<ShardPass> plan;
  if (!build_shard_schedule(geo, g, K, &plan, &e)) return QAA_E_CAP;
  *count = (int64_t)plan.size();
  for (int64_t i = 0; i < (int64_t)plan.size() && i < cap; i++) {
    const ShardPass& sp = plan[(size_t)i];
    int32_t* r = rec + i * QAA_SHARD_RECORD;
    uint32_t pre = 0, post = 0;
    if (sp.kind == SK_PASS) {
      const Group& gr = geo.groups[(size_t)sp.group];
      for (int b = 0; b < TILE_BITS; b++) {
        if ((sp.pre_local >> b) & 1) pre |= 1u << gr.phys[b];
        if ((sp.post_local >> b) & 1) post |= 1u << gr.phys[b];
      }
    }
    r[0] = sp.kind;
    r[1] = sp.group;
    r[2] = (int32_t)sp.pre_step;
    r[3] = (int32_t)sp.d_step;
    r[4] = (int32_t)sp.post_step;
    r[5] = sp.remote;
    r[6] = sp.layout;
    r[7] = (int32_t)pre;
    r[8] = (int32_t)post;
    r[9] = 0;
  }
  return QAA_OK;
}
