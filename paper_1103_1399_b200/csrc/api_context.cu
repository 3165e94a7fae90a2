// api_context.cu -- C-ABI of libqaa (include/qaa.h): context lifetime, options, instance load (A1-A3), initial states (A4), stats.
#include "api_internal.hpp"

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
  CUDA_TRY(superpass_tm_setup());
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
  for (int r = 0; r < 8; r++)
    if (ctx->peer_sync_open[r]) cudaIpcCloseMemHandle(ctx->peer_sync[r]);
  if (ctx->sync_buf) cudaFree(ctx->sync_buf);
  for (int b = 0; b < 2; b++)
    if (ctx->shard_top_eg[b]) cudaFree(ctx->shard_top_eg[b]);
  for (int k = 0; k < 4; k++)
    if (ctx->Eg_tm[k]) cudaFree(ctx->Eg_tm[k]);
  if (ctx->d_pos_tm) cudaFree(ctx->d_pos_tm);
  if (ctx->d_tm_diag) cudaFree(ctx->d_tm_diag);
  if (ctx->d_persist) cudaFree(ctx->d_persist);
  for (int g = 0; g < 4; g++)
    if (ctx->Ewt[g]) cudaFree(ctx->Ewt[g]);
  if (ctx->d_wsweep) cudaFree(ctx->d_wsweep);
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
      if (ctx->loaded && ctx->L > RESIDENT_MAX_L) {
        // everything derived from the tile-group geometry is rebuilt here, before
        // the next evolve: tensor maps, permuted energy tables, L2-blocked chunk
        // plans (single GPU) or the fused layout-swap / top-group plans (sharded)
        if (ctx->poisoned) return fail(ctx, QAA_E_STATE, "context poisoned: %s", ctx->err.c_str());
        Geometry g;
        std::string e;
        if (!build_geometry(ctx->L, (int)value, &g, &e)) return fail(ctx, QAA_E_USAGE, "%s", e.c_str());
        if (ctx->world > 1) {
          std::vector<ShardPass> sp;
          if (!build_shard_schedule(g, ctx->gbits, 1, &sp, &e))
            return fail(ctx, QAA_E_USAGE, "row_bits %lld cannot shard n = %d: %s", (long long)value, ctx->n, e.c_str());
        }
        cudaSetDevice(ctx->device);
        ctx->row_bits = (int)value;
        ctx->geom = g;
        ctx->progs.clear();
        if (ctx->world == 1) return build_tma(ctx);
        build_shard_super(ctx);
        return build_shard_top(ctx);
      }
      ctx->row_bits = (int)value;
      ctx->progs.clear();
      return QAA_OK;
    case QAA_OPT_SUPER_GRID:
      if (value < 0 || value > ctx->num_sms) return fail(ctx, QAA_E_USAGE, "super grid must be in 0..%d", ctx->num_sms);
      ctx->super_grid = (int)value;
      return QAA_OK;
    case QAA_OPT_SUPER_SPLIT:
      if (value < 0 || value >= ctx->num_sms) return fail(ctx, QAA_E_USAGE, "super split must be in 0..%d", ctx->num_sms - 1);
      ctx->super_split = (int)value;
      return QAA_OK;
    case QAA_OPT_SHARD_SYNC:
      if (value < 0 || value > 1) return fail(ctx, QAA_E_USAGE, "shard sync must be 0 (device) or 1 (host)");
      ctx->shard_sync = (int)value;
      return QAA_OK;
    case QAA_OPT_PERSIST:
      if (value < 0 || value > 1) return fail(ctx, QAA_E_USAGE, "persist must be 0 or 1");
      ctx->persist = (int)value;
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
      if (value < 0 || value > 65535) return fail(ctx, QAA_E_USAGE, "super option must be in 0..65535");
      // bit 0: L2-blocked Trotter steps; bit 1: one consumer group per CTA (default two);
      // bits 2-3: L2 eviction hints (0 = evict-last for the group-0 output that the
      // group-k sub-pass reads back + evict-first for dead data; 1 = none; 2 = evict-first only)
      ctx->super_mode = (int)(value & 1);
      ctx->super_groups = (value & 2) ? 1 : 2;
      ctx->super_force = (value & 16) ? 1 : 0;  // also below SUPER_MIN_CHUNKS (tests)
      ctx->super_dynamic = (value & 32) ? 1 : 0;  // dynamic work queue instead of static round robin
      ctx->super_tm = (value & 64) ? 1 : 0;       // 64: tensor-memory exchanges (pass_tmem.cu; measured slower)
      ctx->super_tm_flags = (int)((value >> 7) & 15) | (int)((value >> 9) & 16);  // bits 7-10, 13: pass_tmem.cu switches
      ctx->super_lag = 1 + (int)((value >> 11) & 3);    // bits 11-12: chunk lag - 1 (SuperArgs.lag)
      ctx->super_pw = (value >> 14) & 1;                // bit 14: producer-warp variant (qaa_superpass_pw)
      ctx->super_v2 = ((value >> 15) & 1) ? 0 : 1;      // bit 15: group barriers instead of split-phase WAR + deferred publish
      ctx->super_hints = ((value >> 2) & 3) == 1 ? 0 : (((value >> 2) & 3) == 2 ? 1 : 2);
      return QAA_OK;
    case QAA_OPT_WARPTILE:
      if (value < 0 || value > 3) return fail(ctx, QAA_E_USAGE, "warptile must be 0, 1, 2 or 3");
      ctx->warptile = (int)value;
      return QAA_OK;
    case QAA_OPT_WARP_GRID:
      if (value < 0 || (value && ((value & 15) < 1 || (value & 15) > 8 || (value >> 4) < 1)))
        return fail(ctx, QAA_E_USAGE, "warp grid must be 0 or ctas * 16 + warps (1..8)");
      ctx->warp_grid = (int)value;
      return QAA_OK;
    case QAA_OPT_SUPER_PUB:
      if ((value & 15) < 1 || (value & 15) > 8 || value > 31)
        return fail(ctx, QAA_E_USAGE, "super pub must be batch (1..8) + 16 * early (0/1)");
      ctx->super_pub = (int)value;
      return QAA_OK;
    case QAA_OPT_SWEEP_TUNE:
      if (value < 0 || value >= (4096 << 4)) return fail(ctx, QAA_E_USAGE, "sweep tune must be in 0..65535");
      ctx->sweep_tune = (int)value;
      return QAA_OK;
    case QAA_OPT_SUPER_REV:
      if (value < 0 || value > 1) return fail(ctx, QAA_E_USAGE, "super rev must be 0 or 1");
      ctx->super_rev = (int)value;
      return QAA_OK;
    case QAA_OPT_CLUSTER:
      if (value < 0 || value > 1) return fail(ctx, QAA_E_USAGE, "cluster must be 0 or 1");
      ctx->cluster_evolve = (int)value;
      return QAA_OK;
    case QAA_OPT_DIAG:
      if (value < 0 || value > 127) return fail(ctx, QAA_E_USAGE, "diag must be in 0..127");
      ctx->diag = (int)value;
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

qaa_status qaa_load_instance(qaa_ctx* ctx, int n, int m, const int32_t* lits) {
  QAA_NVTX("qaa_load_instance");
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
  ctx->wt_built = false;  // warp-tile energy tables follow E (built on first use)
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
  QAA_NVTX("qaa_init_uniform");
  CHECK_CTX();
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "init_uniform before load_instance");
  const double a = 1.0 / std::sqrt(std::ldexp(1.0, ctx->n));
  CUDA_TRY(launch_fill(ctx->state, (int64_t)1 << ctx->L, a, 0.0, ctx->num_sms, ctx->stream));
  ctx->stats.kernel_launches_total++;
  ctx->initialized = true;
  return QAA_OK;
}

qaa_status qaa_init_basis(qaa_ctx* ctx, uint64_t x) {
  QAA_NVTX("qaa_init_basis");
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

qaa_status qaa_set_driver(qaa_ctx* ctx, double gx, double gz) {
  if (!ctx) return QAA_E_USAGE;
  if (!std::isfinite(gx) || !std::isfinite(gz)) return fail(ctx, QAA_E_USAGE, "driver weights must be finite");
  ctx->drv_x = gx;
  ctx->drv_z = gz;
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
  if (ctx->d_tm_diag) {
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    CUDA_TRY(cudaMemcpy(s.tm_diag, ctx->d_tm_diag, sizeof s.tm_diag, cudaMemcpyDeviceToHost));
  }
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

}  // extern "C"
