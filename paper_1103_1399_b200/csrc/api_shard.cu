// api_shard.cu -- sharded state: host collectives, IPC shard buffers, layout swaps and the sharded evolve.
#include "api_internal.hpp"

// ------------------------------------------------------------------ sharding helpers
qaa_status comm_barrier(qaa_ctx* ctx) {
  if (ctx->comm.barrier(ctx->comm.user) != 0) return fail(ctx, QAA_E_NCCL, "comm barrier failed");
  return QAA_OK;
}
qaa_status comm_allgather(qaa_ctx* ctx, const void* send, void* recv, size_t bytes) {
  if (ctx->comm.allgather(ctx->comm.user, send, recv, bytes) != 0) return fail(ctx, QAA_E_NCCL, "comm allgather failed");
  return QAA_OK;
}
// sum of `n` doubles over ranks, added in rank order (deterministic)
qaa_status comm_sum(qaa_ctx* ctx, double* v, int n) {
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
qaa_status setup_shard_buffers(qaa_ctx* ctx, size_t bytes) {
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
  // Every rank reaches the allgather below even when its allocation fails: the
  // ranks agree on success (an ok word in the gathered record) and fail together
  // with CAP instead of leaving the others blocked in a collective.
  struct Rec {
    int ok;
    int pad;
    cudaIpcMemHandle_t h[3];
  } mine;
  memset(&mine, 0, sizeof mine);
  mine.ok = 1;
  for (int b = 0; b < 2 && mine.ok; b++)
    if (cudaMalloc(&ctx->bufs[b], bytes) != cudaSuccess) {
      cudaGetLastError();
      ctx->bufs[b] = nullptr;
      mine.ok = 0;
    }
  // the device-side phase barrier's arrival counter (zeroed before any peer can
  // signal: peers first pass the host barrier below)
  if (mine.ok && !ctx->sync_buf) {
    if (cudaMalloc(&ctx->sync_buf, 256) != cudaSuccess || cudaMemset(ctx->sync_buf, 0, 256) != cudaSuccess) {
      cudaGetLastError();
      mine.ok = 0;
    }
    ctx->sync_epoch = 0;
    for (int r = 0; r < 8; r++) {
      if (ctx->peer_sync_open[r]) cudaIpcCloseMemHandle(ctx->peer_sync[r]);
      ctx->peer_sync_open[r] = false;
      ctx->peer_sync[r] = nullptr;
    }
  }
  if (mine.ok) {
    for (int b = 0; b < 2; b++)
      if (cudaIpcGetMemHandle(&mine.h[b], ctx->bufs[b]) != cudaSuccess) mine.ok = 0;
    if (cudaIpcGetMemHandle(&mine.h[2], ctx->sync_buf) != cudaSuccess) mine.ok = 0;
    cudaGetLastError();
  }
  std::vector<Rec> recs((size_t)ctx->world);
  qaa_status st = comm_allgather(ctx, &mine, recs.data(), sizeof mine);
  if (st) return st;
  for (int r = 0; r < ctx->world; r++)
    if (!recs[(size_t)r].ok) {
      for (int b = 0; b < 2; b++) {
        if (ctx->bufs[b]) cudaFree(ctx->bufs[b]);
        ctx->bufs[b] = nullptr;
      }
      return fail(ctx, QAA_E_CAP, "shard buffers of 2 x %zu bytes do not fit on the device of rank %d", bytes, r);
    }
  ctx->buf_cap = bytes;
  std::vector<cudaIpcMemHandle_t> all(3 * (size_t)ctx->world);
  for (int r = 0; r < ctx->world; r++)
    for (int b = 0; b < 3; b++) all[3 * (size_t)r + b] = recs[(size_t)r].h[b];
  for (int r = 0; r < ctx->world; r++) {
    for (int b = 0; b < 2; b++) {
      if (r == ctx->rank) {
        ctx->peers[b][r] = ctx->bufs[b];
        continue;
      }
      void* p = nullptr;
      CUDA_TRY(cudaIpcOpenMemHandle(&p, all[3 * (size_t)r + b], cudaIpcMemLazyEnablePeerAccess));
      ctx->peers[b][r] = (double2*)p;
      ctx->peer_open[b][r] = true;
    }
    if (r == ctx->rank) {
      ctx->peer_sync[r] = ctx->sync_buf;
    } else if (!ctx->peer_sync_open[r]) {
      void* p = nullptr;
      CUDA_TRY(cudaIpcOpenMemHandle(&p, all[3 * (size_t)r + 2], cudaIpcMemLazyEnablePeerAccess));
      ctx->peer_sync[r] = (unsigned*)p;
      ctx->peer_sync_open[r] = true;
    }
  }
  st = comm_barrier(ctx);
  if (st) return st;
  ctx->cur = 0;
  ctx->state = ctx->bufs[0];
  ctx->own_state = false;
  ctx->state_cap_bytes = bytes;
  return QAA_OK;
}

// End of a phase: every rank's peer stores into the others' next buffers are
// complete and visible before anyone reads its next buffer. Default: the
// device-side barrier (enqueued, no host sync: evolve stays asynchronous);
// QAA_OPT_SHARD_SYNC = 1: stream sync + the caller's host barrier.
qaa_status shard_barrier(qaa_ctx* ctx) {
  if (ctx->shard_sync == 1 || !ctx->sync_buf) {
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return comm_barrier(ctx);
  }
  ctx->sync_epoch++;
  CUDA_TRY(launch_shard_barrier(ctx->peer_sync, ctx->sync_buf, ctx->world, ctx->sync_epoch * (unsigned)ctx->world,
                                ctx->stream));
  ctx->stats.kernel_launches_total++;
  return QAA_OK;
}

// one layout swap (A <-> B) of the whole sharded state: stores, barrier, flip
qaa_status shard_remap(qaa_ctx* ctx) {
  CUDA_TRY(launch_remap(ctx->bufs[ctx->cur], ctx->peers[ctx->cur ^ 1], (int64_t)1 << ctx->L, ctx->L - ctx->gbits,
                        ctx->rank, ctx->num_sms, ctx->stream));
  ctx->stats.kernel_launches_total++;
  qaa_status st = shard_barrier(ctx);
  if (st) return st;
  ctx->cur ^= 1;
  ctx->state = ctx->bufs[ctx->cur];
  return QAA_OK;
}


// Sharded evolve (plan.hpp ShardPass): every phase ends with a
// pass whose tiles are stored straight into the peers' other shard buffer
// (the bit swap of the top local and the rank qubits), then one phase barrier
// (device side by default: the whole evolve is enqueued without a host sync).

qaa_status evolve_sharded(qaa_ctx* ctx, int64_t K, const std::vector<StepCoef>& sc, const double2* dphi,
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
        a.v2 = ctx->super_v2;
        a.done_shift = ctx->super_v2 ? 3 : 0;
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
        qaa_status st = shard_barrier(ctx);
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
      qaa_status st = shard_barrier(ctx);
      if (st) return st;
      ctx->cur ^= 1;
      ctx->state = ctx->bufs[ctx->cur];
    }
  }
  (void)P;
  return QAA_OK;
}
