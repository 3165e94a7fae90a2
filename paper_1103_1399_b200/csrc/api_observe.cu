// api_observe.cu -- observables (A9) and state / energy-table copies.
#include "api_internal.hpp"

// ------------------------------------------------------------------ observables
qaa_status ensure_part(qaa_ctx* ctx, size_t doubles) {
  void* p = ctx->d_part;
  qaa_status st = ensure_buffer(ctx, &p, &ctx->d_part_cap, doubles * sizeof(double));
  ctx->d_part = (double*)p;
  return st;
}

extern "C" {

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

// sx[phys] = local pair sums of sigma^x on the rotated bits of every group
static qaa_status obs_sigma_local(qaa_ctx* ctx, double* sx);

// the rank qubits (logical L..n-1, layout A): every rank dots its shard with
// each partner rank's shard read in place over NVLink (16 B/amp per rank qubit,
// nothing moved; round 1 swapped layouts twice: 2 x 16 B/amp of peer stores).
// Device-side barriers on both sides: the peers' states are final before the
// reads, and nobody overwrites its buffer before every rank has read it.
static qaa_status obs_sigma_global(qaa_ctx* ctx, double* sx) {
  const int64_t N = (int64_t)1 << ctx->L;
  PeerDotArgs a;
  memset(&a, 0, sizeof a);
  a.g = ctx->gbits;
  for (int t = 0; t < ctx->gbits; t++) a.peer[t] = ctx->peers[ctx->cur][ctx->rank ^ (1 << t)];
  int grid = ctx->num_sms * RED_BLOCKS_PER_SM;
  if ((int64_t)grid * 256 > N) grid = (int)std::max<int64_t>(1, (N + 255) / 256);
  qaa_status st = ensure_part(ctx, (size_t)grid * 3);
  if (st) return st;
  st = shard_barrier(ctx);
  if (st) return st;
  CUDA_TRY(launch_obs_peer_dot(ctx->state, a, N, ctx->d_part, grid, ctx->stream));
  st = shard_barrier(ctx);
  if (st) return st;
  CUDA_TRY(launch_reduce_partials(ctx->d_part, grid, 3, 3, ctx->d_out, ctx->stream));
  ctx->stats.kernel_launches_total += 2;
  CUDA_TRY(cudaMemcpyAsync(ctx->h_out, ctx->d_out, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  for (int t = 0; t < ctx->gbits; t++) sx[ctx->L + t] = ctx->h_out[t];
  return QAA_OK;
}

// sx[j] = <sigma^x_j> for all n qubits (collective when sharded)
static qaa_status obs_sigma(qaa_ctx* ctx, double* sx) {
  for (int j = 0; j < ctx->n; j++) sx[j] = 0.0;
  qaa_status st = obs_sigma_local(ctx, sx);
  if (st) return st;
  if (ctx->world > 1) {
    st = obs_sigma_global(ctx, sx);
    if (st) return st;
    st = comm_sum(ctx, sx, ctx->n);
    if (st) return st;
  }
  return QAA_OK;
}

static qaa_status obs_sigma_local(qaa_ctx* ctx, double* sx) {
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
      SigmaArgs a;
      memset(&a, 0, sizeof a);
      a.psi = ctx->state;
      a.k = TILE_BITS;
      a.mask = g.rot_local;
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
    for (int j = 0; j < a.k; j++)
      if (a.mask >> j & 1) sx[a.phys[j]] = 2.0 * ctx->h_out[j];
  }
  return QAA_OK;
}

qaa_status qaa_success_prob(qaa_ctx* ctx, double* out) {
  QAA_NVTX("qaa_success_prob");
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
  QAA_NVTX("qaa_norm2");
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
  QAA_NVTX("qaa_sigma_x");
  CHECK_CTX();
  if (!out) return fail(ctx, QAA_E_USAGE, "out is NULL");
  if (!ctx->loaded || !ctx->initialized) return fail(ctx, QAA_E_STATE, "sigma_x before init");
  return obs_sigma(ctx, out);
}

qaa_status qaa_energy(qaa_ctx* ctx, double s, double* out) {
  QAA_NVTX("qaa_energy");
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
  QAA_NVTX("qaa_copy_state");
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
  QAA_NVTX("qaa_set_state");
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

}  // extern "C"
