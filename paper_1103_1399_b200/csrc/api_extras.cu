// api_extras.cu -- NEXT rows: spectrum (F3), energy-table timing (F2), batched sweep (F1), plan description.
#include <algorithm>
#include <vector>

#include "api_internal.hpp"

extern "C" {

qaa_status qaa_spectrum(qaa_ctx* ctx, double s, int kmax, int nev, double* evals, double* overlap, int* iters) {
  QAA_NVTX("qaa_spectrum");
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

qaa_status qaa_time_energy_table(qaa_ctx* ctx, int reps, double* ms) {
  QAA_NVTX("qaa_time_energy_table");
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
  QAA_NVTX("qaa_sweep");
  CHECK_CTX();
  if (!ctx->loaded) return fail(ctx, QAA_E_STATE, "sweep before load_instance");
  const bool wide = (ctx->warptile == 2 && ctx->L <= WARP_MAX_L &&
                     (((int64_t)1 << (ctx->L - 9)) + 7) / 8 <= ctx->num_sms) ||  // warp-tile teams (test hook)
                    (ctx->warptile == 3 && ctx->L <= WARP_MAX_L);                  // quad-warp teams (test hook)
  if (ctx->world != 1 || (ctx->L > SWEEP_MAX_L && !wide))
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
  // replicas are launched longest first (cluster slots free up in order, the
  // longest replica never waits behind short ones); results are mapped back below
  std::vector<int> ord((size_t)nrep);
  for (int r = 0; r < nrep; r++) ord[(size_t)r] = r;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return K[x] > K[y]; });
  int64_t row = 0;
  for (int i = 0; i < nrep; i++) {
    const int r = ord[(size_t)i];
    hK[i] = K[r];
    hoff[i] = row;
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
  const int wteam = ctx->L >= WARP_MIN_L ? (int)((((int64_t)1 << (ctx->L - 9)) + 7) / 8) : 0;
  // quad-warp teams (QAA_OPT_WARPTILE 3, n = 13..21; a test hook: at n = 13..16 measured
  // 4-7e5 replica-steps/s against 4.2-5.3e5 for the default clusters below, but with
  // run-to-run outliers 3-5x slower -- team barriers of ~1000 co-resident CTAs)
  const bool quad = ctx->L >= WARP_MIN_L && ctx->warptile == 3 && ctx->L <= WARP_MAX_L;
  if (quad || (ctx->warptile == 2 && ctx->L >= WARP_MIN_L && ctx->L <= WARP_MAX_L && wteam <= ctx->num_sms)) {
    // teams of CTAs, one replica at a time per team (warp_evolve.cu). Quad-warp
    // teams (qaa_quad_sweep): 128-thread CTAs, several per SM, `tpc` tiles per CTA
    // and pass, tpc chosen to maximise concurrent replicas / (tpc + one barrier).
    // Single-warp teams (qaa_warp_sweep, QAA_OPT_WARPTILE 2): 8 tiles per CTA;
    // measured no faster than the clusters below at n = 13..16, extends to n <= 21.
    qaa_status st = ensure_warp_tables(ctx);
    if (st) return st;
    const int P = warp_group_count(ctx->L);
    int team = wteam, nteams = std::min(nrep, ctx->num_sms / std::max(1, wteam));
    if (quad) {
      const int64_t ntiles = (int64_t)1 << (ctx->L - 9);
      const int64_t slots = (int64_t)ctx->num_sms * std::max(1, quad_sweep_max_active());
      double best = -1.0;
      const int64_t force = (ctx->sweep_tune & 15) ? ((int64_t)1 << ((ctx->sweep_tune & 15) - 1)) : 0;
      for (int64_t tpc = 1; tpc <= ntiles; tpc *= 2) {
        if (force && tpc != force) continue;
        const int64_t tm = ntiles / tpc, nt = std::min<int64_t>(nrep, slots / tm);
        if (nt < 1) continue;
        const double score = (double)nt / (double)(tpc + 1);
        if (score > best) {
          best = score;
          team = (int)tm;
          nteams = (int)nt;
        }
      }
    }
    std::vector<WarpPass> recs;
    std::vector<int64_t> poff((size_t)nrep), plen((size_t)nrep);
    std::vector<PassPlan> plan;
    for (int i = 0; i < nrep; i++) {
      build_pass_schedule(P, hK[i], 1, &plan);
      if (ctx->order == 2) plan.back().d_step = hK[i];
      poff[(size_t)i] = (int64_t)recs.size();
      plen[(size_t)i] = (int64_t)plan.size();
      for (const PassPlan& pp : plan) {
        WarpPass w{pp.group, 0, 0, 0.0, 0.0};
        if (pp.pre_step >= 0) {
          w.flags |= WP_PRE | (hform[hoff[i] + pp.pre_step] ? 8 : 0);
          w.cpre = hcoef[hoff[i] + pp.pre_step];
        }
        if (pp.d_step >= 0) {
          w.flags |= WP_D;
          w.d = hoff[i] + pp.d_step;
        }
        if (pp.post_step >= 0) {
          w.flags |= WP_POST | (hform[hoff[i] + pp.post_step] ? 16 : 0);
          w.cpost = hcoef[hoff[i] + pp.post_step];
        }
        recs.push_back(w);
      }
    }
    const size_t rec_b = recs.size() * sizeof(WarpPass), arr_b = (size_t)nrep * sizeof(int64_t);
    const size_t state_b = (size_t)nteams << ctx->L << 4;
    const size_t part_b = (size_t)nteams * team * 8 * sizeof(double), bar_b = (size_t)nteams * 128;
    const size_t o_off = (rec_b + 255) & ~(size_t)255, o_len = o_off + ((arr_b + 255) & ~(size_t)255),
                 o_state = o_len + ((arr_b + 255) & ~(size_t)255), o_part = o_state + state_b,
                 o_bar = o_part + ((part_b + 255) & ~(size_t)255), need = o_bar + bar_b;
    st = ensure_buffer(ctx, &ctx->d_wsweep, &ctx->d_wsweep_cap, need);
    if (st) return st;
    char* wb = (char*)ctx->d_wsweep;
    CUDA_TRY(cudaMemcpyAsync(wb, recs.data(), rec_b, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(wb + o_off, poff.data(), arr_b, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(wb + o_len, plen.data(), arr_b, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemsetAsync(wb + o_bar, 0, bar_b, ctx->stream));
    WarpSweepArgs wa;
    memset(&wa, 0, sizeof wa);
    wa.L = ctx->L;
    wa.amp0 = a.amp0;
    for (int g = 0; g < ctx->wt_groups; g++) {
      wa.geo[g] = ctx->wgeo[g];
      wa.Eg[g] = ctx->Ewt[g];
    }
    wa.plan = (const WarpPass*)wb;
    wa.plan_off = (const int64_t*)(wb + o_off);
    wa.plan_len = (const int64_t*)(wb + o_len);
    wa.nrep = nrep;
    wa.phi_all = a.phi_all;
    wa.n_phi = n_phi;
    wa.team = team;
    wa.poll_ns = ctx->sweep_tune >> 4;
    wa.scratch = (double2*)(wb + o_state);
    wa.partial = (double*)(wb + o_part);
    wa.bar = (unsigned*)(wb + o_bar);
    wa.out = dout;
    if (quad)
      CUDA_TRY(launch_quad_sweep(wa, nteams * team, ctx->stream));
    else
      CUDA_TRY(launch_warp_sweep(wa, nteams * team, ctx->stream));
    ctx->stats.warp_launches++;
    // the host vectors above must outlive the async copies
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  } else if (ctx->cluster_evolve && ctx->L >= 13 && ctx->L <= 16) {
    // one register-resident cluster of 2^(n-12) CTAs per replica (cluster_evolve.cu)
    ClusterArgs ca;
    memset(&ca, 0, sizeof ca);
    ca.E = ctx->E;
    ca.L = ctx->L;
    ca.amp0 = a.amp0;
    ca.Krep = a.K;
    ca.row_off = a.row_off;
    ca.phi_all = a.phi_all;
    ca.n_phi = n_phi;
    ca.coef = a.coef;
    ca.form = a.form;
    ca.final_d = a.final_d;
    ca.out = dout;
    CUDA_TRY(launch_cluster_evolve(ca, nrep, ctx->stream));
    ctx->stats.cluster_launches++;
  } else if (ctx->L >= 10)  // register phases, one CTA (n <= 13) or one cluster (n = 14..16) per replica
    CUDA_TRY(launch_sweep_cluster(a, nrep, ctx->stream));
  else
    CUDA_TRY(launch_sweep(a, nrep, ctx->stream));
  ctx->stats.kernel_launches_total++;
  double* hres = (double*)ctx->h_out;  // pinned; reused when nrep fits
  std::vector<double> tmp;
  if (nrep > 64) {
    tmp.resize((size_t)nrep);
    hres = tmp.data();
  }
  CUDA_TRY(cudaMemcpyAsync(hres, dout, (size_t)nrep * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < nrep; i++) out[ord[(size_t)i]] = hres[i];
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
