// api_evolve.cu -- qaa_evolve: host coefficient builder (H1), pass plan (H2) and the pass / L2-blocked step launches.
#include "api_internal.hpp"


// One row of the coefficient table: the X coefficient of a step whose H_B
// weight is wb (tan or cot of beta = dt wb / 2) and Phi[e] = e^{-i theta e} *
// (X normalisation)^n. theta is dt wP(s) for Lie-Trotter; Strang passes the
// merged half steps (R7, §4).
void build_step(double T, int64_t K, double wb, double theta, int n, int n_phi, double2* phi_row,
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

qaa_status ensure_events(qaa_ctx* ctx, size_t need) {
  while (ctx->ev_pool.size() < need) {
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreate(&a));
    CUDA_TRY(cudaEventCreate(&b));
    ctx->ev_pool.push_back({a, b});
  }
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
bool super_usable(qaa_ctx* ctx) {
  const size_t P = ctx->geom.groups.size();
  if (!(ctx->super_mode && ctx->world == 1 && use_tma(ctx) && (P == 3 || P == 4) &&
        (int)ctx->emax + 1 <= TMA_MAX_PHI))
    return false;
  for (size_t k = 1; k < P; k++)
    if (!ctx->super_ok[k] || (!ctx->super_force && ctx->super_static[k].nchunks < SUPER_MIN_CHUNKS)) return false;
  return true;
}

static qaa_status launch_super_pair(qaa_ctx* ctx, int k, double t_g0, double t_pre, double t_post,
                                    const double2* phi, int n_phi, bool rev = false) {
  QAA_NVTX(phi ? "qaa_superpass (Trotter step)" : "qaa_superpass (plain pair)");
  int64_t nch = 0;
  for (size_t g = 1; g < ctx->geom.groups.size() && g < 4; g++) nch = std::max(nch, ctx->super_static[g].nchunks);
  const size_t need = 2 * (size_t)nch * sizeof(unsigned) + 256;
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
  a.lag = ctx->super_lag;
  a.queue = ctx->super_dynamic ? (unsigned long long*)ctx->d_super : nullptr;
  a.done = (unsigned*)((char*)ctx->d_super + 256);
  a.doneB = a.done + a.nchunks;
  a.split_a = ctx->super_split;
  a.v2 = ctx->super_v2 && !ctx->super_split;
  a.pub_batch = ctx->super_pub & 15;
  a.early = (ctx->super_pub >> 4) & 1;
  a.tm_flags = ctx->super_tm_flags;  // v2: 1 = publish after the next landed read, 2 = right after the stores
  a.diag = ctx->diag;
  a.rev = rev ? 1 : 0;
  a.done_shift = a.v2 ? 3 : 0;
  CUDA_TRY(cudaMemsetAsync(ctx->d_super, 0, 256 + 2 * (size_t)a.nchunks * sizeof(unsigned), ctx->stream));
  // phi == nullptr: the plain pair of a four-group plan (kernel variant without D)
  const bool bd = phi != nullptr;
  cudaError_t e;
  if (ctx->super_tm && !ctx->tm_built) {
    qaa_status st = build_tm(ctx);
    if (st) return st;
  }
  if (ctx->super_tm && ctx->tm_ok[k] && (!bd || ctx->Eg_tm[k])) {
    if (bd) a.gk.Eg = ctx->Eg_tm[k];
    a.done_shift = 3;  // per-warp publish
    a.split_a = 0;     // split roles: shared-memory kernel only
    a.tm_flags = ctx->super_tm_flags;
    if (a.tm_flags & 8) {  // diagnostics: wait / program cycle counters, read by qaa_get_stats
      if (!ctx->d_tm_diag) {
        CUDA_TRY(cudaMalloc(&ctx->d_tm_diag, 8 * sizeof(unsigned long long)));
        CUDA_TRY(cudaMemsetAsync(ctx->d_tm_diag, 0, 8 * sizeof(unsigned long long), ctx->stream));
      }
      a.dbg = ctx->d_tm_diag;
    }
    // the swizzled map splits the rows off as their own dimension: its own coordinates
    a.gk.ndims = ctx->tm_geo[k].ndims;
    for (int d = 0; d < 5; d++) a.gk.dim_seg[d] = ctx->tm_geo[k].dim_seg[d];
    e = launch_superpass_tm(&ctx->tmaps_sw[k], a, ctx->super_groups, bd, ctx->super_grid ? ctx->super_grid : ctx->num_sms,
                            ctx->stream);
    ctx->stats.tm_launches++;
  } else if (ctx->super_pw) {
    a.qab = (unsigned*)((char*)ctx->d_super + 16);
    a.tm_flags = ctx->super_tm_flags;
    if (a.tm_flags & 8) {
      if (!ctx->d_tm_diag) {
        CUDA_TRY(cudaMalloc(&ctx->d_tm_diag, 8 * sizeof(unsigned long long)));
        CUDA_TRY(cudaMemsetAsync(ctx->d_tm_diag, 0, 8 * sizeof(unsigned long long), ctx->stream));
      }
      a.dbg = ctx->d_tm_diag;
    }
    e = launch_superpass_pw(&ctx->tmaps[(size_t)k], a, (gk.rot_local >> 3) & 1, bd,
                            ctx->super_grid ? ctx->super_grid : ctx->num_sms, ctx->stream);
    ctx->stats.pw_launches++;
  } else {
    if (a.tm_flags & 8) {  // diagnostics: deferred group-k tiles and their wait cycles (tm_diag[5..7])
      if (!ctx->d_tm_diag) {
        CUDA_TRY(cudaMalloc(&ctx->d_tm_diag, 8 * sizeof(unsigned long long)));
        CUDA_TRY(cudaMemsetAsync(ctx->d_tm_diag, 0, 8 * sizeof(unsigned long long), ctx->stream));
      }
      a.dbg = ctx->d_tm_diag;
    }
    e = launch_superpass(&ctx->tmaps[(size_t)k], a, (gk.rot_local >> 3) & 1, ctx->super_groups, bd,
                         ctx->super_grid ? ctx->super_grid : ctx->num_sms, ctx->stream);
  }
  return e == cudaSuccess ? QAA_OK : fail(ctx, QAA_E_CUDA, "superpass launch failed: %s", cudaGetErrorString(e));
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


// Persistent evolve (pass_fast.cu qaa_persist): 13 <= L <= 21 with the
// automatic kernel choice, first-order steps in tangent form, every pass one of
// the compiled-in register programs. One cooperative launch for all K steps
// (the state stays in L2), a grid barrier between passes. Returns false (and
// leaves *st untouched) when not applicable.
static bool pass_fast_prog(const qaa_ctx* ctx, const PassPlan& pp, const std::vector<StepCoef>& sc, int* fp_out) {
  const Group& gr = ctx->geom.groups[(size_t)pp.group];
  const bool pre = pp.pre_step >= 0, d = pp.d_step >= 0, post = pp.post_step >= 0;
  int fp = -1;
  if (pp.group == 0) {
    if (!pre && d && post) fp = FP_G0_DPOST;
    else if (pre && !d && !post) fp = FP_G0_PRE;
    else if (pre && d && post) fp = FP_G0_PRE_D_POST;
  } else if ((gr.rot_local & ~0xFF8u) == 0) {
    if (pre && !d && !post) fp = FP_GK_PRE;
    else if (d && post) fp = FP_GK_PRE_D_POST;
  }
  if ((pre && sc[(size_t)pp.pre_step].form != 0) || (post && sc[(size_t)pp.post_step].form != 0)) fp = -1;
  *fp_out = fp;
  return fp >= 0;
}

static bool try_persist(qaa_ctx* ctx, const std::vector<PassPlan>& plan, const std::vector<StepCoef>& sc,
                        const double2* dphi, const double* dcoef, int n_phi, qaa_status* st) {
  if (!ctx->persist || ctx->world != 1 || ctx->kernel_mode != 2 || ctx->order != 1) return false;
  if (ctx->L < 13 || ctx->L > PERSIST_MAX_L || ctx->geom.groups.size() > 4 || n_phi > 256) return false;
  std::vector<PersistPass> recs(plan.size());
  for (size_t i = 0; i < plan.size(); i++) {
    const PassPlan& pp = plan[i];
    int fp;
    if (!pass_fast_prog(ctx, pp, sc, &fp)) return false;
    const Group& gr = ctx->geom.groups[(size_t)pp.group];
    // LANE3 (rotate tile bit 3 with lane shuffles) exists only for group k > 0 programs
    const int lane3 = pp.group > 0 ? (int)((gr.rot_local >> 3) & 1) : 0;
    recs[i] = PersistPass{fp, lane3, pp.group, (int)pp.pre_step, (int)pp.d_step, (int)pp.post_step};
  }
  const int maxg = persist_max_grid(ctx->num_sms);
  if (maxg <= 0) return false;
  const size_t bytes = recs.size() * sizeof(PersistPass) + 256;
  if (ctx->d_persist_cap < bytes) {
    CUDA_TRY_ST(cudaStreamSynchronize(ctx->stream));
    *st = ensure_buffer(ctx, &ctx->d_persist, &ctx->d_persist_cap, bytes);
    if (*st) return true;
  }
  unsigned* bar = (unsigned*)ctx->d_persist;
  PersistPass* dpass = (PersistPass*)((char*)ctx->d_persist + 256);
  CUDA_TRY_ST(cudaMemsetAsync(bar, 0, 256, ctx->stream));
  CUDA_TRY_ST(cudaMemcpyAsync(dpass, recs.data(), recs.size() * sizeof(PersistPass), cudaMemcpyHostToDevice,
                              ctx->stream));
  PersistLaunch L;
  L.psi = ctx->state;
  L.E = ctx->E;
  L.passes = dpass;
  L.npass = (int)recs.size();
  L.phi_all = dphi;
  L.n_phi = n_phi;
  L.coef = dcoef;
  L.ngroups = (int)ctx->geom.groups.size();
  L.groups = ctx->geom.groups.data();
  L.bar = bar;
  const int grid = (int)std::min<int64_t>(ctx->geom.groups[0].ntiles, maxg);
  size_t ev = ctx->ev_used;
  if (ctx->profile) {
    *st = ensure_events(ctx, ev + 1);
    if (*st) return true;
    CUDA_TRY_ST(cudaEventRecord(ctx->ev_pool[ev].first, ctx->stream));
  }
  CUDA_TRY_ST(launch_persist(L, grid, ctx->stream));
  if (ctx->profile) {
    CUDA_TRY_ST(cudaEventRecord(ctx->ev_pool[ev].second, ctx->stream));
    ctx->ev_used = ev + 1;
  }
  ctx->stats.pass_launches++;
  ctx->stats.persist_launches++;
  ctx->stats.kernel_launches_total++;
  *st = QAA_OK;
  return true;
}

// Warp-tile groups (warp_evolve.cu): group 0 = bits 0..8; group g >= 1 = bits
// {0, 1} + fillers {2, ...} (not rotated) + the next <= 7 bits (rotated)
int warp_group_count(int L) { return 1 + (L - 9 + 6) / 7; }
void build_warp_geo(int L, WarpGeo* out, int* ngroups) {
  int ng = 0;
  WarpGeo g0;
  memset(&g0, 0, sizeof g0);
  for (int b = 0; b < 9; b++) g0.phys[b] = b;
  g0.rot = 0x1FFu;
  out[ng++] = g0;
  for (int next = 9; next < L;) {
    const int hb = std::min(7, L - next);
    WarpGeo g;
    memset(&g, 0, sizeof g);
    int t = 0;
    for (int b = 0; b < 2 + (7 - hb); b++) g.phys[t++] = b;  // row bits + fillers
    for (int b = 0; b < hb; b++) {
      g.rot |= 1u << t;
      g.phys[t++] = next + b;
    }
    next += hb;
    out[ng++] = g;
  }
  for (int k = 0; k < ng; k++) {
    bool in[64] = {false};
    for (int b = 0; b < 9; b++) in[out[k].phys[b]] = true;
    out[k].nfree = 0;
    for (int p = 0; p < L; p++)
      if (!in[p]) out[k].free_bits[out[k].nfree++] = p;
  }
  *ngroups = ng;
}

qaa_status ensure_warp_tables(qaa_ctx* ctx) {
  if (!ctx->wt_built) {
    build_warp_geo(ctx->L, ctx->wgeo, &ctx->wt_groups);
    for (int g = 0; g < ctx->wt_groups; g++) {
      if (ctx->Ewt[g]) cudaFree(ctx->Ewt[g]);
      ctx->Ewt[g] = nullptr;
      CUDA_TRY(cudaMalloc(&ctx->Ewt[g], (size_t)1 << ctx->L));
      CUDA_TRY(launch_warp_energy(ctx->E, ctx->Ewt[g], ctx->wgeo[g], ctx->L, ctx->num_sms, ctx->stream));
      ctx->stats.kernel_launches_total++;
    }
    ctx->wt_built = true;
  }
  return QAA_OK;
}

static qaa_status run_warp_evolve(qaa_ctx* ctx, const WarpPass* dplan, int64_t npass, const double2* dphi,
                                  const double* dcoef, const int32_t* dform, int n_phi) {
  QAA_NVTX("qaa_warp_evolve (all passes)");
  {
    qaa_status st = ensure_warp_tables(ctx);
    if (st) return st;
    st = ensure_buffer(ctx, &ctx->d_persist, &ctx->d_persist_cap, 256);
    if (st) return st;
  }
  WarpEvolveArgs wa;
  memset(&wa, 0, sizeof wa);
  wa.psi = ctx->state;
  wa.L = ctx->L;
  for (int g = 0; g < ctx->wt_groups; g++) {
    wa.geo[g] = ctx->wgeo[g];
    wa.Eg[g] = ctx->Ewt[g];
  }
  wa.plan = dplan;
  wa.npass = npass;
  wa.phi_all = dphi;
  wa.n_phi = n_phi;
  wa.coef = dcoef;
  wa.form = dform;
  wa.bar = (unsigned*)ctx->d_persist;
  CUDA_TRY(cudaMemsetAsync(ctx->d_persist, 0, 16, ctx->stream));
  size_t ev = ctx->ev_used;
  if (ctx->profile) {
    qaa_status st = ensure_events(ctx, ev + 1);
    if (st) return st;
    CUDA_TRY(cudaEventRecord(ctx->ev_pool[ev].first, ctx->stream));
  }
  // grid: fewer, fuller CTAs make the per-pass grid barrier cheaper (tuning hook
  // QAA_OPT_WARP_GRID = ctas * 16 + warps per CTA; 0 = automatic)
  int grid = ctx->num_sms, warps = 8;
  if (ctx->warp_grid) {
    grid = std::min(ctx->num_sms, ctx->warp_grid >> 4);
    warps = ctx->warp_grid & 15;
  }
  if (ctx->warptile == 3 || ctx->warptile == 1) {
    // quad-warp tiles: one 128-thread CTA per tile while they fit co-resident
    const int64_t ntiles = (int64_t)1 << (ctx->L - 9);
    const int cap = ctx->num_sms * std::max(1, quad_evolve_max_active());
    grid = (int)std::min<int64_t>(ntiles, cap);
    if (ctx->warp_grid) grid = std::min(grid, ctx->warp_grid >> 4);
    CUDA_TRY(launch_quad_evolve(wa, grid, ctx->stream));
  } else {
    CUDA_TRY(launch_warp_evolve(wa, grid, warps, ctx->stream));
  }
  if (ctx->profile) {
    CUDA_TRY(cudaEventRecord(ctx->ev_pool[ev].second, ctx->stream));
    ctx->ev_used = ev + 1;
  }
  ctx->stats.pass_launches++;
  ctx->stats.warp_launches++;
  ctx->stats.kernel_launches_total++;
  return QAA_OK;
}

extern "C" {

qaa_status qaa_evolve(qaa_ctx* ctx, double T, int64_t K, const double* schedule) {
  QAA_NVTX("qaa_evolve");
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
  // the warp-tile path stages its pass records behind the coefficients
  const bool use_warp = ctx->warptile && ctx->world == 1 && ctx->kernel_mode == 2 && ctx->L >= WARP_MIN_L &&
                        ctx->L <= (ctx->warptile >= 2 ? WARP_MAX_L : WARP_AUTO_MAX_L);
  std::vector<PassPlan> wplan;
  if (use_warp) {
    build_pass_schedule(warp_group_count(ctx->L), K, 1, &wplan);
    if (ctx->order == 2) wplan.back().d_step = K;  // Strang closing half step
  }
  const size_t wplan_off = (phi_bytes + coef_bytes + form_bytes + 15) & ~(size_t)15;
  const size_t total = (use_warp ? wplan_off + wplan.size() * sizeof(WarpPass) : phi_bytes + coef_bytes + form_bytes) + 256;
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
  if (use_warp) {
    WarpPass* hp = (WarpPass*)((char*)ctx->h_coef + wplan_off);
    for (size_t i = 0; i < wplan.size(); i++) {
      const PassPlan& pp = wplan[i];
      WarpPass w{pp.group, 0, 0, 0.0, 0.0};
      if (pp.pre_step >= 0) {
        w.flags |= WP_PRE | (sc[(size_t)pp.pre_step].form ? 8 : 0);
        w.cpre = sc[(size_t)pp.pre_step].coef;
      }
      if (pp.d_step >= 0) {
        w.flags |= WP_D;
        w.d = pp.d_step;
      }
      if (pp.post_step >= 0) {
        w.flags |= WP_POST | (sc[(size_t)pp.post_step].form ? 16 : 0);
        w.cpost = sc[(size_t)pp.post_step].coef;
      }
      hp[i] = w;
    }
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
  if (use_warp) {
    qaa_status st = run_warp_evolve(ctx, (const WarpPass*)((char*)ctx->d_coef + wplan_off), (int64_t)wplan.size(),
                                    dphi, dcoef, dform, n_phi);
    return st;
  }
  if (ctx->cluster_evolve && ctx->L >= 13 && ctx->L <= 16 && ctx->kernel_mode == 2) {
    // the whole evolution in one launch, state in one cluster's registers
    ClusterArgs ca;
    memset(&ca, 0, sizeof ca);
    ca.psi = ctx->state;
    ca.E = ctx->E;
    ca.L = ctx->L;
    ca.K = K;
    ca.phi_all = dphi;
    ca.n_phi = n_phi;
    ca.coef = dcoef;
    ca.form = dform;
    ca.final_d = ctx->order == 2 ? 1 : 0;
    size_t ev = ctx->ev_used;
    if (ctx->profile) {
      qaa_status st = ensure_events(ctx, ev + 1);
      if (st) return st;
      CUDA_TRY(cudaEventRecord(ctx->ev_pool[ev].first, ctx->stream));
    }
    CUDA_TRY(launch_cluster_evolve(ca, 1, ctx->stream));
    if (ctx->profile) {
      CUDA_TRY(cudaEventRecord(ctx->ev_pool[ev].second, ctx->stream));
      ctx->ev_used = ev + 1;
    }
    ctx->stats.pass_launches++;
    ctx->stats.cluster_launches++;
    ctx->stats.kernel_launches_total++;
    return QAA_OK;
  }
  std::vector<PassPlan> plan;
  build_pass_schedule((int)ctx->geom.groups.size(), K, ctx->step_spanning, &plan);
  // Strang: the closing half step D_K follows the pass that completes X_{K-1}
  // (its program becomes rotate + D; it runs on the generic kernel)
  if (ctx->order == 2) plan.back().d_step = K;
  {
    qaa_status st = QAA_OK;
    if (try_persist(ctx, plan, sc, dphi, dcoef, n_phi, &st)) return st;
  }
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
  const bool rev = sup && ctx->super_rev && ctx->geom.groups.size() == 3 && ctx->super_groups == 2 && ctx->super_v2 &&
                   !ctx->super_tm && !ctx->super_pw && !ctx->super_split && !ctx->diag;
  for (size_t pi = 0; pi < plan.size(); pi++) {
    const PassPlan& pp = plan[pi];
    if (rev && pi + 1 < plan.size()) {
      // reversed pair [group k: (pre j), D_{j+1}, post j+1][group 0: pre j+1] -> one launch
      const PassPlan& pn = plan[pi + 1];
      if (pp.group >= 1 && pp.d_step >= 0 && pp.post_step >= 0 && pn.group == 0 && pn.pre_step == pp.post_step &&
          pn.d_step < 0 && pn.post_step < 0 && ctx->super_ok[(size_t)pp.group] &&
          (pp.pre_step < 0 || sc[(size_t)pp.pre_step].form == 0) && sc[(size_t)pp.post_step].form == 0) {
        if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev_pool[ctx->ev_used].first, ctx->stream));
        qaa_status st = launch_super_pair(ctx, pp.group, sc[(size_t)pn.pre_step].coef,
                                          pp.pre_step >= 0 ? sc[(size_t)pp.pre_step].coef : 0.0,
                                          sc[(size_t)pp.post_step].coef, dphi + (size_t)pp.d_step * n_phi, n_phi, true);
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
    if (sup && !rev && pi + 1 < plan.size()) {
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

}  // extern "C"
