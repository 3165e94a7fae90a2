/*
 * oracle/qaa_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the adiabatic 3-SAT Trotter
 * evolution (arxiv 1103.1399). It is NOT part of the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it. It shares no code, header, table or constant with the CUDA
 * library under paper_1103_1399_b200/ and never imports or links it.
 *
 * Every function follows one row of SURVEY.md §8(c) ("O-1".."O-8") and cites
 * the PAPER.md passage (P:n = line n of /root/reference/PAPER.md) it restates.
 * Arithmetic: IEEE binary64, round-to-nearest; no -ffast-math (R21).
 * Loops are written in the paper's order; OpenMP only splits independent
 * iterations (each output element is computed by exactly one thread with the
 * same arithmetic, so results do not depend on the thread count).
 *
 * Pins (tests/test_oracle_pins.py): brute-force boolean evaluation of the CNF
 * (E and Z), dense Kronecker-product expm products (whole step), closed forms
 * for s=0 / s=1 schedules, H_B spectrum, norm conservation, first-order
 * convergence to the exact evolution. No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_E_USAGE 1
#define ORACLE_E_INPUT 2
/* below this many amplitudes every loop runs on one thread (no OpenMP overhead) */
#define PAR_MIN ((int64_t)1 << 16)

/* O-1: basis index x, bit (j-1) of x holds variable x_j,
 * bit value 1 means "true". */
static int var_value(uint64_t x, int var /* 1-based */) { return (int)((x >> (var - 1)) & 1u); }

/* O-2 (P:84-91 definition of a clause as a disjunction of literals; P:193
 * "energy level proportional to the number of unsatisfied clauses", "sum of
 * smaller energy functions, one for each clause"; constant = 1, R4):
 * E(x) = number of clauses in the list (with multiplicity) in which every
 * literal is false. A literal l is true iff x_{|l|} == (l > 0). */
int oracle_energy_table(int n, int m, const int32_t* lits, uint16_t* E) {
  if (n < 1 || n > 40 || m < 0 || m > 65535) return ORACLE_E_USAGE;
  for (int i = 0; i < 3 * m; i++)
    if (lits[i] == 0 || lits[i] > n || lits[i] < -n) return ORACLE_E_INPUT;
  const int64_t N = (int64_t)1 << n;
#pragma omp parallel for schedule(static) if (N >= PAR_MIN)
  for (int64_t x = 0; x < N; x++) {
    int count = 0;
    for (int c = 0; c < m; c++) {
      int all_false = 1;
      for (int j = 0; j < 3; j++) {
        int32_t l = lits[3 * c + j];
        int var = l > 0 ? l : -l;
        int literal_true = (var_value((uint64_t)x, var) == (l > 0));
        if (literal_true) all_false = 0;
      }
      count += all_false;
    }
    E[x] = (uint16_t)count;
  }
  return ORACLE_OK;
}

/* O-2 at selected assignments: out[i] = E(xs[i]) (same definition as
 * oracle_energy_table, evaluated one x at a time so huge n can be sampled). */
int oracle_energy_at(int n, int m, const int32_t* lits, const uint64_t* xs, int64_t count, uint16_t* out) {
  if (n < 1 || n > 63 || m < 0 || m > 65535) return ORACLE_E_USAGE;
  for (int i = 0; i < 3 * m; i++)
    if (lits[i] == 0 || lits[i] > n || lits[i] < -n) return ORACLE_E_INPUT;
  for (int64_t i = 0; i < count; i++) {
    int count_c = 0;
    for (int c = 0; c < m; c++) {
      int all_false = 1;
      for (int j = 0; j < 3; j++) {
        int32_t l = lits[3 * c + j];
        int var = l > 0 ? l : -l;
        if (var_value(xs[i], var) == (l > 0)) all_false = 0;
      }
      count_c += all_false;
    }
    out[i] = (uint16_t)count_c;
  }
  return ORACLE_OK;
}

/* O-4: psi_g(0) = 2^{-n/2} sum_x |x>, phase 0. psi is interleaved
 * (re, im) pairs, length 2*2^n doubles. */
int oracle_init_uniform(int n, double* psi) {
  if (n < 1 || n > 40) return ORACLE_E_USAGE;
  const int64_t N = (int64_t)1 << n;
  const double a = 1.0 / sqrt(ldexp(1.0, n));
  for (int64_t x = 0; x < N; x++) { psi[2 * x] = a; psi[2 * x + 1] = 0.0; }
  return ORACLE_OK;
}

/* O-6 (P:193 final Hamiltonian H_P = diag(E); Eq. 1 weight s): the diagonal
 * factor exp(-i*dt*s*H_P): psi[x] <- (cos phi - i sin phi) psi[x],
 * phi = (dt*s)*E(x). */
static void apply_D(int n, double* psi, const uint16_t* E, double dt, double s) {
  const int64_t N = (int64_t)1 << n;
  const double theta = dt * s;
#pragma omp parallel for schedule(static) if (N >= PAR_MIN)
  for (int64_t x = 0; x < N; x++) {
    double phi = theta * (double)E[x];
    double c = cos(phi), sn = -sin(phi); /* (c + i sn) = e^{-i phi} */
    double re = psi[2 * x], im = psi[2 * x + 1];
    psi[2 * x] = c * re - sn * im;
    psi[2 * x + 1] = c * im + sn * re;
  }
}

/* O-7 (Eq. 1 weight (1-s); H_B = sum_i (1 - sigma^x_i)/2, whose ground state
 * is the uniform superposition of P:73-76; R1/R2): the factor
 * exp(-i*dt*(1-s)*H_B) = prod_j exp(-i*beta*(1 - sigma^x_j)) with
 * beta = dt*(1-s)/2, and exp(-i beta (1 - sigma^x)) = g*(cos beta I + i sin beta sigma^x),
 * g = e^{-i beta}. So on every pair (x, y = x | 2^j) with bit j of x clear:
 *   (psi[x], psi[y]) <- (A psi[x] + B psi[y], B psi[x] + A psi[y]),
 *   A = g cos beta, B = g * (i sin beta). Qubits j = 0..n-1 ascending. */
static void apply_X(int n, double* psi, double dt, double s) {
  const int64_t N = (int64_t)1 << n;
  const double beta = 0.5 * dt * (1.0 - s);
  const double gr = cos(beta), gi = -sin(beta);            /* g = e^{-i beta} */
  const double Ar = gr * cos(beta), Ai = gi * cos(beta);    /* A = g cos beta */
  const double Br = -gi * sin(beta), Bi = gr * sin(beta);   /* B = g * (i sin beta) */
  for (int j = 0; j < n; j++) {
    const int64_t bit = (int64_t)1 << j;
#pragma omp parallel for schedule(static) if (N >= PAR_MIN)
    for (int64_t x = 0; x < N; x++) {
      if (x & bit) continue;
      int64_t y = x | bit;
      double xr = psi[2 * x], xi = psi[2 * x + 1];
      double yr = psi[2 * y], yi = psi[2 * y + 1];
      /* A*psi[x] + B*psi[y] */
      double nxr = (Ar * xr - Ai * xi) + (Br * yr - Bi * yi);
      double nxi = (Ar * xi + Ai * xr) + (Br * yi + Bi * yr);
      /* B*psi[x] + A*psi[y] */
      double nyr = (Br * xr - Bi * xi) + (Ar * yr - Ai * yi);
      double nyi = (Br * xi + Bi * xr) + (Ar * yi + Ai * yr);
      psi[2 * x] = nxr; psi[2 * x + 1] = nxi;
      psi[2 * y] = nyr; psi[2 * y + 1] = nyi;
    }
  }
}

/* O-5 (Eq. 1: H(s) = (1-s) H_i + s H_f, s = t/tau): K first-order
 * Trotter steps of length dt = T/K; step k uses s_k = sched[k] if given, else
 * the midpoint (k + 0.5)/K (R8). Each step applies D (O-6) first,
 * then X (O-7) (R7). psi is updated in place; no renormalisation. */
int oracle_evolve(int n, const uint16_t* E, double* psi, double T, int64_t K, const double* sched) {
  if (n < 1 || n > 40 || K < 1 || !(T >= 0.0) || !isfinite(T)) return ORACLE_E_USAGE;
  if (sched)
    for (int64_t k = 0; k < K; k++)
      if (!(sched[k] >= 0.0 && sched[k] <= 1.0)) return ORACLE_E_USAGE;
  const double dt = T / (double)K;
  for (int64_t k = 0; k < K; k++) {
    double s = sched ? sched[k] : ((double)k + 0.5) / (double)K;
    apply_D(n, psi, E, dt, s);
    apply_X(n, psi, dt, s);
  }
  return ORACLE_OK;
}

/* NEXT F4: second-order Strang splitting of the same step,
 * exp(-i dt s_k H_P / 2) exp(-i dt (1 - s_k) H_B) exp(-i dt s_k H_P / 2),
 * written literally step by step (no merging of adjacent half steps). */
int oracle_evolve_strang(int n, const uint16_t* E, double* psi, double T, int64_t K, const double* sched) {
  if (n < 1 || n > 40 || K < 1 || !(T >= 0.0) || !isfinite(T)) return ORACLE_E_USAGE;
  if (sched)
    for (int64_t k = 0; k < K; k++)
      if (!(sched[k] >= 0.0 && sched[k] <= 1.0)) return ORACLE_E_USAGE;
  const double dt = T / (double)K;
  for (int64_t k = 0; k < K; k++) {
    double s = sched ? sched[k] : ((double)k + 0.5) / (double)K;
    apply_D(n, psi, E, 0.5 * dt, s);
    apply_X(n, psi, dt, s);
    apply_D(n, psi, E, 0.5 * dt, s);
  }
  return ORACLE_OK;
}

/* NEXT F4 driving term (the paper's "driving Hamiltonian", form not
 * given; R3): H(s) = (1-s) H_B + s H_P + s(1-s)(gx H_B + gz H_P).
 * Step k: exp(-i dt wP H_P) then exp(-i dt wB H_B) with wP = s + gz s(1-s),
 * wB = (1-s) + gx s(1-s), written out like O-6/O-7. */
int oracle_evolve_driven(int n, const uint16_t* E, double* psi, double T, int64_t K, const double* sched,
                         double gx, double gz) {
  if (n < 1 || n > 40 || K < 1 || !(T >= 0.0) || !isfinite(T)) return ORACLE_E_USAGE;
  const int64_t N = (int64_t)1 << n;
  const double dt = T / (double)K;
  for (int64_t k = 0; k < K; k++) {
    double s = sched ? sched[k] : ((double)k + 0.5) / (double)K;
    double wP = s + gz * s * (1.0 - s);
    double wB = (1.0 - s) + gx * s * (1.0 - s);
    /* D: psi[x] <- e^{-i dt wP E(x)} psi[x] */
    for (int64_t x = 0; x < N; x++) {
      double phi = dt * wP * (double)E[x];
      double c = cos(phi), sn = -sin(phi);
      double re = psi[2 * x], im = psi[2 * x + 1];
      psi[2 * x] = c * re - sn * im;
      psi[2 * x + 1] = c * im + sn * re;
    }
    /* X: beta = dt wB / 2 on every qubit, as in O-7 */
    double beta = 0.5 * dt * wB;
    double gr = cos(beta), gi = -sin(beta);
    double Ar = gr * cos(beta), Ai = gi * cos(beta);
    double Br = -gi * sin(beta), Bi = gr * sin(beta);
    for (int j = 0; j < n; j++) {
      int64_t bit = (int64_t)1 << j;
      for (int64_t x = 0; x < N; x++) {
        if (x & bit) continue;
        int64_t y = x | bit;
        double xr = psi[2 * x], xi = psi[2 * x + 1], yr = psi[2 * y], yi = psi[2 * y + 1];
        psi[2 * x] = (Ar * xr - Ai * xi) + (Br * yr - Bi * yi);
        psi[2 * x + 1] = (Ar * xi + Ai * xr) + (Br * yi + Bi * yr);
        psi[2 * y] = (Br * xr - Bi * xi) + (Ar * yr - Ai * yi);
        psi[2 * y + 1] = (Br * xi + Bi * xr) + (Ar * yi + Ai * yr);
      }
    }
  }
  return ORACLE_OK;
}

/* O-8 helpers: pairwise (recursive halving) summation of f over [lo, hi) in a
 * fixed order, so the error grows like log2(N) * eps rather than N * eps. */
typedef double (*term_fn)(const void* ctx, int64_t x);
static double pairwise_sum(term_fn f, const void* ctx, int64_t lo, int64_t hi) {
  if (hi - lo <= 64) {
    double s = 0.0;
    for (int64_t x = lo; x < hi; x++) s += f(ctx, x);
    return s;
  }
  int64_t mid = lo + (hi - lo) / 2;
  double a, b;
  if (hi - lo >= ((int64_t)1 << 20)) {
#pragma omp task shared(a)
    a = pairwise_sum(f, ctx, lo, mid);
#pragma omp task shared(b)
    b = pairwise_sum(f, ctx, mid, hi);
#pragma omp taskwait
  } else {
    a = pairwise_sum(f, ctx, lo, mid);
    b = pairwise_sum(f, ctx, mid, hi);
  }
  return a + b;
}
static double sum_over(term_fn f, const void* ctx, int64_t N) {
  double r = 0.0;
#pragma omp parallel if (N >= PAR_MIN)
#pragma omp single
  r = pairwise_sum(f, ctx, 0, N);
  return r;
}

typedef struct { const double* psi; const uint16_t* E; int64_t bit; } obs_ctx;
static double t_norm2(const void* c, int64_t x) {
  const obs_ctx* o = (const obs_ctx*)c;
  return o->psi[2 * x] * o->psi[2 * x] + o->psi[2 * x + 1] * o->psi[2 * x + 1];
}
static double t_hp(const void* c, int64_t x) { /* E(x) |psi[x]|^2 */
  const obs_ctx* o = (const obs_ctx*)c;
  return (double)o->E[x] * t_norm2(c, x);
}
static double t_succ(const void* c, int64_t x) { /* [E(x) == 0] |psi[x]|^2 (O-3) */
  const obs_ctx* o = (const obs_ctx*)c;
  return o->E[x] == 0 ? t_norm2(c, x) : 0.0;
}
static double t_sx(const void* c, int64_t x) { /* 2 Re(conj(psi[x]) psi[x ^ 2^j]) for bit j of x clear */
  const obs_ctx* o = (const obs_ctx*)c;
  if (x & o->bit) return 0.0;
  int64_t y = x | o->bit;
  return 2.0 * (o->psi[2 * x] * o->psi[2 * y] + o->psi[2 * x + 1] * o->psi[2 * y + 1]);
}

/* O-8 (P:66 <psi|H|psi>): raw (unnormalised) observables.
 * out[0] = ||psi||^2, out[1] = sum_x E(x)|psi[x]|^2 = <H_P>,
 * out[2] = P_succ = sum_{E(x)=0} |psi[x]|^2, out[3 + j] = <sigma^x_j>, j < n. */
int oracle_observables(int n, const uint16_t* E, const double* psi, double* out) {
  if (n < 1 || n > 40) return ORACLE_E_USAGE;
  const int64_t N = (int64_t)1 << n;
  obs_ctx o = {psi, E, 0};
  out[0] = sum_over(t_norm2, &o, N);
  out[1] = sum_over(t_hp, &o, N);
  out[2] = sum_over(t_succ, &o, N);
  for (int j = 0; j < n; j++) {
    o.bit = (int64_t)1 << j;
    out[3 + j] = sum_over(t_sx, &o, N);
  }
  return ORACLE_OK;
}

/* O-8 / A9: <psi|H(s)|psi> = (1-s) sum_j (||psi||^2 - <sigma^x_j>)/2 + s <H_P>
 * (Eq. 1 with H_B = sum_j (1 - sigma^x_j)/2). */
int oracle_energy(int n, const uint16_t* E, const double* psi, double s, double* out) {
  if (!(s >= 0.0 && s <= 1.0)) return ORACLE_E_USAGE;
  double* o = (double*)malloc(sizeof(double) * (size_t)(3 + n));
  if (!o) return ORACLE_E_USAGE;
  int st = oracle_observables(n, E, psi, o);
  if (st) { free(o); return st; }
  double hb = 0.0;
  for (int j = 0; j < n; j++) hb += 0.5 * (o[0] - o[3 + j]);
  *out = (1.0 - s) * hb + s * o[1];
  free(o);
  return ORACLE_OK;
}
