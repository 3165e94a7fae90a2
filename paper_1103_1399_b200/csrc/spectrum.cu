// spectrum.cu -- NEXT F3: the adiabatic-theorem diagnostic of
// the low spectrum of H(s) and the ground-state overlap -- from a
// Lanczos iteration on the matrix-free H(s) psi (never a dense matrix).
//
//   (H psi)[x] = wB(s) * (n/2 psi[x] - 1/2 sum_j psi[x ^ 2^j]) + wP(s) * E[x] psi[x]
//
// with the same weights as the evolution (Eq. 1, optional driving term).
// Lanczos with full re-orthogonalisation against every stored basis vector
// (so no ghost copies of converged eigenvalues), tridiagonal eigenvalues by
// Sturm-sequence bisection, Ritz vectors for the overlap. Deterministic
// reductions (fixed grid, fixed trees). Single GPU, n <= 24.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "kernels.cuh"

namespace qaa {
namespace {

constexpr int SP_THREADS = 256;

__global__ void __launch_bounds__(SP_THREADS) hmatvec_kernel(const double2* x, const uint8_t* E, double2* y, int n,
                                                            int64_t N, double wb, double wp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    double sr = 0.0, si = 0.0;
    for (int j = 0; j < n; j++) {
      const double2 v = x[i ^ ((int64_t)1 << j)];
      sr += v.x;
      si += v.y;
    }
    const double2 v = x[i];
    const double d = wb * 0.5 * (double)n + wp * (double)E[i];
    y[i] = make_double2(fma(d, v.x, -0.5 * wb * sr), fma(d, v.y, -0.5 * wb * si));
  }
}

// partial[b] = sum over this block's fixed index set of conj(a) * b  (re, im)
__global__ void __launch_bounds__(SP_THREADS) dot_kernel(const double2* a, const double2* b, int64_t N,
                                                        double* partial) {
  __shared__ double sh[2][SP_THREADS / 32];
  double re = 0.0, im = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 u = a[i], v = b[i];
    re = fma(u.x, v.x, fma(u.y, v.y, re));
    im = fma(u.x, v.y, fma(-u.y, v.x, im));
  }
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sh[0][w] = re;
    sh[1][w] = im;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0, s = 0.0;
    for (int k = 0; k < SP_THREADS / 32; k++) {
      r += sh[0][k];
      s += sh[1][k];
    }
    partial[2 * blockIdx.x] = r;
    partial[2 * blockIdx.x + 1] = s;
  }
}

// deterministic pseudo-random start vector (splitmix64 of the index)
__device__ __forceinline__ double hash01(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
}
__global__ void random_start_kernel(double2* v, int64_t N) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = make_double2(hash01(2 * (uint64_t)i), hash01(2 * (uint64_t)i + 1));
}

// y <- y - c * x   (complex c)
__global__ void axpy_kernel(double2* y, const double2* x, int64_t N, double cr, double ci) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = x[i];
    double2 w = y[i];
    w.x -= cr * v.x - ci * v.y;
    w.y -= cr * v.y + ci * v.x;
    y[i] = w;
  }
}

__global__ void scale_kernel(double2* dst, const double2* src, int64_t N, double s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = src[i];
    dst[i] = make_double2(v.x * s, v.y * s);
  }
}

// number of eigenvalues of the symmetric tridiagonal (a, b) below x (Sturm)
int sturm_count(const std::vector<double>& a, const std::vector<double>& b, double x) {
  int c = 0;
  double q = 1.0;
  for (size_t i = 0; i < a.size(); i++) {
    const double bb = i ? b[i - 1] * b[i - 1] : 0.0;
    q = (a[i] - x) - (i ? bb / q : 0.0);
    if (q == 0.0) q = -1e-300;
    if (q < 0) c++;
  }
  return c;
}

// k-th smallest eigenvalue (0-based) by bisection on [lo, hi]
double tri_eig(const std::vector<double>& a, const std::vector<double>& b, int k, double lo, double hi) {
  for (int it = 0; it < 200 && hi - lo > 1e-15 * std::max(1.0, std::fabs(lo) + std::fabs(hi)); it++) {
    const double mid = 0.5 * (lo + hi);
    if (sturm_count(a, b, mid) > k)
      hi = mid;
    else
      lo = mid;
  }
  return 0.5 * (lo + hi);
}

// eigenvector of the tridiagonal for eigenvalue lam (inverse iteration, 3 sweeps)
std::vector<double> tri_vec(const std::vector<double>& a, const std::vector<double>& b, double lam) {
  const size_t m = a.size();
  std::vector<double> v(m, 1.0), w(m);
  for (int sweep = 0; sweep < 3; sweep++) {
    // solve (T - lam I - eps) w = v with the Thomas algorithm
    std::vector<double> c(m), d(m);
    const double shift = lam + 1e-10 * std::max(1.0, std::fabs(lam));
    double den = a[0] - shift;
    if (den == 0.0) den = 1e-300;
    c[0] = m > 1 ? b[0] / den : 0.0;
    d[0] = v[0] / den;
    for (size_t i = 1; i < m; i++) {
      den = (a[i] - shift) - b[i - 1] * c[i - 1];
      if (den == 0.0) den = 1e-300;
      c[i] = i + 1 < m ? b[i] / den : 0.0;
      d[i] = (v[i] - b[i - 1] * d[i - 1]) / den;
    }
    w[m - 1] = d[m - 1];
    for (size_t i = m - 1; i-- > 0;) w[i] = d[i] - c[i] * w[i + 1];
    double nrm = 0.0;
    for (double x : w) nrm += x * x;
    nrm = std::sqrt(nrm);
    for (size_t i = 0; i < m; i++) v[i] = w[i] / nrm;
  }
  return v;
}

}  // namespace

cudaError_t lanczos_spectrum(const LanczosArgs& p, cudaStream_t st, double* evals, double* overlap, int* iters) {
  const int64_t N = (int64_t)1 << p.n;
  int grid = p.num_sms * 4;
  if ((int64_t)grid * SP_THREADS > N) grid = (int)std::max<int64_t>(1, (N + SP_THREADS - 1) / SP_THREADS);
  double* partial = p.scratch;  // 2 * grid doubles
  std::vector<double> hpart(2 * (size_t)grid);
  cudaError_t e;
  auto dot = [&](const double2* a, const double2* b, double* re, double* im) -> cudaError_t {
    dot_kernel<<<grid, SP_THREADS, 0, st>>>(a, b, N, partial);
    cudaError_t er = cudaMemcpyAsync(hpart.data(), partial, hpart.size() * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (er != cudaSuccess) return er;
    er = cudaStreamSynchronize(st);
    if (er != cudaSuccess) return er;
    double r = 0.0, s = 0.0;
    for (int b2 = 0; b2 < grid; b2++) {  // fixed order: deterministic
      r += hpart[2 * (size_t)b2];
      s += hpart[2 * (size_t)b2 + 1];
    }
    *re = r;
    *im = s;
    return cudaGetLastError();
  };
  // start vector: deterministic pseudo-random (overlaps every eigenvector)
  random_start_kernel<<<grid, SP_THREADS, 0, st>>>(p.basis, N);
  double nr, ni;
  if ((e = dot(p.basis, p.basis, &nr, &ni)) != cudaSuccess) return e;
  scale_kernel<<<grid, SP_THREADS, 0, st>>>(p.basis, p.basis, N, 1.0 / std::sqrt(nr));
  std::vector<double> alpha, beta;
  int m = 0;
  for (; m < p.kmax; m++) {
    double2* v = p.basis + (size_t)m * N;
    double2* w = p.basis + (size_t)(m + 1) * N;
    hmatvec_kernel<<<grid, SP_THREADS, 0, st>>>(v, p.E, w, p.n, N, p.wb, p.wp);
    double ar, ai;
    if ((e = dot(v, w, &ar, &ai)) != cudaSuccess) return e;
    alpha.push_back(ar);
    // full re-orthogonalisation (twice) against v_0..v_m
    for (int pass = 0; pass < 2; pass++)
      for (int i = 0; i <= m; i++) {
        double cr, ci;
        const double2* vi = p.basis + (size_t)i * N;
        if ((e = dot(vi, w, &cr, &ci)) != cudaSuccess) return e;
        axpy_kernel<<<grid, SP_THREADS, 0, st>>>(w, vi, N, cr, ci);
      }
    double br, bi;
    if ((e = dot(w, w, &br, &bi)) != cudaSuccess) return e;
    const double b = std::sqrt(std::max(br, 0.0));
    if (m + 1 == p.kmax || b < 1e-12 * std::max(1.0, std::fabs(ar))) {
      m++;
      break;
    }
    beta.push_back(b);
    scale_kernel<<<grid, SP_THREADS, 0, st>>>(w, w, N, 1.0 / b);
  }
  *iters = m;
  // eigenvalues of the m x m tridiagonal: Gershgorin bounds + bisection
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < m; i++) {
    const double r = (i ? beta[i - 1] : 0.0) + (i + 1 < m ? beta[i] : 0.0);
    lo = std::min(lo, alpha[i] - r);
    hi = std::max(hi, alpha[i] + r);
  }
  beta.resize((size_t)std::max(0, m - 1));
  for (int k = 0; k < p.nev; k++) evals[k] = k < m ? tri_eig(alpha, beta, k, lo, hi) : NAN;
  if (overlap && p.state) {
    // Ritz ground vector g = sum_i y_i v_i; overlap |<g|psi>|^2 / <psi|psi>
    std::vector<double> y = tri_vec(alpha, beta, evals[0]);
    double ovr = 0.0, ovi = 0.0, sr, si;
    for (int i = 0; i < m; i++) {
      double cr, ci;
      if ((e = dot(p.basis + (size_t)i * N, p.state, &cr, &ci)) != cudaSuccess) return e;
      ovr += y[(size_t)i] * cr;
      ovi += y[(size_t)i] * ci;
    }
    if ((e = dot(p.state, p.state, &sr, &si)) != cudaSuccess) return e;
    *overlap = (ovr * ovr + ovi * ovi) / sr;
  }
  return cudaGetLastError();
}

}  // namespace qaa
