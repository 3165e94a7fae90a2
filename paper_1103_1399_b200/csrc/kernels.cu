// kernels.cu -- sm_100a kernels of libqaa.
//
//  K4 qaa_pass_kernel     fused Trotter pass: one HBM round trip over the state
//                         applies, per 2^12-amplitude tile, the X rotations of
//                         up to 2 x 12 qubits and optionally the diagonal D
//                         (BASELINE north_star).
//  -- qaa_resident_kernel all K steps for L <= 12 in one CTA's shared memory.
//  K1 energy_table_kernel E[x] = #violated clauses.
//  K2 compact_zeros       Z = {x : E[x] = 0}.
//  K3 fill / set_one      initial states.
//  K5 obs_* / reduce      deterministic fp64 reductions (A9).
//
// Rotation algebra (R2, §4): exp(-i beta (1 - sigma^x)) =
// g (cos beta I + i sin beta sigma^x), g = e^{-i beta}. With |tan beta| <= 1
// the pass applies (I + i t sigma^x), t = tan beta ("tangent form": one FMA
// per real component); otherwise (u I + i sigma^x), u = cot beta. The scalar
// (g cos beta)^n (resp. (g sin beta)^n) of a whole step is folded into that
// step's diagonal table Phi_k[e] = e^{-i dt s_k e} * scale_k, computed on the
// host (R11).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace qaa {

#define FULL_MASK 0xffffffffu

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ int swz(int l) {
  // XOR-fold the three 3-bit groups above bit 3 into the low 3 bits: every
  // register pattern's first three lane bits then hit 8 distinct 16-byte
  // bank groups, so 128-bit LDS/STS are conflict free.
  return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7);
}

__device__ __forceinline__ int thread_local_index(int pat, int lane, int warp) {
  // PA: lanes {0..4} warps {5,6,7}; PB: lanes {0,1,2,3,8} warps {9,10,11};
  // PC: lanes {4..8} warps {9,10,11} (see plan.hpp)
  return pat == PA ? (lane | (warp << 5))
                   : (pat == PB ? ((lane & 15) | ((lane >> 4) << 8) | (warp << 9)) : ((lane << 4) | (warp << 9)));
}

template <int PAT>
struct RegShift {
  static constexpr int value = PAT == PA ? 8 : (PAT == PB ? 4 : 0);
};

struct PatOff {
  int64_t thr;
  int64_t s[4];
};

__device__ __forceinline__ PatOff make_patoff(const int (&phys)[TILE_BITS], int pat, int lane, int warp) {
  PatOff p;
  const int tl = thread_local_index(pat, lane, warp);
  int64_t o = 0;
#pragma unroll
  for (int b = 0; b < TILE_BITS; b++)
    if ((tl >> b) & 1) o += (int64_t)1 << phys[b];
  p.thr = o;
#pragma unroll
  for (int i = 0; i < 4; i++) p.s[i] = (int64_t)1 << (pat == PA ? phys[8 + i] : (pat == PB ? phys[4 + i] : phys[i]));
  return p;
}

__device__ __forceinline__ int64_t reg_off(const PatOff& p, int r) {
  int64_t o = p.thr;
  if (r & 1) o += p.s[0];
  if (r & 2) o += p.s[1];
  if (r & 4) o += p.s[2];
  if (r & 8) o += p.s[3];
  return o;
}

__device__ __forceinline__ int64_t tile_base(const PassArgs& a, int64_t T) {
  int64_t base = 0;
#pragma unroll
  for (int s = 0; s < MAX_SEGS; s++)
    if (s < a.nseg) base += ((T >> a.seg_src[s]) & (((int64_t)1 << a.seg_len[s]) - 1)) << a.seg_dst[s];
  return base;
}

// (a, b) <- (a + i c b, b + i c a)  [FORM 0]   or   (c a + i b, c b + i a)  [FORM 1]
template <int FORM>
__device__ __forceinline__ void rot_pair(double2& a, double2& b, double c) {
  double2 na, nb;
  if (FORM == 0) {
    na = make_double2(fma(-c, b.y, a.x), fma(c, b.x, a.y));
    nb = make_double2(fma(-c, a.y, b.x), fma(c, a.x, b.y));
  } else {
    na = make_double2(fma(c, a.x, -b.y), fma(c, a.y, b.x));
    nb = make_double2(fma(c, b.x, -a.y), fma(c, b.y, a.x));
  }
  a = na;
  b = nb;
}

template <int I, int FORM>
__device__ __forceinline__ void rot_reg(double2 (&v)[RPT], double c) {
#pragma unroll
  for (int r = 0; r < RPT; r++)
    if (!(r & (1 << I))) rot_pair<FORM>(v[r], v[r | (1 << I)], c);
}

template <int FORM>
__device__ __forceinline__ void rot_lane(double2 (&v)[RPT], int mask, double c) {
#pragma unroll
  for (int r = 0; r < RPT; r++) {
    const double px = __shfl_xor_sync(FULL_MASK, v[r].x, mask);
    const double py = __shfl_xor_sync(FULL_MASK, v[r].y, mask);
    if (FORM == 0)
      v[r] = make_double2(fma(-c, py, v[r].x), fma(c, px, v[r].y));
    else
      v[r] = make_double2(fma(c, v[r].x, -py), fma(c, v[r].y, px));
  }
}

template <int PAT>
__device__ __forceinline__ void sts_pat(double2* xb, const double2 (&v)[RPT], int tl) {
#pragma unroll
  for (int r = 0; r < RPT; r++) xb[swz(tl | (r << RegShift<PAT>::value))] = v[r];
}
template <int PAT>
__device__ __forceinline__ void lds_pat(const double2* xb, double2 (&v)[RPT], int tl) {
#pragma unroll
  for (int r = 0; r < RPT; r++) v[r] = xb[swz(tl | (r << RegShift<PAT>::value))];
}

__device__ __forceinline__ void apply_diag(double2 (&v)[RPT], const uint32_t (&ep)[4], const double2* phis) {
#pragma unroll
  for (int r = 0; r < RPT; r++) {
    const int e = (ep[r >> 2] >> ((r & 3) * 8)) & 0xff;
    const double2 f = phis[e];
    const double2 x = v[r];
    v[r] = make_double2(fma(f.x, x.x, -f.y * x.y), fma(f.x, x.y, f.y * x.x));
  }
}

// Runs the pass program (plan.cpp build_program) on one tile held in registers.
__device__ __forceinline__ void run_program(const PassArgs& a, const Op* ops, double2 (&v)[RPT],
                                            const uint32_t (&ep)[4], double2* xb, const double2* phis, int lane,
                                            int warp) {
  int pat = PA;
  const int nops = a.nops;
  for (int i = 0; i < nops; i++) {
    const Op op = ops[i];
    const double c = op.slot ? a.coef[1] : a.coef[0];
    const int f = op.slot ? a.form[1] : a.form[0];
    switch (op.kind) {
      case OP_ROT_REG:
        switch (op.arg * 2 + f) {
          case 0: rot_reg<0, 0>(v, c); break;
          case 1: rot_reg<0, 1>(v, c); break;
          case 2: rot_reg<1, 0>(v, c); break;
          case 3: rot_reg<1, 1>(v, c); break;
          case 4: rot_reg<2, 0>(v, c); break;
          case 5: rot_reg<2, 1>(v, c); break;
          case 6: rot_reg<3, 0>(v, c); break;
          default: rot_reg<3, 1>(v, c); break;
        }
        break;
      case OP_ROT_LANE:
        if (f == 0)
          rot_lane<0>(v, 1 << op.arg, c);
        else
          rot_lane<1>(v, 1 << op.arg, c);
        break;
      case OP_XCHG: {
        const int to = op.arg;
        const int tlf = thread_local_index(pat, lane, warp);
        if (pat == PA)
          sts_pat<PA>(xb, v, tlf);
        else if (pat == PB)
          sts_pat<PB>(xb, v, tlf);
        else
          sts_pat<PC>(xb, v, tlf);
        __syncthreads();
        const int tlt = thread_local_index(to, lane, warp);
        if (to == PA)
          lds_pat<PA>(xb, v, tlt);
        else if (to == PB)
          lds_pat<PB>(xb, v, tlt);
        else
          lds_pat<PC>(xb, v, tlt);
        __syncthreads();
        pat = to;
        break;
      }
      case OP_DIAG:
        apply_diag(v, ep, phis);
        break;
      default:
        break;
    }
  }
}

__device__ __forceinline__ void load_tile(const PassArgs& a, const PatOff& pa, const PatOff& pe, int64_t T,
                                          double2 (&v)[RPT], uint32_t (&ep)[4]) {
  const int64_t base = tile_base(a, T);
  const double2* src = a.psi + base;
#pragma unroll
  for (int r = 0; r < RPT; r++) v[r] = src[reg_off(pa, r)];
  if (a.e_pattern >= 0) {
    const uint8_t* eb = a.E + base;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      uint32_t w = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) w |= (uint32_t)eb[reg_off(pe, q * 4 + j)] << (8 * j);
      ep[q] = w;
    }
  }
}

__device__ __forceinline__ void store_tile(const PassArgs& a, const PatOff& pf, int64_t T, const double2 (&v)[RPT]) {
  double2* dst = a.psi + tile_base(a, T);
#pragma unroll
  for (int r = 0; r < RPT; r++) dst[reg_off(pf, r)] = v[r];
}

__global__ void __launch_bounds__(NTHREADS, 1) qaa_pass_kernel(const PassArgs a) {
  extern __shared__ double2 smem[];
  double2* xb = smem;            // TILE exchange buffer (64 KiB)
  double2* phis = smem + TILE;   // D row (<= 256 entries)
  __shared__ Op ops[MAX_OPS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int i = 0; i < MAX_OPS; i++)
    if (tid == i && i < a.nops) ops[i] = a.ops[i];
  if (a.e_pattern >= 0)
    for (int e = tid; e < a.n_phi; e += NTHREADS) phis[e] = a.phi[e];
  __syncthreads();

  const PatOff pa = make_patoff(a.phys, PA, lane, warp);
  const PatOff pf = make_patoff(a.phys, a.final_pattern, lane, warp);
  const PatOff pe = make_patoff(a.phys, a.e_pattern >= 0 ? a.e_pattern : PA, lane, warp);

  double2 va[RPT], vb[RPT];
  uint32_t ea[4] = {0, 0, 0, 0}, eb[4] = {0, 0, 0, 0};
  int64_t T = blockIdx.x;
  const int64_t stride = gridDim.x;
  if (T < a.ntiles) load_tile(a, pa, pe, T, va, ea);
  while (T < a.ntiles) {
    int64_t Tn = T + stride;
    if (Tn < a.ntiles) load_tile(a, pa, pe, Tn, vb, eb);  // prefetch next tile
    run_program(a, ops, va, ea, xb, phis, lane, warp);
    store_tile(a, pf, T, va);
    T = Tn;
    if (T >= a.ntiles) break;
    Tn = T + stride;
    if (Tn < a.ntiles) load_tile(a, pa, pe, Tn, va, ea);
    run_program(a, ops, vb, eb, xb, phis, lane, warp);
    store_tile(a, pf, T, vb);
    T = Tn;
  }
}

cudaError_t pass_kernel_setup() {
  return cudaFuncSetAttribute(qaa_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PASS_SMEM_BYTES);
}

cudaError_t launch_pass(const PassArgs& a, int grid, cudaStream_t st) {
  qaa_pass_kernel<<<grid, NTHREADS, PASS_SMEM_BYTES, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------ resident (L <= 12)
__global__ void __launch_bounds__(1024, 1) qaa_resident_kernel(const ResidentArgs a) {
  extern __shared__ double2 smem[];
  double2* s = smem;
  uint8_t* e = reinterpret_cast<uint8_t*>(smem + (1 << a.L));
  const int N = 1 << a.L, half = N >> 1, tid = threadIdx.x, nt = blockDim.x;
  for (int x = tid; x < N; x += nt) {
    s[x] = a.psi[x];
    e[x] = a.E[x];
  }
  __syncthreads();
  for (int64_t k = 0; k < a.K; k++) {
    const double2* phi = a.phi_all + k * a.n_phi;
    for (int x = tid; x < N; x += nt) {  // D_k
      const double2 f = phi[e[x]], v = s[x];
      s[x] = make_double2(fma(f.x, v.x, -f.y * v.y), fma(f.x, v.y, f.y * v.x));
    }
    __syncthreads();
    const double c = a.coef[k];
    const int form = a.form[k];
    for (int j = 0; j < a.L; j++) {  // X_k, qubit by qubit
      for (int p = tid; p < half; p += nt) {
        const int x = ((p >> j) << (j + 1)) | (p & ((1 << j) - 1));
        const int y = x | (1 << j);
        double2 u = s[x], w = s[y];
        if (form == 0)
          rot_pair<0>(u, w, c);
        else
          rot_pair<1>(u, w, c);
        s[x] = u;
        s[y] = w;
      }
      __syncthreads();
    }
  }
  if (a.final_d) {  // Strang: closing half step D(s_{K-1})^{1/2}
    const double2* phi = a.phi_all + a.K * a.n_phi;
    for (int x = tid; x < N; x += nt) {
      const double2 f = phi[e[x]], v = s[x];
      s[x] = make_double2(fma(f.x, v.x, -f.y * v.y), fma(f.x, v.y, f.y * v.x));
    }
    __syncthreads();
  }
  for (int x = tid; x < N; x += nt) a.psi[x] = s[x];
}

cudaError_t launch_resident(const ResidentArgs& a, cudaStream_t st) {
  const size_t smem = (sizeof(double2) + 1) * ((size_t)1 << a.L);
  cudaError_t e = cudaFuncSetAttribute(qaa_resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int threads = a.L >= 10 ? 1024 : ((1 << a.L) < 64 ? 64 : (1 << a.L));
  qaa_resident_kernel<<<1, threads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int NV>
__device__ __forceinline__ void block_reduce(double (&acc)[NV], double* sh);

// Batched sweep: block r evolves its own copy of the uniform
// state (L <= 12, resident in shared memory) with its own step count and
// coefficient rows, then reduces P_succ = sum_{E=0} |psi|^2 (fixed tree).
__global__ void __launch_bounds__(512) qaa_sweep_kernel(const SweepArgs a) {
  extern __shared__ double2 smem[];
  double2* s = smem;
  uint8_t* e = reinterpret_cast<uint8_t*>(smem + (1 << a.L));
  __shared__ double red[32];
  const int r = blockIdx.x;
  const int N = 1 << a.L, half = N >> 1, tid = threadIdx.x, nt = blockDim.x;
  const int64_t K = a.K[r], off = a.row_off[r];
  for (int x = tid; x < N; x += nt) {
    s[x] = make_double2(a.amp0, 0.0);
    e[x] = a.E[x];
  }
  __syncthreads();
  for (int64_t k = 0; k < K + (a.final_d ? 1 : 0); k++) {
    const double2* phi = a.phi_all + (off + k) * a.n_phi;
    for (int x = tid; x < N; x += nt) {
      const double2 f = phi[e[x]], v = s[x];
      s[x] = make_double2(fma(f.x, v.x, -f.y * v.y), fma(f.x, v.y, f.y * v.x));
    }
    __syncthreads();
    if (k == K) break;  // Strang closing half step: no X after it
    const double c = a.coef[off + k];
    const int form = a.form[off + k];
    for (int j = 0; j < a.L; j++) {
      for (int p = tid; p < half; p += nt) {
        const int x = ((p >> j) << (j + 1)) | (p & ((1 << j) - 1));
        const int y = x | (1 << j);
        double2 u = s[x], w = s[y];
        if (form == 0)
          rot_pair<0>(u, w, c);
        else
          rot_pair<1>(u, w, c);
        s[x] = u;
        s[y] = w;
      }
      __syncthreads();
    }
  }
  double acc[1] = {0.0};
  for (int x = tid; x < N; x += nt)
    if (e[x] == 0) acc[0] += fma(s[x].x, s[x].x, s[x].y * s[x].y);
  block_reduce<1>(acc, red);
  if (tid == 0) a.out[r] = acc[0];
}

cudaError_t launch_sweep(const SweepArgs& a, int nrep, cudaStream_t st) {
  const size_t smem = (sizeof(double2) + 1) * ((size_t)1 << a.L);
  cudaError_t e = cudaFuncSetAttribute(qaa_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int threads = a.L >= 9 ? 512 : ((1 << a.L) < 64 ? 64 : (1 << a.L));
  qaa_sweep_kernel<<<nrep, threads, smem, st>>>(a);
  return cudaGetLastError();
}

// Batched sweep for 13 <= L <= 16 (SURVEY §8(f) F1 as specified there: each
// replica's state resident in one thread-block cluster's shared memory, all K
// steps in one launch, zero HBM traffic). Cluster = 2^(L-13) CTAs; CTA q holds
// the 2^13 amplitudes whose top L-13 bits are q (128 KiB + its 8 KiB energy
// slice). Per step: D fused into the first of four register phases over the 13
// local bits (16 amplitudes per thread: bits {0-3}, {4-7}, {8-11}, {12}), then
// one DSMEM phase per cluster bit (own' from own and the partner CTA's
// amplitude at the same local index; cluster barriers before the remote reads
// and before the writes). DSMEM bandwidth (~20 B/clk/SM) bounds these phases:
// ~6.5 us per cluster bit; reading all 2^cb - 1 other CTAs at once (two
// barriers per step instead of two per bit) was measured 4x slower at n = 16. Shared memory holds amplitude x at x ^ ((x>>4)&7):
// every phase's quarter-warp then hits 8 distinct 16-byte bank groups.
namespace cg = cooperative_groups;
constexpr int SWEEP_LB = 13;  // max local bits per CTA (2^13 amplitudes, 128 KiB)

__device__ __forceinline__ int sw_pos(int x) { return x ^ ((x >> 4) & 7); }
__device__ __forceinline__ uint32_t dsmem_map(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(r)
               : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ double2 ld_dsmem(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}
// amplitude index of register r of thread t in the phase whose register bits
// are R[0..3] (the LB-4 thread bits fill the other local bits in increasing order)
template <int LB>
__device__ __forceinline__ int sw_index(int t, int r, const int (&R)[4]) {
  int x = 0, tb = 0;
#pragma unroll
  for (int b = 0; b < LB; b++) {
    int rb = -1;
#pragma unroll
    for (int i = 0; i < 4; i++)
      if (R[i] == b) rb = i;
    if (rb >= 0)
      x |= ((r >> rb) & 1) << b;
    else
      x |= ((t >> tb++) & 1) << b;
  }
  return x;
}

// one register phase: 16 amplitudes per thread whose indices differ in the
// register bits R; the first nrot of them are rotated (D fused when phi != 0)
template <int FORM, int LB>
__device__ __forceinline__ void sw_phase(double2* s, const uint8_t* e, const double2* phi, int t, int nrot,
                                         const int (&R)[4], double c) {
  double2 v[16];
  int pos[16];
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int x = sw_index<LB>(t, r, R);
    pos[r] = sw_pos(x);
    v[r] = s[pos[r]];
    if (phi) {  // D_k (first phase): psi[x] <- Phi_k[E[x]] psi[x]
      const double2 f = phi[e[x]];
      v[r] = make_double2(fma(f.x, v[r].x, -f.y * v[r].y), fma(f.x, v[r].y, f.y * v[r].x));
    }
  }
#pragma unroll
  for (int i = 0; i < 4; i++)
    if (i < nrot)
#pragma unroll
      for (int r = 0; r < 16; r++)
        if (!(r & (1 << i))) rot_pair<FORM>(v[r], v[r | (1 << i)], c);
#pragma unroll
  for (int r = 0; r < 16; r++) s[pos[r]] = v[r];
}

// one Trotter step of a replica: D fused into the first of the register
// phases over the LB local bits ({0-3} {4-7} {8-11} {12}; the last phase of an
// LB < 12 state re-uses lower bits unrotated), then one DSMEM phase per cluster bit
template <int FORM, int LB>
__device__ __forceinline__ void sw_step(double2* s, const uint8_t* e, const double2* phi, int t, double c,
                                        cg::cluster_group& cl, int cb, int q) {
  constexpr int NT = 1 << (LB - 4);
  const int R0[4] = {0, 1, 2, 3}, R1[4] = {4, 5, 6, 7};
  const int R2[4] = {8, LB > 9 ? 9 : 4, LB > 10 ? 10 : 5, LB > 11 ? 11 : (LB > 10 ? 7 : 6)};
  const int R3[4] = {12, 9, 10, 11};
  sw_phase<FORM, LB>(s, e, phi, t, 4, R0, c);
  __syncthreads();
  sw_phase<FORM, LB>(s, e, nullptr, t, 4, R1, c);
  __syncthreads();
  sw_phase<FORM, LB>(s, e, nullptr, t, LB >= 12 ? 4 : LB - 8, R2, c);
  if (LB == 13) {
    __syncthreads();
    sw_phase<FORM, LB>(s, e, nullptr, t, 1, R3, c);
  }
  for (int b = 0; b < cb; b++) {
    cl.sync();  // every CTA's phase writes are visible
    // partner CTA's copy of my positions, through the shared::cluster window
    const uint32_t rbase = dsmem_map(s, (uint32_t)(q ^ (1 << b)));
    double2 v[16];
#pragma unroll
    for (int i = 0; i < 16; i++) {
      const int p = t + NT * i;  // any bijection: own and partner amplitude share the position
      const double2 a = s[p], w = ld_dsmem(rbase + 16u * (uint32_t)p);
      v[i] = FORM == 0 ? make_double2(fma(-c, w.y, a.x), fma(c, w.x, a.y))
                       : make_double2(fma(c, a.x, -w.y), fma(c, a.y, w.x));
    }
    cl.sync();  // the partner has read my old values
#pragma unroll
    for (int i = 0; i < 16; i++) s[t + NT * i] = v[i];
  }
  __syncthreads();  // the next step's first phase reads other threads' amplitudes
}

template <int LB>
__global__ void __launch_bounds__(1 << (LB - 4), 1) qaa_sweep_cluster_kernel(const SweepArgs a) {
  constexpr int NT = 1 << (LB - 4), N = 1 << LB;
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks(), q = (int)cl.block_rank();
  const int cb = a.L - LB, r = blockIdx.x / C, t = threadIdx.x;
  extern __shared__ double2 smem[];
  double2* s = smem;
  uint8_t* e = reinterpret_cast<uint8_t*>(smem + N);
  __shared__ double red[32];
  __shared__ double part;
  const int64_t K = a.K[r], off = a.row_off[r];
  for (int x = t; x < N; x += NT) {
    s[x] = make_double2(a.amp0, 0.0);
    e[x] = a.E[((int64_t)q << LB) | x];
  }
  __syncthreads();
  for (int64_t k = 0; k < K; k++) {
    const double2* phi = a.phi_all + (off + k) * a.n_phi;
    if (a.form[off + k] == 0)
      sw_step<0, LB>(s, e, phi, t, a.coef[off + k], cl, cb, q);
    else
      sw_step<1, LB>(s, e, phi, t, a.coef[off + k], cl, cb, q);
  }
  if (a.final_d) {  // Strang: closing half step D(s_{K-1})^{1/2}
    const double2* phi = a.phi_all + (off + K) * a.n_phi;
    for (int x = t; x < N; x += NT) {
      const double2 f = phi[e[x]], v = s[sw_pos(x)];
      s[sw_pos(x)] = make_double2(fma(f.x, v.x, -f.y * v.y), fma(f.x, v.y, f.y * v.x));
    }
    __syncthreads();
  }
  double acc[1] = {0.0};
  for (int x = t; x < N; x += NT)
    if (e[x] == 0) {
      const double2 v = s[sw_pos(x)];
      acc[0] += fma(v.x, v.x, v.y * v.y);
    }
  block_reduce<1>(acc, red);
  if (t == 0) part = acc[0];
  cl.sync();
  if (q == 0 && t == 0) {  // fixed order over the cluster's CTAs
    double sum = 0.0;
    for (int j = 0; j < C; j++) sum += *cl.map_shared_rank(&part, j);
    a.out[r] = sum;
  }
  cl.sync();  // keep every CTA's shared memory alive until rank 0 has read it
}

// Single evolution resident in one CTA for 10 <= L <= 12 (qaa_evolve): the
// sweep's register phases over a swizzled shared-memory copy of the state,
// loaded from and stored back to psi (SURVEY §7 hard part 5).
template <int LB>
__global__ void __launch_bounds__(1 << (LB - 4), 1) qaa_resident_phase_kernel(const ResidentArgs a) {
  constexpr int NT = 1 << (LB - 4), N = 1 << LB;
  cg::cluster_group cl = cg::this_cluster();  // a cluster of one: sw_step's cluster phase is empty
  extern __shared__ double2 smem[];
  double2* s = smem;
  uint8_t* e = reinterpret_cast<uint8_t*>(smem + N);
  const int t = threadIdx.x;
  for (int x = t; x < N; x += NT) {
    s[sw_pos(x)] = a.psi[x];
    e[x] = a.E[x];
  }
  __syncthreads();
  for (int64_t k = 0; k < a.K; k++) {
    const double2* phi = a.phi_all + k * a.n_phi;
    if (a.form[k] == 0)
      sw_step<0, LB>(s, e, phi, t, a.coef[k], cl, 0, 0);
    else
      sw_step<1, LB>(s, e, phi, t, a.coef[k], cl, 0, 0);
  }
  if (a.final_d) {  // Strang: closing half step D(s_{K-1})^{1/2}
    const double2* phi = a.phi_all + a.K * a.n_phi;
    for (int x = t; x < N; x += NT) {
      const double2 f = phi[e[x]], v = s[sw_pos(x)];
      s[sw_pos(x)] = make_double2(fma(f.x, v.x, -f.y * v.y), fma(f.x, v.y, f.y * v.x));
    }
    __syncthreads();
  }
  for (int x = t; x < N; x += NT) a.psi[x] = s[sw_pos(x)];
}

template <int LB>
static cudaError_t launch_resident_lb(const ResidentArgs& a, cudaStream_t st) {
  const size_t smem = (sizeof(double2) + 1) * ((size_t)1 << LB);
  cudaError_t e =
      cudaFuncSetAttribute(qaa_resident_phase_kernel<LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  qaa_resident_phase_kernel<LB><<<1, 1 << (LB - 4), smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_resident_phases(const ResidentArgs& a, cudaStream_t st) {
  switch (a.L) {
    case 10: return launch_resident_lb<10>(a, st);
    case 11: return launch_resident_lb<11>(a, st);
    case 12: return launch_resident_lb<12>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int LB>
static cudaError_t launch_sweep_lb(const SweepArgs& a, int nrep, cudaStream_t st) {
  const size_t smem = (sizeof(double2) + 1) * ((size_t)1 << LB);
  cudaError_t e =
      cudaFuncSetAttribute(qaa_sweep_cluster_kernel<LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int C = 1 << (a.L - LB);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nrep * C));
  cfg.blockDim = dim3(1u << (LB - 4));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, qaa_sweep_cluster_kernel<LB>, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_sweep_cluster(const SweepArgs& a, int nrep, cudaStream_t st) {
  switch (a.L < SWEEP_LB ? a.L : SWEEP_LB) {
    case 10: return launch_sweep_lb<10>(a, nrep, st);
    case 11: return launch_sweep_lb<11>(a, nrep, st);
    case 12: return launch_sweep_lb<12>(a, nrep, st);
    case 13: return launch_sweep_lb<13>(a, nrep, st);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------ energy table
// Clause record (host-built, api_context.cu): {M_hi, V_hi, spread[4]}: the clause
// is violated by x iff (x & M) == V. For 16 consecutive x = x0 | i the high
// part (bits >= 4) is one test, and spread[] holds, byte i, the outcome of the
// low part for x0 | i, so one predicated 4-word add counts 16 assignments.
struct ClauseRec {
  uint64_t mhi, vhi;
  uint32_t spread[4];
};

// Each thread handles NB groups of 16 assignments (grid-stride apart, so every
// store instruction stays coalesced) per pass over the clause list: one clause
// record load (a shared-memory broadcast) serves NB tests. W32: every
// assignment fits 32 bits (n <= 32), so the test is one AND + one compare.
template <bool W32, int NB>
__global__ void __launch_bounds__(256) energy_table_kernel(uint8_t* E, int64_t N, uint64_t x_offset,
                                                            const ClauseRec* recs, int m, unsigned* d_max,
                                                            unsigned long long* d_zeros, int lowbits, int hishift) {
  // local index p -> global assignment x = (p mod 2^lowbits) | x_offset | ((p >> lowbits) << hishift)
  // (layout A: lowbits = L; layout B of the sharded state: lowbits = L - g, hishift = L)
  const uint64_t lowmask = (lowbits >= 64) ? ~0ull : ((1ull << lowbits) - 1);
  __shared__ ClauseRec sr[256];
  for (int i = threadIdx.x; i < m; i += blockDim.x) sr[i] = recs[i];
  __syncthreads();
  unsigned mx = 0;
  unsigned long long zeros = 0;
  const int64_t ngroups = N >> 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g0 < ngroups; g0 += NB * stride) {
    uint64_t x0[NB];
    uint32_t c[NB][4];
#pragma unroll
    for (int b = 0; b < NB; b++) {
      const uint64_t p0 = (uint64_t)(g0 + b * stride) << 4;
      x0[b] = (p0 & lowmask) | x_offset | ((p0 >> lowbits) << hishift);
      c[b][0] = c[b][1] = c[b][2] = c[b][3] = 0;
    }
    for (int k = 0; k < m; k++) {
      const ClauseRec r = sr[k];
#pragma unroll
      for (int b = 0; b < NB; b++) {
        const bool hit = W32 ? (((uint32_t)x0[b] & (uint32_t)r.mhi) == (uint32_t)r.vhi) : ((x0[b] & r.mhi) == r.vhi);
        if (hit) {
          c[b][0] += r.spread[0];
          c[b][1] += r.spread[1];
          c[b][2] += r.spread[2];
          c[b][3] += r.spread[3];
        }
      }
    }
#pragma unroll
    for (int b = 0; b < NB; b++) {
      if (g0 + b * stride >= ngroups) break;
      reinterpret_cast<uint4*>(E)[g0 + b * stride] = make_uint4(c[b][0], c[b][1], c[b][2], c[b][3]);
#pragma unroll
      for (int q = 0; q < 4; q++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const unsigned v = (c[b][q] >> (8 * j)) & 0xff;
          mx = v > mx ? v : mx;
          zeros += v == 0;
        }
    }
  }
  // block reduce (integers: order-independent)
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned om = __shfl_xor_sync(FULL_MASK, mx, o);
    mx = om > mx ? om : mx;
    zeros += __shfl_xor_sync(FULL_MASK, zeros, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(d_max, mx);
    atomicAdd(d_zeros, zeros);
  }
}

// tail for N < 16 (tiny instances): one thread per x
__global__ void energy_table_small_kernel(uint8_t* E, int64_t N, uint64_t x_offset, const ClauseRec* recs, int m,
                                          unsigned* d_max, unsigned long long* d_zeros) {
  const int64_t x = threadIdx.x;
  if (x >= N) return;
  const uint64_t xg = x_offset + (uint64_t)x;
  unsigned cnt = 0;
  for (int c = 0; c < m; c++) {
    const ClauseRec r = recs[c];
    if ((xg & r.mhi) == r.vhi) cnt += (r.spread[(xg & 15) >> 2] >> (8 * (xg & 3))) & 0xff;
  }
  E[x] = (uint8_t)cnt;
  atomicMax(d_max, cnt);
  if (cnt == 0) atomicAdd(d_zeros, 1ull);
}

cudaError_t launch_energy_table(uint8_t* E, int64_t N, uint64_t x_offset, const uint64_t* MV, int m, unsigned* d_max,
                                unsigned long long* d_zeros, int num_sms, cudaStream_t st, int lowbits, int hishift,
                                bool force_w64) {
  const ClauseRec* recs = reinterpret_cast<const ClauseRec*>(MV);
  if (N < 16) {
    energy_table_small_kernel<<<1, 32, 0, st>>>(E, N, x_offset, recs, m, d_max, d_zeros);
  } else {
    const int64_t groups = N >> 4;
    int64_t grid = (groups + 255) / 256;
    const int64_t cap = (int64_t)num_sms * 8;
    if (grid > cap) grid = cap;
    // every assignment x < x_offset + N fits 32 bits when the highest one does
    const uint64_t xmax = (uint64_t)(N - 1) | x_offset | (hishift < 64 && lowbits < 64 ?
                              (((uint64_t)(N - 1) >> lowbits) << hishift) : 0ull);
    const bool w32 = (xmax >> 32) == 0 && !force_w64;
    if (w32)
      energy_table_kernel<true, 4><<<(int)grid, 256, 0, st>>>(E, N, x_offset, recs, m, d_max, d_zeros, lowbits, hishift);
    else
      energy_table_kernel<false, 4><<<(int)grid, 256, 0, st>>>(E, N, x_offset, recs, m, d_max, d_zeros, lowbits, hishift);
  }
  return cudaGetLastError();
}

__global__ void compact_zeros_kernel(const uint8_t* E, int64_t N, uint64_t x_offset, uint64_t* Z,
                                     unsigned long long* d_count) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N; x += (int64_t)gridDim.x * blockDim.x)
    if (E[x] == 0) Z[atomicAdd(d_count, 1ull)] = x_offset + (uint64_t)x;
}

cudaError_t launch_compact_zeros(const uint8_t* E, int64_t N, uint64_t x_offset, uint64_t* Z,
                                 unsigned long long* d_count, int num_sms, cudaStream_t st) {
  int64_t grid = (N + 255) / 256;
  if (grid > (int64_t)num_sms * 8) grid = (int64_t)num_sms * 8;
  compact_zeros_kernel<<<(int)grid, 256, 0, st>>>(E, N, x_offset, Z, d_count);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ init
__global__ void fill_kernel(double2* psi, int64_t N, double re, double im) {
  const double2 v = make_double2(re, im);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N; x += (int64_t)gridDim.x * blockDim.x)
    psi[x] = v;
}
cudaError_t launch_fill(double2* psi, int64_t N, double re, double im, int num_sms, cudaStream_t st) {
  int64_t grid = (N + 255) / 256;
  if (grid > (int64_t)num_sms * 16) grid = (int64_t)num_sms * 16;
  fill_kernel<<<(int)grid, 256, 0, st>>>(psi, N, re, im);
  return cudaGetLastError();
}
__global__ void set_one_kernel(double2* psi, int64_t idx) { psi[idx] = make_double2(1.0, 0.0); }
cudaError_t launch_set_one(double2* psi, int64_t idx, cudaStream_t st) {
  set_one_kernel<<<1, 1, 0, st>>>(psi, idx);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ reductions
// Deterministic block reduction of NV doubles: xor-butterfly inside each warp
// (every lane ends with the same fixed-order sum), then warp 0 combines the
// per-warp sums the same way. Result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_reduce(double (&acc)[NV], double* sh /* >= 32*NV */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; j++)
    for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(FULL_MASK, acc[j], o);
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NV; j++) sh[warp * NV + j] = acc[j];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < NV; j++) {
      double v = lane < nw ? sh[lane * NV + j] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
      acc[j] = v;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) obs_basic_kernel(const double2* psi, const uint8_t* E, int64_t N,
                                                         double* partial) {
  __shared__ double sh[32 * 3];
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N; x += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = psi[x];
    const double p = fma(v.x, v.x, v.y * v.y);
    const unsigned e = E[x];
    acc[0] += p;
    acc[1] += (double)e * p;
    acc[2] += e == 0 ? p : 0.0;
  }
  block_reduce<3>(acc, sh);
  if (threadIdx.x == 0)
    for (int j = 0; j < 3; j++) partial[blockIdx.x * 3 + j] = acc[j];
}

cudaError_t launch_obs_basic(const double2* psi, const uint8_t* E, int64_t N, double* partial, int grid,
                             cudaStream_t st) {
  obs_basic_kernel<<<grid, 256, 0, st>>>(psi, E, N, partial);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) obs_peer_dot_kernel(const double2* psi, const PeerDotArgs a, int64_t N,
                                                            double* partial) {
  __shared__ double sh[32 * 3];
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N; x += (int64_t)gridDim.x * blockDim.x) {
    const double2 u = psi[x];
#pragma unroll
    for (int t = 0; t < 3; t++)
      if (t < a.g) {
        const double2 w = __ldcg(a.peer[t] + x);  // another GPU's memory: no L1 reuse
        acc[t] += fma(u.x, w.x, u.y * w.y);
      }
  }
  block_reduce<3>(acc, sh);
  if (threadIdx.x == 0)
    for (int j = 0; j < 3; j++) partial[blockIdx.x * 3 + j] = acc[j];
}

cudaError_t launch_obs_peer_dot(const double2* psi, const PeerDotArgs& a, int64_t N, double* partial, int grid,
                                cudaStream_t st) {
  obs_peer_dot_kernel<<<grid, 256, 0, st>>>(psi, a, N, partial);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) obs_sigma_kernel(const SigmaArgs a, double* partial) {
  extern __shared__ double2 tile[];
  __shared__ double sh[32 * TILE_BITS];
  double acc[TILE_BITS];
#pragma unroll
  for (int j = 0; j < TILE_BITS; j++) acc[j] = 0.0;
  const int tsize = 1 << a.k, half = tsize >> 1;
  for (int64_t T = blockIdx.x; T < a.ntiles; T += gridDim.x) {
    int64_t base = 0;
#pragma unroll
    for (int s = 0; s < MAX_SEGS; s++)
      if (s < a.nseg) base += ((T >> a.seg_src[s]) & (((int64_t)1 << a.seg_len[s]) - 1)) << a.seg_dst[s];
    for (int l = threadIdx.x; l < tsize; l += blockDim.x) {
      int64_t o = base;
#pragma unroll
      for (int b = 0; b < TILE_BITS; b++)
        if (b < a.k && ((l >> b) & 1)) o += (int64_t)1 << a.phys[b];
      tile[l] = a.psi[o];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < TILE_BITS; j++) {
      if (j < a.k && ((a.mask >> j) & 1)) {
        for (int p = threadIdx.x; p < half; p += blockDim.x) {
          const int x = ((p >> j) << (j + 1)) | (p & ((1 << j) - 1));
          const double2 u = tile[x], w = tile[x | (1 << j)];
          acc[j] += fma(u.x, w.x, u.y * w.y);
        }
      }
    }
    __syncthreads();
  }
  block_reduce<TILE_BITS>(acc, sh);
  if (threadIdx.x == 0)
    for (int j = 0; j < TILE_BITS; j++) partial[blockIdx.x * TILE_BITS + j] = acc[j];
}

cudaError_t launch_obs_sigma(const SigmaArgs& a, double* partial, int grid, cudaStream_t st) {
  const size_t smem = sizeof(double2) * ((size_t)1 << a.k);
  cudaError_t e = cudaFuncSetAttribute(obs_sigma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double2) * TILE));
  if (e != cudaSuccess) return e;
  obs_sigma_kernel<<<grid, 256, smem, st>>>(a, partial);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) gather_success_kernel(const double2* psi, const uint64_t* Z, int64_t nz,
                                                              uint64_t x_offset, double* out) {
  __shared__ double sh[32];
  double acc[1] = {0.0};
  for (int64_t i = threadIdx.x; i < nz; i += blockDim.x) {
    const double2 v = psi[Z[i] - x_offset];
    acc[0] += fma(v.x, v.x, v.y * v.y);
  }
  block_reduce<1>(acc, sh);
  if (threadIdx.x == 0) out[0] = acc[0];
}

cudaError_t launch_gather_success(const double2* psi, const uint64_t* Z, int64_t nz, uint64_t x_offset, double* out,
                                  cudaStream_t st) {
  gather_success_kernel<<<1, 256, 0, st>>>(psi, Z, nz, x_offset, out);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) reduce_partials_kernel(const double* partial, int nblocks, int stride,
                                                               int nvals, double* out) {
  __shared__ double sh[32];
  for (int j = 0; j < nvals; j++) {
    double acc[1] = {0.0};
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) acc[0] += partial[(int64_t)b * stride + j];
    block_reduce<1>(acc, sh);
    if (threadIdx.x == 0) out[j] = acc[0];
  }
}

cudaError_t launch_reduce_partials(const double* partial, int nblocks, int stride, int nvals, double* out,
                                   cudaStream_t st) {
  reduce_partials_kernel<<<1, 256, 0, st>>>(partial, nblocks, stride, nvals, out);
  return cudaGetLastError();
}

}  // namespace qaa

namespace qaa {
// Eg[T*4096 + pack(l)] = E[tbase(T) + off(l)]: the energy slice of tile T of a group,
// contiguous so the TMA pass can bulk-copy it next to the amplitudes.
struct PermArgs {
  int phys[TILE_BITS];
  int nseg;
  int seg_src[MAX_SEGS], seg_dst[MAX_SEGS], seg_len[MAX_SEGS];
  int64_t ntiles;
  int pb3;
};
__global__ void __launch_bounds__(256) permute_energy_kernel(const uint8_t* E, uint8_t* Eg, const PermArgs a,
                                                             const uint16_t* pos) {
  for (int64_t T = blockIdx.x; T < a.ntiles; T += gridDim.x) {
    int64_t base = 0;
#pragma unroll
    for (int s = 0; s < MAX_SEGS; s++)
      if (s < a.nseg) base += ((T >> a.seg_src[s]) & (((int64_t)1 << a.seg_len[s]) - 1)) << a.seg_dst[s];
    for (int l = threadIdx.x; l < TILE; l += blockDim.x) {
      int64_t o = base;
#pragma unroll
      for (int b = 0; b < TILE_BITS; b++)
        if ((l >> b) & 1) o += (int64_t)1 << a.phys[b];
      // packed for the D of the group-k programs (pass_tma.cu diag): thread
      // t = lane + 32 warp holds register r at byte 16 t + r, in pattern PB, or
      // PB3 (tile bits 3 and 7 swapped between register and lane bit 3) when
      // the group rotates tile bit 3
      int lane = (l & 15) | (((l >> 8) & 1) << 4), r = (l >> 4) & 15;
      if (a.pb3) {
        lane = (l & 7) | (((l >> 7) & 1) << 3) | (((l >> 8) & 1) << 4);
        r = ((l >> 4) & 7) | (((l >> 3) & 1) << 3);
      }
      const int warp = l >> 9;
      Eg[T * TILE + (pos ? (int)pos[l] : (((lane + 32 * warp) << 4) | r))] = E[o];
    }
  }
}
cudaError_t launch_permute_energy(const uint8_t* E, uint8_t* Eg, const int (&phys)[TILE_BITS], int nseg,
                                  const int* seg_src, const int* seg_dst, const int* seg_len, int64_t ntiles,
                                  int pb3, int num_sms, cudaStream_t st, const uint16_t* pos) {
  PermArgs a;
  a.pb3 = pb3;
  for (int b = 0; b < TILE_BITS; b++) a.phys[b] = phys[b];
  a.nseg = nseg;
  for (int s = 0; s < MAX_SEGS; s++) {
    a.seg_src[s] = s < nseg ? seg_src[s] : 0;
    a.seg_dst[s] = s < nseg ? seg_dst[s] : 0;
    a.seg_len[s] = s < nseg ? seg_len[s] : 0;
  }
  a.ntiles = ntiles;
  int64_t grid = ntiles < (int64_t)num_sms * 8 ? ntiles : (int64_t)num_sms * 8;
  permute_energy_kernel<<<(int)grid, 256, 0, st>>>(E, Eg, a, pos);
  return cudaGetLastError();
}
// ------------------------------------------------------------------ sharded phase barrier (device side)
// One thread: release this rank's prior stores at system scope, add 1 to every
// rank's arrival counter (CUDA-IPC-mapped; peers' counters over NVLink), then
// wait until the own counter reaches `target` = epoch * world. Kernels queued
// behind it on the stream see every peer's pre-barrier stores. A bounded wait:
// a rank that never arrives becomes a trap (launch error), not a hang.
struct ShardSyncArgs {
  unsigned* peer[8];
  unsigned* mine;
  int world;
  unsigned target;
};
__global__ void shard_barrier_kernel(const ShardSyncArgs a) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int r = 0; r < a.world; r++) asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(a.peer[r]) : "memory");
  for (unsigned long long it = 0;; it++) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a.mine) : "memory");
    if ((int)(v - a.target) >= 0) break;
    __nanosleep(100);
    if (it > (1ull << 31)) __trap();
  }
  __threadfence_system();
}
cudaError_t launch_shard_barrier(unsigned* const* peer_flags, unsigned* my_flag, int world, unsigned target,
                                 cudaStream_t st) {
  ShardSyncArgs a;
  for (int r = 0; r < 8; r++) a.peer[r] = r < world ? peer_flags[r] : nullptr;
  a.mine = my_flag;
  a.world = world;
  a.target = target;
  shard_barrier_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}
}  // namespace qaa
