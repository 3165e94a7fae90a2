// api_tma.cu -- per-group TMA tensor maps, permuted energy tables and the L2-blocked chunk plans (single GPU and sharded).
#include "api_internal.hpp"

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
static bool encode_group(qaa_ctx* ctx, const Group& gr, void* base, CUtensorMap* mapp, TmaArgs* tp,
                         bool swz128 = false) {
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
          // 128-byte swizzle: the inner box dim is exactly one 128-byte row (3 bits)
          const int lim = nd == 0 ? (swz128 ? 3 : 7) : 8;
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
                       box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
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
qaa_status build_shard_top(qaa_ctx* ctx) {
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

void build_shard_super(qaa_ctx* ctx) {
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

qaa_status build_tma(qaa_ctx* ctx) {
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
  // the tensor-memory variant's tables are built on its first use (build_tm)
  ctx->tm_built = false;
  for (int k = 0; k < 4; k++) ctx->tm_ok[k] = 0;
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return QAA_OK;
}

// Tensor-memory L2-blocked step (pass_tmem.cu): per paired group k a tensor map
// with the 128-byte swizzle (the landed tile is read conflict-free in pattern
// K1) and, when the pair carries D (three-group plans), the energy slices
// packed for pattern K3. Needs the group's tile bits 0..2 to be the three
// 128-byte-row bits (row_bits = 3; unrotated padding bits above them are
// fine). Missing pieces leave tm_ok[k] = 0 (legacy kernel).
qaa_status build_tm(qaa_ctx* ctx) {
  ctx->tm_built = true;
  for (int k = 0; k < 4; k++) ctx->tm_ok[k] = 0;
  const int P = (int)ctx->geom.groups.size();
  const size_t N = (size_t)1 << ctx->L;
  if (!(P == 3 || P == 4)) return QAA_OK;
  if (!ctx->d_pos_tm) {
    std::vector<uint16_t> pos(TILE);
    superpass_tm_energy_positions(pos.data());
    CUDA_TRY(cudaMalloc(&ctx->d_pos_tm, TILE * sizeof(uint16_t)));
    CUDA_TRY(cudaMemcpy(ctx->d_pos_tm, pos.data(), TILE * sizeof(uint16_t), cudaMemcpyHostToDevice));
  }
  for (int k = 1; k < P; k++) {
    if (!ctx->super_ok[k]) continue;
    const Group& gr = ctx->geom.groups[(size_t)k];
    if (gr.phys[0] != 0 || gr.phys[1] != 1 || gr.phys[2] != 2) continue;  // 128-byte rows
    TmaArgs& t = ctx->tm_geo[k];
    if (!encode_group(ctx, gr, (void*)ctx->state, &ctx->tmaps_sw[k], &t, true) || t.contiguous) continue;
    if (P == 3) {  // the pair carries D: packed energies for pattern K3
      if (ctx->Eg_tm_cap[k] < N) {
        if (ctx->Eg_tm[k]) cudaFree(ctx->Eg_tm[k]);
        ctx->Eg_tm[k] = nullptr;
        ctx->Eg_tm_cap[k] = 0;
        if (cudaMalloc(&ctx->Eg_tm[k], N) != cudaSuccess) {
          cudaGetLastError();
          ctx->Eg_tm[k] = nullptr;
          continue;
        }
        ctx->Eg_tm_cap[k] = N;
      }
      CUDA_TRY(launch_permute_energy(ctx->E, ctx->Eg_tm[k], gr.phys, gr.nseg, gr.seg_src, gr.seg_dst, gr.seg_len,
                                     gr.ntiles, 0, ctx->num_sms, ctx->stream, ctx->d_pos_tm));
      ctx->stats.kernel_launches_total++;
    }
    ctx->tm_ok[k] = 1;
  }
  return QAA_OK;
}
