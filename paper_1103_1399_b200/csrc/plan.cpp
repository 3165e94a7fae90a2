// plan.cpp -- see plan.hpp. Pure host code.
#include "plan.hpp"

#include <algorithm>
#include <cstring>

namespace qaa {

static const int kRegLocal[NPAT][4] = {{8, 9, 10, 11}, {4, 5, 6, 7}, {0, 1, 2, 3}};
static const int kLaneLocal[NPAT][5] = {{0, 1, 2, 3, 4}, {0, 1, 2, 3, 8}, {4, 5, 6, 7, 8}};
static const int kWarpLocal[NPAT][3] = {{5, 6, 7}, {9, 10, 11}, {9, 10, 11}};

int pattern_reg_local(int pat, int i) { return kRegLocal[pat][i]; }
int pattern_lane_local(int pat, int i) { return kLaneLocal[pat][i]; }
int pattern_warp_local(int pat, int i) { return kWarpLocal[pat][i]; }
bool pattern_storable(int pat) { return pat == PA || pat == PB; }

static uint32_t lane_mask(int pat) {
  uint32_t m = 0;
  for (int i = 0; i < 5; i++) m |= 1u << kLaneLocal[pat][i];
  return m;
}

bool build_geometry(int L, int row_bits, Geometry* g, std::string* err) {
  if (row_bits < 1 || row_bits > 5) {
    if (err) *err = "row_bits must be in 1..5";
    return false;
  }
  if (L <= TILE_BITS) {
    if (err) *err = "geometry needs L > 12 (smaller states use the resident kernel)";
    return false;
  }
  g->L = L;
  g->row_bits = row_bits;
  g->groups.clear();
  const int c = row_bits;
  const int q = TILE_BITS - c;  // rotated bits per later group
  // remaining bits [12, L) split into the fewest chunks of <= q, balanced
  const int R = L - TILE_BITS;
  const int nchunks = (R + q - 1) / q;
  std::vector<std::vector<int>> chunks;
  int next = TILE_BITS;
  for (int i = 0; i < nchunks; i++) {
    int len = R / nchunks + (i < R % nchunks ? 1 : 0);
    std::vector<int> ch;
    for (int b = 0; b < len; b++) ch.push_back(next++);
    chunks.push_back(ch);
  }
  auto finish = [&](Group& gr) {
    bool in_tile[64] = {false};
    for (int b = 0; b < TILE_BITS; b++) in_tile[gr.phys[b]] = true;
    std::vector<int> rest;
    for (int p = 0; p < L; p++)
      if (!in_tile[p]) rest.push_back(p);
    gr.nseg = 0;
    for (size_t i = 0; i < rest.size();) {
      size_t j = i;
      while (j + 1 < rest.size() && rest[j + 1] == rest[j] + 1) j++;
      gr.seg_src[gr.nseg] = (int)i;
      gr.seg_dst[gr.nseg] = rest[i];
      gr.seg_len[gr.nseg] = (int)(j - i + 1);
      gr.nseg++;
      i = j + 1;
    }
    gr.ntiles = (int64_t)1 << (L - TILE_BITS);
    gr.rot_phys = 0;
    for (int b = 0; b < TILE_BITS; b++)
      if (gr.rot_local >> b & 1) gr.rot_phys |= 1ull << gr.phys[b];
  };
  Group g0;
  for (int b = 0; b < TILE_BITS; b++) g0.phys[b] = b;
  g0.rot_local = (1u << TILE_BITS) - 1;
  finish(g0);
  g->groups.push_back(g0);
  for (auto& ch : chunks) {
    Group gr;
    std::vector<int> bits;
    for (int b = 0; b < c; b++) bits.push_back(b);
    // padding: the lowest non-row bits (rotated by group 0, not here); keeping
    // them next to the rows lengthens the contiguous runs of short chunks.
    int pad = q - (int)ch.size();
    for (int b = 0; b < pad; b++) bits.push_back(c + b);
    for (int p : ch) bits.push_back(p);
    std::sort(bits.begin(), bits.end());
    gr.rot_local = 0;
    for (int b = 0; b < TILE_BITS; b++) {
      gr.phys[b] = bits[b];
      if (std::find(ch.begin(), ch.end(), bits[b]) != ch.end()) gr.rot_local |= 1u << b;
    }
    finish(gr);
    g->groups.push_back(gr);
  }
  return true;
}

void build_pass_schedule(int P, int64_t K, int step_spanning, std::vector<PassPlan>* out) {
  out->clear();
  if (K <= 0 || P <= 0) return;
  if (step_spanning == 2 && P >= 3) {
    // Group 0 never hosts D: D_{k+1} always rides on a strided group g >= 1
    // (rotate step k, D_{k+1}, rotate step k+1 on its tile), and every step
    // visits group 0 with a plain contiguous pass. Same pass count as the
    // cyclic schedule (K (P-1) + 1) but without the 4-transpose group-0 D pass
    // and without plain passes over 128-byte-row tiles when P = 3.
    int dg = 1;
    out->push_back({1, -1, 0, 0});
    for (int64_t k = 0; k < K; k++) {
      std::vector<int> rem{0};
      for (int g = 1; g < P; g++)
        if (g != dg) rem.push_back(g);
      int next = dg;
      for (size_t i = 0; i < rem.size(); i++) {
        const int g = rem[i];
        if (i + 1 == rem.size() && k + 1 < K) {
          out->push_back({g, k, k + 1, k + 1});
          next = g;
        } else {
          out->push_back({g, k, -1, -1});
        }
      }
      dg = next;
    }
    return;
  }
  if (!step_spanning || P == 1) {
    for (int64_t k = 0; k < K; k++)
      for (int g = 0; g < P; g++) out->push_back({g, g == 0 ? -1 : k, g == 0 ? k : -1, g == 0 ? k : -1});
    return;
  }
  // pass 0: D_0 then X_0 on group 0
  out->push_back({0, -1, 0, 0});
  int64_t step = 0;
  int done = 1;  // groups of X_step applied so far (cyclic order starting after D_step's group)
  int g = 0;
  while (true) {
    g = (g + 1) % P;
    done++;
    if (done == P) {
      // this pass finishes X_step on group g
      if (step + 1 < K) {
        out->push_back({g, step, step + 1, step + 1});
        step++;
        done = 1;
      } else {
        out->push_back({g, step, -1, -1});
        break;
      }
    } else {
      out->push_back({g, step, -1, -1});
    }
  }
}

bool build_shard_schedule(const Geometry& geo, int gbits, int64_t K, std::vector<ShardPass>* out, std::string* err) {
  out->clear();
  const int P = (int)geo.groups.size();
  const int L = geo.L;
  if (P < 2) {
    if (err) *err = "sharding needs at least two tile groups (n - log2(world) >= 13)";
    return false;
  }
  const Group& top = geo.groups[(size_t)P - 1];
  const Group& last = geo.groups[(size_t)P - 2];
  uint32_t carried = 0;
  for (int b = 0; b < TILE_BITS; b++) {
    if (top.phys[b] >= L - gbits) carried |= 1u << b;
    if (last.phys[b] >= L - gbits) {
      if (err) *err = "remote group holds a carried bit";
      return false;
    }
  }
  int nc = 0;
  for (int b = 0; b < TILE_BITS; b++) nc += (carried >> b) & 1;
  if (nc != gbits || (carried & ~top.rot_local)) {
    if (err) *err = "top tile group does not rotate every carried qubit (n too small for this world)";
    return false;
  }
  for (int64_t k = 0; k < K; k++) {
    const int layout = (int)(k & 1);
    ShardPass f{SK_PASS, P - 1, k >= 1 ? k - 1 : -1, k >= 1 ? carried : 0u, k, k, top.rot_local, 0, layout};
    out->push_back(f);
    // groups 1..P-3, then 0, then P-2 (remote): group 0 right before the
    // layout-swap pass, so the pair [0][P-2] can run as one L2-blocked launch
    for (int i = 0; i <= P - 2; i++) {
      const int g = i < P - 3 ? i + 1 : (i == P - 3 ? 0 : P - 2);
      out->push_back({SK_PASS, g, k, geo.groups[(size_t)g].rot_local, -1, -1, 0u, g == P - 2 ? 1 : 0, layout});
    }
  }
  const int lay = (int)(K & 1);
  out->push_back({SK_PASS, P - 1, K - 1, carried, -1, -1, 0u, 0, lay});
  if (lay == 1) out->push_back({SK_REMAP, -1, -1, 0u, -1, -1, 0u, 1, 1});
  return true;
}

// ---------------------------------------------------------------- programs
namespace {
struct Best {
  double cost = 1e30;
  std::vector<Op> ops;
  int e_pattern = -1, final_pattern = -1, n_exch = 0, n_shfl = 0;
};

constexpr double kExchCost = 1.0;
constexpr double kShflCost = 0.5;

void search(int pat, uint32_t rem_pre, bool has_d, bool d_done, uint32_t rem_post, double cost, int n_exch,
            int n_shfl, int e_pat, std::vector<Op>& ops, Best& best, int depth) {
  if (cost >= best.cost) return;
  // visit `pat`: rotate registers for free, then optional lane shuffles.
  const uint32_t lm = lane_mask(pat);
  size_t mark = ops.size();
  uint32_t pre = rem_pre, post = rem_post;
  bool dd = d_done;
  int ep = e_pat;
  auto emit_regs = [&](uint32_t& rem, uint8_t slot) {
    for (int i = 0; i < 4; i++) {
      int lb = pattern_reg_local(pat, i);
      if (rem >> lb & 1) {
        ops.push_back({OP_ROT_REG, (uint8_t)i, slot, 0});
        rem &= ~(1u << lb);
      }
    }
  };
  // enumerate which lane bits of the pending phase to shuffle here
  auto lanes_of = [&](uint32_t rem) { return rem & lm; };
  // phase pre
  emit_regs(pre, 0);
  uint32_t lp = lanes_of(pre);
  // try all subsets of lane bits for pre (usually 0..2 bits)
  std::vector<uint32_t> subs_pre;
  for (uint32_t s = lp;; s = (s - 1) & lp) {
    subs_pre.push_back(s);
    if (s == 0) break;
  }
  for (uint32_t sp : subs_pre) {
    size_t m2 = ops.size();
    uint32_t pre2 = pre & ~sp;
    int sh = 0;
    for (int i = 0; i < 5; i++)
      if (sp >> pattern_lane_local(pat, i) & 1) {
        ops.push_back({OP_ROT_LANE, (uint8_t)i, 0, 0});
        sh++;
      }
    bool dd2 = dd;
    int ep2 = ep;
    uint32_t post2 = post;
    std::vector<uint32_t> subs_post{0};
    if (pre2 == 0 && has_d && !dd2) {
      ops.push_back({OP_DIAG, 0, 0, 0});
      dd2 = true;
      ep2 = pat;
    }
    size_t m3 = ops.size();
    if (pre2 == 0 && (dd2 || !has_d)) {
      emit_regs(post2, 1);
      uint32_t lq = lanes_of(post2);
      subs_post.clear();
      for (uint32_t s = lq;; s = (s - 1) & lq) {
        subs_post.push_back(s);
        if (s == 0) break;
      }
    }
    size_t m4 = ops.size();
    for (uint32_t sq : subs_post) {
      uint32_t post3 = post2 & ~sq;
      int sh2 = 0;
      for (int i = 0; i < 5; i++)
        if (sq >> pattern_lane_local(pat, i) & 1) {
          ops.push_back({OP_ROT_LANE, (uint8_t)i, 1, 0});
          sh2++;
        }
      double c2 = cost + kShflCost * (sh + sh2);
      bool complete = pre2 == 0 && (dd2 || !has_d) && post3 == 0;
      if (complete && pattern_storable(pat)) {
        if (c2 < best.cost) {
          best.cost = c2;
          best.ops = ops;
          best.e_pattern = ep2;
          best.final_pattern = pat;
          best.n_exch = n_exch;
          best.n_shfl = n_shfl + sh + sh2;
        }
      } else if (depth < 6) {
        for (int np = 0; np < NPAT; np++) {
          if (np == pat) continue;
          ops.push_back({OP_XCHG, (uint8_t)np, 0, 0});
          search(np, pre2, has_d, dd2, post3, c2 + kExchCost, n_exch + 1, n_shfl + sh + sh2, ep2, ops, best,
                 depth + 1);
          ops.pop_back();
        }
      }
      ops.resize(m4);
    }
    ops.resize(m3);
    ops.resize(m2);
  }
  ops.resize(mark);
}
}  // namespace

bool build_program(uint32_t pre_local, bool has_d, uint32_t post_local, Program* prog) {
  Best best;
  std::vector<Op> ops;
  search(PA, pre_local, has_d, false, post_local, 0.0, 0, 0, -1, ops, best, 0);
  if (best.final_pattern < 0 || (int)best.ops.size() > MAX_OPS) return false;
  prog->nops = (int)best.ops.size();
  for (int i = 0; i < prog->nops; i++) prog->ops[i] = best.ops[i];
  prog->e_pattern = has_d ? best.e_pattern : -1;
  prog->final_pattern = best.final_pattern;
  prog->n_exch = best.n_exch;
  prog->n_shfl = best.n_shfl;
  return true;
}

}  // namespace qaa
