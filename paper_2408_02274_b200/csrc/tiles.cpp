// Host-side (plan time) owner partition and MMA row tiles of one propagation
// level: the native builder behind octree.row_tiles.  Pure integer work on
// the accumulation plan (reference _accum_types, ifgf.py:705-749), threaded
// over parent rows.
//
// Per parent segment row (<= 8 instances, one per child box):
//  1. signature order: nodes stably sorted by the key that packs, 4 bits per
//     instance slot, the node's sigma group under each child (0xF for absent
//     slots), so nodes that share child segments under every child are
//     adjacent;
//  2. warp cuts: the order is split into WARP_PARTS contiguous sets, cut k in
//     [15k - R, 15k + R] (sets of 7..23 nodes), chosen by a small DP that
//     minimises the largest per-warp tile count over the row's instances
//     (the CTA waits for its slowest warp before the K3 transform), ties by
//     the row's total tile count, then by the earliest cut;
//  3. tiles: per (instance, warp) the owned slots are stably grouped by sigma
//     group and cut into runs of <= 8 rows.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ifgfb.h"

namespace ifgfb {
void set_error(const std::string& msg);
}

namespace {

constexpr int NN = 75, WP = 5, PER = 15, MAX_R = 4, MAX_SET = 24, MAX_INST = 8;
constexpr int MAX_GROUPS = NN;   // a type's 75 nodes fall into <= 75 child segments

struct RowIn {
  const int64_t* inst_off;
  const int64_t* inst_type;
  const uint8_t* group_id;   // (n_types, 75)
};

// order + cuts of row r; returns false on malformed input
// Wide-warp cuts (IFGFB_K4=wide): W contiguous sets of the signature order,
// cut k within +-R of the even position 75k/W, every set 1..32 nodes (one
// lane per node).  The wide kernel runs up to 4 row tiles of one sigma group
// together, so what a split costs is executed DMMA work: the DP minimises
// balance_w * W * (largest per-warp tile count) + total_w * (the row's tile
// count) (weights 1/0: the 5-warp rule; 0/1: fewest tiles), ties by the
// other term, then by the earliest cuts.  One (max, total) label per DP
// state: exact for the two pure objectives, a heuristic (within ~1% of the
// brute-force optimum, tests/test_plan.py) for mixed weights.
bool wide_cuts(int ni, const uint8_t (*gs)[NN], int W, int R, int total_w, int balance_w,
               uint8_t* cuts, int pass_w = 0) {
  constexpr int MAXW = 5, MAXR = 8, NO = 2 * MAXR + 1, WIDE_SET = 32;
  if (W < 1 || W > MAXW || R < 0 || R > MAXR) return false;
  auto sweep = [&](int a, int bmax, int* tiles_upto) {
    uint8_t cnt[MAX_INST][MAX_GROUPS];
    std::memset(cnt, 0, sizeof(cnt));
    int tot = 0;
    tiles_upto[0] = 0;
    // cost in quarter tiles: 4 per row tile + pass_w per pass (a pass = up to
    // 2 row tiles of one sigma group: its B-load latency and tile formation)
    for (int b = a; b < bmax; ++b) {
      for (int i = 0; i < ni; ++i) {
        const int c = cnt[i][gs[i][b]]++;
        if (c % 8 == 0) tot += 4;
        if (c % 16 == 0) tot += pass_w;
      }
      tiles_upto[b + 1 - a] = tot;
    }
  };
  int pos[MAXW + 1][NO], npos[MAXW + 1];
  int bmax_[MAXW + 1][NO], btot_[MAXW + 1][NO], from[MAXW + 1][NO];
  npos[0] = 1; pos[0][0] = 0; bmax_[0][0] = 0; btot_[0][0] = 0;
  for (int k = 1; k <= W; ++k) {
    npos[k] = 0;
    if (k < W) {
      const int even = (NN * k) / W;
      for (int o = -R; o <= R; ++o) {
        const int c = even + o;
        if (c >= k && c <= NN - (W - k)) pos[k][npos[k]++] = c;
      }
    } else {
      pos[k][npos[k]++] = NN;
    }
    for (int c = 0; c < npos[k]; ++c) { bmax_[k][c] = INT32_MAX; btot_[k][c] = INT32_MAX; from[k][c] = -1; }
    for (int pidx = 0; pidx < npos[k - 1]; ++pidx) {
      if (bmax_[k - 1][pidx] == INT32_MAX) continue;
      const int a = pos[k - 1][pidx];
      const int bmax = std::min(pos[k][npos[k] - 1], a + WIDE_SET);
      if (bmax <= a) continue;
      int upto[WIDE_SET + 1];
      sweep(a, bmax, upto);
      for (int c = 0; c < npos[k]; ++c) {
        const int b = pos[k][c];
        if (b - a < 1 || b - a > WIDE_SET) continue;
        const int t = upto[b - a];
        const int m = std::max(bmax_[k - 1][pidx], t), tt = btot_[k - 1][pidx] + t;
        const int64_t score = (int64_t)balance_w * W * m + (int64_t)total_w * tt;
        const int64_t best = bmax_[k][c] == INT32_MAX ? INT64_MAX
            : (int64_t)balance_w * W * bmax_[k][c] + (int64_t)total_w * btot_[k][c];
        const bool better = score < best ||
            (score == best && (m < bmax_[k][c] || (m == bmax_[k][c] && tt < btot_[k][c])));
        if (better) { bmax_[k][c] = m; btot_[k][c] = tt; from[k][c] = pidx; }
      }
    }
  }
  if (from[W][0] < 0) return false;
  cuts[0] = 0;
  cuts[W] = NN;
  int c = 0;
  for (int k = W; k >= 2; --k) {
    c = from[k][c];
    cuts[k - 1] = (uint8_t)pos[k - 1][c];
  }
  for (int k = W + 1; k <= WP; ++k) cuts[k] = NN;   // unused entries of the 6-byte record
  return true;
}

bool row_partition(const RowIn& in, int64_t r, int R, uint8_t* order, uint8_t* cuts,
                   int wide_w = 0, int total_w = 0, int balance_w = 1, int pass_w = 0) {
  const int64_t i0 = in.inst_off[r], ni = in.inst_off[r + 1] - i0;
  if (ni < 0 || ni > MAX_INST) return false;
  int64_t key[NN];
  for (int n = 0; n < NN; ++n) {
    int64_t k = 0;
    for (int i = 0; i < MAX_INST; ++i) {
      const int64_t g = i < ni ? in.group_id[in.inst_type[i0 + i] * NN + n] : 0xF;
      k |= g << (4 * (7 - i));
    }
    key[n] = k;
  }
  int idx[NN];
  std::iota(idx, idx + NN, 0);
  std::stable_sort(idx, idx + NN, [&](int a, int b) { return key[a] < key[b]; });
  for (int n = 0; n < NN; ++n) order[n] = (uint8_t)idx[n];
  // groups in row order per instance
  uint8_t gs[MAX_INST][NN];
  for (int i = 0; i < ni; ++i) {
    const uint8_t* g = in.group_id + in.inst_type[i0 + i] * NN;
    for (int n = 0; n < NN; ++n) gs[i][n] = g[idx[n]];
  }
  if (wide_w > 0) return wide_cuts((int)ni, gs, wide_w, R, total_w, balance_w, cuts, pass_w);
  // tiles of [a, b) summed over instances, for b swept upward from a
  auto sweep = [&](int a, int bmax, int* tiles_upto /* index b - a */) {
    uint8_t cnt[MAX_INST][MAX_GROUPS];
    std::memset(cnt, 0, sizeof(cnt));
    int tot = 0;
    tiles_upto[0] = 0;
    for (int b = a; b < bmax; ++b) {
      for (int i = 0; i < ni; ++i)
        if (cnt[i][gs[i][b]]++ % 8 == 0) ++tot;
      tiles_upto[b + 1 - a] = tot;
    }
  };
  // DP over cut positions: stage k chooses cut c_k (c_0 = 0, c_5 = 75)
  constexpr int NO = 2 * MAX_R + 1;
  int best_max[NO], best_tot[NO], from[WP][NO];
  int prev_pos[NO], n_prev = 1;
  prev_pos[0] = 0;
  int pmax[NO] = {0}, ptot[NO] = {0};
  for (int k = 1; k <= WP; ++k) {
    int cur_pos[NO], n_cur = 0;
    if (k < WP) {
      for (int o = -R; o <= R; ++o) cur_pos[n_cur++] = PER * k + o;
    } else {
      cur_pos[n_cur++] = NN;
    }
    for (int c = 0; c < n_cur; ++c) { best_max[c] = INT32_MAX; best_tot[c] = INT32_MAX; }
    for (int p = 0; p < n_prev; ++p) {
      const int a = prev_pos[p], bmax = cur_pos[n_cur - 1];
      int upto[NN + 1];
      sweep(a, bmax, upto);
      for (int c = 0; c < n_cur; ++c) {
        const int b = cur_pos[c];
        if (b - a < 1 || b - a > MAX_SET - 1) continue;
        const int t = upto[b - a];
        const int m = std::max(pmax[p], t), tt = ptot[p] + t;
        if (m < best_max[c] || (m == best_max[c] && tt < best_tot[c])) {
          best_max[c] = m;
          best_tot[c] = tt;
          from[k - 1][c] = p;
        }
      }
    }
    for (int c = 0; c < n_cur; ++c) {
      prev_pos[c] = cur_pos[c];
      pmax[c] = best_max[c];
      ptot[c] = best_tot[c];
    }
    n_prev = n_cur;
  }
  // backtrack: from[k-1][c] = index of the stage k-1 cut; stage positions
  // are PER*k + (index - R)
  cuts[0] = 0;
  cuts[WP] = NN;
  int c = 0;
  for (int k = WP; k >= 2; --k) {
    c = from[k - 1][c];
    cuts[k - 1] = (uint8_t)(PER * (k - 1) + c - R);
  }
  return true;
}

// tiles of (instance i of row r, warp w): writes up to MAX_SET records when
// out != nullptr; returns the count
int warp_tiles(const RowIn& in, int64_t inst, const uint8_t* order, const uint8_t* cuts,
               int w, uint8_t* out) {
  const int lo = cuts[w], hi = cuts[w + 1];
  const uint8_t* g = in.group_id + in.inst_type[inst] * NN;
  int slots[MAX_SET];
  const int n = hi - lo;
  for (int s = 0; s < n; ++s) slots[s] = s;
  std::stable_sort(slots, slots + n,
                   [&](int a, int b) { return g[order[lo + a]] < g[order[lo + b]]; });
  int count = 0, run = 0, prev = -1;
  uint8_t* rec = nullptr;
  for (int s = 0; s < n; ++s) {
    const int gr = g[order[lo + slots[s]]];
    if (gr != prev || run == 8) {
      if (out) {
        rec = out + 16 * count;
        std::memset(rec, 0xFF, 16);
        rec[0] = (uint8_t)gr;
        rec[1] = 0;
      }
      ++count;
      run = 0;
      prev = gr;
    }
    if (out) {
      rec[2 + run] = (uint8_t)slots[s];
      rec[1] = (uint8_t)(run + 1);
    }
    ++run;
  }
  return count;
}

template <class F>
void parallel_rows(int64_t n_rows, int n_threads, F&& f) {
  if (n_threads <= 0) n_threads = (int)std::max(1u, std::thread::hardware_concurrency());
  n_threads = (int)std::min<int64_t>(n_threads, std::max<int64_t>(1, n_rows / 256));
  std::vector<std::thread> pool;
  const int64_t chunk = (n_rows + n_threads - 1) / n_threads;
  for (int t = 0; t < n_threads; ++t) {
    const int64_t r0 = t * chunk, r1 = std::min(n_rows, r0 + chunk);
    if (r0 >= r1) break;
    pool.emplace_back([=, &f] { f(r0, r1); });
  }
  for (auto& th : pool) th.join();
}

bool check_groups(const uint8_t* group_id, int64_t n_types) {
  for (int64_t i = 0; i < n_types * NN; ++i)
    if (group_id[i] >= MAX_GROUPS) return false;
  return true;
}

}  // namespace

extern "C" {

int ifgfb_row_tiles_plan(int64_t n_rows, const int64_t* inst_off, const int64_t* inst_type,
                         int64_t n_types, const uint8_t* group_id, uint8_t* row_order,
                         uint8_t* row_cuts, int64_t* tile_off, int32_t cut_radius,
                         int32_t n_threads) {
  // tile_off == NULL: order and cuts only (tile-free plans form the tiles on
  // the device)
  if (n_rows < 0 || !inst_off || (n_rows && (!row_order || !row_cuts)) ||
      cut_radius < 0 || cut_radius > MAX_R) {
    ifgfb::set_error("ifgfb_row_tiles_plan: bad arguments");
    return IFGFB_ERR_ARG;
  }
  if (!check_groups(group_id, n_types)) {
    ifgfb::set_error("ifgfb_row_tiles_plan: sigma group id >= 75");
    return IFGFB_ERR_ARG;
  }
  const int64_t ni = inst_off[n_rows] - inst_off[0];
  for (int64_t i = 0; i < ni; ++i)
    if (inst_type[inst_off[0] + i] < 0 || inst_type[inst_off[0] + i] >= n_types) {
      ifgfb::set_error("ifgfb_row_tiles_plan: inst_type out of range");
      return IFGFB_ERR_ARG;
    }
  RowIn in{inst_off, inst_type, group_id};
  std::atomic<bool> bad{false};
  // pass 1: order, cuts and per-(instance, warp) tile counts into tile_off[1..]
  parallel_rows(n_rows, n_threads, [&](int64_t r0, int64_t r1) {
    for (int64_t r = r0; r < r1; ++r) {
      uint8_t* ord = row_order + r * NN;
      uint8_t* cut = row_cuts + r * (WP + 1);
      if (!row_partition(in, r, cut_radius, ord, cut)) { bad = true; continue; }
      if (!tile_off) continue;
      for (int64_t i = inst_off[r]; i < inst_off[r + 1]; ++i)
        for (int w = 0; w < WP; ++w)
          tile_off[(i - inst_off[0]) * WP + w + 1] = warp_tiles(in, i, ord, cut, w, nullptr);
    }
  });
  if (bad) {
    ifgfb::set_error("ifgfb_row_tiles_plan: more than 8 instances in a parent row");
    return IFGFB_ERR_ARG;
  }
  if (!tile_off) return IFGFB_OK;
  tile_off[0] = 0;
  for (int64_t k = 1; k <= ni * WP; ++k) tile_off[k] += tile_off[k - 1];
  return IFGFB_OK;
}

int ifgfb_row_cuts_wide(int64_t n_rows, const int64_t* inst_off, const int64_t* inst_type,
                        int64_t n_types, const uint8_t* group_id, uint8_t* row_order,
                        uint8_t* row_cuts, int32_t n_warps, int32_t cut_radius,
                        int32_t total_weight, int32_t balance_weight, int32_t n_threads) {
  if (n_rows < 0 || !inst_off || (n_rows && (!row_order || !row_cuts)) || n_warps < 1 ||
      n_warps > WP || (NN + n_warps - 1) / n_warps > 32 || cut_radius < 0 || cut_radius > 8 ||
      total_weight < 0 || balance_weight < 0 || total_weight + balance_weight == 0) {
    ifgfb::set_error("ifgfb_row_cuts_wide: bad arguments");
    return IFGFB_ERR_ARG;
  }
  if (!check_groups(group_id, n_types)) {
    ifgfb::set_error("ifgfb_row_cuts_wide: sigma group id >= 75");
    return IFGFB_ERR_ARG;
  }
  const int64_t ni = inst_off[n_rows] - inst_off[0];
  for (int64_t i = 0; i < ni; ++i)
    if (inst_type[inst_off[0] + i] < 0 || inst_type[inst_off[0] + i] >= n_types) {
      ifgfb::set_error("ifgfb_row_cuts_wide: inst_type out of range");
      return IFGFB_ERR_ARG;
    }
  RowIn in{inst_off, inst_type, group_id};
  std::atomic<bool> bad{false};
  // cost of a pass relative to a row tile, in quarter tiles (experiment knob;
  // 0 = tiles only, the documented objective)
  const char* pw_env = std::getenv("IFGFB_WIDE_PW");
  const int pass_w = pw_env ? std::max(0, std::min(16, std::atoi(pw_env))) : 0;
  parallel_rows(n_rows, n_threads, [&](int64_t r0, int64_t r1) {
    for (int64_t r = r0; r < r1; ++r)
      if (!row_partition(in, r, cut_radius, row_order + r * NN, row_cuts + r * (WP + 1),
                         n_warps, total_weight, balance_weight, pass_w))
        bad = true;
  });
  if (bad) {
    ifgfb::set_error("ifgfb_row_cuts_wide: more than 8 instances in a parent row, or no "
                     "feasible cuts");
    return IFGFB_ERR_ARG;
  }
  return IFGFB_OK;
}

int ifgfb_row_tiles_fill(int64_t n_rows, const int64_t* inst_off, const int64_t* inst_type,
                         int64_t n_types, const uint8_t* group_id, const uint8_t* row_order,
                         const uint8_t* row_cuts, const int64_t* tile_off, uint8_t* tiles,
                         int32_t n_threads) {
  if (n_rows < 0 || !inst_off || !check_groups(group_id, n_types)) {
    ifgfb::set_error("ifgfb_row_tiles_fill: bad arguments");
    return IFGFB_ERR_ARG;
  }
  RowIn in{inst_off, inst_type, group_id};
  parallel_rows(n_rows, n_threads, [&](int64_t r0, int64_t r1) {
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t i = inst_off[r]; i < inst_off[r + 1]; ++i)
        for (int w = 0; w < WP; ++w) {
          const int64_t k = (i - inst_off[0]) * WP + w;
          warp_tiles(in, i, row_order + r * NN, row_cuts + r * (WP + 1), w,
                     tiles + 16 * tile_off[k]);
        }
  });
  return IFGFB_OK;
}

}  // extern "C"
