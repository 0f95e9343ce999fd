// C ABI of libifgfb200: plan construction (host arrays -> device), entry
// points and error reporting.  See include/ifgfb.h for the contract.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"

namespace ifgfb {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

int far_setup_kernels();

static bool to_i32(const int64_t* src, size_t n, std::vector<int>& out,
                   const char* what) {
  out.resize(n);
  for (size_t i = 0; i < n; ++i) {
    if (src[i] < INT32_MIN || src[i] > INT32_MAX) {
      set_error(std::string(what) + ": index exceeds int32");
      return false;
    }
    out[i] = static_cast<int>(src[i]);
  }
  return true;
}

#define CHECK_ARG IFGFB_CHECK_ARG
#define RC IFGFB_RC

// (re)size the two coefficient ping-pong buffers to exactly `need` segments
static int resize_coef(Plan& p, size_t need) {
  if (need == p.coef_cap) return IFGFB_OK;
  for (int i = 0; i < 2; ++i) {
    if (p.coef[i]) {
      auto it = std::find(p.allocations.begin(), p.allocations.end(), (void*)p.coef[i]);
      if (it != p.allocations.end()) p.allocations.erase(it);
      IFGFB_CUDA(cudaFree(p.coef[i]));
      p.bytes -= p.coef_cap * SEG_DOUBLES * sizeof(double);
      p.coef[i] = nullptr;
    }
  }
  for (int i = 0; i < 2; ++i) IFGFB_RC(dev_alloc(p, &p.coef[i], need * SEG_DOUBLES));
  p.coef_cap = need;
  return IFGFB_OK;
}

// size of the coefficient buffers the current mode needs
int ensure_coef(Plan& p) {
  size_t need = 1;
  if (!p.stream_parts.empty()) {
    for (const auto& part : p.stream_parts)
      for (int d = 3; d <= p.depth; ++d)
        need = std::max(need, (size_t)(part[d].seg_hi - part[d].seg_lo));
  } else {
    for (int d = 3; d <= p.depth; ++d)
      need = std::max(need, (size_t)(p.levels[d].seg_hi() - p.levels[d].seg_lo()));
  }
  return resize_coef(p, need);
}

}  // namespace ifgfb

using namespace ifgfb;

extern "C" {

int ifgfb_abi_version(void) { return IFGFB_ABI_VERSION; }
const char* ifgfb_last_error(void) { return g_err.c_str(); }

int ifgfb_device_info(char* buf, size_t len) {
  int dev = 0;
  IFGFB_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  IFGFB_CUDA(cudaGetDeviceProperties(&prop, dev));
  snprintf(buf, len, "%s sm_%d%d SMs=%d", prop.name, prop.major, prop.minor,
           prop.multiProcessorCount);
  return IFGFB_OK;
}

int ifgfb_plan_create(const ifgfb_tree_desc* t, ifgfb_plan** out) {
  CHECK_ARG(t && out, "null argument");
  CHECK_ARG(t->n_points > 0 && t->depth >= 1, "bad tree sizes");
  CHECK_ARG(t->p_s == PS && t->p_a == PA,
            "only p_s=3, p_a=5 (IfgfConfig defaults) are compiled");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error("no CUDA device available (libifgfb200 has no CPU fallback)");
    return IFGFB_ERR_CUDA;
  }
  auto* h = new ifgfb_plan();
  Plan& p = h->p;
  IFGFB_CUDA(cudaGetDevice(&p.device));
  p.n = t->n_points;
  p.depth = t->depth;
  p.levels.resize(p.depth + 1);
  int rc = dev_upload(p, &p.points_tree, t->points_tree, (size_t)p.n * 3);
  std::vector<int> perm;
  if (rc == IFGFB_OK && !to_i32(t->perm, p.n, perm, "perm")) rc = IFGFB_ERR_ARG;
  if (rc == IFGFB_OK) rc = dev_upload(p, &p.perm, perm.data(), perm.size());
  if (rc == IFGFB_OK) rc = far_setup_kernels();
  if (rc != IFGFB_OK) {
    ifgfb_plan_destroy(h);
    return rc;
  }
  *out = h;
  return IFGFB_OK;
}

int ifgfb_plan_add_level(ifgfb_plan* h, const ifgfb_level_desc* d) {
  CHECK_ARG(h && d, "null argument");
  Plan& p = h->p;
  CHECK_ARG(!p.finalized, "plan already finalized");
  CHECK_ARG(d->level >= 3 && d->level <= p.depth, "level out of range");
  Level& L = p.levels[d->level];
  L.d = d->level;
  L.n_boxes = d->n_boxes;
  L.n_s = d->n_s;
  L.n_a = d->n_a;
  L.side = d->side;
  L.h = d->h;
  L.delta_s = d->delta_s;
  L.delta_a = d->delta_a;
  CHECK_ARG(d->n_segments <= INT32_MAX, "too many segments for int32 rows");
  L.n_seg = (int)d->n_segments;
  RC(dev_upload(p, &L.centers, d->centers, (size_t)L.n_boxes * 3));
  std::vector<int> tmp;
  if (!to_i32(d->pt_start, L.n_boxes, tmp, "pt_start")) return IFGFB_ERR_ARG;
  RC(dev_upload(p, &L.pt_start, tmp.data(), tmp.size()));
  if (!to_i32(d->pt_count, L.n_boxes, tmp, "pt_count")) return IFGFB_ERR_ARG;
  RC(dev_upload(p, &L.pt_count, tmp.data(), tmp.size()));
  std::vector<int> sbox(L.n_seg), sid(L.n_seg);
  for (int b = 0; b < L.n_boxes; ++b) {
    CHECK_ARG(d->seg_off[b] <= d->seg_off[b + 1], "seg_off not monotone");
    for (int64_t r = d->seg_off[b]; r < d->seg_off[b + 1]; ++r) sbox[r] = b;
  }
  CHECK_ARG(d->seg_off[L.n_boxes] == L.n_seg, "seg_off end != n_segments");
  if (!to_i32(d->seg_ids, L.n_seg, sid, "seg_ids")) return IFGFB_ERR_ARG;
  RC(dev_upload(p, &L.seg_box, sbox.data(), sbox.size()));
  RC(dev_upload(p, &L.seg_id, sid.data(), sid.size()));
  std::vector<double> tabs;
  tabs.insert(tabs.end(), d->s_nodes, d->s_nodes + L.n_s * PS);
  tabs.insert(tabs.end(), d->sin_t, d->sin_t + L.n_a * PA);
  tabs.insert(tabs.end(), d->cos_t, d->cos_t + L.n_a * PA);
  tabs.insert(tabs.end(), d->sin_p, d->sin_p + 2 * L.n_a * PA);
  tabs.insert(tabs.end(), d->cos_p, d->cos_p + 2 * L.n_a * PA);
  RC(dev_upload(p, &L.tabs, tabs.data(), tabs.size()));
  p.max_seg = std::max(p.max_seg, L.n_seg);
  return IFGFB_OK;
}

int ifgfb_plan_set_emission(ifgfb_plan* h, const ifgfb_emit_desc* e) {
  CHECK_ARG(h && e, "null argument");
  Plan& p = h->p;
  CHECK_ARG(!p.finalized, "plan already finalized");
  CHECK_ARG(e->level >= 3 && e->level <= p.depth, "level out of range");
  Level& L = p.levels[e->level];
  CHECK_ARG(L.d == e->level, "add_level must precede set_emission");
  const int64_t np_ = e->n_pairs;
  CHECK_ARG(np_ >= 0 && np_ < INT32_MAX, "pair count out of range");
  L.n_pairs = np_;
  L.has_disp = e->geom_disp != nullptr;
  // sort pairs by segment row (stable counting sort, O(pairs + rows)) ->
  // per-row tiles of <= 4 pairs
  std::vector<int> order(np_);
  std::vector<int64_t> rstart((size_t)L.n_seg + 1, 0);
  for (int64_t i = 0; i < np_; ++i) {
    CHECK_ARG(e->row[i] >= 0 && e->row[i] < L.n_seg, "emission row out of range");
    CHECK_ARG(e->target[i] >= 0 && e->target[i] < p.n, "emission target out of range");
    rstart[e->row[i] + 1]++;
  }
  for (int64_t r = 0; r < L.n_seg; ++r) rstart[r + 1] += rstart[r];
  for (int64_t i = 0; i < np_; ++i) order[rstart[e->row[i]]++] = (int)i;
  std::vector<double4> g(np_), gd(L.has_disp ? np_ : 0);
  std::vector<int4> tiles;
  for (int64_t s = 0; s < np_; ++s) {
    const int i = order[s];
    g[s] = make_double4(e->geom[4 * i], e->geom[4 * i + 1], e->geom[4 * i + 2],
                        e->geom[4 * i + 3]);
    if (L.has_disp)
      gd[s] = make_double4(e->geom_disp[4 * i], e->geom_disp[4 * i + 1],
                           e->geom_disp[4 * i + 2], e->geom_disp[4 * i + 3]);
  }
  int64_t s = 0;
  while (s < np_) {
    const int64_t row = e->row[order[s]];
    int64_t t = s;
    while (t < np_ && e->row[order[t]] == row) ++t;
    for (int64_t q = s; q < t; q += 4)
      tiles.push_back(make_int4((int)row, (int)q, (int)std::min<int64_t>(4, t - q), 0));
    s = t;
  }
  L.n_etiles = (int)tiles.size();
  L.etile_rows.resize(tiles.size());
  for (size_t i = 0; i < tiles.size(); ++i) L.etile_rows[i] = tiles[i].x;
  RC(dev_upload(p, &L.pair_id, order.data(), order.size()));
  RC(dev_upload(p, &L.geom, g.data(), g.size()));
  if (L.has_disp) RC(dev_upload(p, &L.geom_disp, gd.data(), gd.size()));
  RC(dev_upload(p, &L.etiles, tiles.data(), tiles.size()));
  // per-target CSR of pair indices (box-major pair order == box order)
  std::vector<int> off(p.n + 1, 0), lst(np_);
  for (int64_t i = 0; i < np_; ++i) off[e->target[i] + 1]++;
  for (int t = 0; t < p.n; ++t) off[t + 1] += off[t];
  std::vector<int> fill(off.begin(), off.end() - 1);
  for (int64_t i = 0; i < np_; ++i) lst[fill[e->target[i]]++] = (int)i;
  RC(dev_upload(p, &L.tgt_off, off.data(), off.size()));
  RC(dev_upload(p, &L.tgt_pairs, lst.data(), lst.size()));
  p.max_pairs = std::max<int64_t>(p.max_pairs, np_);
  return IFGFB_OK;
}

int ifgfb_plan_add_accum(ifgfb_plan* h, const ifgfb_accum_desc* a) {
  CHECK_ARG(h && a, "null argument");
  Plan& p = h->p;
  CHECK_ARG(!p.finalized, "plan already finalized");
  CHECK_ARG(a->level >= 4 && a->level <= p.depth, "accum level out of range");
  Level& L = p.levels[a->level];
  Level& U = p.levels[a->level - 1];
  CHECK_ARG(L.d == a->level && U.d == a->level - 1,
            "add_level(d) and add_level(d-1) must precede add_accum(d)");
  CHECK_ARG(a->n_parent_rows == U.n_seg, "n_parent_rows != segments of level d-1");
  const int64_t nt = a->n_types;
  L.n_types = nt;
  std::vector<int> tmp;
  const int64_t ni = a->n_instances;
  const bool tile_free = a->tiles == nullptr;
  CHECK_ARG(!tile_free || a->group_id != nullptr, "tiles or group_id required");
  if (!tile_free) {
    if (!to_i32(a->tile_off, ni * WARP_PARTS + 1, tmp, "tile_off")) return IFGFB_ERR_ARG;
    CHECK_ARG(a->tile_off[ni * WARP_PARTS] == a->n_tiles, "tile_off end != n_tiles");
    RC(dev_upload(p, &L.tile_off, tmp.data(), tmp.size()));
    for (int64_t i = 0; i < a->n_tiles; ++i) {
      const uint8_t* t = a->tiles + 16 * i;
      CHECK_ARG(t[1] >= 1 && t[1] <= 8, "tile row count out of range");
      for (int r = 0; r < t[1]; ++r)
        CHECK_ARG(t[2 + r] < MAX_SET, "tile slot out of range");
    }
    RC(dev_upload(p, &L.tiles, reinterpret_cast<const uint4*>(a->tiles), (size_t)a->n_tiles));
  }
  if (a->group_id) RC(dev_upload(p, &L.gid, a->group_id, (size_t)nt * NN));
  for (int64_t i = 0; i < a->n_parent_rows * NN; ++i)
    CHECK_ARG(a->row_order[i] < NN, "row_order entry out of range");
  RC(dev_upload(p, &L.row_order, a->row_order, (size_t)a->n_parent_rows * NN));
  CHECK_ARG(a->row_cuts != nullptr, "row_cuts missing");
  // 5-warp kernels: 5 sets of 1..23 nodes; wide-warp kernel
  // (ifgfb_row_cuts_wide): W <= 5 sets of 1..32 nodes, then 75s
  L.cut_warps = 0;
  L.cut_max_set = 0;
  for (int64_t r = 0; r < a->n_parent_rows; ++r) {
    const uint8_t* c = a->row_cuts + r * (WARP_PARTS + 1);
    CHECK_ARG(c[0] == 0 && c[WARP_PARTS] == NN, "row_cuts must start at 0 and end at 75");
    int used = 0;
    for (int w = 0; w < WARP_PARTS; ++w) {
      if (c[w] == NN) {
        CHECK_ARG(c[w + 1] == NN, "row_cuts: entries after 75 must be 75");
        continue;
      }
      CHECK_ARG(c[w + 1] > c[w] && c[w + 1] - c[w] <= 32, "row_cuts: warp set size out of 1..32");
      L.cut_max_set = std::max(L.cut_max_set, (int)(c[w + 1] - c[w]));
      ++used;
    }
    CHECK_ARG(L.cut_warps == 0 || used == L.cut_warps, "row_cuts: rows differ in their number of sets");
    L.cut_warps = used;
  }
  RC(dev_upload(p, &L.row_cuts, a->row_cuts, (size_t)a->n_parent_rows * (WARP_PARTS + 1)));
  L.otf = a->geometry_on_device != 0;
  if (L.otf) {
    CHECK_ARG(a->type_octant != nullptr, "geometry_on_device needs type_octant");
    for (int64_t t = 0; t < nt; ++t) CHECK_ARG(a->type_octant[t] < 8, "type_octant out of range");
    RC(dev_upload(p, &L.type_octant, a->type_octant, (size_t)nt));
  } else {
    CHECK_ARG(a->node_geom != nullptr && a->node_r != nullptr, "node_geom / node_r missing");
    RC(dev_upload(p, &L.node_geom, a->node_geom, (size_t)nt * NN * 3));
    RC(dev_upload(p, &L.node_r, a->node_r, (size_t)nt * NN * 2));
    RC(dev_alloc(p, &L.ratio, (size_t)nt * NN * 4));
  }
  if (!to_i32(a->inst_off, a->n_parent_rows + 1, tmp, "inst_off")) return IFGFB_ERR_ARG;
  RC(dev_upload(p, &L.inst_off, tmp.data(), tmp.size()));
  if (L.otf) L.h_inst_off = tmp;
  L.n_instances = a->n_instances;
  for (int64_t i = 0; i < a->n_instances; ++i)
    CHECK_ARG(a->inst_type[i] >= 0 && a->inst_type[i] < nt, "inst_type out of range");
  if (!to_i32(a->inst_type, a->n_instances, tmp, "inst_type")) return IFGFB_ERR_ARG;
  RC(dev_upload(p, &L.inst_type, tmp.data(), tmp.size()));
  if (!to_i32(a->inst_crow_off, a->n_instances + 1, tmp, "inst_crow_off")) return IFGFB_ERR_ARG;
  RC(dev_upload(p, &L.inst_crow_off, tmp.data(), tmp.size()));
  const int64_t ncrow = a->inst_crow_off[a->n_instances];
  for (int64_t i = 0; i < ncrow; ++i)
    CHECK_ARG(a->crow[i] >= 0 && a->crow[i] < L.n_seg, "crow out of range");
  if (!to_i32(a->crow, ncrow, tmp, "crow")) return IFGFB_ERR_ARG;
  RC(dev_upload(p, &L.crow, tmp.data(), tmp.size()));
  // capacities of the kernel's per-warp staging (far.cu WarpStage)
  for (int64_t r = 0; r < a->n_parent_rows; ++r)
    CHECK_ARG(a->inst_off[r + 1] - a->inst_off[r] <= 31, "more than 31 instances per row");
  std::vector<int> type_groups(a->group_id ? nt : 0, -1);
  for (int64_t i = 0; i < ni; ++i) {
    const int64_t ng = a->inst_crow_off[i + 1] - a->inst_crow_off[i];
    CHECK_ARG(ng >= 0 && ng <= NN, "more than 75 child segments in one instance");
    L.max_groups = std::max(L.max_groups, (int)ng);
    if (a->group_id) {   // every node's group indexes the instance's crow list
      int& tg = type_groups[a->inst_type[i]];
      if (tg < 0) {
        int gmax = -1;
        for (int n = 0; n < NN; ++n)
          gmax = std::max(gmax, (int)a->group_id[a->inst_type[i] * NN + n]);
        tg = gmax + 1;
      }
      CHECK_ARG(tg == ng, "group_id inconsistent with the instance's child rows");
    }
    if (tile_free) continue;
    for (int w = 0; w < WARP_PARTS; ++w) {
      const int64_t k0 = a->tile_off[i * WARP_PARTS + w], k1 = a->tile_off[i * WARP_PARTS + w + 1];
      CHECK_ARG(k1 - k0 >= 0 && k1 - k0 <= MAX_SET, "more than 23 tiles per (instance, warp)");
      for (int64_t k = k0; k < k1; ++k)
        CHECK_ARG(a->tiles[16 * k] < ng, "tile group out of range for its instance");
    }
  }
  L.has_accum = true;
  return IFGFB_OK;
}

int ifgfb_plan_finalize(ifgfb_plan* h) {
  CHECK_ARG(h, "null argument");
  Plan& p = h->p;
  CHECK_ARG(!p.finalized, "plan already finalized");
  for (int d = 3; d <= p.depth; ++d) {
    if (p.levels[d].d != d) {
      set_error("level " + std::to_string(d) + " missing");
      return IFGFB_ERR_STATE;
    }
    if (d >= 4 && !p.levels[d].has_accum) {
      set_error("accumulation plan for level " + std::to_string(d) + " missing");
      return IFGFB_ERR_STATE;
    }
  }
  const size_t n = p.n;
  RC(dev_alloc(p, &p.wt, n * NCOL * 2));
  // coefficient ping-pong buffers are sized on first use (ensure_coef):
  // full levels, a rank's owned rows, or the largest streaming part
  p.coef_cap = 0;
  RC(dev_alloc(p, &p.partial, std::max<int64_t>(p.max_pairs, 1) * 2 * NCOL * 2));
  RC(dev_alloc(p, &p.out_tree, n * NCOL * 2));
  RC(dev_alloc(p, &p.out_disp_tree, n * NCOL * 2));
  p.finalized = true;
  return IFGFB_OK;
}

int ifgfb_plan_set_streaming(ifgfb_plan* h, const ifgfb_partition_desc* parts,
                             int n_parts) {
  CHECK_ARG(h && parts && n_parts >= 1, "bad argument");
  Plan& p = h->p;
  CHECK_ARG(p.finalized, "finalize the plan before setting streaming");
  std::vector<std::vector<StreamRange>> sp(n_parts, std::vector<StreamRange>(p.depth + 1));
  size_t need = 1;
  for (int q = 0; q < n_parts; ++q) {
    const ifgfb_partition_desc& d = parts[q];
    CHECK_ARG(d.n_levels == std::max(0, p.depth - 2), "need one entry per level 3..depth");
    for (int i = 0; i < d.n_levels; ++i) {
      const ifgfb_level_part& lp = d.levels[i];
      CHECK_ARG(lp.level >= 3 && lp.level <= p.depth, "stream level out of range");
      Level& L = p.levels[lp.level];
      CHECK_ARG(0 <= lp.seg_lo && lp.seg_lo <= lp.seg_hi && lp.seg_hi <= L.n_seg,
                "segment range out of bounds");
      CHECK_ARG(0 <= lp.pair_lo && lp.pair_lo <= lp.pair_hi && lp.pair_hi <= L.n_pairs,
                "pair range out of bounds");
      StreamRange& r = sp[q][lp.level];
      r.seg_lo = (int)lp.seg_lo;
      r.seg_hi = (int)lp.seg_hi;
      r.pair_lo = (int)lp.pair_lo;
      r.pair_hi = (int)lp.pair_hi;
      r.tile_lo = (int)(std::lower_bound(L.etile_rows.begin(), L.etile_rows.end(),
                                         (int)lp.seg_lo) - L.etile_rows.begin());
      r.tile_hi = (int)(std::lower_bound(L.etile_rows.begin(), L.etile_rows.end(),
                                         (int)lp.seg_hi) - L.etile_rows.begin());
      need = std::max(need, (size_t)(lp.seg_hi - lp.seg_lo));
    }
  }
  p.stream_parts.swap(sp);
  (void)need;
  RC(ensure_coef(p));
  return IFGFB_OK;
}

int ifgfb_plan_destroy(ifgfb_plan* h) {
  if (!h) return IFGFB_OK;
  for (void* ptr : h->p.allocations) cudaFree(ptr);
  if (h->p.host_stage) cudaFreeHost(h->p.host_stage);
  for (cudaEvent_t e : h->p.sync_events) cudaEventDestroy(e);
  if (h->p.aux) cudaStreamDestroy(h->p.aux);
  delete h;
  return IFGFB_OK;
}

int64_t ifgfb_plan_device_bytes(const ifgfb_plan* h) {
  return h ? (int64_t)h->p.bytes : 0;
}

int ifgfb_plan_set_timing(ifgfb_plan* h, int enable) {
  CHECK_ARG(h, "null argument");
  h->p.timer.reset();
  h->p.timer.on = enable != 0;
  return IFGFB_OK;
}

int ifgfb_plan_kernel_times(ifgfb_plan* h, double* ms, int64_t* counts) {
  CHECK_ARG(h && ms && counts, "null argument");
  h->p.timer.collect();
  for (int k = 0; k < K_NKINDS; ++k) {
    ms[k] = h->p.timer.ms[k];
    counts[k] = h->p.timer.count[k];
  }
  return IFGFB_OK;
}

int ifgfb_plan_level_times(ifgfb_plan* h, int max_levels, double* ms, int64_t* counts) {
  CHECK_ARG(h && ms && counts && max_levels >= 0, "null argument");
  h->p.timer.collect();
  for (int d = 0; d < max_levels; ++d) {
    const bool in = d < KTimer::MAXLV;
    ms[d] = in ? h->p.timer.lvl_ms[d] : 0.0;
    counts[d] = in ? h->p.timer.lvl_count[d] : 0;
  }
  return IFGFB_OK;
}

int64_t ifgfb_plan_last_launches(const ifgfb_plan* h) {
  return h ? h->p.launches : 0;
}

int ifgfb_far_apply(ifgfb_plan* h, const double* w, int nch,
                    const double* kappas, int nk, double* out,
                    double* out_disp, void* stream) {
  CHECK_ARG(h && w && kappas && out, "null argument");
  Plan& p = h->p;
  if (!p.finalized) {
    set_error("plan not finalized");
    return IFGFB_ERR_STATE;
  }
  if (p.rank_mode) {
    set_error("plan is one rank's share: ifgfb_far_apply would return a rank-local "
              "partial sum");
    return IFGFB_ERR_STATE;
  }
  double kap[4] = {kappas[0], kappas[1], nk > 1 ? kappas[2] : 0.0,
                   nk > 1 ? kappas[3] : 0.0};
  p.launches = 0;
  return far_apply(p, w, nch, kap, nk, out, out_disp,
                   static_cast<cudaStream_t>(stream));
}

}  // extern "C"
