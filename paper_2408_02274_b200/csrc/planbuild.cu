// Plan-time cone hierarchy on the device (native plan
// builder).  Replaces the host numpy relevance pass of
// octree.build_cone_hierarchy (reference ifgf.py:417-482): per box, the
// relevant cone segments are those holding a cousin point or a node of a
// relevant parent segment (ifgf.py:452-473), sorted per box.
//
// Exactness.  Segment ids are integer decisions made from floating point:
// the device replays the reference's numpy expressions operation by
// operation with correctly rounded IEEE ops in numpy's order (node
// positions c + r*(st*cp) from the host's own sin/cos tables, dx, the norm
// ((dx^2 + dy^2) + dz^2), s = (sqrt(3)/2 * side) / r, dz / r, the mod 2 pi
// of atan2), so every value is bit-identical to numpy's except arccos and
// arctan2 (numpy's SIMD libm vs CUDA's: a few ulp apart).  Wherever a few
// ulp could move theta or phi across a segment edge (|v/delta - edge| <
// 1e-14 (|v| + 1) / delta) the evaluation is not decided on the device: its
// (box, dx) is returned and the host decides it with numpy's own
// arccos/arctan2 (ifgfb_cones_set).  The result is the numpy builder's,
// bit for bit (tests/test_gpu_planbuild.py).
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace ifgfb {

struct ConeBuild {
  int n_s = 0, n_a = 0;
  double delta_s = 0, delta_a = 0, s_num = 0;
  int64_t n_boxes = 0, words = 0;        // 32-bit bitmap words per box
  uint32_t* bits = nullptr;              // n_boxes * words
  int64_t* amb_box = nullptr;            // ambiguous evaluations
  double* amb_dx = nullptr;
  unsigned long long* amb_n = nullptr;
  int64_t amb_cap = 0;
};

struct ConeArgs {
  int n_s, n_a;
  double delta_s, delta_a, s_num;        // s_num = np.sqrt(3.0) / 2.0 * side
  int64_t words;
  uint32_t* bits;
  int64_t* amb_box; double* amb_dx; unsigned long long* amb_n; int64_t amb_cap;
};

__device__ __forceinline__ bool edge_ambiguous(double v, double delta) {
  const double tol = 1e-14 * (fabs(v) + 1.0);
  return floor(__ddiv_rn(v - tol, delta)) != floor(__ddiv_rn(v + tol, delta));
}

// numpy cone_coords + seg_index on dx (ifgf.py:305-317, :349-354); returns
// the flat id, or -1 when a few ulp of arccos / arctan2 could change it
__device__ __forceinline__ int64_t cone_key(const ConeArgs& a, double dx, double dy,
                                            double dz) {
  const double r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                        __dmul_rn(dz, dz)));
  const double s = __ddiv_rn(a.s_num, r);
  const double cz = fmin(fmax(__ddiv_rn(dz, r), -1.0), 1.0);
  const double th = acos(cz);
  double ph = atan2(dy, dx);
  // np.mod(phi, 2 pi): fmod(phi, 2 pi) == phi here; negative -> + 2 pi;
  // zero -> +0
  if (ph < 0.0) ph = __dadd_rn(ph, 6.283185307179586);
  else if (ph == 0.0) ph = 0.0;
  if (edge_ambiguous(th, a.delta_a) || edge_ambiguous(ph, a.delta_a)) return -1;
  const int64_t i_s = min((int64_t)__ddiv_rn(s, a.delta_s), (int64_t)a.n_s - 1);
  const int64_t i_t = min((int64_t)__ddiv_rn(th, a.delta_a), (int64_t)a.n_a - 1);
  const int64_t i_p = min((int64_t)__ddiv_rn(ph, a.delta_a), 2 * (int64_t)a.n_a - 1);
  return (i_s * a.n_a + i_t) * (2 * a.n_a) + i_p;
}

__device__ __forceinline__ void mark(const ConeArgs& a, int64_t box, double dx, double dy,
                                     double dz) {
  const int64_t key = cone_key(a, dx, dy, dz);
  if (key >= 0) {
    atomicOr(a.bits + box * a.words + (key >> 5), 1u << (key & 31));
    return;
  }
  const unsigned long long slot = atomicAdd(a.amb_n, 1ull);
  if ((int64_t)slot < a.amb_cap) {
    a.amb_box[slot] = box;
    a.amb_dx[3 * slot] = dx;
    a.amb_dx[3 * slot + 1] = dy;
    a.amb_dx[3 * slot + 2] = dz;
  }
}

// cousin points: pair q of the box-major CSR (box of pair q = pair_box[q])
__global__ void cone_points_kernel(ConeArgs a, int64_t n_pairs, const int* __restrict__ pair_box,
                                   const int* __restrict__ pair_pt,
                                   const double* __restrict__ points,
                                   const double* __restrict__ centers) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_pairs;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = pair_box[q], t = pair_pt[q];
    mark(a, b, __dsub_rn(points[3 * t], centers[3 * b]),
         __dsub_rn(points[3 * t + 1], centers[3 * b + 1]),
         __dsub_rn(points[3 * t + 2], centers[3 * b + 2]));
  }
}

// parent nodes: instance i = (child box, parent segment row) in box-major
// order (inst_off per box); thread = (instance, node)
struct ParentArgs {
  int64_t n_inst, n_boxes;
  const int64_t* inst_off;       // n_boxes + 1
  const int64_t* row0;           // per box: first parent row of its parent box
  const int* pbox;               // per box: parent box
  const int* pseg;               // parent rows: segment id
  const double* pcenters;        // parent boxes x 3
  const double* centers;         // boxes x 3
  const double* ptabs;           // s_nodes | sin_t | cos_t | sin_p | cos_p
  int pn_s, pn_a;
  double ph;
};

__global__ void cone_parents_kernel(ConeArgs a, ParentArgs P) {
  const double* s_nodes = P.ptabs;
  const double* sin_t = s_nodes + P.pn_s * PS;
  const double* cos_t = sin_t + P.pn_a * PA;
  const double* sin_p = cos_t + P.pn_a * PA;
  const double* cos_p = sin_p + 2 * P.pn_a * PA;
  const int two_na = 2 * P.pn_a;
  const int64_t total = P.n_inst * NN;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t inst = e / NN;
    const int node = (int)(e - inst * NN);
    // box of the instance: last b with inst_off[b] <= inst
    int64_t lo = 0, hi = P.n_boxes;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (P.inst_off[mid] <= inst) lo = mid; else hi = mid;
    }
    const int64_t b = lo;
    const int pb = P.pbox[b];
    const int id = P.pseg[P.row0[b] + (inst - P.inst_off[b])];
    const int i_p = id % two_na, rest = id / two_na;
    const int i_t = rest % P.pn_a, i_s = rest / P.pn_a;
    const int na = node / (PA * PA), nb = (node / PA) % PA, nc = node % PA;
    const double r = __ddiv_rn(P.ph, s_nodes[i_s * PS + na]);
    const double st = sin_t[i_t * PA + nb], ct = cos_t[i_t * PA + nb];
    const double sp = sin_p[i_p * PA + nc], cp = cos_p[i_p * PA + nc];
    const double x = __dadd_rn(P.pcenters[3 * pb], __dmul_rn(r, __dmul_rn(st, cp)));
    const double y = __dadd_rn(P.pcenters[3 * pb + 1], __dmul_rn(r, __dmul_rn(st, sp)));
    const double z = __dadd_rn(P.pcenters[3 * pb + 2], __dmul_rn(r, ct));
    mark(a, b, __dsub_rn(x, P.centers[3 * b]), __dsub_rn(y, P.centers[3 * b + 1]),
         __dsub_rn(z, P.centers[3 * b + 2]));
  }
}

__global__ void cone_set_kernel(ConeArgs a, int64_t n, const int64_t* __restrict__ box,
                                const int64_t* __restrict__ key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicOr(a.bits + box[i] * a.words + (key[i] >> 5), 1u << (key[i] & 31));
}

// one warp per box: set-bit count
__global__ void cone_count_kernel(const uint32_t* __restrict__ bits, int64_t n_boxes,
                                  int64_t words, int64_t* __restrict__ count) {
  const int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= n_boxes) return;
  int64_t c = 0;
  for (int64_t w = lane; w < words; w += 32) c += __popc(bits[b * words + w]);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) count[b] = c;
}

// one warp per box: ascending set-bit positions (segment ids) from off[b]
__global__ void cone_ids_kernel(const uint32_t* __restrict__ bits, int64_t n_boxes,
                                int64_t words, const int64_t* __restrict__ off,
                                int64_t* __restrict__ ids) {
  const int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= n_boxes) return;
  int64_t base = off[b];
  for (int64_t w0 = 0; w0 < words; w0 += 32) {
    const int64_t w = w0 + lane;
    uint32_t v = w < words ? bits[b * words + w] : 0u;
    const int c = __popc(v);
    int incl = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int64_t pos = base + incl - c;
    while (v) {
      const int bit = __ffs(v) - 1;
      ids[pos++] = w * 32 + bit;
      v &= v - 1;
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
}

static ConeArgs args_of(const ConeBuild& c) {
  return ConeArgs{c.n_s, c.n_a, c.delta_s, c.delta_a, c.s_num, c.words, c.bits,
                  c.amb_box, c.amb_dx, c.amb_n, c.amb_cap};
}

static int grid_for(int64_t n, int threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 64));
}

template <typename T>
static int upload(T** dst, const T* src, size_t n, std::vector<void*>& owned) {
  *dst = nullptr;
  if (n == 0) return IFGFB_OK;
  IFGFB_CUDA(cudaMalloc(dst, n * sizeof(T)));
  owned.push_back(*dst);
  IFGFB_CUDA(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return IFGFB_OK;
}

static void free_all(std::vector<void*>& owned) {
  for (void* p : owned) cudaFree(p);
  owned.clear();
}

}  // namespace ifgfb

using namespace ifgfb;

struct ifgfb_cone_build {
  ConeBuild c;
};

extern "C" {

int ifgfb_cones_begin(const ifgfb_cone_level_desc* d, ifgfb_cone_build** out) {
  IFGFB_CHECK_ARG(d && out, "null argument");
  IFGFB_CHECK_ARG(d->n_s >= 1 && d->n_a >= 1 && d->n_boxes >= 0, "bad cone level");
  const int64_t full = (int64_t)d->n_s * d->n_a * 2 * d->n_a;
  IFGFB_CHECK_ARG(full < ((int64_t)1 << 40), "cone level too large");
  auto* h = new ifgfb_cone_build();
  ConeBuild& c = h->c;
  c.n_s = d->n_s;
  c.n_a = d->n_a;
  c.delta_s = d->delta_s;
  c.delta_a = d->delta_a;
  c.s_num = d->s_num;
  c.n_boxes = d->n_boxes;
  c.words = (full + 31) / 32;
  c.amb_cap = std::max<int64_t>(1 << 16, d->amb_capacity);
  int rc = IFGFB_OK;
  if (cudaMalloc(&c.bits, sizeof(uint32_t) * std::max<int64_t>(1, c.n_boxes * c.words)) !=
          cudaSuccess ||
      cudaMemset(c.bits, 0, sizeof(uint32_t) * std::max<int64_t>(1, c.n_boxes * c.words)) !=
          cudaSuccess ||
      cudaMalloc(&c.amb_box, sizeof(int64_t) * c.amb_cap) != cudaSuccess ||
      cudaMalloc(&c.amb_dx, sizeof(double) * 3 * c.amb_cap) != cudaSuccess ||
      cudaMalloc(&c.amb_n, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(c.amb_n, 0, sizeof(unsigned long long)) != cudaSuccess) {
    set_error("ifgfb_cones_begin: device allocation failed");
    rc = IFGFB_ERR_CUDA;
  }
  if (rc != IFGFB_OK) {
    ifgfb_cones_free(h);
    return rc;
  }
  *out = h;
  return IFGFB_OK;
}

int ifgfb_cones_mark_points(ifgfb_cone_build* h, int64_t n_pairs, const int32_t* pair_box,
                            const int32_t* pair_pt, int64_t n_points, const double* points,
                            const double* centers) {
  IFGFB_CHECK_ARG(h && n_pairs >= 0, "bad argument");
  if (n_pairs == 0) return IFGFB_OK;
  ConeBuild& c = h->c;
  std::vector<void*> owned;
  int *db = nullptr, *dp = nullptr;
  double *dpts = nullptr, *dctr = nullptr;
  int rc = upload(&db, pair_box, n_pairs, owned);
  if (!rc) rc = upload(&dp, pair_pt, n_pairs, owned);
  if (!rc) rc = upload(&dpts, points, 3 * (size_t)n_points, owned);
  if (!rc) rc = upload(&dctr, centers, 3 * (size_t)c.n_boxes, owned);
  if (!rc) {
    cone_points_kernel<<<grid_for(n_pairs, 256), 256>>>(args_of(c), n_pairs, db, dp, dpts, dctr);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      set_error("cone_points_kernel failed");
      rc = IFGFB_ERR_CUDA;
    }
  }
  free_all(owned);
  return rc;
}

int ifgfb_cones_mark_parents(ifgfb_cone_build* h, const ifgfb_cone_parent_desc* d) {
  IFGFB_CHECK_ARG(h && d, "null argument");
  ConeBuild& c = h->c;
  IFGFB_CHECK_ARG(d->n_boxes == c.n_boxes, "box count mismatch");
  const int64_t n_inst = d->inst_off[c.n_boxes];
  if (n_inst == 0) return IFGFB_OK;
  std::vector<void*> owned;
  ParentArgs P{};
  P.n_inst = n_inst;
  P.n_boxes = c.n_boxes;
  P.pn_s = d->pn_s;
  P.pn_a = d->pn_a;
  P.ph = d->ph;
  int64_t *io = nullptr, *r0 = nullptr;
  int *pb = nullptr, *ps = nullptr;
  double *pc = nullptr, *cc = nullptr, *tb = nullptr;
  const size_t ntab = (size_t)d->pn_s * PS + 2 * (size_t)d->pn_a * PA + 4 * (size_t)d->pn_a * PA;
  int rc = upload(&io, d->inst_off, c.n_boxes + 1, owned);
  if (!rc) rc = upload(&r0, d->row0, c.n_boxes, owned);
  if (!rc) rc = upload(&pb, d->parent_box, c.n_boxes, owned);
  if (!rc) rc = upload(&ps, d->parent_seg_ids, d->n_parent_rows, owned);
  if (!rc) rc = upload(&pc, d->parent_centers, 3 * (size_t)d->n_parent_boxes, owned);
  if (!rc) rc = upload(&cc, d->centers, 3 * (size_t)c.n_boxes, owned);
  if (!rc) rc = upload(&tb, d->parent_tabs, ntab, owned);
  if (!rc) {
    P.inst_off = io; P.row0 = r0; P.pbox = pb; P.pseg = ps; P.pcenters = pc;
    P.centers = cc; P.ptabs = tb;
    cone_parents_kernel<<<grid_for(n_inst * NN, 256), 256>>>(args_of(c), P);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      set_error("cone_parents_kernel failed");
      rc = IFGFB_ERR_CUDA;
    }
  }
  free_all(owned);
  return rc;
}

int ifgfb_cones_ambiguous(ifgfb_cone_build* h, int64_t* n, int64_t* box, double* dx) {
  IFGFB_CHECK_ARG(h && n, "null argument");
  ConeBuild& c = h->c;
  unsigned long long cnt = 0;
  IFGFB_CUDA(cudaMemcpy(&cnt, c.amb_n, sizeof(cnt), cudaMemcpyDeviceToHost));
  if ((int64_t)cnt > c.amb_cap) {
    set_error("ifgfb_cones_ambiguous: more edge cases than the capacity "
              "(raise amb_capacity)");
    *n = (int64_t)cnt;
    return IFGFB_ERR_STATE;
  }
  *n = (int64_t)cnt;
  if (box && cnt) IFGFB_CUDA(cudaMemcpy(box, c.amb_box, sizeof(int64_t) * cnt,
                                        cudaMemcpyDeviceToHost));
  if (dx && cnt) IFGFB_CUDA(cudaMemcpy(dx, c.amb_dx, sizeof(double) * 3 * cnt,
                                       cudaMemcpyDeviceToHost));
  return IFGFB_OK;
}

int ifgfb_cones_set(ifgfb_cone_build* h, int64_t n, const int64_t* box, const int64_t* key) {
  IFGFB_CHECK_ARG(h && n >= 0, "bad argument");
  if (n == 0) return IFGFB_OK;
  ConeBuild& c = h->c;
  for (int64_t i = 0; i < n; ++i)
    IFGFB_CHECK_ARG(box[i] >= 0 && box[i] < c.n_boxes && key[i] >= 0 && key[i] < 32 * c.words,
                    "ifgfb_cones_set: entry out of range");
  std::vector<void*> owned;
  int64_t *db = nullptr, *dk = nullptr;
  int rc = upload(&db, box, n, owned);
  if (!rc) rc = upload(&dk, key, n, owned);
  if (!rc) {
    cone_set_kernel<<<grid_for(n, 256), 256>>>(args_of(c), n, db, dk);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      set_error("cone_set_kernel failed");
      rc = IFGFB_ERR_CUDA;
    }
  }
  free_all(owned);
  return rc;
}

int ifgfb_cones_finish(ifgfb_cone_build* h, int64_t* seg_off, int64_t** seg_ids_dev,
                       int64_t* n_segments) {
  IFGFB_CHECK_ARG(h && seg_off && n_segments, "null argument");
  ConeBuild& c = h->c;
  std::vector<void*> owned;
  int64_t* cnt = nullptr;
  const int64_t nb = c.n_boxes;
  seg_off[0] = 0;
  if (nb == 0) {
    *n_segments = 0;
    return IFGFB_OK;
  }
  IFGFB_CUDA(cudaMalloc(&cnt, sizeof(int64_t) * nb));
  owned.push_back(cnt);
  const int threads = 256, grid = (int)((nb * 32 + threads - 1) / threads);
  cone_count_kernel<<<grid, threads>>>(c.bits, nb, c.words, cnt);
  std::vector<int64_t> hc(nb);
  if (cudaMemcpy(hc.data(), cnt, sizeof(int64_t) * nb, cudaMemcpyDeviceToHost) != cudaSuccess) {
    free_all(owned);
    set_error("cone_count_kernel failed");
    return IFGFB_ERR_CUDA;
  }
  for (int64_t b = 0; b < nb; ++b) seg_off[b + 1] = seg_off[b] + hc[b];
  *n_segments = seg_off[nb];
  if (seg_ids_dev) *seg_ids_dev = nullptr;
  free_all(owned);
  return IFGFB_OK;
}

int ifgfb_cones_ids(ifgfb_cone_build* h, const int64_t* seg_off, int64_t* seg_ids) {
  IFGFB_CHECK_ARG(h && seg_off && seg_ids, "null argument");
  ConeBuild& c = h->c;
  const int64_t nb = c.n_boxes, total = seg_off[nb];
  if (total == 0) return IFGFB_OK;
  std::vector<void*> owned;
  int64_t *doff = nullptr, *dids = nullptr;
  int rc = upload(&doff, seg_off, nb + 1, owned);
  if (!rc && cudaMalloc(&dids, sizeof(int64_t) * total) != cudaSuccess) {
    set_error("ifgfb_cones_ids: allocation failed");
    rc = IFGFB_ERR_CUDA;
  }
  if (!rc) {
    owned.push_back(dids);
    const int threads = 256, grid = (int)((nb * 32 + threads - 1) / threads);
    cone_ids_kernel<<<grid, threads>>>(c.bits, nb, c.words, doff, dids);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpy(seg_ids, dids, sizeof(int64_t) * total, cudaMemcpyDeviceToHost) !=
            cudaSuccess) {
      set_error("cone_ids_kernel failed");
      rc = IFGFB_ERR_CUDA;
    }
  }
  free_all(owned);
  return rc;
}

int ifgfb_cones_free(ifgfb_cone_build* h) {
  if (!h) return IFGFB_OK;
  ConeBuild& c = h->c;
  if (c.bits) cudaFree(c.bits);
  if (c.amb_box) cudaFree(c.amb_box);
  if (c.amb_dx) cudaFree(c.amb_dx);
  if (c.amb_n) cudaFree(c.amb_n);
  delete h;
  return IFGFB_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------
// Propagation types on the device (reference _AccumType.__init__,
// ifgf.py:686-702, vectorised host form octree._type_geometry): per type
// (parent segment gamma, child octant) the 75 parent nodes seen from the
// child centre (-offset + r * dir), their child segment (sigma, an integer
// decision: replayed exactly as above, edge cases flagged for the host), the
// sigma groups (distinct child segments, ascending) and, on request, the
// continuous node geometry (local coordinates in the child segment, r_parent,
// r_child) -- those from CUDA's acos / atan2, a few ulp from numpy's (as the
// on-device geometry of the propagation kernel).
namespace ifgfb {

struct TypeArgs {
  int64_t n_types;
  const int* gamma; const unsigned char* octant;
  const double* ptabs; int pn_s, pn_a; double ph;     // parent level
  int n_s, n_a; double delta_s, delta_a, s_num;       // child level
  double half;                                        // 0.5 * child side
  unsigned char* gid; int* sigma; unsigned char* nsig; unsigned char* amb;
  double* geom; double* node_r;                       // optional
};

__global__ void __launch_bounds__(128) accum_types_kernel(TypeArgs a) {
  __shared__ int64_t sf[4][NN];
  __shared__ unsigned char first[4][NN];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * 4 + w;
  if (t >= a.n_types) return;
  const double* s_nodes = a.ptabs;
  const double* sin_t = s_nodes + a.pn_s * PS;
  const double* cos_t = sin_t + a.pn_a * PA;
  const double* sin_p = cos_t + a.pn_a * PA;
  const double* cos_p = sin_p + 2 * a.pn_a * PA;
  const int two_na = 2 * a.pn_a;
  const int id = a.gamma[t], oct = a.octant[t];
  const int i_p = id % two_na, rest = id / two_na;
  const int i_t = rest % a.pn_a, i_s = rest / a.pn_a;
  // center = -offset, offset = 0.5 side (2 bit - 1) (ifgf.py:687-688)
  const double cx = (oct >> 2) & 1 ? -a.half : a.half;
  const double cy = (oct >> 1) & 1 ? -a.half : a.half;
  const double cz = oct & 1 ? -a.half : a.half;
  ConeArgs ca{a.n_s, a.n_a, a.delta_s, a.delta_a, a.s_num, 0, nullptr, nullptr, nullptr,
              nullptr, 0};
  bool bad = false;
  for (int n = lane; n < NN; n += 32) {
    const int na = n / (PA * PA), nb = (n / PA) % PA, nc = n % PA;
    const double rp = __ddiv_rn(a.ph, s_nodes[i_s * PS + na]);
    const double st = sin_t[i_t * PA + nb], ct = cos_t[i_t * PA + nb];
    const double sp = sin_p[i_p * PA + nc], cp = cos_p[i_p * PA + nc];
    const double x = __dadd_rn(cx, __dmul_rn(rp, __dmul_rn(st, cp)));
    const double y = __dadd_rn(cy, __dmul_rn(rp, __dmul_rn(st, sp)));
    const double z = __dadd_rn(cz, __dmul_rn(rp, ct));
    const int64_t key = cone_key(ca, x, y, z);
    bad |= key < 0;
    sf[w][n] = key;
    if (a.geom) {
      const double rc = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)),
                                             __dmul_rn(z, z)));
      const double s = __ddiv_rn(a.s_num, rc);
      const double th = acos(fmin(fmax(__ddiv_rn(z, rc), -1.0), 1.0));
      double ph = atan2(y, x);
      if (ph < 0.0) ph = __dadd_rn(ph, 6.283185307179586);
      const int64_t f = key < 0 ? 0 : key;
      const int two = 2 * a.n_a;
      const int64_t jp = f % two, jr = f / two, jt = jr % a.n_a, js = jr / a.n_a;
      double* g = a.geom + (t * NN + n) * 3;
      g[0] = 2.0 * (s / a.delta_s - js) - 1.0;
      g[1] = 2.0 * (th / a.delta_a - jt) - 1.0;
      g[2] = 2.0 * (ph / a.delta_a - jp) - 1.0;
      a.node_r[(t * NN + n) * 2] = rp;
      a.node_r[(t * NN + n) * 2 + 1] = rc;
    }
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) a.amb[t] = bad ? 1 : 0;
  if (bad) return;     // decided on the host
  __syncwarp();
  for (int n = lane; n < NN; n += 32) {
    bool f = true;
    for (int k = 0; k < n; ++k) f &= sf[w][k] != sf[w][n];
    first[w][n] = f;
  }
  __syncwarp();
  int cnt_first = 0;
  for (int n = lane; n < NN; n += 32) {
    const int64_t v = sf[w][n];
    int g = 0;
    for (int j = 0; j < NN; ++j) g += (first[w][j] && sf[w][j] < v) ? 1 : 0;
    a.gid[t * NN + n] = (unsigned char)g;
    if (first[w][n]) {
      a.sigma[t * NN + g] = (int)v;
      ++cnt_first;
    }
  }
  for (int o = 16; o > 0; o >>= 1) cnt_first += __shfl_xor_sync(0xffffffffu, cnt_first, o);
  if (lane == 0) a.nsig[t] = (unsigned char)cnt_first;
  for (int g = cnt_first + lane; g < NN; g += 32) a.sigma[t * NN + g] = -1;
}

}  // namespace ifgfb

extern "C" int ifgfb_accum_types(const ifgfb_accum_types_desc* d, uint8_t* gid, int32_t* sigma,
                                 uint8_t* nsig, uint8_t* ambiguous, double* node_geom,
                                 double* node_r) {
  IFGFB_CHECK_ARG(d && gid && sigma && nsig && ambiguous, "null argument");
  IFGFB_CHECK_ARG((node_geom == nullptr) == (node_r == nullptr), "node_geom / node_r: both or none");
  const int64_t nt = d->n_types;
  if (nt == 0) return IFGFB_OK;
  std::vector<void*> owned;
  int* dg = nullptr;
  unsigned char *doc = nullptr, *dgid = nullptr, *dns = nullptr, *damb = nullptr;
  double *dtab = nullptr, *dgeo = nullptr, *dr = nullptr;
  int* dsig = nullptr;
  const size_t ntab = (size_t)d->pn_s * PS + 2 * (size_t)d->pn_a * PA + 4 * (size_t)d->pn_a * PA;
  int rc = upload(&dg, d->gamma, nt, owned);
  if (!rc) rc = upload(&doc, d->octant, nt, owned);
  if (!rc) rc = upload(&dtab, d->parent_tabs, ntab, owned);
  auto alloc = [&](auto** p, size_t n) {
    if (rc) return;
    if (cudaMalloc(p, n * sizeof(**p)) != cudaSuccess) {
      set_error("ifgfb_accum_types: allocation failed");
      rc = IFGFB_ERR_CUDA;
      return;
    }
    owned.push_back(*p);
  };
  alloc(&dgid, (size_t)nt * NN);
  alloc(&dsig, (size_t)nt * NN);
  alloc(&dns, (size_t)nt);
  alloc(&damb, (size_t)nt);
  if (node_geom) {
    alloc(&dgeo, (size_t)nt * NN * 3);
    alloc(&dr, (size_t)nt * NN * 2);
  }
  if (!rc) {
    TypeArgs a{nt, dg, doc, dtab, d->pn_s, d->pn_a, d->ph, d->n_s, d->n_a, d->delta_s,
               d->delta_a, d->s_num, d->half, dgid, dsig, dns, damb, dgeo, dr};
    accum_types_kernel<<<(unsigned)((nt + 3) / 4), 128>>>(a);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      set_error("accum_types_kernel failed");
      rc = IFGFB_ERR_CUDA;
    }
  }
  auto down = [&](void* h, const void* dptr, size_t bytes) {
    if (!rc && cudaMemcpy(h, dptr, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) {
      set_error("ifgfb_accum_types: copy failed");
      rc = IFGFB_ERR_CUDA;
    }
  };
  down(gid, dgid, (size_t)nt * NN);
  down(sigma, dsig, sizeof(int) * (size_t)nt * NN);
  down(nsig, dns, (size_t)nt);
  down(ambiguous, damb, (size_t)nt);
  if (node_geom) {
    down(node_geom, dgeo, sizeof(double) * (size_t)nt * NN * 3);
    down(node_r, dr, sizeof(double) * (size_t)nt * NN * 2);
  }
  free_all(owned);
  return rc;
}
