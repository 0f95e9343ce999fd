// Shared device helpers and the plan object of libifgfb200.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/ifgfb.h"

namespace ifgfb {

constexpr int PS = 3;          // radial interpolation order
constexpr int PA = 5;          // angular interpolation order
constexpr int NN = PS * PA * PA;  // 75 nodes per cone segment
constexpr int NCOL = 16;       // complex columns carried per traversal
constexpr int NRCOL = 2 * NCOL;   // 32 real columns
// Coefficients of one segment are stored in DMMA B-fragment order:
// [ks 0..18][half 0..1][lane 0..31][2] doubles, column tile nt = 2*half + j,
// column = 8*nt + (lane>>2) of the 32 real columns (re/im of 16 complex).
// K dimension: the 75 coefficients i = (a*PA + b)*PA + c = ab*PA + c packed
// into 19 k-steps of 4 (76 rows, one zero row), tig = lane&3:
//   ks = 5q + c (q < 3, c < 5): ab = 4q + tig, this c;
//   ks = 15 + s (s < 4):        (ab, c) = (12 + tig, s) for tig < 3,
//                               (12 + s, 4) for tig = 3 (s = 3: zero row).
// A k-step's fragments are two fully contiguous 512-byte warp loads (16
// bytes per lane).
constexpr int KSTEPS = 19;
constexpr int KMAIN = 15;                     // k-steps of the (q, c) block
constexpr int SEG_DOUBLES = KSTEPS * 32 * 4;  // 2432 doubles = 19 KB per segment
constexpr int WARP_PARTS = 5;                 // propagation: node owners per CTA
constexpr int PART_NODES = NN / WARP_PARTS;   // 15 parent nodes per warp (mean)
constexpr int MAX_SET = 23;                   // largest warp-owned node set

void set_error(const std::string& msg);

#define IFGFB_CUDA(call)                                                  \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess) {                                              \
      ::ifgfb::set_error(std::string(#call) + ": " + cudaGetErrorString(e_)); \
      return IFGFB_ERR_CUDA;                                              \
    }                                                                     \
  } while (0)

// ---- exact (non-contracted) arithmetic, used wherever the reference's
//      numpy expression order must be reproduced bit for bit
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// exp(i * kappa * x) for complex kappa = (kr, ki): exp(-ki x) (cos(kr x), sin(kr x))
// following numpy's evaluation of np.exp(1j * kappa * x).
__device__ __forceinline__ double2 cexp_ikx(double kr, double ki, double x) {
  double s, c;
  sincos(mul_rn(kr, x), &s, &c);
  if (ki != 0.0) {
    double m = exp(-mul_rn(ki, x));
    return make_double2(c * m, s * m);
  }
  return make_double2(c, s);
}

// Chebyshev T_0..T_{n-1} by the reference's recurrence (chebyshev.py:82-95):
// T_i = (2.0 * x) * T_{i-1} - T_{i-2}, each op rounded (no FMA contraction).
template <int N>
__device__ __forceinline__ void cheb_exact(double x, double (&t)[N]) {
  t[0] = 1.0;
  if (N > 1) t[1] = x;
  const double x2 = mul_rn(2.0, x);
#pragma unroll
  for (int i = 2; i < N; ++i) t[i] = sub_rn(mul_rn(x2, t[i - 1]), t[i - 2]);
}

// 8x8x4 FP64 tensor-core MMA (the only FP64 tensor path on sm_100a; tcgen05
// has no f64 kind).  a: A[row=lane>>2][k=lane&3], b: B[k=lane&3][col=lane>>2],
// c0/c1: C[row=lane>>2][col=2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Device-side bounds checks of the hand-written staging and index
// arithmetic (build with -DIFGFB_DEVICE_CHECKS: tools/device_checks.sh).
// compute-sanitizer is not available on the GPU pool, so these asserts are
// the memory-safety net: a violated check prints and traps.
#ifdef IFGFB_DEVICE_CHECKS
#define IFGFB_DCHECK(cond)                                                     \
  do {                                                                         \
    if (!(cond)) {                                                             \
      printf("IFGFB_DEVICE_CHECKS: %s failed at %s:%d (block %d thread %d)\n", \
             #cond, __FILE__, __LINE__, (int)blockIdx.x, (int)threadIdx.x);    \
      __trap();                                                                \
    }                                                                          \
  } while (0)
#else
#define IFGFB_DCHECK(cond) do { } while (0)
#endif

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
struct DevArray {
  T* ptr = nullptr;
  size_t n = 0;
};

// ------------------------------------------------------- kernel timing --
// Optional CUDA-event timing of every kernel class (enabled through
// ifgfb_plan_set_timing); events are recorded on the launching stream.
enum KernelKind {
  K_LEAF = 0, K_ACCUM, K_EMIT, K_REDUCE, K_NEAR, K_PACK, K_ASSEMBLE, K_OTHER,
  K_NKINDS
};

struct KTimer {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<int> kinds;
  std::vector<int> lvls;
  double ms[K_NKINDS] = {};
  int64_t count[K_NKINDS] = {};
  static constexpr int MAXLV = 32;
  double lvl_ms[MAXLV] = {};          // propagation (K_ACCUM) per child level
  int64_t lvl_count[MAXLV] = {};

  cudaEvent_t next() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  // returns a token (index of the start event) or -1 when off
  int begin(int kind, cudaStream_t st, int level = -1) {
    if (!on) return -1;
    const int tok = (int)used;
    cudaEventRecord(next(), st);
    kinds.push_back(kind);
    lvls.push_back(level);
    return tok;
  }
  void end(int tok, cudaStream_t st) {
    if (tok < 0) return;
    cudaEventRecord(next(), st);
  }
  // fold recorded pairs into the accumulators (synchronises the events)
  void collect() {
    for (size_t i = 0; i < kinds.size(); ++i) {
      float t = 0.f;
      cudaEventSynchronize(pool[2 * i + 1]);
      cudaEventElapsedTime(&t, pool[2 * i], pool[2 * i + 1]);
      ms[kinds[i]] += t;
      count[kinds[i]] += 1;
      if (lvls[i] >= 0 && lvls[i] < MAXLV) {
        lvl_ms[lvls[i]] += t;
        lvl_count[lvls[i]] += 1;
      }
    }
    kinds.clear();
    lvls.clear();
    used = 0;
  }
  void reset() {
    collect();
    for (int k = 0; k < K_NKINDS; ++k) { ms[k] = 0; count[k] = 0; }
    for (int k = 0; k < MAXLV; ++k) { lvl_ms[k] = 0; lvl_count[k] = 0; }
  }
};

// ------------------------------------------------------------------ plan --
struct Level {
  int d = 0, n_boxes = 0, n_s = 0, n_a = 0;
  double side = 0, h = 0, delta_s = 0, delta_a = 0;
  int n_seg = 0;
  double* centers = nullptr;   // n_boxes*3
  int* pt_start = nullptr;     // n_boxes
  int* pt_count = nullptr;
  int* seg_box = nullptr;      // n_seg
  int* seg_id = nullptr;       // n_seg
  double* tabs = nullptr;      // s_nodes | sin_t | cos_t | sin_p | cos_p
  // emission (pairs pre-sorted by segment row)
  int64_t n_pairs = 0;
  bool has_disp = false;
  int* pair_id = nullptr;      // sorted pos -> pair index (box-major)
  double4* geom = nullptr;     // sorted pos
  double4* geom_disp = nullptr;
  int n_etiles = 0;
  int4* etiles = nullptr;      // (row, first sorted pos, count<=4, 0)
  int* tgt_off = nullptr;      // N+1 (tree order targets)
  int* tgt_pairs = nullptr;    // pair indices, per target in box order
  // accumulation from this level (as child) into level d-1
  bool has_accum = false;
  int64_t n_types = 0;
  int* tile_off = nullptr;     // n_instances*WARP_PARTS+1
  unsigned char* row_order = nullptr;  // parent rows x NN
  unsigned char* row_cuts = nullptr;   // parent rows x (WARP_PARTS+1)
  int cut_warps = 0, cut_max_set = 0;  // sets per row / largest set of row_cuts
  int max_groups = 0;                  // most child segments of one instance
  bool otf = false;                    // node geometry computed on the device
  unsigned char* type_octant = nullptr;  // per type (otf levels)
  uint4* tiles = nullptr;      // 16-byte tile records (null: tile-free)
  unsigned char* gid = nullptr;  // per type x NN: sigma group of each node
  double* node_geom = nullptr; // n_types*NN*3 (parent node order)
  double* node_r = nullptr;    // n_types*NN*2 (r_parent, r_child)
  double* ratio = nullptr;     // workspace n_types*NN*2 complex
  int* inst_off = nullptr;     // parent rows + 1
  std::vector<int> h_inst_off; // host copy (on-device-geometry levels: row chunks of the node-table pre-pass)
  int* inst_type = nullptr;
  int* inst_crow_off = nullptr;
  int* crow = nullptr;
  int64_t n_instances = 0;
  // multi-GPU partition (defaults: everything)
  int part_seg_lo = 0, part_seg_hi = -1;     // -1: n_seg
  int part_pair_lo = 0, part_pair_hi = -1;   // -1: n_pairs
  int part_tile_lo = 0, part_tile_hi = -1;   // -1: n_etiles
  std::vector<int> etile_rows;               // host copy (sorted by row)
  int seg_lo() const { return part_seg_lo; }
  int seg_hi() const { return part_seg_hi < 0 ? n_seg : part_seg_hi; }
  int tile_lo() const { return part_tile_lo; }
  int tile_hi() const { return part_tile_hi < 0 ? n_etiles : part_tile_hi; }
  int pair_lo() const { return part_pair_lo; }
  int pair_hi() const { return part_pair_hi < 0 ? (int)n_pairs : part_pair_hi; }
};

struct StreamRange {
  int seg_lo = 0, seg_hi = 0, pair_lo = 0, pair_hi = 0, tile_lo = 0, tile_hi = 0;
};

struct Plan {
  int device = 0;
  int n = 0, depth = 0;
  double* points_tree = nullptr;   // N*3
  int* perm = nullptr;             // tree slot -> original
  std::vector<Level> levels;       // index d (0..depth); only d>=3 used
  bool finalized = false;
  // work buffers
  double* wt = nullptr;            // N * 8 complex (tree order, channels)
  double* coef[2] = {nullptr, nullptr};
  size_t coef_cap = 0;             // segments
  // node tables of on-device-geometry levels, tabulated per (instance, node)
  // for one chunk of parent rows ahead of its propagation launch (far.cu)
  double* otf_geom = nullptr;      // otf_cap * NN * 3
  double* otf_ratio = nullptr;     // otf_cap * NN * 2 complex
  int64_t otf_cap = 0;             // instances; -1: allocation failed / disabled
  double* partial = nullptr;       // max pairs * 2 * NCOL complex
  // emission overlap: a level's emission (K5 + reduce) runs on `aux`
  // concurrently with the next propagation step on the apply stream
  cudaStream_t aux = nullptr;
  std::vector<cudaEvent_t> sync_events;
  bool overlap_emit = false;
  double* out_tree = nullptr;      // N * NCOL complex
  double* out_disp_tree = nullptr;
  int64_t max_pairs = 0;
  int max_seg = 0;
  // surface / operator
  bool has_surface = false;
  int n_patches = 0, n_c = 0;
  double* sdata = nullptr;         // packed surface arrays
  double* pts = nullptr; double* nrm = nullptr; double* wq = nullptr;
  double* jac = nullptr; double* eu = nullptr; double* ev = nullptr;
  double* t1 = nullptr; double* t2 = nullptr; double* dmat = nullptr;
  double* cmat = nullptr;
  double eps_e[2], mu_e[2], eps_i[2], mu_i[2], omega = 0, kappa[4], fd_step = 1e-6;
  // near field
  bool has_near = false;
  int64_t n_mom = 0, n_direct = 0;
  int* mom_off = nullptr; int* mom_patch = nullptr; double* moments = nullptr;
  int* dir_off = nullptr; int* dir_src = nullptr;
  // muller workspaces
  double* phi = nullptr;        // 8*N complex
  double* phiw = nullptr;       // 8*N complex (phi * weights)
  double* pcoef = nullptr;      // 8*P*n_c^2 complex
  double* phi_pm = nullptr;     // N * [phi(8) | phi*w(8)] complex (point-major)
  double* far_out = nullptr;    // 16*N complex (8 ch x 2 k, original order)
  double* far_disp = nullptr;
  double* s_val = nullptr;      // 8*2*N complex
  double* d_val = nullptr;      // 6*2*N complex
  double* host_stage = nullptr; // pinned 2 * 4N complex
  double* dev_y = nullptr;      // 4N complex
  double* dev_out = nullptr;    // 4N complex
  int64_t launches = 0;
  KTimer timer;
  // rank mode (multi-GPU, ifgfb_plan_set_rank): the plan holds one rank's
  // window of level-3 subtrees; the far phase leaves the PARTIAL far field of
  // its sources in xfar (point-major, padded: n_ranks*chunk rows of 32
  // complex = 16 far + 16 displaced), the caller reduce-scatters it into
  // xfar_mine (chunk rows), the near phase writes the owned result rows
  // into xout_mine (chunk rows of 4 complex), the caller all-gathers them
  // into xout and ifgfb_rank_unpack writes the 4N y-layout vector.
  bool rank_mode = false;
  int rank = 0, n_ranks = 1;
  int64_t chunk = 0;
  double* xfar = nullptr;
  double* xfar_mine = nullptr;
  double* xout_mine = nullptr;
  double* xout = nullptr;
  // streaming: per part, per level (index d) the ranges of one group of
  // level-3 subtrees; empty = single pass
  std::vector<std::vector<StreamRange>> stream_parts;
  int part_t_lo = 0, part_t_hi = -1;         // owned targets (original order)
  int t_lo() const { return part_t_lo; }
  int t_hi() const { return part_t_hi < 0 ? n : part_t_hi; }
  size_t bytes = 0;
  std::vector<void*> allocations;
};

template <typename T>
inline int dev_upload(Plan& p, T** dst, const T* src, size_t n) {
  *dst = nullptr;
  if (n == 0) return IFGFB_OK;
  void* ptr = nullptr;
  IFGFB_CUDA(cudaMalloc(&ptr, n * sizeof(T)));
  p.allocations.push_back(ptr);
  p.bytes += n * sizeof(T);
  if (src) IFGFB_CUDA(cudaMemcpy(ptr, src, n * sizeof(T), cudaMemcpyHostToDevice));
  *dst = static_cast<T*>(ptr);
  return IFGFB_OK;
}

template <typename T>
inline int dev_alloc(Plan& p, T** dst, size_t n) {
  return dev_upload<T>(p, dst, nullptr, n);
}

#define IFGFB_CHECK_ARG(cond, msg) \
  do {                             \
    if (!(cond)) {                 \
      ::ifgfb::set_error(msg);     \
      return IFGFB_ERR_ARG;        \
    }                              \
  } while (0)

#define IFGFB_RC(x)                  \
  do {                               \
    int rc_ = (x);                   \
    if (rc_ != IFGFB_OK) return rc_; \
  } while (0)

// pm_stride == 0: out / out_disp are (nch*nk, N) channel-major (original
// order); pm_stride > 0: point-major, out[ell * pm_stride + m]
int far_apply(Plan& p, const double* w, int nch, const double* kappas, int nk,
              double* out, double* out_disp, cudaStream_t st, int pm_stride = 0);
int potentials(Plan& p, const double* phi, double* s_val, double* d_val,
               cudaStream_t st);
int muller_apply(Plan& p, const double* y, double* out, cudaStream_t st);
int muller_far_phase(Plan& p, const double* y, cudaStream_t st);
int muller_near_phase(Plan& p, const double* y, double* out, cudaStream_t st);

}  // namespace ifgfb

struct ifgfb_plan {
  ifgfb::Plan p;
};
