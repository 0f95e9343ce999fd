// Far-field IFGF traversal on sm_100a: leaf direct spectra (K2), value ->
// Chebyshev coefficient transform (K3, fused), child -> parent
// re-interpolation on FP64 tensor cores (K4), cousin emission on FP64 tensor
// cores (K5) and the deterministic per-target reduction.
//
// Reference: ifgf.py:788-882 (propagate_and_emit), ifgf.py:535-554 (K2),
// ifgf.py:502-522 (K3), ifgf.py:752-785 (K4), ifgf.py:630-673 (K5).
//
// Data layout in HBM: per level one coefficient array of 19 KB segments in
// DMMA fragment order (see SEG_DOUBLES), holding the rows this rank owns
// (all rows without a partition; buffers are addressed through a base
// pointer shifted by the first owned row); two arrays are live (child level
// / parent level ping-pong).
#include "common.cuh"

#include <algorithm>
#include <cstdlib>

namespace ifgfb {

__constant__ double c_ms[PS * PS];   // chebyshev transform_matrix(3)
__constant__ double c_ma[PA * PA];   // chebyshev transform_matrix(5)

static bool g_const_ready = false;

static void host_transform_matrix(int n, double* out) {
  // (2/n) T_i(x_j), row 0 halved (reference chebyshev.py:98-105)
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double x = cos((j + 0.5) * M_PI / n);
      double t0 = 1.0, t1 = x, ti = (i == 0) ? 1.0 : x;
      for (int q = 2; q <= i; ++q) {
        ti = 2.0 * x * t1 - t0;
        t0 = t1;
        t1 = ti;
      }
      out[i * n + j] = (2.0 / n) * ti * (i == 0 ? 0.5 : 1.0);
    }
}

int init_constants() {
  if (g_const_ready) return IFGFB_OK;
  double ms[PS * PS], ma[PA * PA];
  host_transform_matrix(PS, ms);
  host_transform_matrix(PA, ma);
  IFGFB_CUDA(cudaMemcpyToSymbol(c_ms, ms, sizeof(ms)));
  IFGFB_CUDA(cudaMemcpyToSymbol(c_ma, ma, sizeof(ma)));
  g_const_ready = true;
  return IFGFB_OK;
}

// ---------------------------------------------------------------- K3 ----
// Node (a, b, c) -> row of a segment buffer in shared memory.  Standard
// layout: (a*PA + b)*PA + c.  OWNER layout (propagation kernel): the row of
// node n is its position inv[n] in the CTA's warp-owned node order.
template <bool OWNER>
__device__ __forceinline__ int node_row(const unsigned char* inv, int a, int b, int c) {
  return OWNER ? (int)inv[(a * PA + b) * PA + c] : (a * PA + b) * PA + c;
}

// In-place node values -> coefficients for one segment held in shared memory
// (rows per node_row<OWNER>, NCOL complex columns, row stride RS complex):
// three axis transforms (reference ifgf.py:502-522).
// CTA-wide barrier of the threads running the transform: all threads
// (__syncthreads) or, in the K4 ring kernel, the 160 consumer threads only
// (named barrier 1; the producer warp never joins)
template <bool NAMED>
__device__ __forceinline__ void k3_sync() {
  if (NAMED) asm volatile("bar.sync 1, %0;\n" :: "n"(32 * WARP_PARTS) : "memory");
  else __syncthreads();
}

// One axis transform c = M v (values at the Chebyshev nodes -> coefficients,
// M = (2/n) T_i(x_j), row 0 halved) using the node symmetry x_{n-1-j} = -x_j:
// T_i(x_{n-1-j}) = (-1)^i T_i(x_j), so even rows act on v_j + v_{n-1-j} and
// odd rows on v_j - v_{n-1-j} (and T_i(0) = 0 for odd i): 14 / 34 FP64
// operations per complex value for n = 3 / 5 instead of 18 / 50.
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 rfma(double m, double2 v, double2 acc) {
  return make_double2(fma(m, v.x, acc.x), fma(m, v.y, acc.y));
}
__device__ __forceinline__ double2 rmul(double m, double2 v) { return make_double2(m * v.x, m * v.y); }

__device__ __forceinline__ void xform3(double2 (&v)[PS]) {
  const double2 s = cadd(v[0], v[2]), d = csub(v[0], v[2]), mid = v[1];
  v[0] = rfma(c_ms[0], s, rmul(c_ms[1], mid));
  v[1] = rmul(c_ms[PS], d);
  v[2] = rfma(c_ms[2 * PS], s, rmul(c_ms[2 * PS + 1], mid));
}

__device__ __forceinline__ void xform5(double2 (&v)[PA]) {
  const double2 s0 = cadd(v[0], v[4]), s1 = cadd(v[1], v[3]);
  const double2 d0 = csub(v[0], v[4]), d1 = csub(v[1], v[3]), mid = v[2];
#pragma unroll
  for (int i = 0; i < PA; ++i) {
    if (i & 1) v[i] = rfma(c_ma[i * PA], d0, rmul(c_ma[i * PA + 1], d1));
    else v[i] = rfma(c_ma[i * PA], s0, rfma(c_ma[i * PA + 1], s1, rmul(c_ma[i * PA + 2], mid)));
  }
}

template <bool OWNER, int RS = NCOL, bool NAMED = false>
__device__ void to_coeffs_smem(double2* V, const unsigned char* inv, int tid, int nthr) {
  for (int task = tid; task < PA * PA * NCOL; task += nthr) {
    const int bc = task / NCOL, m = task % NCOL;
    const int b = bc / PA, c = bc % PA;
    double2 v[PS];
    int row[PS];
#pragma unroll
    for (int a = 0; a < PS; ++a) {
      row[a] = node_row<OWNER>(inv, a, b, c) * RS + m;
      v[a] = V[row[a]];
    }
    xform3(v);
#pragma unroll
    for (int a = 0; a < PS; ++a) V[row[a]] = v[a];
  }
  k3_sync<NAMED>();
  for (int task = tid; task < PS * PA * NCOL; task += nthr) {
    const int ac = task / NCOL, m = task % NCOL;
    const int a = ac / PA, c = ac % PA;
    double2 v[PA];
    int row[PA];
#pragma unroll
    for (int b = 0; b < PA; ++b) {
      row[b] = node_row<OWNER>(inv, a, b, c) * RS + m;
      v[b] = V[row[b]];
    }
    xform5(v);
#pragma unroll
    for (int b = 0; b < PA; ++b) V[row[b]] = v[b];
  }
  k3_sync<NAMED>();
  for (int task = tid; task < PS * PA * NCOL; task += nthr) {
    const int ab = task / NCOL, m = task % NCOL;
    const int a = ab / PA, b = ab % PA;
    double2 v[PA];
    int row[PA];
#pragma unroll
    for (int c = 0; c < PA; ++c) {
      row[c] = node_row<OWNER>(inv, a, b, c) * RS + m;
      v[c] = V[row[c]];
    }
    xform5(v);
#pragma unroll
    for (int c = 0; c < PA; ++c) V[row[c]] = v[c];
  }
  k3_sync<NAMED>();
}

// Write one segment's coefficients V[i][m] (rows per node_row<OWNER>, row
// stride RS complex) in DMMA B-fragment order (see SEG_DOUBLES): coalesced
// stores, padding zeroed.  RS = 20 spreads the 4 rows a warp reads over both
// bank halves (conflict-free); the K4 accumulators keep RS = NCOL.
template <bool OWNER, int RS = NCOL>
__device__ __forceinline__ void store_segment(double* dst, const double2* V,
                                              const unsigned char* inv, int tid,
                                              int nthr) {
  for (int idx = tid; idx < SEG_DOUBLES; idx += nthr) {
    const int ks = idx >> 7, lane = (idx >> 1) & 31, nt = ((idx >> 5) & 2) | (idx & 1);
    int ab, c;
    if (ks < KMAIN) {
      const int q = ks / PA;
      c = ks - PA * q;
      ab = 4 * q + (lane & 3);
    } else {
      const int t = lane & 3, st = ks - KMAIN;
      ab = t < 3 ? 12 + t : (st < 3 ? 12 + st : PS * PA);   // (s=3, tig=3): zero row
      c = t < 3 ? st : PA - 1;
    }
    double v = 0.0;
    if (ab < PS * PA) {
      const int col = 8 * nt + (lane >> 2);
      const double2 z = V[node_row<OWNER>(inv, ab / PA, ab % PA, c) * RS + (col >> 1)];
      v = (col & 1) ? z.y : z.x;
    }
    dst[idx] = v;
  }
}

// The same store for CTAs of exactly 128 threads: element idx = 128 ks + tid,
// so a thread's fragment lane and column tile are fixed and the k-step loop
// unrolls into one shared load and one coalesced store per k-step (the
// generic loop spends ~37 instructions per element on index arithmetic).
template <bool OWNER, int RS = NCOL>
__device__ __forceinline__ void store_segment128(double* dst, const double2* V,
                                                 const unsigned char* inv, int tid) {
  const int lane = (tid >> 1) & 31, nt = ((tid >> 5) & 2) | (tid & 1);
  const int tig = lane & 3, col = 8 * nt + (lane >> 2);
  const double* Vd = reinterpret_cast<const double*>(V) + (col >> 1) * 2 + (col & 1);
#pragma unroll
  for (int ks = 0; ks < KSTEPS; ++ks) {
    int ab, c;
    if (ks < KMAIN) {
      ab = 4 * (ks / PA) + tig;
      c = ks % PA;
    } else {
      const int st = ks - KMAIN;
      ab = tig < 3 ? 12 + tig : (st < 3 ? 12 + st : PS * PA);   // (s=3, tig=3): zero row
      c = tig < 3 ? st : PA - 1;
    }
    double v = 0.0;
    if (ab < PS * PA) {
      const int node = ab * PA + c;
      v = Vd[(OWNER ? (int)inv[node] : node) * (RS * 2)];
    }
    dst[ks * 128 + tid] = v;
  }
}

// ------------------------------------------------------------ weights ----
// wt[t][c] = w[c][perm[t]] (tree order, CH channel slots, zero padded)
__global__ void pack_weights(const double2* __restrict__ w, int nch, int n,
                             const int* __restrict__ perm, int ch,
                             double2* __restrict__ wt) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * ch) return;
  const int t = idx / ch, c = idx % ch;
  wt[idx] = (c < nch) ? w[(size_t)c * n + perm[t]] : make_double2(0.0, 0.0);
}

// ---------------------------------------------------------------- K2 ----
struct LeafArgs {
  const int* seg_box; const int* seg_id; const double* centers;
  const int* pt_start; const int* pt_count; const double* tabs;
  int n_s, n_a; double h;
  const double* points;  // tree order
  const double2* wt;     // [N][CH]
  double kr[2], ki[2];
  double* coef;
  int row0;              // first segment row handled (partition)
};

// One CTA per finest-level segment: node values
//   F[node][c*NK+k] = sum_{src in box} (r/d) exp(i kappa_k (d - r)) w[c][src]
// (reference _direct_spectra_box, ifgf.py:535-554), then the K3 transform.
// Thread (node, k) owns the CH columns of one wavenumber: 75*NK busy threads,
// CH accumulators each (the per-value arithmetic and source order are those
// of one thread per node, so the result does not depend on the split).
constexpr int LEAF_RS = 20;   // padded row stride of the leaf's node values
template <int NK>
constexpr int leaf_threads() { return ((NN * NK + 31) / 32) * 32; }

#ifndef IFGFB_LEAF_MINB   // 6 CTAs/SM (64 registers, 40 B spill): 1.833 -> 1.739 ms at (4,10)
#define IFGFB_LEAF_MINB 6
#endif
template <int NK>
__global__ void __launch_bounds__(leaf_threads<NK>(), IFGFB_LEAF_MINB) leaf_kernel(LeafArgs a) {
  constexpr int CH = NCOL / NK;
  __shared__ double2 V[NN * LEAF_RS];
  const int row = blockIdx.x + a.row0, tid = threadIdx.x;
  const int box = a.seg_box[row], id = a.seg_id[row];
  if (tid < NN * NK) {
    const int node = tid / NK, k = NK > 1 ? tid % NK : 0;
    const int two_na = 2 * a.n_a;
    const int i_p = id % two_na, rest = id / two_na;
    const int i_t = rest % a.n_a, i_s = rest / a.n_a;
    const int na = node / (PA * PA), nb = (node / PA) % PA, nc = node % PA;
    const double* s_nodes = a.tabs;
    const double* sin_t = s_nodes + a.n_s * PS;
    const double* cos_t = sin_t + a.n_a * PA;
    const double* sin_p = cos_t + a.n_a * PA;
    const double* cos_p = sin_p + two_na * PA;
    const double r = a.h / s_nodes[i_s * PS + na];
    const double st = sin_t[i_t * PA + nb], ct = cos_t[i_t * PA + nb];
    const double sp = sin_p[i_p * PA + nc], cp = cos_p[i_p * PA + nc];
    const double x = add_rn(a.centers[3 * box + 0], mul_rn(r, mul_rn(st, cp)));
    const double y = add_rn(a.centers[3 * box + 1], mul_rn(r, mul_rn(st, sp)));
    const double z = add_rn(a.centers[3 * box + 2], mul_rn(r, ct));
    const double kr = (NK > 1 && k) ? a.kr[1] : a.kr[0];
    const double ki = (NK > 1 && k) ? a.ki[1] : a.ki[0];
    double2 acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = make_double2(0.0, 0.0);
    const int s0 = a.pt_start[box], s1 = s0 + a.pt_count[box];
    for (int s = s0; s < s1; ++s) {
      const double dx = x - a.points[3 * s], dy = y - a.points[3 * s + 1],
                   dz = z - a.points[3 * s + 2];
      const double d = sqrt(dx * dx + dy * dy + dz * dz);
      const double q = r / d;
      const double2 e = cexp_ikx(kr, ki, d - r);
      const double2 g = make_double2(q * e.x, q * e.y);
      const double2* wv = a.wt + (size_t)s * CH;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const double2 p = cmul(g, wv[c]);
        acc[c].x += p.x;
        acc[c].y += p.y;
      }
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) V[node * LEAF_RS + c * NK + k] = acc[c];
  }
  __syncthreads();
  to_coeffs_smem<false, LEAF_RS>(V, nullptr, tid, blockDim.x);
  // unrolled store by the first 128 threads (element 128 ks + tid): 6 instead
  // of 37 instructions per element of the generic index arithmetic
  constexpr int LEAF_THREADS = ((NN * NK + 31) / 32) * 32;
  if (LEAF_THREADS >= 128) {
    if (tid < 128) store_segment128<false, LEAF_RS>(a.coef + (size_t)row * SEG_DOUBLES, V, nullptr, tid);
  } else {
    store_segment<false, LEAF_RS>(a.coef + (size_t)row * SEG_DOUBLES, V, nullptr, tid,
                                  blockDim.x);
  }
}

// ------------------------------------------------------- DMMA helpers ----
// Tensor-product Chebyshev basis of one interpolation point, consumed as the
// A operand of m8n8k4 f64 MMAs (K = 75 coefficients in 19 k-steps, see
// SEG_DOUBLES).  Main block, k-step 5q + c (q < 3): coefficient
// (ab = 4q + tig, c), A value tst[q] * tp[c] with tst[q] = T_a(xs) T_b(xt).
// Tail, k-step 15 + s: tig < 3 holds (ab, c) = (12 + tig, s), tig = 3 holds
// (12 + s, 4) (s < 3; s = 3 is the zero row); u = T_2(xs) T_{2+min(tig,2)}(xt)
// and the tig = 3 lanes take T_{12+s} from lane s of their group by shuffle.
// Products in numpy's order (T_a T_b) T_c.
struct BasisA {
  double tst[3];
  double tp[PA];
  double u;
};

template <bool EXACT>
__device__ __forceinline__ BasisA make_basis(double xs, double xt, double xp,
                                             int tig) {
  double ts[PS], tt[PA];
  BasisA B;
  if (EXACT) {
    cheb_exact<PS>(xs, ts);
    cheb_exact<PA>(xt, tt);
    cheb_exact<PA>(xp, B.tp);
  } else {
    ts[0] = 1.0; ts[1] = xs; ts[2] = 2.0 * xs * xs - 1.0;
    tt[0] = 1.0; tt[1] = xt;
    B.tp[0] = 1.0; B.tp[1] = xp;
#pragma unroll
    for (int i = 2; i < PA; ++i) {
      tt[i] = 2.0 * xt * tt[i - 1] - tt[i - 2];
      B.tp[i] = 2.0 * xp * B.tp[i - 1] - B.tp[i - 2];
    }
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int ab = 4 * q + tig;
    const int ia = ab / PA, ib = ab - PA * ia;
    const double va = (ia == 0) ? ts[0] : (ia == 1) ? ts[1] : ts[2];
    const double vb = (ib == 0) ? tt[0] : (ib == 1) ? tt[1] : (ib == 2) ? tt[2]
                    : (ib == 3) ? tt[3] : tt[4];
    B.tst[q] = EXACT ? mul_rn(va, vb) : va * vb;
  }
  const double vu = (tig == 0) ? tt[2] : (tig == 1) ? tt[3] : tt[4];
  B.u = EXACT ? mul_rn(ts[2], vu) : ts[2] * vu;
  return B;
}

// dst += c * r (complex) in 4 FMAs: the K4 accumulate of one re-interpolated
// value times the re-centering ratio.  (The separate multiply-then-add took
// 6 FP64 instructions; scalar FP64 shares the DMMA pipe and costs ~5 pipe
// cycles each when interleaved with DMMAs, tools/dmma_mix.cu.)
__device__ __forceinline__ void cmul_acc(double2& dst, double c_re, double c_im, double2 r) {
  dst.x = fma(c_re, r.x, fma(-c_im, r.y, dst.x));
  dst.y = fma(c_re, r.y, fma(c_im, r.x, dst.y));
}

// acc[nt] (+)= sum_i basis_i * C[i][8nt + grp]: 19 k-steps x 4 column tiles
// of DMMA; the B fragments of a k-step are two contiguous 512-byte warp
// loads from the fragment-ordered segment.
#ifndef IFGFB_ACC_QUNROLL
#define IFGFB_ACC_QUNROLL 3
#endif
#ifndef IFGFB_ACC_MINB
#define IFGFB_ACC_MINB 6
#endif
#ifndef IFGFB_ACC_ROWS
#define IFGFB_ACC_ROWS 1
#endif

__device__ __forceinline__ void dmma4(double (&c0)[4], double (&c1)[4], double av,
                                      const double2* F, int ks) {
  const double2 b01 = F[ks * 64], b23 = F[ks * 64 + 32];
  dmma(c0[0], c1[0], av, b01.x);
  dmma(c0[1], c1[1], av, b01.y);
  dmma(c0[2], c1[2], av, b23.x);
  dmma(c0[3], c1[3], av, b23.y);
}

// K4: software L1 prefetch of the B fragments IFGFB_ACC_PF k-steps ahead
// (prefetch.global.L1 takes no registers; 0 = off).  Measured at (4,10):
// 0 / 2 / 4 / 6 / 8 / 12 / 16 -> propagate 22.98 / 23.06 / 23.07 / 22.67 /
// 22.58 / 22.52 / 23.40 ms (tools/ab_variants.sh, profiles/ab_r01_prefetch.txt).
#ifndef IFGFB_ACC_PF
#define IFGFB_ACC_PF 12
#endif
#ifndef IFGFB_EMIT_PF   // same for the emission kernel (K5): 1.198 -> 1.046 ms at 8
#define IFGFB_EMIT_PF 8
#endif
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];\n" :: "l"(p));
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" :: "l"(p));
}
#ifndef IFGFB_ACC_L2PF   // K4: L2 prefetch of the next instance's child blocks
#define IFGFB_ACC_L2PF 0
#endif

template <bool EXACT, int QU = 3>
__device__ __forceinline__ void basis_times_block(const BasisA& B,
                                                  const double* __restrict__ C,
                                                  int lane, double (&c0)[4],
                                                  double (&c1)[4]) {
  const double2* F = reinterpret_cast<const double2*>(C) + lane;
#pragma unroll QU
  for (int q = 0; q < 3; ++q) {
#pragma unroll
    for (int c = 0; c < PA; ++c) {
      const int ks = 5 * q + c;
      constexpr int PF = EXACT ? IFGFB_EMIT_PF : IFGFB_ACC_PF;
      if (PF > 0 && ks + PF < KSTEPS) {
        prefetch_l1(F + (ks + PF) * 64);
        prefetch_l1(F + (ks + PF) * 64 + 32);
      }
      dmma4(c0, c1, EXACT ? mul_rn(B.tst[q], B.tp[c]) : B.tst[q] * B.tp[c], F, ks);
    }
  }
  const int tig = lane & 3;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const double us = __shfl_sync(0xffffffffu, B.u, (lane & ~3) | (s < 3 ? s : 0));
    const double x = tig < 3 ? B.u : us, y = tig < 3 ? B.tp[s] : B.tp[PA - 1];
    const double av = (tig < 3 || s < 3) ? (EXACT ? mul_rn(x, y) : x * y) : 0.0;
    dmma4(c0, c1, av, F, KMAIN + s);
  }
}

// ---------------------------------------------------------------- K4 ----
// ratio[t][j][k] = (r_p / r_c) exp(i kappa_k (r_c - r_p)) per type and parent
// node (reference ifgf.py:772-773), tabulated once per apply and level.
template <int NK>
__global__ void ratio_kernel(int64_t n, const double* __restrict__ node_r,
                             double kr0, double ki0, double kr1, double ki1,
                             double2* __restrict__ ratio) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const double rp = node_r[2 * idx], rc = node_r[2 * idx + 1];
  const double q = rp / rc;
  const double2 e0 = cexp_ikx(kr0, ki0, rc - rp);
  ratio[idx * NK] = make_double2(q * e0.x, q * e0.y);
  if (NK > 1) {
    const double2 e1 = cexp_ikx(kr1, ki1, rc - rp);
    ratio[idx * NK + 1] = make_double2(q * e1.x, q * e1.y);
  }
}

// Node geometry computed on the device per (instance, node) instead of the
// per-type tables node_geom / ratio (levels whose type tables do not fit;
// coarse levels of large configurations have about one type per instance).
// Continuous values only: the sigma assignment of every node stays the
// host's (exact, reference expressions); these coordinates differ from the
// host's by a few ulps (libdevice acos/atan2 vs numpy), far inside the
// interpolation accuracy.
struct OtfGeom {
  const unsigned char* type_octant;   // per type: child octant
  const int* parent_seg_id;           // per parent row: flat segment id
  const double* ptabs;                // parent level node tables (see LeafArgs)
  int pn_s, pn_a;
  double ph;                          // parent level h
  const int* child_seg_id;            // per child row: flat segment id
  int cn_a;
  double c_delta_s, c_delta_a, child_side;
  double kr[2], ki[2];
};

// Parent node `node` of parent segment `pseg` seen from the centre of the
// child in octant `oct` (reference _AccumType, ifgf.py:686-702; node layout
// ifgf.py:369-387; cone_coords ifgf.py:305-317; local_coords ifgf.py:361-367)
// -> local coordinates in child segment `csid` and the re-centering ratio
// (r_p / r_c) exp(i kappa (r_c - r_p)) (ifgf.py:772-773).
template <int NK>
__device__ __forceinline__ void otf_node(const OtfGeom& o, int pseg, int oct, int node,
                                         int csid, double* geom, double2* ratio) {
  const int two_na = 2 * o.pn_a;
  const int i_p = pseg % two_na, rest = pseg / two_na;
  const int i_t = rest % o.pn_a, i_s = rest / o.pn_a;
  const int na = node / (PA * PA), nb = (node / PA) % PA, nc = node % PA;
  const double* s_nodes = o.ptabs;
  const double* sin_t = s_nodes + o.pn_s * PS;
  const double* cos_t = sin_t + o.pn_a * PA;
  const double* sin_p = cos_t + o.pn_a * PA;
  const double* cos_p = sin_p + two_na * PA;
  const double rp = o.ph / s_nodes[i_s * PS + na];
  const double st = sin_t[i_t * PA + nb], ct = cos_t[i_t * PA + nb];
  const double sp = sin_p[i_p * PA + nc], cp = cos_p[i_p * PA + nc];
  const double half = 0.5 * o.child_side;
  const double x = ((oct >> 2) & 1 ? -half : half) + rp * (st * cp);
  const double y = ((oct >> 1) & 1 ? -half : half) + rp * (st * sp);
  const double z = (oct & 1 ? -half : half) + rp * ct;
  const double rc = sqrt((x * x + y * y) + z * z);
  const double sv = (0.8660254037844386 * o.child_side) / rc;
  const double th = acos(fmin(fmax(z / rc, -1.0), 1.0));
  double ph = atan2(y, x);
  const int two_cna = 2 * o.cn_a;
  const int j_p = csid % two_cna, crest = csid / two_cna;
  const int j_t = crest % o.cn_a, j_s = crest / o.cn_a;
  // phi in [0, 2 pi) as np.mod does; across the seam take the branch of the
  // host-assigned interval
  if (ph < 0.0) ph += 2.0 * M_PI;
  const double lp = ph / o.c_delta_a - j_p;
  if (lp > o.cn_a) ph -= 2.0 * M_PI;
  else if (lp < -o.cn_a) ph += 2.0 * M_PI;
  geom[0] = 2.0 * (sv / o.c_delta_s - j_s) - 1.0;
  geom[1] = 2.0 * (th / o.c_delta_a - j_t) - 1.0;
  geom[2] = 2.0 * (ph / o.c_delta_a - j_p) - 1.0;
  const double q = rp / rc;
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const double2 e = cexp_ikx(o.kr[k], o.ki[k], rc - rp);
    ratio[k] = make_double2(q * e.x, q * e.y);
  }
}

struct AccArgs {
  const int* inst_off; const int* inst_type; const int* inst_crow_off;
  const int* crow; const int* tile_off; const uint4* tiles;
  const unsigned char* row_order; const unsigned char* row_cuts;
  const double* node_geom; const double2* ratio;
  const double* coef_child; double* coef_parent;
  int row0;              // first parent row handled (partition)
  int row_end;           // one past the last parent row handled
  int rows_per_cta;      // consecutive parent rows per CTA
  OtfGeom o;             // OTF instantiation only
  const unsigned char* gid;   // tile-free ring kernel: sigma group per (type, node)
  int child_lo, child_hi;     // child rows present in coef_child (checks)
  // PRE instantiation of the wide kernel: node_geom / ratio hold one row per
  // (instance, node), instance index relative to inst_base (otf_tables_kernel)
  int inst_base = 0;
};

// cp.async (LDGSTS) helpers: global -> shared without a register round trip
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n"
               :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n"
               :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n"
               :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" :: "n"(N));
}

// Staging of one instance for the CTA: everything the tiles read besides the
// child coefficients.  Indexed by node position in the row order, so warp w
// fills and reads only its own slice [cuts[w], cuts[w+1]) (a warp has at
// most as many tiles as nodes) and no cross-warp synchronisation is needed.
#ifndef IFGFB_STAGE_GROUPS
#define IFGFB_STAGE_GROUPS 32
#endif
constexpr int MAX_GROUPS = IFGFB_STAGE_GROUPS;  // staged child rows per instance (more: global)
struct __align__(16) RowStage {
  uint4 tiles[NN];                    // warp w: tiles[cuts[w] ..]
  double2 ratio[NN * 2];              // [position][kappa]
  double geom[NN * 3];                // [position][xs, xt, xp]
  int crow[WARP_PARTS][MAX_GROUPS];   // per-warp copy of the instance's child rows
};

// Row (lane group grp) of a K4 row tile: the warp-set slot it owns; rows past
// the tile's count duplicate slot 0 and are dropped.
__device__ __forceinline__ int tile_slot(const uint4& tl, int grp, bool& valid) {
  const int nrows = (tl.x >> 8) & 0xff;
  const int byte = 2 + grp;
  const unsigned word = byte < 4 ? tl.x : byte < 8 ? tl.y : tl.z;
  valid = grp < nrows;
  return valid ? (int)((word >> (8 * (byte & 3))) & 0xff) : (int)((tl.x >> 16) & 0xff);
}

// One CTA (5 warps) per parent segment row, owner computes: warp w owns the
// parent nodes at positions row_cuts[w]..row_cuts[w+1]-1 (7..23 nodes) of the
// row's signature order (octree.row_tiles, csrc/tiles.cpp) and keeps their
// 16-column accumulators in its own shared slice (no atomics, no inter-warp hazards; every warp walks every (parent
// segment, child) instance).  Per instance each warp re-interpolates the
// child's coefficients at its nodes: row tiles of <= 8 nodes sharing a child
// segment sigma, 20 k-steps x 4 column tiles of FP64 DMMA, times the
// re-centering ratio.  The instance's tile records, child rows, node
// geometry and ratios are staged by cp.async one instance ahead, so the
// only global loads on a tile's critical path are the B fragments.  The
// summed values are transformed to coefficients (K3) and written once.
// WIDE: some instance of the level has more than MAX_GROUPS child segments
// (coarse levels of large configurations); the extra rows are read from
// global memory.  Kept out of the common instantiation (costs ~2%).
// TILEFREE: no tile records in the plan; each warp forms its row tiles per
// sigma group from its slots' group ids (gid per type and node): distinct
// groups ascending (__reduce_min_sync), slots of a group in slot order
// (ballot), runs of <= 8 -- exactly the records ifgfb_row_tiles_fill writes,
// so the result is bitwise the tile-record kernel's.
template <int NK, bool WIDE, bool OTF, bool TILEFREE = false>
__global__ void __launch_bounds__(160, IFGFB_ACC_MINB) accum_kernel(AccArgs a) {
  __shared__ double2 acc[NN * NCOL];                        // 19.2 KB
  __shared__ RowStage stage[2];                             // 11.8 KB
  __shared__ unsigned char ord[NN], inv[NN], sgrp[NN];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, tig = lane & 3;
  const int pbeg = a.row0 + blockIdx.x * a.rows_per_cta;
  const int pend = min(pbeg + a.rows_per_cta, a.row_end);
  for (int p = pbeg; p < pend; ++p) {
  const int pos0 = a.row_cuts[(size_t)p * (WARP_PARTS + 1) + warp];
  const int nset = a.row_cuts[(size_t)p * (WARP_PARTS + 1) + warp + 1] - pos0;
  double2* mine = acc + pos0 * NCOL;
  const unsigned char* word = ord + pos0;
  if (lane < nset)               // each warp loads its own part of the order
    ord[pos0 + lane] = a.row_order[(size_t)p * NN + pos0 + lane];
  for (int i = lane; i < nset * NCOL; i += 32) mine[i] = make_double2(0.0, 0.0);
  // the row's instance scalars, lane j <-> instance i0 + j (<= 8 per row)
  const int i0 = a.inst_off[p], ni = a.inst_off[p + 1] - i0;
  int my_t = 0, my_ks = 0, my_ke = 0, my_co = 0;
  if (lane < ni) {
    my_t = a.inst_type[i0 + lane];
    if (!TILEFREE) {
      my_ks = a.tile_off[(i0 + lane) * WARP_PARTS + warp];
      my_ke = a.tile_off[(i0 + lane) * WARP_PARTS + warp + 1];
    }
  }
  if (lane <= ni) my_co = a.inst_crow_off[i0 + lane];
  __syncwarp();
  // TILEFREE: sigma group of the lane's slot (0xFFFFFFFF: no slot), one
  // instance ahead
  auto slot_group = [&](int j) -> unsigned {
    if (!TILEFREE || j >= ni) return 0xFFFFFFFFu;       // warp-uniform
    const int t = __shfl_sync(0xffffffffu, my_t, j);    // all lanes
    return lane < nset ? (unsigned)__ldg(a.gid + (size_t)t * NN + word[lane]) : 0xFFFFFFFFu;
  };
  auto stage_inst = [&](int j, RowStage& S) {
    const int t = __shfl_sync(0xffffffffu, my_t, j);
    const int ks = __shfl_sync(0xffffffffu, my_ks, j);
    const int ke = __shfl_sync(0xffffffffu, my_ke, j);
    const int cs = __shfl_sync(0xffffffffu, my_co, j);
    const int ce = __shfl_sync(0xffffffffu, my_co, j + 1);
    const size_t tb = (size_t)t * NN;
    if (!OTF) {
      for (int e = lane; e < nset * 3; e += 32)
        cp_async8(&S.geom[3 * pos0 + e], a.node_geom + (tb + word[e / 3]) * 3 + e % 3);
      for (int e = lane; e < nset * NK; e += 32)
        cp_async16(&S.ratio[NK * pos0 + e], a.ratio + (tb + word[e / NK]) * NK + e % NK);
    }
    if (!TILEFREE && lane < ke - ks) cp_async16(&S.tiles[pos0 + lane], a.tiles + ks + lane);
    if (lane < min(ce - cs, MAX_GROUPS)) cp_async4(&S.crow[warp][lane], a.crow + cs + lane);
    cp_async_commit();
    if (IFGFB_ACC_L2PF) {   // warp w warms L2 with groups w, w + 5, ...
      for (int g = warp; g < ce - cs; g += WARP_PARTS) {
        const double* blk = a.coef_child + (size_t)__ldg(a.crow + cs + g) * SEG_DOUBLES;
        for (int off = lane * 16; off < SEG_DOUBLES; off += 32 * 16) prefetch_l2(blk + off);
      }
    }
  };
  unsigned g_next = slot_group(0);
  if (ni > 0) stage_inst(0, stage[0]);
  for (int j = 0; j < ni; ++j) {
    RowStage& S = stage[j & 1];
    const unsigned g_cur = g_next;
    if (j + 1 < ni) {
      stage_inst(j + 1, stage[(j + 1) & 1]);
      g_next = slot_group(j + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const int ntile = __shfl_sync(0xffffffffu, my_ke - my_ks, j);
    const int* crow_g = a.crow + __shfl_sync(0xffffffffu, my_co, j);
    if (OTF && TILEFREE) {   // each lane: geometry of its own slot
      const int pseg = a.o.parent_seg_id[p];
      const int oct = a.o.type_octant[__shfl_sync(0xffffffffu, my_t, j)];
      if (lane < nset) {
        const int g = (int)g_cur;
        const int cr = (!WIDE || g < MAX_GROUPS) ? S.crow[warp][g] : crow_g[g];
        otf_node<NK>(a.o, pseg, oct, word[lane], a.o.child_seg_id[cr],
                     &S.geom[(pos0 + lane) * 3], &S.ratio[(pos0 + lane) * NK]);
      }
      __syncwarp();
    } else if (OTF) {   // slot -> sigma group from the tile records, then geometry
      for (int e = lane; e < ntile * 8; e += 32) {
        const uint4 tl = S.tiles[pos0 + (e >> 3)];
        const int r = e & 7;
        if (r < (int)((tl.x >> 8) & 0xff)) {
          const int byte = 2 + r;
          const unsigned w = byte < 4 ? tl.x : byte < 8 ? tl.y : tl.z;
          sgrp[pos0 + ((w >> (8 * (byte & 3))) & 0xff)] = (unsigned char)(tl.x & 0xff);
        }
      }
      __syncwarp();
      const int pseg = a.o.parent_seg_id[p];
      const int oct = a.o.type_octant[__shfl_sync(0xffffffffu, my_t, j)];
      for (int e = lane; e < nset; e += 32) {
        const int g = sgrp[pos0 + e];
        const int cr = (!WIDE || g < MAX_GROUPS) ? S.crow[warp][g] : crow_g[g];
        otf_node<NK>(a.o, pseg, oct, word[e], a.o.child_seg_id[cr], &S.geom[(pos0 + e) * 3],
                     &S.ratio[(pos0 + e) * NK]);
      }
      __syncwarp();
    }
    unsigned g_at = TILEFREE ? __reduce_min_sync(0xffffffffu, g_cur) : 0u;
    unsigned mask = TILEFREE && g_at != 0xFFFFFFFFu
                        ? __ballot_sync(0xffffffffu, g_cur == g_at) : 0u;
    for (int k = 0; TILEFREE ? (mask != 0u) : (k < ntile); ++k) {
      bool valid;
      int slot, g;
      if (TILEFREE) {
        // row grp of this tile = the grp-th slot of group g_at (slot order)
        unsigned m = mask;
        for (int i = 0; i < grp; ++i) m &= m - 1;
        valid = m != 0u;
        slot = valid ? __ffs(m) - 1 : __ffs(mask) - 1;
        g = (int)g_at;
        if (__popc(mask) > 8) {
          for (int i = 0; i < 8; ++i) mask &= mask - 1;
        } else {   // next distinct group of the warp's slots
          g_at = __reduce_min_sync(0xffffffffu, g_cur > g_at ? g_cur : 0xFFFFFFFFu);
          mask = g_at != 0xFFFFFFFFu ? __ballot_sync(0xffffffffu, g_cur == g_at) : 0u;
        }
      } else {
        const uint4 tl = S.tiles[pos0 + k];
        slot = tile_slot(tl, grp, valid);
        g = tl.x & 0xff;
      }
#ifdef IFGFB_ACC_FAKEB   // diagnostic only: every tile reads the first owned child row
      const int crow_used = S.crow[warp][0] & 0;
#else
      const int crow_used = (!WIDE || g < MAX_GROUPS) ? S.crow[warp][g] : crow_g[g];
      IFGFB_DCHECK(crow_used >= a.child_lo && crow_used < a.child_hi && slot < nset);
#endif
#if IFGFB_ACC_PF > 0 && defined(IFGFB_ACC_PFNEXT)
      if (!TILEFREE && k + 1 < ntile) {   // warm L1 with the next tile's first k-steps
        const int gn = S.tiles[pos0 + k + 1].x & 0xff;
        const int crn = (!WIDE || gn < MAX_GROUPS) ? S.crow[warp][gn] : crow_g[gn];
        const double2* Fn = reinterpret_cast<const double2*>(
            a.coef_child + (size_t)crn * SEG_DOUBLES) + lane;
#pragma unroll
        for (int q = 0; q < IFGFB_ACC_PF; ++q) {
          prefetch_l1(Fn + q * 64);
          prefetch_l1(Fn + q * 64 + 32);
        }
      }
#endif
      const double* ng = S.geom + (pos0 + slot) * 3;
      const BasisA B = make_basis<false>(ng[0], ng[1], ng[2], tig);
      double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
      basis_times_block<false, IFGFB_ACC_QUNROLL>(
          B, a.coef_child + (size_t)crow_used * SEG_DOUBLES, lane, c0, c1);
      if (valid) {
        const double2 r0 = S.ratio[(pos0 + slot) * NK];
        const double2 r1 = NK > 1 ? S.ratio[(pos0 + slot) * NK + NK - 1] : r0;
        double2* dst = mine + slot * NCOL;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const int m = 4 * nt + tig;
          cmul_acc(dst[m], c0[nt], c1[nt], (NK > 1 && (tig & 1)) ? r1 : r0);
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (threadIdx.x < NN) inv[ord[threadIdx.x]] = (unsigned char)threadIdx.x;
  __syncthreads();
  to_coeffs_smem<true>(acc, inv, threadIdx.x, 32 * WARP_PARTS);
  store_segment<true>(a.coef_parent + (size_t)p * SEG_DOUBLES, acc, inv, threadIdx.x,
                      32 * WARP_PARTS);
  __syncthreads();
  }
}

// ------------------------------------------------- K4, wide warps ----
// The same owner-computes propagation with FEWER, WIDER owner warps
// (IFGFB_K4=wide): WW warps per parent row, each owning NN/WW (25 for WW = 3)
// consecutive positions of the row's signature order.  A parent row's 75
// nodes fall into only 2-3 child segments per child (tools/group_analysis.py),
// so a warp's nodes of one sigma group fill up to 4 MMA row tiles; the warp
// runs them TOGETHER: one pair of 512-byte B-fragment loads per k-step feeds
// 4 x NT DMMAs (NT = 1..4 row tiles), instead of every 8-row tile pulling
// its own copy of the 19 KB child block through L1 (the 5-warp kernel moves
// ~4.5 KB of L2 -> SM traffic per DMMA k-step and sits at 72% of the L2
// bandwidth; this one ~1/NT of it).  The Chebyshev values of a node
// (T_0..2(xs), T_0..4(xt), T_0..4(xp)) are computed once per (instance,
// node) into shared memory by the node's owner lane; a tile's A values are
// two shared loads and two multiplies per k-step (the 5-warp kernel
// recomputes the recurrences in all 4 lanes of a row, per tile).  Tiles are
// formed in the kernel from the nodes' sigma groups (tile-free plans).  The
// per-node arithmetic (basis products, k order, accumulation order over the
// row's instances) is the 5-warp kernel's, so results are bitwise equal.
#ifndef IFGFB_WIDE_WARPS
#define IFGFB_WIDE_WARPS 4
#endif
#ifndef IFGFB_WIDE_MINB
#define IFGFB_WIDE_MINB 5
#endif
#ifndef IFGFB_WIDE_MAXNT   // row tiles of one sigma group run together (1..4)
#define IFGFB_WIDE_MAXNT 2
#endif
constexpr int WW = IFGFB_WIDE_WARPS;
constexpr int WIDE_MAXNT = IFGFB_WIDE_MAXNT;
#ifndef IFGFB_WIDE_RS   // accumulator row stride in complex values: 17 spreads the 8 rows of a
#define IFGFB_WIDE_RS 17   // tile over the banks (16: every row on the same 64 bytes)
#endif
constexpr int WIDE_RS = IFGFB_WIDE_RS;
static_assert(WIDE_MAXNT >= 1 && WIDE_MAXNT <= 4, "1..4 row tiles per pass");
constexpr int NT_STRIDE = PS + 2 * PA;   // 13 doubles per node
static_assert((NN + WW - 1) / WW <= 32, "a wide warp owns at most 32 nodes");

struct __align__(16) WideStage {
  double2 ratio[NN * 2];        // [position][kappa]
  double geom[NN * 3];          // [position][xs, xt, xp]
  int crow[WW][MAX_GROUPS];     // per-warp copy of the instance's child rows
};

// A operand of k-step KS for the node whose Chebyshev values are T (see
// BasisA): main block ks = 5q + c -> (T_a(xs) T_b(xt)) T_c(xp) with ab = 4q +
// tig; tail ks = 15 + s -> (ab, c) = (12 + tig, s) for tig < 3, (12 + s, 4) for
// tig = 3 (s = 3: the zero row).  tst caches T_a T_b of the current q.
#ifndef IFGFB_WIDE_PF    // L1 prefetch distance of the B fragments, in k-steps
#define IFGFB_WIDE_PF IFGFB_ACC_PF
#endif
#ifndef IFGFB_WIDE_PIN   // pin the A-value multiplies between the DMMA groups
#define IFGFB_WIDE_PIN 1
#endif
__device__ __forceinline__ double wide_mul(double a, double b) {
#if IFGFB_WIDE_PIN
  double r;
  asm volatile("mul.rn.f64 %0, %1, %2;\n" : "=d"(r) : "d"(a), "d"(b));
  return r;
#else
  return a * b;
#endif
}

template <int KS>
__device__ __forceinline__ double wide_tst(const double* T, int tig) {
  if (KS < KMAIN) {
    const int ab = 4 * (KS / PA) + tig;
    const int ia = ab / PA, ib = ab - PA * ia;
    return wide_mul(T[ia], T[PS + ib]);
  }
  const int s = KS - KMAIN;
  return wide_mul(T[2], T[PS + 2 + (tig < 3 ? tig : (s < 3 ? s : 0))]);
}

template <int KS>
__device__ __forceinline__ double wide_av(const double* T, double tst, int tig) {
  if (KS < KMAIN) return wide_mul(tst, T[PS + PA + KS % PA]);
  const int s = KS - KMAIN;
  const double av = wide_mul(tst, T[PS + PA + (tig < 3 ? s : PA - 1)]);
  return (s == 3 && tig == 3) ? 0.0 : av;
}

// one k-step of NT row tiles: the 4 x NT DMMAs of k-step KS, each tile's A
// value for k-step KS + 1 computed right behind its DMMAs (its latency hides
// under the next tile's), the B fragments of KS + 1 loaded ahead
template <int NT, int KS>
__device__ __forceinline__ void wide_kstep(const double2* F, const double* const (&T)[NT],
                                           double (&tst)[NT], double (&av)[NT],
                                           double2& b01, double2& b23,
                                           double (&c0)[NT][4], double (&c1)[NT][4], int tig) {
  if (IFGFB_WIDE_PF > 0 && KS + IFGFB_WIDE_PF < KSTEPS) {
    prefetch_l1(F + (KS + IFGFB_WIDE_PF) * 64);
    prefetch_l1(F + (KS + IFGFB_WIDE_PF) * 64 + 32);
  }
  double2 n01 = b01, n23 = b23;
  if (KS + 1 < KSTEPS) {
    n01 = F[(KS + 1) * 64];
    n23 = F[(KS + 1) * 64 + 32];
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    dmma(c0[i][0], c1[i][0], av[i], b01.x);
    dmma(c0[i][1], c1[i][1], av[i], b01.y);
    dmma(c0[i][2], c1[i][2], av[i], b23.x);
    dmma(c0[i][3], c1[i][3], av[i], b23.y);
    if (KS + 1 < KSTEPS) {
      if ((KS + 1) % PA == 0 || KS + 1 >= KMAIN) tst[i] = wide_tst<KS + 1>(T[i], tig);
      av[i] = wide_av<KS + 1>(T[i], tst[i], tig);
    }
  }
  b01 = n01;
  b23 = n23;
  if constexpr (KS + 1 < KSTEPS)
    wide_kstep<NT, KS + 1>(F, T, tst, av, b01, b23, c0, c1, tig);
}

// NT row tiles of one sigma group against the group's child block: 19
// k-steps, per k-step one B fragment pair and 4 x NT DMMAs
template <int NT, int NK>
__device__ __forceinline__ void wide_pass(const double* __restrict__ C, const double* T0,
                                          const int (&slot)[4], int nrows,
                                          const double2* ratio, double2* mine,
                                          int lane) {
  const int grp = lane >> 2, tig = lane & 3;
  const double2* F = reinterpret_cast<const double2*>(C) + lane;
  double2 b01 = F[0], b23 = F[32];
  double c0[NT][4], c1[NT][4], tst[NT], av[NT];
  const double* T[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    T[i] = T0 + slot[i] * NT_STRIDE;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) c0[i][nt] = c1[i][nt] = 0.0;
    tst[i] = wide_tst<0>(T[i], tig);
    av[i] = wide_av<0>(T[i], tst[i], tig);
  }
#ifndef IFGFB_DIAG_NODMMA
  wide_kstep<NT, 0>(F, T, tst, av, b01, b23, c0, c1, tig);
#else
#pragma unroll
  for (int i = 0; i < NT; ++i) c0[i][0] = av[i] + b01.x + b23.y;
#endif
#ifndef IFGFB_DIAG_NOACC
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    if (8 * i + grp < nrows) {
      const double2 r0 = ratio[slot[i] * NK];
      const double2 r1 = NK > 1 ? ratio[slot[i] * NK + NK - 1] : r0;
      double2* dst = mine + slot[i] * WIDE_RS;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int m = 4 * nt + tig;
        cmul_acc(dst[m], c0[i][nt], c1[i][nt], (NK > 1 && (tig & 1)) ? r1 : r0);
      }
    }
  }
#else
  if (c0[0][0] == 1.2345e300) mine[0].x = c1[NT - 1][3];
#endif
}

template <int NK, bool WIDE, bool OTF, bool PRE = false>
__global__ void __launch_bounds__(32 * WW, IFGFB_WIDE_MINB) accum_wide_kernel(AccArgs a) {
  static_assert(!(OTF && PRE), "PRE reads tabulated node geometry");
  __shared__ double2 acc[NN * WIDE_RS];                     // 20.4 KB (padded rows)
  __shared__ WideStage stage[2];                            // 9.2 KB
  __shared__ double nodeT[NN * NT_STRIDE];                  // 7.8 KB
  __shared__ unsigned char ord[NN], inv[NN];
  __shared__ unsigned char rank2slot[WW][32];
  __shared__ unsigned char sgid[8][NN];                     // [instance][position]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2;
  const int p = a.row0 + blockIdx.x;
  if (p >= a.row_end) return;
  // warp w owns positions cuts[w] .. cuts[w+1]-1 of the signature order
  // (ifgfb_row_cuts_wide: <= 32 nodes, first WW + 1 entries of the 6-byte record)
  const int pos0 = a.row_cuts[(size_t)p * (WARP_PARTS + 1) + warp];
  const int nset = a.row_cuts[(size_t)p * (WARP_PARTS + 1) + warp + 1] - pos0;
  IFGFB_DCHECK(nset >= 1 && nset <= 32 && pos0 + nset <= NN);
  double2* mine = acc + pos0 * WIDE_RS;
  const unsigned char* word = ord + pos0;
  if (lane < nset) ord[pos0 + lane] = a.row_order[(size_t)p * NN + pos0 + lane];
  for (int i = lane; i < nset * WIDE_RS; i += 32) mine[i] = make_double2(0.0, 0.0);
  // the row's instance scalars, lane j <-> instance i0 + j (<= 8 per row)
  const int i0 = a.inst_off[p], ni = a.inst_off[p + 1] - i0;
  int my_t = 0, my_co = 0;
  if (lane < ni) my_t = a.inst_type[i0 + lane];
  if (lane <= ni) my_co = a.inst_crow_off[i0 + lane];
  __syncwarp();
  // sigma group of every owned slot under every instance of the row: the
  // (<= 8) loads of a lane are independent and complete under the first
  // instance's staging; each warp reads only what it wrote
  {
    unsigned char gv[8];
    const int node = lane < nset ? word[lane] : 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {   // all loads first, then the stores
      const int t = __shfl_sync(0xffffffffu, my_t, j);
      gv[j] = (j < ni && lane < nset) ? __ldg(a.gid + (size_t)t * NN + node) : 0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < ni && lane < nset) sgid[j][pos0 + lane] = gv[j];
  }
  auto stage_inst = [&](int j, WideStage& S) {
    const int t = __shfl_sync(0xffffffffu, my_t, j);
    const int cs = __shfl_sync(0xffffffffu, my_co, j);
    const int ce = __shfl_sync(0xffffffffu, my_co, j + 1);
    const size_t tb = PRE ? (size_t)(i0 + j - a.inst_base) * NN : (size_t)t * NN;
    if (!OTF && lane < nset) {   // one lane per owned node
      const size_t nd = tb + word[lane];
#pragma unroll
      for (int k = 0; k < 3; ++k) cp_async8(&S.geom[3 * (pos0 + lane) + k], a.node_geom + nd * 3 + k);
#pragma unroll
      for (int k = 0; k < NK; ++k) cp_async16(&S.ratio[NK * (pos0 + lane) + k], a.ratio + nd * NK + k);
    }
    if (lane < min(ce - cs, MAX_GROUPS)) cp_async4(&S.crow[warp][lane], a.crow + cs + lane);
    cp_async_commit();
  };
  if (ni > 0) stage_inst(0, stage[0]);
  __syncwarp();
  for (int j = 0; j < ni; ++j) {
    WideStage& S = stage[j & 1];
    const unsigned g_cur = lane < nset ? (unsigned)sgid[j][pos0 + lane] : 0xFFFFFFFFu;
    if (j + 1 < ni) {
      stage_inst(j + 1, stage[(j + 1) & 1]);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const int* crow_g = a.crow + __shfl_sync(0xffffffffu, my_co, j);
    if (OTF) {   // each lane: geometry of its own slot
      const int pseg = a.o.parent_seg_id[p];
      const int oct = a.o.type_octant[__shfl_sync(0xffffffffu, my_t, j)];
      if (lane < nset) {
        const int g = (int)g_cur;
        const int cr = (!WIDE || g < MAX_GROUPS) ? S.crow[warp][g] : crow_g[g];
        otf_node<NK>(a.o, pseg, oct, word[lane], a.o.child_seg_id[cr],
                     &S.geom[(pos0 + lane) * 3], &S.ratio[(pos0 + lane) * NK]);
      }
    }
    if (lane < nset) {   // Chebyshev values of the lane's node (make_basis<false>)
      const double* ng = S.geom + (pos0 + lane) * 3;
      const double xs = ng[0], xt = ng[1], xp = ng[2];
      double* T = nodeT + (pos0 + lane) * NT_STRIDE;
      double tt[PA], tp[PA];
      tt[0] = 1.0; tt[1] = xt;
      tp[0] = 1.0; tp[1] = xp;
#pragma unroll
      for (int i = 2; i < PA; ++i) {
        tt[i] = 2.0 * xt * tt[i - 1] - tt[i - 2];
        tp[i] = 2.0 * xp * tp[i - 1] - tp[i - 2];
      }
      T[0] = 1.0; T[1] = xs; T[2] = 2.0 * xs * xs - 1.0;
#pragma unroll
      for (int i = 0; i < PA; ++i) { T[PS + i] = tt[i]; T[PS + PA + i] = tp[i]; }
    }
    __syncwarp();
    unsigned g_at = __reduce_min_sync(0xffffffffu, g_cur);
    while (g_at != 0xFFFFFFFFu) {
      const unsigned mask = __ballot_sync(0xffffffffu, g_cur == g_at);
      const int nrows = __popc(mask);
      if (g_cur == g_at) rank2slot[warp][__popc(mask & ((1u << lane) - 1u))] = (unsigned char)lane;
      __syncwarp();
      const int g = (int)g_at;
      const int crow_used = (!WIDE || g < MAX_GROUPS) ? S.crow[warp][g] : crow_g[g];
      IFGFB_DCHECK(crow_used >= a.child_lo && crow_used < a.child_hi && nrows <= nset);
      const double* C = a.coef_child + (size_t)crow_used * SEG_DOUBLES;
      const double* T0 = nodeT + pos0 * NT_STRIDE;
      const double2* rt = S.ratio + pos0 * NK;
      for (int r0 = 0; r0 < nrows; r0 += 8 * WIDE_MAXNT) {   // one pass unless MAXNT < 4
        const int nr = min(nrows - r0, 8 * WIDE_MAXNT);
        int slot[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          slot[i] = rank2slot[warp][r0 + (8 * i + grp < nr ? 8 * i + grp : 0)];
        if (nr <= 8) wide_pass<1, NK>(C, T0, slot, nr, rt, mine, lane);
        else if (WIDE_MAXNT < 3 || nr <= 16) wide_pass<2, NK>(C, T0, slot, nr, rt, mine, lane);
        else if (WIDE_MAXNT < 4 || nr <= 24) wide_pass<3, NK>(C, T0, slot, nr, rt, mine, lane);
        else wide_pass<4, NK>(C, T0, slot, nr, rt, mine, lane);
      }
      __syncwarp();
      g_at = __reduce_min_sync(0xffffffffu, g_cur > g_at ? g_cur : 0xFFFFFFFFu);
    }
  }
  __syncthreads();
  if (threadIdx.x < NN) inv[ord[threadIdx.x]] = (unsigned char)threadIdx.x;
  __syncthreads();
#ifndef IFGFB_DIAG_NOK3      // diagnostic builds only (tools/ab_wide.sh): timing without a phase
  to_coeffs_smem<true, WIDE_RS>(acc, inv, threadIdx.x, 32 * WW);
#endif
#ifndef IFGFB_DIAG_NOSTORE
  if (WW == 4) store_segment128<true, WIDE_RS>(a.coef_parent + (size_t)p * SEG_DOUBLES, acc, inv, threadIdx.x);
  else store_segment<true, WIDE_RS>(a.coef_parent + (size_t)p * SEG_DOUBLES, acc, inv, threadIdx.x, 32 * WW);
#endif
}

// Node tables of an on-device-geometry level for the parent rows
// [row0, row_end): geometry and re-centering ratio of every (instance, node),
// exactly what the OTF instantiations compute per owner lane (otf_node), but
// with every lane busy and off the propagation kernel's FP64/DMMA critical
// path.  The propagation then runs its table instantiation (PRE) on the
// chunk.  One CTA per parent row (<= 8 instances x 75 nodes).
template <int NK>
__global__ void __launch_bounds__(128) otf_tables_kernel(AccArgs a, double* __restrict__ geom,
                                                         double2* __restrict__ ratio) {
  const int p = a.row0 + blockIdx.x;
  if (p >= a.row_end) return;
  const int i0 = a.inst_off[p], ni = a.inst_off[p + 1] - i0;
  const int pseg = a.o.parent_seg_id[p];
  for (int e = threadIdx.x; e < ni * NN; e += blockDim.x) {
    const int j = e / NN, node = e - j * NN;
    const int t = a.inst_type[i0 + j];
    const int oct = a.o.type_octant[t];
    const int g = a.gid[(size_t)t * NN + node];
    const int cr = a.crow[a.inst_crow_off[i0 + j] + g];
    const size_t o = (size_t)(i0 + j - a.inst_base) * NN + node;
    otf_node<NK>(a.o, pseg, oct, node, a.o.child_seg_id[cr], geom + o * 3, ratio + o * NK);
  }
}

// ------------------------------------------------- K4, ring-staged ----
// The same owner-computes propagation with the child coefficient blocks
// staged in shared memory: a producer warp streams every (instance, sigma
// group) block of the CTA's rows, in the order the owner warps consume them,
// into a ring of NSLOT 19 KB slots with one cp.async.bulk (TMA, UBLKCP) per
// block and an mbarrier per slot (full: transaction bytes landed; empty: all
// five owner warps done with it).  Each block crosses L2 -> SMEM once per
// CTA; the owner warps read their B fragments with LDS.128 instead of each
// pulling the block through L1 (round-1 ncu: L1 hit 30%, long-scoreboard the
// second stall).  CTAs are persistent (rows blockIdx.x, +gridDim.x, ...), so
// the producer fills the next row's first blocks during the K3 epilogue.
constexpr int SEG_BYTES = SEG_DOUBLES * 8;   // 19,456 B, a multiple of 16

struct __align__(16) InstStage {
  uint4 tiles[NN];          // warp w: tiles[cuts[w] ..]
  double2 ratio[NN * 2];    // [position][kappa]
  double geom[NN * 3];      // [position][xs, xt, xp]
};

template <int NSLOT>
struct __align__(128) RingSmem {
  double ring[NSLOT][SEG_DOUBLES];
  double2 acc[NN * NCOL];
  InstStage stage[2];
  unsigned long long full[NSLOT], empty[NSLOT];
  unsigned char ord[NN], inv[NN], sgrp[NN];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared (TMA), completing transaction bytes on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// Plain loads (the pointer is derived from the kernel's shared array, so
// they compile to LDS.128): unlike volatile asm they can be hoisted ahead of
// the (volatile) DMMAs, which hides the shared-memory latency; they stay
// behind the mbarrier wait, whose asm clobbers memory.
__device__ __forceinline__ double2 lds128(const double2* p) { return *p; }

// acc (+)= basis x block for a block resident in shared memory
__device__ __forceinline__ void basis_times_smem(const BasisA& B, const double* C, int lane,
                                                 double (&c0)[4], double (&c1)[4]) {
  const double2* F = reinterpret_cast<const double2*>(C) + lane;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
#pragma unroll
    for (int c = 0; c < PA; ++c) {
      const int ks = 5 * q + c;
      const double2 b01 = lds128(F + ks * 64), b23 = lds128(F + ks * 64 + 32);
      const double av = B.tst[q] * B.tp[c];
      dmma(c0[0], c1[0], av, b01.x);
      dmma(c0[1], c1[1], av, b01.y);
      dmma(c0[2], c1[2], av, b23.x);
      dmma(c0[3], c1[3], av, b23.y);
    }
  }
  const int tig = lane & 3;
#pragma unroll
  for (int st = 0; st < 4; ++st) {
    const double us = __shfl_sync(0xffffffffu, B.u, (lane & ~3) | (st < 3 ? st : 0));
    const double x = tig < 3 ? B.u : us, y = tig < 3 ? B.tp[st] : B.tp[PA - 1];
    const double av = (tig < 3 || st < 3) ? x * y : 0.0;
    const int ks = KMAIN + st;
    const double2 b01 = lds128(F + ks * 64), b23 = lds128(F + ks * 64 + 32);
    dmma(c0[0], c1[0], av, b01.x);
    dmma(c0[1], c1[1], av, b01.y);
    dmma(c0[2], c1[2], av, b23.x);
    dmma(c0[3], c1[3], av, b23.y);
  }
}

#ifndef IFGFB_RING_SLOTS
#define IFGFB_RING_SLOTS 2
#endif
#ifndef IFGFB_RING_MINB
#define IFGFB_RING_MINB 3
#endif
constexpr int RING_THREADS = 32 * (WARP_PARTS + 1);

// TILEFREE: no tile records; each warp forms its row tiles per sigma group
// from the group ids of its slots (ballot, runs of <= 8 in slot order: the
// tiles ifgfb_row_tiles_fill would have written).
template <int NK, bool OTF, int NSLOT, bool TILEFREE>
__global__ void __launch_bounds__(RING_THREADS, IFGFB_RING_MINB) accum_ring_kernel(AccArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RingSmem<NSLOT>& S = *reinterpret_cast<RingSmem<NSLOT>*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], WARP_PARTS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == WARP_PARTS) {
    // ---------------- producer: one lane streams the blocks in consumption order
    if (lane == 0) {
      uint32_t seq = 0;
      for (int p = a.row0 + blockIdx.x; p < a.row_end; p += gridDim.x) {
        const int i0 = a.inst_off[p], i1 = a.inst_off[p + 1];
        for (int i = i0; i < i1; ++i) {
          const int c0 = a.inst_crow_off[i], c1 = a.inst_crow_off[i + 1];
          for (int c = c0; c < c1; ++c, ++seq) {
            IFGFB_DCHECK(a.crow[c] >= a.child_lo && a.crow[c] < a.child_hi);
            const int slot = seq % NSLOT;
            const uint32_t use = seq / NSLOT;
            if (use > 0) mbar_wait(&S.empty[slot], (use - 1) & 1);
            mbar_expect_tx(&S.full[slot], SEG_BYTES);
            bulk_g2s(S.ring[slot], a.coef_child + (size_t)__ldg(a.crow + c) * SEG_DOUBLES,
                     SEG_BYTES, &S.full[slot]);
          }
        }
      }
    }
    return;
  }
  // ---------------- owner warps
  const int grp = lane >> 2, tig = lane & 3;
  uint32_t seq = 0;
  for (int p = a.row0 + blockIdx.x; p < a.row_end; p += gridDim.x) {
    const int pos0 = a.row_cuts[(size_t)p * (WARP_PARTS + 1) + warp];
    const int nset = a.row_cuts[(size_t)p * (WARP_PARTS + 1) + warp + 1] - pos0;
    double2* mine = S.acc + pos0 * NCOL;
    const unsigned char* word = S.ord + pos0;
    if (lane < nset) S.ord[pos0 + lane] = a.row_order[(size_t)p * NN + pos0 + lane];
    for (int i = lane; i < nset * NCOL; i += 32) mine[i] = make_double2(0.0, 0.0);
    const int i0 = a.inst_off[p], ni = a.inst_off[p + 1] - i0;
    int my_t = 0, my_ks = 0, my_ke = 0, my_co = 0;
    if (lane < ni) {
      my_t = a.inst_type[i0 + lane];
      if (!TILEFREE) {
        my_ks = a.tile_off[(i0 + lane) * WARP_PARTS + warp];
        my_ke = a.tile_off[(i0 + lane) * WARP_PARTS + warp + 1];
      }
    }
    if (lane <= ni) my_co = a.inst_crow_off[i0 + lane];
    __syncwarp();
    // TILEFREE: sigma group of the lane's slot, loaded one instance ahead
    auto slot_group = [&](int j) -> int {
      if (!TILEFREE || j >= ni) return 0xFF;            // warp-uniform
      const int t = __shfl_sync(0xffffffffu, my_t, j);  // all lanes
      return lane < nset ? (int)__ldg(a.gid + (size_t)t * NN + word[lane]) : 0xFF;
    };
    auto stage_inst = [&](int j, InstStage& T) {
      const int t = __shfl_sync(0xffffffffu, my_t, j);
      const int ks = __shfl_sync(0xffffffffu, my_ks, j);
      const int ke = __shfl_sync(0xffffffffu, my_ke, j);
      const size_t tb = (size_t)t * NN;
      if (!OTF) {
        for (int e = lane; e < nset * 3; e += 32)
          cp_async8(&T.geom[3 * pos0 + e], a.node_geom + (tb + word[e / 3]) * 3 + e % 3);
        for (int e = lane; e < nset * NK; e += 32)
          cp_async16(&T.ratio[NK * pos0 + e], a.ratio + (tb + word[e / NK]) * NK + e % NK);
      }
      if (!TILEFREE && lane < ke - ks) cp_async16(&T.tiles[pos0 + lane], a.tiles + ks + lane);
      cp_async_commit();
    };
    __syncwarp();
    int g_next = slot_group(0);
    if (ni > 0) stage_inst(0, S.stage[0]);
    for (int j = 0; j < ni; ++j) {
      InstStage& T = S.stage[j & 1];
      const int g_cur = g_next;
      if (j + 1 < ni) {
        stage_inst(j + 1, S.stage[(j + 1) & 1]);
        g_next = slot_group(j + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      const int ntile = __shfl_sync(0xffffffffu, my_ke - my_ks, j);
      const int cs = __shfl_sync(0xffffffffu, my_co, j);
      const int ng = __shfl_sync(0xffffffffu, my_co, j + 1) - cs;
      IFGFB_DCHECK(ng >= 0 && ng <= NN && nset >= 1 && nset <= MAX_SET && pos0 + nset <= NN);
      IFGFB_DCHECK(!TILEFREE || lane >= nset || g_cur < ng);
      if (OTF && TILEFREE) {
        const int pseg = a.o.parent_seg_id[p];
        const int oct = a.o.type_octant[__shfl_sync(0xffffffffu, my_t, j)];
        if (lane < nset) {
          const int cr = a.crow[cs + g_cur];
          otf_node<NK>(a.o, pseg, oct, word[lane], a.o.child_seg_id[cr],
                       &T.geom[(pos0 + lane) * 3], &T.ratio[(pos0 + lane) * NK]);
        }
        __syncwarp();
      } else if (OTF) {   // slot -> sigma group from the tile records, then geometry
        for (int e = lane; e < ntile * 8; e += 32) {
          const uint4 tl = T.tiles[pos0 + (e >> 3)];
          const int r = e & 7;
          if (r < (int)((tl.x >> 8) & 0xff)) {
            const int byte = 2 + r;
            const unsigned w = byte < 4 ? tl.x : byte < 8 ? tl.y : tl.z;
            S.sgrp[pos0 + ((w >> (8 * (byte & 3))) & 0xff)] = (unsigned char)(tl.x & 0xff);
          }
        }
        __syncwarp();
        const int pseg = a.o.parent_seg_id[p];
        const int oct = a.o.type_octant[__shfl_sync(0xffffffffu, my_t, j)];
        for (int e = lane; e < nset; e += 32) {
          const int cr = a.crow[cs + S.sgrp[pos0 + e]];
          otf_node<NK>(a.o, pseg, oct, word[e], a.o.child_seg_id[cr], &T.geom[(pos0 + e) * 3],
                       &T.ratio[(pos0 + e) * NK]);
        }
        __syncwarp();
      }
      int k = 0;
      for (int g = 0; g < ng; ++g, ++seq) {
        const int slot = seq % NSLOT;
        mbar_wait(&S.full[slot], (seq / NSLOT) & 1);
        const double* blk = S.ring[slot];
        unsigned mask = TILEFREE ? __ballot_sync(0xffffffffu, g_cur == g) : 0u;
        for (;;) {
          bool valid;
          int slot_n;
          if (TILEFREE) {
            if (!mask) break;
            // tile row grp = the grp-th owned slot of group g (slot order)
            unsigned m = mask;
            for (int i = 0; i < grp; ++i) m &= m - 1;
            valid = m != 0u;
            slot_n = valid ? __ffs(m) - 1 : __ffs(mask) - 1;
            if (__popc(mask) > 8) {
              for (int i = 0; i < 8; ++i) mask &= mask - 1;
            } else {
              mask = 0u;
            }
          } else {
            if (k >= ntile) break;
            const uint4 tl = T.tiles[pos0 + k];
            if ((int)(tl.x & 0xff) != g) break;
            slot_n = tile_slot(tl, grp, valid);
            ++k;
          }
          IFGFB_DCHECK(slot_n >= 0 && slot_n < nset);
          const double* ng3 = T.geom + (pos0 + slot_n) * 3;
          const BasisA B = make_basis<false>(ng3[0], ng3[1], ng3[2], tig);
          double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
          basis_times_smem(B, blk, lane, c0, c1);
          if (valid) {
            const double2 r0 = T.ratio[(pos0 + slot_n) * NK];
            const double2 r1 = NK > 1 ? T.ratio[(pos0 + slot_n) * NK + NK - 1] : r0;
            double2* dst = mine + slot_n * NCOL;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              const int m = 4 * nt + tig;
              cmul_acc(dst[m], c0[nt], c1[nt], (NK > 1 && (tig & 1)) ? r1 : r0);
            }
          }
          __syncwarp();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[slot]);
      }
    }
    k3_sync<true>();
    if (threadIdx.x < NN) S.inv[S.ord[threadIdx.x]] = (unsigned char)threadIdx.x;
    k3_sync<true>();
    to_coeffs_smem<true, NCOL, true>(S.acc, S.inv, threadIdx.x, 32 * WARP_PARTS);
    store_segment<true>(a.coef_parent + (size_t)p * SEG_DOUBLES, S.acc, S.inv, threadIdx.x,
                        32 * WARP_PARTS);
    k3_sync<true>();
  }
}

template <int NK, bool OTF, bool TILEFREE>
static int launch_ring(const AccArgs& aa, int nrows, cudaStream_t st) {
  constexpr int NS = IFGFB_RING_SLOTS;
  auto kern = accum_ring_kernel<NK, OTF, NS, TILEFREE>;
  const int smem = (int)sizeof(RingSmem<NS>);
  static bool attr = false;
  static int per_sm = 0, n_sm = 0;
  if (!attr) {
    IFGFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    IFGFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RING_THREADS, smem));
    int dev = 0;
    IFGFB_CUDA(cudaGetDevice(&dev));
    IFGFB_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    attr = true;
  }
  const int grid = std::max(1, std::min(nrows, std::max(1, per_sm) * n_sm));
  kern<<<grid, RING_THREADS, smem, st>>>(aa);
  return IFGFB_OK;
}

// ---------------------------------------------------------------- K5 ----
struct EmitArgs {
  const int4* tiles; int tile0, tile_end;
  const int* pair_id; const double4* geom; const double4* geom_disp;
  const double* coef;
  double kr[2], ki[2];
  double2* partial;   // [pair][2][NCOL]
};

// One warp per tile of <= 4 (box, target) pairs sharing a segment row; the 8
// MMA rows are (pair, point) with point 0 = x_t, 1 = x_t + h n_t (same
// segment polynomial, reference ifgf.py:647-653).  The basis is formed
// exactly as numpy does ((T_a T_b) T_c, unfused recurrences).  A bitwise
// replica of the reference's contraction order (sequential FMA chain, as
// OpenBLAS evaluates these dgemm shapes) was measured 3x slower and does not
// tighten D_far parity: D_far = (S(x+hn) - S(x))/h is a chaotic function of
// the last bits of the coefficients themselves.
template <int NK>
__global__ void __launch_bounds__(128) emit_kernel(EmitArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = a.tile0 + blockIdx.x * 4 + warp;
  if (tile >= a.tile_end) return;
  const int grp = lane >> 2, tig = lane & 3;
  const int4 td = a.tiles[tile];
  const int pp = grp >> 1, pt = grp & 1;
  const bool has_disp = a.geom_disp != nullptr;
  const bool valid = pp < td.z && (pt == 0 || has_disp);
  const int pos = td.y + min(pp, td.z - 1);
  const double4 gm = (pt && has_disp) ? a.geom_disp[pos] : a.geom[pos];
  const BasisA B = make_basis<true>(gm.x, gm.y, gm.z, tig);
  double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
  basis_times_block<true>(B, a.coef + (size_t)td.x * SEG_DOUBLES, lane, c0, c1);
  if (!valid) return;
  const double r = gm.w;
  // G_k = exp(i kappa r) / (4 pi r); numpy divides a complex by a real as a
  // multiplication by the reciprocal (ifgf.py:660-663)
  const double rec = 1.0 / mul_rn(4.0 * M_PI, r);
  double2 gk[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const double2 e = cexp_ikx(a.kr[k], a.ki[k], r);
    gk[k] = make_double2(mul_rn(e.x, rec), mul_rn(e.y, rec));
  }
  double2* dst = a.partial + ((size_t)a.pair_id[pos] * 2 + pt) * NCOL;
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    const int m = 4 * nt + tig;
    dst[m] = cmul(make_double2(c0[nt], c1[nt]),
                  (NK > 1 && (tig & 1)) ? gk[NK - 1] : gk[0]);
  }
}

// out_tree[t][m] += sum of t's pair partials in box order (reference
// per-box scatter-add, ifgf.py:664-673; levels D..3 in turn).
__global__ void emit_reduce(int n, int pair_lo, int pair_hi,
                            const int* __restrict__ tgt_off,
                            const int* __restrict__ tgt_pairs,
                            const double2* __restrict__ partial,
                            double2* __restrict__ out,
                            double2* __restrict__ out_disp) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * NCOL) return;
  const int t = idx / NCOL, m = idx % NCOL;
  int q0 = tgt_off[t], q1 = tgt_off[t + 1];
  if (q0 == q1) return;
  // a target's pairs are in box (= pair index) order, so the pairs of the
  // active range [pair_lo, pair_hi) (a streaming part) are one contiguous run
  // of its list: binary search both ends instead of scanning every pair
  // once per part
  if (tgt_pairs[q0] < pair_lo || tgt_pairs[q1 - 1] >= pair_hi) {
    int lo = q0, hi = q1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (tgt_pairs[mid] < pair_lo) lo = mid + 1; else hi = mid;
    }
    int lo2 = lo, hi2 = q1;
    while (lo2 < hi2) {
      const int mid = (lo2 + hi2) >> 1;
      if (tgt_pairs[mid] < pair_hi) lo2 = mid + 1; else hi2 = mid;
    }
    q0 = lo;
    q1 = lo2;
    if (q0 == q1) return;
  }
  double2 s = out[idx];
  double2 sd = out_disp ? out_disp[idx] : make_double2(0.0, 0.0);
  for (int q = q0; q < q1; ++q) {
    const int pq = tgt_pairs[q];
    const size_t pr = pq;
    const double2 v = partial[(pr * 2) * NCOL + m];
    s.x += v.x;
    s.y += v.y;
    if (out_disp) {
      const double2 vd = partial[(pr * 2 + 1) * NCOL + m];
      sd.x += vd.x;
      sd.y += vd.y;
    }
  }
  out[idx] = s;
  if (out_disp) out_disp[idx] = sd;
}

// out[(c*nk + k)][ell] = out_tree[iperm[ell]][c*NK + k]  (original order);
// pm_stride > 0: point-major out[ell * pm_stride + m] (rank exchange rows)
__global__ void unpermute(int n, int ncols, const int* __restrict__ perm,
                          const double2* __restrict__ src,
                          double2* __restrict__ dst, int pm_stride) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * ncols) return;
  const int t = idx / ncols, m = idx % ncols;
  const size_t o = pm_stride ? (size_t)perm[t] * pm_stride + m : (size_t)m * n + perm[t];
  dst[o] = src[(size_t)t * NCOL + m];
}

// ------------------------------------------------------------ driver -----
// Streaming: make part `part` the active per-level row / pair / tile ranges.
static void apply_stream_part(Plan& p, int part) {
  for (int d = 3; d <= p.depth; ++d) {
    const StreamRange& r = p.stream_parts[part][d];
    Level& L = p.levels[d];
    L.part_seg_lo = r.seg_lo;
    L.part_seg_hi = r.seg_hi;
    L.part_pair_lo = r.pair_lo;
    L.part_pair_hi = r.pair_hi;
    L.part_tile_lo = r.tile_lo;
    L.part_tile_hi = r.tile_hi;
  }
}

int ensure_coef(Plan& p);

// Emission overlap (Plan::overlap_emit, opt-in: env IFGFB_OVERLAP_EMIT=1).
// Measured at (4,10): 26.27 -> 26.10 ms per matvec (0.7%); off by default
// because per-kernel event times of the overlapped emission then include
// the time its CTAs wait for SMs held by the propagation.
// level d's emission reads only level d's coefficients, so it runs on the
// plan's aux stream while the apply stream propagates d -> d-1.  The
// propagation that overwrites level d's ping-pong buffer (d-1 -> d-2, or
// the next streaming part's leaf) first waits for that emission.
struct EmitSync {
  Plan& p;
  cudaStream_t st;
  size_t next = 0;
  bool on;
  EmitSync(Plan& p_, cudaStream_t st_) : p(p_), st(st_), on(p_.overlap_emit && p_.aux) {}
  cudaEvent_t ev() {
    if (next == p.sync_events.size()) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      p.sync_events.push_back(e);
    }
    return p.sync_events[next++];
  }
  // aux waits for everything issued so far on st
  void fork() {
    if (!on) return;
    cudaEvent_t e = ev();
    cudaEventRecord(e, st);
    cudaStreamWaitEvent(p.aux, e, 0);
  }
  // st waits for everything issued so far on aux
  void join() {
    if (!on) return;
    cudaEvent_t e = ev();
    cudaEventRecord(e, p.aux);
    cudaStreamWaitEvent(st, e, 0);
  }
  cudaStream_t emit_stream() const { return on ? p.aux : st; }
};

// K4 implementation (env IFGFB_K4, see engine.k4_mode): the L1-streaming
// kernel (default "l1free" / "l1") or the ring-staged kernel ("ringfree" /
// "ring": measured 45% slower, DESIGN 4); "...free" plans hold no tile
// records (the host side decides, plan time)
static bool use_ring() {
  static const bool ring = [] {
    const char* v = std::getenv("IFGFB_K4");
    return v && v[0] == 'r';
  }();
  return ring;
}

static int ensure_aux(Plan& p) {
  static const bool env_on = [] {
    const char* v = std::getenv("IFGFB_OVERLAP_EMIT");
    return v && v[0] == '1';
  }();
  p.overlap_emit = env_on;
  if (p.overlap_emit && !p.aux)
    IFGFB_CUDA(cudaStreamCreateWithFlags(&p.aux, cudaStreamNonBlocking));
  return IFGFB_OK;
}

// Scratch for the node-table pre-pass of on-device-geometry levels
// (otf_tables_kernel): IFGFB_OTF_PRE_MB MiB (default 4096, 0 = off: geometry
// inside the propagation kernel), at most a quarter of the free device
// memory.  Returns false when the pre-pass is off or the scratch does not fit.
static bool ensure_otf_tables(Plan& p) {
  if (p.otf_cap != 0) return p.otf_cap > 0;
  p.otf_cap = -1;
  const char* v = std::getenv("IFGFB_OTF_PRE_MB");
  size_t want = (size_t)(v ? std::max(0L, std::atol(v)) : 4096L) << 20;
  size_t free_b = 0, total_b = 0;
  if (want == 0 || cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return false;
  want = std::min(want, free_b / 4);
  const size_t per_inst = (size_t)NN * (3 + 4) * sizeof(double);
  // at least a few thousand rows per chunk, or the launches stop filling the GPU
  int64_t cap = (int64_t)(want / per_inst);
  if (cap < 65536) return false;
  int64_t most = 0;   // no more than the largest on-device-geometry level needs
  for (const Level& L : p.levels)
    if (L.otf) most = std::max(most, L.n_instances);
  cap = std::min(cap, std::max<int64_t>(most, 31));
  // tests: capacity in instances (>= 31, the most one row can hold), to
  // force several chunks on small plans
  if (const char* ci = std::getenv("IFGFB_OTF_PRE_INST")) cap = std::max(31L, std::atol(ci));
  if (dev_alloc(p, &p.otf_geom, (size_t)cap * NN * 3) != IFGFB_OK ||
      dev_alloc(p, &p.otf_ratio, (size_t)cap * NN * 4) != IFGFB_OK) {
    cudaGetLastError();
    return false;
  }
  p.otf_cap = cap;
  return true;
}

template <int NK>
static int far_apply_t(Plan& p, const double* w, int nch, const double* kap,
                       double* out, double* out_disp, cudaStream_t st, int pm_stride) {
  if (p.coef_cap == 0) IFGFB_RC(ensure_coef(p));
  IFGFB_RC(ensure_aux(p));
  EmitSync sync(p, st);
  constexpr int CH = NCOL / NK;
  const int n = p.n;
  const int threads = 256;
  int64_t launches = 0;
  pack_weights<<<(n * CH + threads - 1) / threads, threads, 0, st>>>(
      reinterpret_cast<const double2*>(w), nch, n, p.perm, CH,
      reinterpret_cast<double2*>(p.wt));
  ++launches;
  IFGFB_CUDA(cudaMemsetAsync(p.out_tree, 0, sizeof(double2) * n * NCOL, st));
  if (out_disp)
    IFGFB_CUDA(cudaMemsetAsync(p.out_disp_tree, 0, sizeof(double2) * n * NCOL, st));
  double kr[2] = {kap[0], NK > 1 ? kap[2] : 0.0};
  double ki[2] = {kap[1], NK > 1 ? kap[3] : 0.0};
  const int D = p.depth;
  if (D >= 3) {
    // re-centering ratios, once per apply and level (kappa dependent)
    for (int d = 4; d <= D; ++d) {
      Level& L = p.levels[d];
      if (!L.has_accum || L.otf) continue;
      const int64_t nr = L.n_types * NN;
      const int tk = p.timer.begin(K_OTHER, st);
      ratio_kernel<NK><<<(unsigned)((nr + 255) / 256), 256, 0, st>>>(
          nr, L.node_r, kr[0], ki[0], kr[1], ki[1], reinterpret_cast<double2*>(L.ratio));
      p.timer.end(tk, st);
      ++launches;
    }
    // one pass over the owned subtrees, or (streaming) one pass per group of
    // Morton-contiguous level-3 subtrees, accumulating into out_tree
    const int n_parts = p.stream_parts.empty() ? 1 : (int)p.stream_parts.size();
    for (int part = 0; part < n_parts; ++part) {
      if (!p.stream_parts.empty()) apply_stream_part(p, part);
      int cur = 0;
      {
        Level& L = p.levels[D];
        LeafArgs la{L.seg_box, L.seg_id, L.centers, L.pt_start, L.pt_count, L.tabs,
                    L.n_s, L.n_a, L.h, p.points_tree,
                    reinterpret_cast<const double2*>(p.wt), {kr[0], kr[1]},
                    {ki[0], ki[1]}, p.coef[cur] - (size_t)L.seg_lo() * SEG_DOUBLES,
                    L.seg_lo()};
        if (L.seg_hi() > L.seg_lo()) {
          const int tk = p.timer.begin(K_LEAF, st);
          leaf_kernel<NK><<<L.seg_hi() - L.seg_lo(), leaf_threads<NK>(), 0, st>>>(la);
          p.timer.end(tk, st);
          ++launches;
        }
      }
      cudaEvent_t prev_done = nullptr;   // emission of level d + 1 finished
      for (int d = D; d >= 3; --d) {
        Level& L = p.levels[d];
        // level d's coefficients (coef[cur]) are complete on st
        sync.fork();
        const cudaStream_t est = sync.emit_stream();
        if (L.tile_hi() > L.tile_lo()) {
          EmitArgs ea{L.etiles, L.tile_lo(), L.tile_hi(), L.pair_id, L.geom,
                      out_disp ? L.geom_disp : nullptr,
                      p.coef[cur] - (size_t)L.seg_lo() * SEG_DOUBLES,
                      {kr[0], kr[1]}, {ki[0], ki[1]},
                      reinterpret_cast<double2*>(p.partial)};
          int tk = p.timer.begin(K_EMIT, est);
          emit_kernel<NK><<<(L.tile_hi() - L.tile_lo() + 3) / 4, 128, 0, est>>>(ea);
          p.timer.end(tk, est);
          tk = p.timer.begin(K_REDUCE, est);
          emit_reduce<<<(n * NCOL + threads - 1) / threads, threads, 0, est>>>(
              n, L.pair_lo(), L.pair_hi(), L.tgt_off, L.tgt_pairs,
              reinterpret_cast<const double2*>(p.partial),
              reinterpret_cast<double2*>(p.out_tree),
              out_disp ? reinterpret_cast<double2*>(p.out_disp_tree) : nullptr);
          p.timer.end(tk, est);
          launches += 2;
        }
        // the propagation below overwrites coef[cur ^ 1], which holds level
        // d + 1: wait for level d + 1's emission first
        cudaEvent_t done_d = nullptr;
        if (sync.on) {
          done_d = sync.ev();
          cudaEventRecord(done_d, p.aux);
          if (prev_done) cudaStreamWaitEvent(st, prev_done, 0);
          prev_done = done_d;
        }
        if (d > 3 && L.has_accum) {
          Level& U = p.levels[d - 1];
          if (U.seg_hi() > U.seg_lo()) {
            AccArgs aa{L.inst_off, L.inst_type, L.inst_crow_off, L.crow, L.tile_off,
                       L.tiles, L.row_order, L.row_cuts, L.node_geom,
                       reinterpret_cast<const double2*>(L.ratio),
                       p.coef[cur] - (size_t)L.seg_lo() * SEG_DOUBLES,
                       p.coef[cur ^ 1] - (size_t)U.seg_lo() * SEG_DOUBLES, U.seg_lo()};
            aa.row_end = U.seg_hi();
            aa.rows_per_cta = IFGFB_ACC_ROWS;
            aa.child_lo = L.seg_lo();
            aa.child_hi = L.seg_hi();
            const int nrows = U.seg_hi() - U.seg_lo();
            const int tk = p.timer.begin(K_ACCUM, st, d);
            const int grid = (nrows + IFGFB_ACC_ROWS - 1) / IFGFB_ACC_ROWS;
            const bool wide = L.max_groups > MAX_GROUPS;
            if (L.otf)
              aa.o = OtfGeom{L.type_octant, U.seg_id, U.tabs, U.n_s, U.n_a, U.h, L.seg_id,
                             L.n_a, L.delta_s, L.delta_a, L.side, {kr[0], kr[1]}, {ki[0], ki[1]}};
            aa.gid = L.gid;
            const bool tf = L.tiles == nullptr;   // tile-free plan
            const dim3 blk(32 * WARP_PARTS);
            if (tf && WW != WARP_PARTS && L.cut_warps == WW) {
              // the level's rows were cut for the wide-warp kernel
              // (ifgfb_row_cuts_wide; the plan builder decides per level)
              const dim3 wblk(32 * WW);
              if (L.otf && ensure_otf_tables(p)) {
                // node tables of a chunk of rows, then its propagation from them
                const std::vector<int>& io = L.h_inst_off;
                AccArgs ab = aa;
                ab.node_geom = p.otf_geom;
                ab.ratio = reinterpret_cast<const double2*>(p.otf_ratio);
                for (int r0 = U.seg_lo(); r0 < U.seg_hi();) {
                  const int64_t lim = (int64_t)io[r0] + p.otf_cap;
                  int r1 = (int)(std::upper_bound(io.begin() + r0 + 1, io.begin() + U.seg_hi() + 1,
                                                  lim, [](int64_t v, int x) { return v < x; })
                                 - io.begin()) - 1;
                  r1 = std::min(std::max(r1, r0 + 1), U.seg_hi());
                  ab.row0 = r0;
                  ab.row_end = r1;
                  ab.inst_base = io[r0];
                  otf_tables_kernel<NK><<<r1 - r0, 128, 0, st>>>(
                      ab, p.otf_geom, reinterpret_cast<double2*>(p.otf_ratio));
                  if (wide) accum_wide_kernel<NK, true, false, true><<<r1 - r0, wblk, 0, st>>>(ab);
                  else accum_wide_kernel<NK, false, false, true><<<r1 - r0, wblk, 0, st>>>(ab);
                  launches += 2;
                  r0 = r1;
                }
                --launches;   // the common ++launches below
              } else if (L.otf) {
                if (wide) accum_wide_kernel<NK, true, true><<<nrows, wblk, 0, st>>>(aa);
                else accum_wide_kernel<NK, false, true><<<nrows, wblk, 0, st>>>(aa);
              } else {
                if (wide) accum_wide_kernel<NK, true, false><<<nrows, wblk, 0, st>>>(aa);
                else accum_wide_kernel<NK, false, false><<<nrows, wblk, 0, st>>>(aa);
              }
            } else if (L.cut_warps != WARP_PARTS || L.cut_max_set > MAX_SET) {
              set_error("the 5-warp propagation kernels need 5 row sets of <= 23 nodes "
                        "(this plan was cut for IFGFB_K4=wide)");
              return IFGFB_ERR_STATE;
            } else if (use_ring()) {
              if (L.otf) IFGFB_RC(tf ? (launch_ring<NK, true, true>(aa, nrows, st))
                                     : (launch_ring<NK, true, false>(aa, nrows, st)));
              else IFGFB_RC(tf ? (launch_ring<NK, false, true>(aa, nrows, st))
                               : (launch_ring<NK, false, false>(aa, nrows, st)));
            } else if (tf) {
              if (L.otf) {
                if (wide) accum_kernel<NK, true, true, true><<<grid, blk, 0, st>>>(aa);
                else accum_kernel<NK, false, true, true><<<grid, blk, 0, st>>>(aa);
              } else {
                if (wide) accum_kernel<NK, true, false, true><<<grid, blk, 0, st>>>(aa);
                else accum_kernel<NK, false, false, true><<<grid, blk, 0, st>>>(aa);
              }
            } else if (L.otf) {
              if (wide) accum_kernel<NK, true, true><<<grid, blk, 0, st>>>(aa);
              else accum_kernel<NK, false, true><<<grid, blk, 0, st>>>(aa);
            } else {
              if (wide) accum_kernel<NK, true, false><<<grid, blk, 0, st>>>(aa);
              else accum_kernel<NK, false, false><<<grid, blk, 0, st>>>(aa);
            }
            p.timer.end(tk, st);
            ++launches;
          }
          cur ^= 1;
        }
      }
      // the next part's leaf overwrites coef[0]; unpermute reads out_tree
      sync.join();
    }
  }
  const int ncols = nch * NK;
  unpermute<<<(n * ncols + threads - 1) / threads, threads, 0, st>>>(
      n, ncols, p.perm, reinterpret_cast<const double2*>(p.out_tree),
      reinterpret_cast<double2*>(out), pm_stride);
  ++launches;
  if (out_disp) {
    unpermute<<<(n * ncols + threads - 1) / threads, threads, 0, st>>>(
        n, ncols, p.perm, reinterpret_cast<const double2*>(p.out_disp_tree),
        reinterpret_cast<double2*>(out_disp), pm_stride);
    ++launches;
  }
  IFGFB_CUDA(cudaGetLastError());
  p.launches += launches;
  return IFGFB_OK;
}

int far_setup_kernels() { return init_constants(); }

int far_apply(Plan& p, const double* w, int nch, const double* kappas, int nk,
              double* out, double* out_disp, cudaStream_t st, int pm_stride) {
  if (nk == 1) {
    if (nch < 1 || nch > NCOL) { set_error("far_apply: 1 <= nch <= 16 for nk=1"); return IFGFB_ERR_ARG; }
    return far_apply_t<1>(p, w, nch, kappas, out, out_disp, st, pm_stride);
  }
  if (nk == 2) {
    if (nch < 1 || nch > NCOL / 2) { set_error("far_apply: 1 <= nch <= 8 for nk=2"); return IFGFB_ERR_ARG; }
    return far_apply_t<2>(p, w, nch, kappas, out, out_disp, st, pm_stride);
  }
  set_error("far_apply: nk must be 1 or 2");
  return IFGFB_ERR_ARG;
}

}  // namespace ifgfb

extern "C" int ifgfb_wide_warps(void) { return ifgfb::WW; }
