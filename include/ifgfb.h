/*
 * ifgfb.h -- C ABI of the B200-native IFGF N-Muller matvec (libifgfb200.so).
 *
 * Drop-in boundary for the hot path of arXiv 2408.02274's reference
 * (`emscat`, pure Python).  The reference has no FFI; each entry point below
 * replaces one Python function of its operator API, cited as file:line
 * (paths under the reference's pkg/src/emscat/):
 *
 *   ifgfb_far_apply      <- ifgf.py:885-923        ifgf_apply(tree, hier, weights,
 *                                                   kappas, mode, displaced_normals,
 *                                                   displaced_step)
 *   ifgfb_potentials     <- operators.py:321-350   MullerOperator.potentials(dens)
 *   ifgfb_muller_apply   <- operators.py:399-403   MullerOperator.apply(y)
 *   ifgfb_muller_apply_host  same, host buffers in/out (copies inside)
 *   ifgfb_zdotc/ifgfb_zaxpy/ifgfb_dznrm2/ifgfb_zscal
 *                        <- solver.py:61-66         GMRES vector ops (np.vdot, axpy,
 *                                                   np.linalg.norm, w/h)
 *
 * Plan construction (reference ifgf.py:176-482, ifgf.py:676-749,
 * quadrature.py:97-525, all plan-time) is done on the host by the Python
 * package; its arrays are handed over ONCE through the ifgfb_plan_* calls
 * (host pointers, copied to device memory owned by the plan).
 *
 * Conventions
 *  - complex128 values are interleaved (re, im) doubles ("double2").
 *  - "tree order" = the octree's Morton order (reference BoxTree.perm);
 *    "original order" = surface point order ell = j + n_c*i + p*n_c^2.
 *  - every function returns IFGFB_OK (0) or a negative error code; the
 *    message is available from ifgfb_last_error() (thread-local).
 *  - device pointers are raw CUDA global-memory pointers (e.g. a torch
 *    tensor's data_ptr()); `stream` is a cudaStream_t (NULL = legacy default).
 *  - a plan is bound to the device current at ifgfb_plan_create; it is not
 *    re-entrant (one apply at a time per plan), plans are independent.
 *  - there is no CPU fallback: without a usable sm_100 device every compute
 *    entry point fails with IFGFB_ERR_CUDA.
 */
#ifndef IFGFB_H
#define IFGFB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IFGFB_ABI_VERSION 8

enum {
  IFGFB_OK = 0,
  IFGFB_ERR_ARG = -1,      /* bad argument / shape (Python: ValueError)     */
  IFGFB_ERR_CUDA = -2,     /* CUDA failure (Python: RuntimeError)           */
  IFGFB_ERR_STATE = -3,    /* plan incomplete or used out of order          */
  IFGFB_ERR_UNSUPPORTED = -4
};

typedef struct ifgfb_plan ifgfb_plan;

/* ---- global geometry of the IFGF tree (reference BoxTree, ifgf.py:139-173) */
typedef struct {
  int32_t n_points;          /* N */
  int32_t depth;             /* D; levels 3..D carry cone segments */
  int32_t p_s, p_a;          /* interpolation orders (only 3, 5 compiled) */
  const double* points_tree; /* N*3, tree order (BoxTree.points) */
  const int64_t* perm;       /* N: tree slot -> original index (BoxTree.perm) */
} ifgfb_tree_desc;

/* ---- one cone level d (reference LevelBoxes + ConeLevel, ifgf.py:109-126,
 *      ifgf.py:324-387).  Node tables are the per-cell Chebyshev nodes and
 *      their sin/cos (host-evaluated, so node positions match the reference). */
typedef struct {
  int32_t level;
  int32_t n_boxes;
  int32_t n_s, n_a;
  double side, h, delta_s, delta_a;
  const double* centers;     /* n_boxes*3 */
  const int64_t* pt_start;   /* n_boxes, tree-order point ranges */
  const int64_t* pt_count;   /* n_boxes */
  int64_t n_segments;
  const int64_t* seg_off;    /* n_boxes+1 (ConeLevel.seg_off) */
  const int64_t* seg_ids;    /* n_segments (ConeLevel.seg_ids) */
  const double* s_nodes;     /* n_s*p_s    (ConeLevel.s_nodes) */
  const double* sin_t;       /* n_a*p_a    sin(ang_nodes_t) */
  const double* cos_t;       /* n_a*p_a    cos(ang_nodes_t) */
  const double* sin_p;       /* 2n_a*p_a   sin(ang_nodes_p) */
  const double* cos_p;       /* 2n_a*p_a   cos(ang_nodes_p) */
} ifgfb_level_desc;

/* ---- emission pairs of level d (reference _emit_level, ifgf.py:630-673):
 *      one entry per (box, cousin point), box-major as ConeLevel.cpt_idx. */
typedef struct {
  int32_t level;
  int64_t n_pairs;
  const int64_t* row;        /* segment row of the pair */
  const int64_t* target;     /* target point, tree order */
  const double* geom;        /* n_pairs*4: xs, xt, xp, r   of x_t */
  const double* geom_disp;   /* n_pairs*4 of x_t + h n_t, or NULL */
} ifgfb_emit_desc;

/* ---- propagation child level d -> parent level d-1 (reference _AccumType /
 *      _accum_types / _accumulate_level, ifgf.py:676-785), regrouped per
 *      parent segment row (owner computes).  Each CTA owns one parent
 *      segment row; its 75 nodes, in row_order, are split into 5 contiguous
 *      warp-owned sets (warp w owns positions row_cuts[w] .. row_cuts[w+1]-1,
 *      at most 23 nodes).  Per (instance, warp) the owned nodes are grouped
 *      by child segment into MMA row tiles of <= 8 nodes.  row_order,
 *      row_cuts, tile_off and tiles are what ifgfb_row_tiles_plan/_fill
 *      produce. */
typedef struct {
  int32_t level;             /* child level d */
  int64_t n_types;
  const double* node_geom;   /* n_types*75*3: xs, xt, xp of each parent node
                                in its child segment (parent node order) */
  const double* node_r;      /* n_types*75*2: r_parent, r_child */
  int64_t n_parent_rows;     /* segments of level d-1 */
  const uint8_t* row_order;  /* n_parent_rows*75 */
  const uint8_t* row_cuts;   /* n_parent_rows*6: 0 = c0 < c1 < ... < c5 = 75 */
  const int64_t* inst_off;   /* n_parent_rows+1 */
  int64_t n_instances;
  const int64_t* inst_type;  /* n_instances */
  const int64_t* inst_crow_off; /* n_instances+1 into crow */
  const int64_t* crow;       /* child segment row per sigma group */
  const int64_t* tile_off;   /* n_instances*5+1: tiles of (instance, warp) */
  int64_t n_tiles;
  const uint8_t* tiles;      /* n_tiles*16: [local sigma group, n_rows,
                                slot0..slot7 (position in the warp's set,
                                0xFF pad), 6 pad] */
  int32_t geometry_on_device;/* 1: node_geom / node_r unused (may be NULL);
                                the kernel recomputes each node's local
                                coordinates and radii from the parent
                                segment, node and child octant (memory-lean
                                coarse levels of large configurations) */
  const uint8_t* type_octant;/* n_types: child octant of each type (used
                                when geometry_on_device) */
  const uint8_t* group_id;   /* n_types*75: sigma group (index into the
                                instance's crow list) of each parent node,
                                or NULL.  Given group_id, tile_off / tiles
                                may be NULL (n_tiles 0): the ring-staged
                                kernel forms each warp's row tiles on the fly
                                (same tiles as ifgfb_row_tiles_fill) and the
                                plan holds no tile records */
} ifgfb_accum_desc;

/* ---- surface + operator data (reference SurfaceDiscretization,
 *      geometry.py:128-184; MaterialPair operators.py:58-101) */
typedef struct {
  int32_t n_patches, n_c;
  const double* points;      /* N*3 original order */
  const double* normals;     /* N*3 */
  const double* weights;     /* N   (Fejer x Jacobian) */
  const double* jacobians;   /* N */
  const double* e_u;         /* N*3 */
  const double* e_v;         /* N*3 */
  const double* tangent1;    /* N*3 */
  const double* tangent2;    /* N*3 */
  const double* diff_matrix; /* n_c*n_c (chebyshev.diff_matrix) */
  const double* coeff_matrix;/* n_c*n_c (chebyshev.transform_matrix) */
  const double* eps_e; const double* mu_e;  /* complex (2 doubles each) */
  const double* eps_i; const double* mu_i;
  double omega;
  const double* kappas;      /* 2 complex: kappa_e, kappa_i */
  double fd_step;            /* OperatorConfig.fd_step */
} ifgfb_surface_desc;

/* ---- near field (reference quadrature.py:251-525, operators.py:255-319):
 *      per target (original order) its singular-moment pairs and one signed
 *      direct-interaction list (+ neighbour-box sources off the singular
 *      patches, - correction sources). */
typedef struct {
  int64_t n_mom;
  const int64_t* mom_off;    /* N+1 */
  const int64_t* mom_patch;  /* n_mom */
  const double* moments;     /* n_mom*4*n_c*n_c complex: beta_s[k=0,1], beta_d[k=0,1] */
  int64_t n_direct;
  const int64_t* dir_off;    /* N+1 */
  const int64_t* dir_src;    /* n_direct: source index (original order), or
                                -(src+1) for a subtracted correction entry */
} ifgfb_near_desc;

int ifgfb_abi_version(void);
const char* ifgfb_last_error(void);
int ifgfb_device_info(char* buf, size_t len);

/* Plan-time owner partition and MMA row tiles of one propagation level
 * (host only; octree.row_tiles; csrc/tiles.cpp).  Inputs are the
 * accumulation plan regrouped per parent row (reference _accum_types,
 * ifgf.py:705-749): inst_off (n_rows+1), inst_type (instances), group_id
 * (n_types*75: sigma group of each parent node under the type, < 75).
 * _plan writes row_order (n_rows*75), row_cuts (n_rows*6) and tile_off
 * (n_instances*5+1; tile_off[n_instances*5] = number of tiles);
 * cut_radius 0..4 (0 = equal sets of 15).  _fill then writes the 16-byte
 * tile records.  n_threads <= 0: all hardware threads. */
int ifgfb_row_tiles_plan(int64_t n_rows, const int64_t* inst_off,
                         const int64_t* inst_type, int64_t n_types,
                         const uint8_t* group_id, uint8_t* row_order,
                         uint8_t* row_cuts, int64_t* tile_off,
                         int32_t cut_radius, int32_t n_threads);
/* Wide-warp propagation kernel (IFGFB_K4=wide): the same signature order,
 * cut into n_warps (= ifgfb_wide_warps()) contiguous sets of <= 32 nodes,
 * cut k within +-cut_radius (<= 8) of 75k/n_warps, minimising
 * balance_weight * n_warps * (largest per-warp tile count) + total_weight *
 * (the row's tile count).  row_cuts keeps the 6-byte record per row:
 * entries 0..n_warps are the cuts, the rest 75. */
int ifgfb_row_cuts_wide(int64_t n_rows, const int64_t* inst_off,
                        const int64_t* inst_type, int64_t n_types,
                        const uint8_t* group_id, uint8_t* row_order,
                        uint8_t* row_cuts, int32_t n_warps, int32_t cut_radius,
                        int32_t total_weight, int32_t balance_weight,
                        int32_t n_threads);
/* owner warps per parent row the wide propagation kernel was built with */
int ifgfb_wide_warps(void);
int ifgfb_row_tiles_fill(int64_t n_rows, const int64_t* inst_off,
                         const int64_t* inst_type, int64_t n_types,
                         const uint8_t* group_id, const uint8_t* row_order,
                         const uint8_t* row_cuts, const int64_t* tile_off,
                         uint8_t* tiles, int32_t n_threads);

/* Plan-time singular moments on the device (reference quadrature.py:271-331,
 * compute_moments; graded clustered grid quadrature.py:163-228).  For each
 * (target, singular patch) pair i: target point / normal (3 doubles each),
 * patch index, closest (u0, v0).  patch_coeffs holds per patch 9 tensor
 * Chebyshev coefficient blocks of n_p x n_p (position x,y,z; d/du x,y,z;
 * d/dv x,y,z; reference Patch.coeffs / coeffs_du / coeffs_dv).  base /
 * weights: the n_beta Chebyshev nodes and Fejer weights; grading: the map
 * order d.  out (HOST, n_pairs*4*n_c*n_c complex) receives per pair
 * beta_s[k=0], beta_s[k=1], beta_d[k=0], beta_d[k=1] (n_c x n_c each, row
 * m = u-degree) -- the layout of ifgfb_near_desc.moments. */
typedef struct {
  int64_t n_pairs;
  const double* target_xyz;     /* n_pairs*3 */
  const double* target_nrm;     /* n_pairs*3 */
  const int32_t* patch;         /* n_pairs */
  const double* uv;             /* n_pairs*2 */
  int32_t n_patches, n_p;
  const double* patch_coeffs;   /* n_patches*9*n_p*n_p */
  int32_t n_c, n_beta, grading;
  const double* base;           /* n_beta */
  const double* weights;        /* n_beta */
  const double* kappas;         /* 2 complex */
  /* ABI 7, exact mode: when nodes is non-null it holds per pair the graded
   * nodes the reference computes on the host (quadrature.py:203-228
   * clustered_nodes: np.power is not reproducible on the device) as
   * [xi_u, dxi_u, xi_v, dxi_v] x n_beta, and the device evaluates the patch
   * geometry in the reference's float64 operation order (numpy elementwise,
   * OpenBLAS dgemm: sequential FMA over k, except result columns >= gemm_tail
   * which use 8 k-interleaved lanes + a pairwise tree; 0 = no tail), so beta_d
   * matches the reference to rounding instead of to its ~1e-7 conditioning.
   * nodes == NULL: graded map on the device (uv used). */
  const double* nodes;          /* n_pairs*4*n_beta, or NULL */
  int32_t gemm_tail_u;          /* u contraction (tu @ coeff): column of the tail, 0 = none */
  int32_t gemm_tail_v;          /* v contraction ((.) @ tv^T): column of the tail, 0 = none */
} ifgfb_moment_desc;
int ifgfb_singular_moments(const ifgfb_moment_desc* desc, double* out);

/* Off-surface layer fields (replaces reference reference.py:285-312
 * _layer_fields, called by evaluate_fields :315-347): for n_tgt targets
 * tgt[3*t] and n_src sources src[15*s] = (x, y, z, m_w[3] complex, j_w[3]
 * complex) (densities already times the quadrature weights), with
 * G = exp(i kappa r)/(4 pi r) and kappa = (kappa[0], kappa[1]) complex:
 *   out[f][t][c] (complex, f = 0..3) = curl S[m], curl S[j],
 *   curlcurl S[m], curlcurl S[j]  (reference row order);
 * min_dist[t] (optional) = min_s |tgt_t - src_s| (the reference's
 * near-surface guard).  Host buffers; deterministic summation order. */
int ifgfb_layer_fields(int64_t n_src, const double* src, int64_t n_tgt,
                       const double* tgt, const double* kappa, double* out,
                       double* min_dist);

int ifgfb_plan_create(const ifgfb_tree_desc* tree, ifgfb_plan** out);
int ifgfb_plan_add_level(ifgfb_plan* plan, const ifgfb_level_desc* lvl);
int ifgfb_plan_add_accum(ifgfb_plan* plan, const ifgfb_accum_desc* acc);
int ifgfb_plan_set_emission(ifgfb_plan* plan, const ifgfb_emit_desc* em);
int ifgfb_plan_set_surface(ifgfb_plan* plan, const ifgfb_surface_desc* s);
int ifgfb_plan_set_near(ifgfb_plan* plan, const ifgfb_near_desc* nf);
int ifgfb_plan_finalize(ifgfb_plan* plan);
int ifgfb_plan_destroy(ifgfb_plan* plan);
/* bytes of device memory held by the plan (static + workspace) */
int64_t ifgfb_plan_device_bytes(const ifgfb_plan* plan);

/* Far-field sums for every surface point over the sources outside its
 * finest-level neighbour boxes (reference ifgf_apply, ifgf.py:885-923).
 *   w        device, nch*N complex, ORIGINAL order, row c = channel c
 *   kappas   host, nk complex (nk = 1 or 2)
 *   out      device, nch*nk*N complex, layout (nch, nk, N) original order
 *   out_disp device, same layout (evaluation at x + h n), or NULL
 * nch*nk <= 16.  Result identical for mode "vec"/"seq" (the device always
 * carries every channel-kernel column through one traversal). */
int ifgfb_far_apply(ifgfb_plan* plan, const double* w, int nch,
                    const double* kappas, int nk, double* out,
                    double* out_disp, void* stream);

/* S (8,2,N) and D (6,2,N) potentials of packed densities phi (8,N)
 * (reference MullerOperator.potentials, operators.py:321-350). */
int ifgfb_potentials(ifgfb_plan* plan, const double* phi, double* s_val,
                     double* d_val, void* stream);

/* y (4N complex, device) -> A y (4N complex, device)
 * (reference MullerOperator.apply, operators.py:399-403). */
int ifgfb_muller_apply(ifgfb_plan* plan, const double* y, double* out,
                       void* stream);
/* same with host buffers; copies (pinned staging) are inside the call and
 * the call returns after the result is in `out_host`. */
int ifgfb_muller_apply_host(ifgfb_plan* plan, const double* y_host,
                            double* out_host, void* stream);

/* GMRES vector primitives on device vectors of n complex entries
 * (reference solver.py:61-66, :91-92).  Scalars are host complex. */
int ifgfb_zdotc(const double* x, const double* y, int64_t n, double* result,
                void* stream);              /* sum conj(x) y  (np.vdot)   */
int ifgfb_dznrm2(const double* x, int64_t n, double* result, void* stream);
int ifgfb_zaxpy(const double* alpha, const double* x, double* y, int64_t n,
                void* stream);              /* y += alpha x               */
int ifgfb_zscal_div(double* y, const double* x, double denom, int64_t n,
                    void* stream);          /* y = x / denom (real)       */

/* One modified Gram-Schmidt Arnoldi step (reference solver.py:61-67) on a
 * device basis V (vectors of n complex, stride ld complex between vectors):
 *   for i in 0..k: h[i] = vdot(V[i], w); w -= h[i] V[i]
 *   h[k+1] = ||w||;  V[k+1] = w / h[k+1]  (skipped when h[k+1] == 0)
 * h is a device array of >= k+2 complex; nothing is synchronised. */
int ifgfb_arnoldi_mgs(double* basis, int64_t ld, int k, int64_t n, double* w,
                      double* h, void* stream);
/* x = sum_{j<k} y[j] V[j]   (reference solver.py:92), y device k complex */
int ifgfb_basis_combine(const double* basis, int64_t ld, int k, int64_t n,
                        const double* y, double* x, void* stream);
/* The same two operations on a basis given as a host table of row pointers
 * (rows[i] = V[i]; device memory or pinned host memory, which sm_100
 * kernels address directly under UVA), so the Krylov basis can grow in
 * chunks and spill to host memory instead of being preallocated
 * (max_iter+1) x n on the device.  v_next receives w / h[k+1]. */
int ifgfb_arnoldi_mgs_rows(const double* const* rows, int k, int64_t n, double* w,
                           double* h, double* v_next, void* stream);
int ifgfb_basis_combine_rows(const double* const* rows, int k, int64_t n,
                             const double* y, double* x, void* stream);

/* Per-kernel-class CUDA-event timing (recorded on the launching stream).
 * Classes: 0 leaf (K2+K3), 1 propagation (K4+K3), 2 emission (K5),
 * 3 emission reduce, 4 near field (K6), 5 density pack (K1),
 * 6 assembly (K7), 7 other.  set_timing resets the accumulators;
 * kernel_times synchronises and returns total ms and launch counts. */
#define IFGFB_KERNEL_KINDS 8
int ifgfb_plan_set_timing(ifgfb_plan* plan, int enable);
int ifgfb_plan_kernel_times(ifgfb_plan* plan, double* ms, int64_t* counts);
/* Propagation (class 1) time split by CHILD level d (ms[d], counts[d] for
 * d < max_levels; levels whose K4 writes level d-1), same accumulators. */
int ifgfb_plan_level_times(ifgfb_plan* plan, int max_levels, double* ms, int64_t* counts);

/* Number of kernels launched by the last apply on this plan. */
int64_t ifgfb_plan_last_launches(const ifgfb_plan* plan);

/* ---- streaming and multi-GPU ranks.
 *
 * Windows: a plan may be built for a Morton range of level-3 subtrees only
 * (the host builds the window's cones, propagation and emission plans; the
 * device plan is a complete plan over that forest: levels <= 2 carry no
 * cones, reference ifgf.py:433, so no parent lies outside the window).  Its
 * far field is then the PARTIAL sum of the window's sources at all N
 * targets.
 *
 * Single-GPU streaming: run the upward pass as n_parts sequential passes,
 * one per group of Morton-contiguous level-3 subtrees of the plan,
 * accumulating the far field; the coefficient buffers shrink to the largest
 * part, so levels larger than half the HBM fit (cfg 5 on one B200). */
typedef struct {
  int32_t level;
  int64_t seg_lo, seg_hi;     /* segment rows of this level in the part */
  int64_t pair_lo, pair_hi;   /* (box, cousin point) pairs of this level */
} ifgfb_level_part;

typedef struct {
  int32_t n_levels;                 /* entries for levels 3..depth */
  const ifgfb_level_part* levels;
  int64_t target_lo, target_hi;     /* unused (kept for layout) */
} ifgfb_partition_desc;

int ifgfb_plan_set_streaming(ifgfb_plan* plan, const ifgfb_partition_desc* parts,
                             int n_parts);

/* Rank mode (one process per GPU).  The plan is rank `rank`'s window (far
 * field sources) and its near-field plan covers the owned targets
 * [target_lo, target_hi) = [rank*chunk, min((rank+1)*chunk, N)) (original
 * order, patch aligned); exchange buffers are point-major and padded to
 * n_ranks*chunk rows so each rank's rows are one contiguous, equal-size
 * chunk (NCCL reduce-scatter / all-gather):
 *   ifgfb_muller_far_phase  -> xfar (n_ranks*chunk rows x 32 complex: the 8
 *                              channels x 2 kernels far field, then the same
 *                              at x + h n) = this rank's PARTIAL sums;
 *   caller: reduce-scatter(sum) xfar -> xfar_mine (chunk rows);
 *   ifgfb_muller_near_phase -> xout_mine (chunk rows x 4 complex: the owned
 *                              result rows of y = [m1, m2, j1, j2]);
 *   caller: all-gather xout_mine -> xout (n_ranks*chunk rows x 4);
 *   ifgfb_rank_unpack       -> out (4N, the apply's y layout).
 * Replaces the reference's single-process MullerOperator.apply
 * (operators.py:399-403); the whole-plan entry points (ifgfb_muller_apply,
 * _host, ifgfb_potentials, ifgfb_far_apply) refuse a rank plan. */
typedef struct {
  int64_t target_lo, target_hi;
  int64_t chunk;
  int32_t rank, n_ranks;
} ifgfb_rank_desc;

int ifgfb_plan_set_rank(ifgfb_plan* plan, const ifgfb_rank_desc* rank);
int ifgfb_plan_rank_buffers(ifgfb_plan* plan, double** xfar, double** xfar_mine,
                            double** xout_mine, double** xout, int64_t* chunk);
int ifgfb_rank_unpack(ifgfb_plan* plan, double* out, void* stream);
/* density packing (all points) + far field of the plan's sources (whole plan:
 * into the internal far buffers; rank mode: into xfar) */
int ifgfb_muller_far_phase(ifgfb_plan* plan, const double* y, void* stream);
/* near field + assembly of the owned targets (whole plan: all, into out;
 * rank mode: into xout_mine, out may be NULL).  Without a rank,
 * far_phase + near_phase == ifgfb_muller_apply. */
int ifgfb_muller_near_phase(ifgfb_plan* plan, const double* y, double* out,
                            void* stream);

/* ---- plan-time cone hierarchy on the device (native plan builder,
 * SURVEY 8(f) rank 1; replaces the relevance pass of
 * build_cone_hierarchy, reference ifgf.py:417-482).  Per cone level:
 *   begin -> mark_points (cousin points) -> mark_parents (nodes of the
 *   parent level's relevant segments) -> ambiguous (evaluations whose
 *   arccos / arctan2 sit within a few ulp of a segment edge: the caller
 *   decides them with the reference's own expressions and returns them
 *   through cones_set) -> finish (per-box counts -> seg_off) -> ids
 *   (ascending segment ids per box) -> free.
 * Every other floating-point step replays numpy's operation order with
 * correctly rounded ops, so the result equals the host builder bit for
 * bit.  Synchronous; host arrays in, host arrays out. */
typedef struct ifgfb_cone_build ifgfb_cone_build;

typedef struct {
  int32_t n_s, n_a;            /* cone counts of the level */
  double delta_s, delta_a;     /* ETA / n_s, pi / n_a */
  double s_num;                /* np.sqrt(3.0) / 2.0 * side */
  int64_t n_boxes;
  int64_t amb_capacity;        /* edge cases buffered (>= 65536 used) */
} ifgfb_cone_level_desc;

typedef struct {
  int64_t n_boxes;             /* boxes of the level (== the build's) */
  const int64_t* inst_off;     /* n_boxes + 1: (box, parent row) instances */
  const int64_t* row0;         /* n_boxes: first segment row of the parent box */
  const int32_t* parent_box;   /* n_boxes */
  int64_t n_parent_rows;
  const int32_t* parent_seg_ids;   /* parent level segment ids */
  int64_t n_parent_boxes;
  const double* parent_centers;    /* n_parent_boxes x 3 */
  const double* centers;           /* n_boxes x 3 */
  int32_t pn_s, pn_a;              /* parent cone counts */
  double ph;                       /* parent level h */
  const double* parent_tabs;       /* s_nodes | sin_t | cos_t | sin_p | cos_p */
} ifgfb_cone_parent_desc;

int ifgfb_cones_begin(const ifgfb_cone_level_desc* level, ifgfb_cone_build** out);
int ifgfb_cones_mark_points(ifgfb_cone_build* b, int64_t n_pairs, const int32_t* pair_box,
                            const int32_t* pair_point, int64_t n_points,
                            const double* points, const double* centers);
int ifgfb_cones_mark_parents(ifgfb_cone_build* b, const ifgfb_cone_parent_desc* parents);
int ifgfb_cones_ambiguous(ifgfb_cone_build* b, int64_t* n, int64_t* box, double* dx);
int ifgfb_cones_set(ifgfb_cone_build* b, int64_t n, const int64_t* box, const int64_t* key);
int ifgfb_cones_finish(ifgfb_cone_build* b, int64_t* seg_off, int64_t** reserved,
                       int64_t* n_segments);
int ifgfb_cones_ids(ifgfb_cone_build* b, const int64_t* seg_off, int64_t* seg_ids);
int ifgfb_cones_free(ifgfb_cone_build* b);

/* Propagation types of one level on the device (reference _AccumType,
 * ifgf.py:686-702): per type (parent segment id gamma, child octant) the
 * sigma group of each of the 75 parent nodes (gid), the groups' child
 * segment ids ascending (sigma, -1 padded to 75), their count and, if
 * node_geom / node_r are given, the nodes' local coordinates and radii.
 * ambiguous[t] = 1: some node of type t lies within a few ulp of a child
 * segment edge; its row is NOT filled and must be decided on the host with
 * the reference's own expressions. */
typedef struct {
  int64_t n_types;
  const int32_t* gamma;        /* parent segment id per type */
  const uint8_t* octant;       /* child octant per type */
  int32_t pn_s, pn_a;          /* parent cone counts */
  double ph;                   /* parent level h */
  const double* parent_tabs;   /* s_nodes | sin_t | cos_t | sin_p | cos_p */
  int32_t n_s, n_a;            /* child cone counts */
  double delta_s, delta_a;     /* child level */
  double s_num;                /* np.sqrt(3.0) / 2.0 * child_side */
  double half;                 /* 0.5 * child_side */
} ifgfb_accum_types_desc;

int ifgfb_accum_types(const ifgfb_accum_types_desc* d, uint8_t* gid, int32_t* sigma,
                      uint8_t* nsig, uint8_t* ambiguous, double* node_geom, double* node_r);

#ifdef __cplusplus
}
#endif
#endif /* IFGFB_H */
