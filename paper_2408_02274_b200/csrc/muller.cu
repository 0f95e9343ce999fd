// N-Muller operator around the far field: density packing (K1), near field
// (K6), surface assembly (K7), the apply driver and GMRES vector primitives.
//
// Reference: operators.py:230-245 (decode/encode), :121-128 + :148-189
// (DensityBlock.from_currents, surface_divergence), :249-253 (_patch_coeffs),
// :321-350 (potentials), :354-397 (apply_block), quadrature.py:343-360
// (apply_singular_block), :457-487 (CorrectionSet), operators.py:279-319
// (_neighbor_sums), solver.py:61-66 (GMRES vector ops).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace ifgfb {

constexpr int MAXNC = 16;       // largest patch grid n_c supported on device

struct SurfPtrs {
  int n, n_c, n_patches;
  const double* pts; const double* nrm; const double* wq; const double* jac;
  const double* eu; const double* ev; const double* t1; const double* t2;
  const double* dmat; const double* cmat;
};

__device__ __forceinline__ double2 cscale(double s, double2 a) {
  return make_double2(s * a.x, s * a.y);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}

// ---------------------------------------------------------------- K1 ----
// One CTA per patch (n_c^2 threads): y -> (m, j) Cartesian, surface
// divergences, phi (8,N), phi * weights (8,N) and per-patch Chebyshev
// coefficient grids of phi (8,P,n_c,n_c).
// Also writes phi_pm, point-major rows [phi(8) | phi*w(8)] (256 B per point)
// for the near field's source gathers: one row per direct entry instead of
// 8 channel-strided loads.
__global__ void pack_kernel(SurfPtrs s, const double2* __restrict__ y,
                            const double2* __restrict__ phi_in,
                            double2* __restrict__ phi, double2* __restrict__ phiw,
                            double2* __restrict__ pcoef, double2* __restrict__ phi_pm) {
  extern __shared__ double2 sh[];
  const int nc = s.n_c, n2 = nc * nc;
  double2* gu = sh;            // 2 x n2 : J f^u for (j, m)
  double2* gv = gu + 2 * n2;   // 2 x n2 : J f^v
  double2* gp = gv + 2 * n2;   // 8 x n2 : phi grid
  double2* gx = gp + 8 * n2;   // 8 x n2 : T @ phi
  const int p = blockIdx.x, loc = threadIdx.x;
  const int n = s.n;
  const int ell = p * n2 + loc;
  const bool act = loc < n2;
  double2 J[3], M[3];
  double e = 0, f = 0, g = 0, det = 1, jac = 1;
  if (act && phi_in) {
    // densities given directly (potentials(dens)): skip decode/divergence
    const double wq = s.wq[ell];
    for (int c = 0; c < 8; ++c) {
      const double2 v = phi_in[(size_t)c * n + ell];
      phi[(size_t)c * n + ell] = v;
      phiw[(size_t)c * n + ell] = cscale(wq, v);
      phi_pm[(size_t)ell * 16 + c] = v;
      phi_pm[(size_t)ell * 16 + 8 + c] = cscale(wq, v);
      gp[c * n2 + loc] = v;
    }
  }
  if (act && !phi_in) {
    const double2 y1 = y[ell], y2 = y[n + ell], y3 = y[2 * n + ell], y4 = y[3 * n + ell];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double a = s.t1[3 * ell + c], b = s.t2[3 * ell + c];
      M[c] = cadd(cscale(a, y1), cscale(b, y2));
      J[c] = cadd(cscale(a, y3), cscale(b, y4));
    }
    const double* eu = s.eu + 3 * ell;
    const double* ev = s.ev + 3 * ell;
    e = eu[0] * eu[0] + eu[1] * eu[1] + eu[2] * eu[2];
    f = eu[0] * ev[0] + eu[1] * ev[1] + eu[2] * ev[2];
    g = ev[0] * ev[0] + ev[1] * ev[1] + ev[2] * ev[2];
    det = e * g - f * f;
    jac = s.jac[ell];
    for (int q = 0; q < 2; ++q) {
      const double2* V = q == 0 ? J : M;
      double2 cu = make_double2(0, 0), cv = make_double2(0, 0);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        cu = cadd(cu, cscale(eu[c], V[c]));
        cv = cadd(cv, cscale(ev[c], V[c]));
      }
      const double2 fu = cscale(1.0 / det, csub(cscale(g, cu), cscale(f, cv)));
      const double2 fv = cscale(1.0 / det, csub(cscale(e, cv), cscale(f, cu)));
      gu[q * n2 + loc] = cscale(jac, fu);
      gv[q * n2 + loc] = cscale(jac, fv);
    }
  }
  __syncthreads();
  if (act && !phi_in) {
    const int i = loc / nc, jj = loc % nc;
    double2 div[2];
    for (int q = 0; q < 2; ++q) {
      double2 du = make_double2(0, 0), dv = make_double2(0, 0);
      for (int k = 0; k < nc; ++k) {
        du = cadd(du, cscale(s.dmat[i * nc + k], gu[q * n2 + k * nc + jj]));
        dv = cadd(dv, cscale(s.dmat[jj * nc + k], gv[q * n2 + i * nc + k]));
      }
      div[q] = cscale(1.0 / jac, cadd(du, dv));
    }
    double2 vals[8] = {J[0], J[1], J[2], M[0], M[1], M[2], div[0], div[1]};
    const double wq = s.wq[ell];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      phi[(size_t)c * n + ell] = vals[c];
      phiw[(size_t)c * n + ell] = cscale(wq, vals[c]);
      phi_pm[(size_t)ell * 16 + c] = vals[c];
      phi_pm[(size_t)ell * 16 + 8 + c] = cscale(wq, vals[c]);
      gp[c * n2 + loc] = vals[c];
    }
  }
  __syncthreads();
  // coefficient grids: X = T @ Phi, A = X @ T^T  (reference _patch_coeffs)
  if (act) {
    const int i = loc / nc, jj = loc % nc;
    for (int c = 0; c < 8; ++c) {
      double2 x = make_double2(0, 0);
      for (int k = 0; k < nc; ++k) x = cadd(x, cscale(s.cmat[i * nc + k], gp[c * n2 + k * nc + jj]));
      gx[c * n2 + loc] = x;
    }
  }
  __syncthreads();
  if (act) {
    const int i = loc / nc, jj = loc % nc;
    for (int c = 0; c < 8; ++c) {
      double2 a = make_double2(0, 0);
      for (int k = 0; k < nc; ++k) a = cadd(a, cscale(s.cmat[jj * nc + k], gx[c * n2 + i * nc + k]));
      pcoef[((size_t)c * s.n_patches + p) * n2 + loc] = a;
    }
  }
}

// ---------------------------------------------------------------- K6 ----
struct NearArgs {
  SurfPtrs s;
  const int* mom_off; const int* mom_patch; const double2* moments;
  const int* dir_off; const int* dir_src;
  const double2* phi; const double2* phiw; const double2* pcoef;
  const double2* phi_pm;                        // [N][phi(8) | phi*w(8)]
  const double2* far; const double2* far_disp;  // (8,2,N)
  double kr[2], ki[2];
  double fd_step;
  double2* s_val; double2* d_val;
  int t_lo, t_hi;        // owned targets (original order)
  int far_pm;            // rank mode: far = xfar_mine, row (ell - t_lo) x 32
};


// S kernel e^{i k r}/(4 pi r) and its target-normal derivative factor.
__device__ __forceinline__ void kernel_pair(double kr, double ki, double r,
                                            double ndx, double2& gk,
                                            double2& qk) {
  const double2 e = cexp_ikx(kr, ki, r);
  const double inv = 1.0 / (4.0 * M_PI * r);
  gk = make_double2(e.x * inv, e.y * inv);
  // (ndx * (i kappa r - 1) / r^2): i*kappa*r = (-ki r, kr r)
  const double2 f = make_double2(ndx * (-ki * r - 1.0) / (r * r), ndx * (kr * r) / (r * r));
  qk = cmul(gk, f);
}

// Sums 28 complex per-lane partials over the warp; lane c*2+k keeps the
// totals of channel c, kernel k (S in tot_s, D in tot_d for c < 6).
__device__ __forceinline__ void warp_reduce_owned(const double2 (&s)[8][2],
                                                  const double2 (&d)[6][2],
                                                  int lane, double2& tot_s,
                                                  double2& tot_d) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double2 ts = make_double2(warp_sum(s[c][k].x), warp_sum(s[c][k].y));
      if (lane == c * 2 + k) tot_s = ts;
      if (c < 6) {
        const double2 td = make_double2(warp_sum(d[c][k].x), warp_sum(d[c][k].y));
        if (lane == c * 2 + k) tot_d = td;
      }
    }
}

// One warp per target: singular moments (S, D), neighbour-box direct sums
// (+ entries) and local corrections (- entries), then the reference's
// combination with the far field (operators.py:341-350), including
// D_far = (S_disp - S) / h.  Three phases keep 28 complex accumulators live.
#ifndef IFGFB_NEAR_MINB
#define IFGFB_NEAR_MINB 3   // 168 registers, 3 CTAs/SM: 1.20 -> 1.08 ms at (8,10), 10.1 -> 8.8 ms on the (48,6,3) slab
#endif
__global__ void __launch_bounds__(128, IFGFB_NEAR_MINB) near_kernel(NearArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int n = a.s.n, n2 = a.s.n_c * a.s.n_c;
  const int ell = warp + a.t_lo;
  if (ell >= a.t_hi) return;
  double2 S[8][2], D[6][2];
  double2 near_s = make_double2(0, 0), near_d = make_double2(0, 0);
  double2 nb_s = make_double2(0, 0), nb_d = make_double2(0, 0);
  double2 cr_s = make_double2(0, 0), cr_d = make_double2(0, 0);
  auto zero = [&]() {
#pragma unroll
    for (int c = 0; c < 8; ++c) S[c][0] = S[c][1] = make_double2(0, 0);
#pragma unroll
    for (int c = 0; c < 6; ++c) D[c][0] = D[c][1] = make_double2(0, 0);
  };
  // ---- phase 1: singular moments (quadrature.py:343-360)
  zero();
  for (int q = a.mom_off[ell]; q < a.mom_off[ell + 1]; ++q) {
    const int p = a.mom_patch[q];
    const double2* beta = a.moments + (size_t)q * 4 * n2;
    for (int mn = lane; mn < n2; mn += 32) {
      const double2 bs0 = beta[mn], bs1 = beta[n2 + mn];
      const double2 bd0 = beta[2 * n2 + mn], bd1 = beta[3 * n2 + mn];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double2 co = a.pcoef[((size_t)c * a.s.n_patches + p) * n2 + mn];
        S[c][0] = cadd(S[c][0], cmul(bs0, co));
        S[c][1] = cadd(S[c][1], cmul(bs1, co));
        if (c < 6) {
          D[c][0] = cadd(D[c][0], cmul(bd0, co));
          D[c][1] = cadd(D[c][1], cmul(bd1, co));
        }
      }
    }
  }
  warp_reduce_owned(S, D, lane, near_s, near_d);
  const double x0 = a.s.pts[3 * ell], x1 = a.s.pts[3 * ell + 1], x2 = a.s.pts[3 * ell + 2];
  const double n0 = a.s.nrm[3 * ell], n1 = a.s.nrm[3 * ell + 1], n2v = a.s.nrm[3 * ell + 2];
  const int e0 = a.dir_off[ell], e1 = a.dir_off[ell + 1];
  // ---- phases 2/3: + neighbour sources (operators.py:279-319, phi*w),
  //                  - corrections (quadrature.py:457-487, (G*jw)*phi)
#pragma unroll 1
  for (int phase = 0; phase < 2; ++phase) {
    zero();
    for (int e = e0 + lane; e < e1; e += 32) {
      const int code = a.dir_src[e];
      const bool neg = code < 0;
      if (neg != (phase == 1)) continue;
      const int src = neg ? -code - 1 : code;
      const double dx = x0 - a.s.pts[3 * src], dy = x1 - a.s.pts[3 * src + 1],
                   dz = x2 - a.s.pts[3 * src + 2];
      const double r = sqrt(dx * dx + dy * dy + dz * dz);
      const double ndx = dx * n0 + dy * n1 + dz * n2v;
      double2 gk[2], qk[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) kernel_pair(a.kr[k], a.ki[k], r, ndx, gk[k], qk[k]);
      const double jw = neg ? a.s.wq[src] : 1.0;
      const double2* wrow = a.phi_pm + (size_t)src * 16 + (neg ? 0 : 8);
      if (neg) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          gk[k] = cscale(jw, gk[k]);
          qk[k] = cscale(jw, qk[k]);
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double2 w = wrow[c];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          S[c][k] = cadd(S[c][k], cmul(gk[k], w));
          if (c < 6) D[c][k] = cadd(D[c][k], cmul(qk[k], w));
        }
      }
    }
    if (phase == 0) warp_reduce_owned(S, D, lane, nb_s, nb_d);
    else warp_reduce_owned(S, D, lane, cr_s, cr_d);
  }
  if (lane < 16) {
    const int c = lane >> 1;
    const size_t o = (size_t)lane * n + ell;   // (c*2+k)*N + ell
    const size_t of = a.far_pm ? (size_t)(ell - a.t_lo) * 32 + lane : o;
    const double2 s_if = a.far[of];
    a.s_val[o] = cadd(near_s, csub(cadd(s_if, nb_s), cr_s));
    if (c < 6) {
      const double2 sd = a.far_pm ? a.far[of + 16] : a.far_disp[o];
      // numpy's complex / real: multiply by the reciprocal (Smith, rat = 0)
      const double scl = 1.0 / a.fd_step;
      const double2 d_if = make_double2(mul_rn(sd.x - s_if.x, scl),
                                        mul_rn(sd.y - s_if.y, scl));
      a.d_val[o] = cadd(near_d, csub(cadd(d_if, nb_d), cr_d));
    }
  }
}

// ------------------------------------------------- K6, split (default) ----
// K6a: singular moments (quadrature.py:343-360).  One warp per target; lane
// L < 28 owns one output, S(c, k) for L < 16 (L = 2c + k) and D(c, k) for
// L >= 16, and streams the target's moment blocks in mn order (each block
// 4 x n_c^2 complex, read once, coalesced per k-step through L1) against the
// patch coefficient grids (L2 resident).  No cross-lane reduction and ~40
// registers, against 28 warp reductions and 220 registers of the fused form.
__global__ void __launch_bounds__(128) near_moments_kernel(NearArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int n = a.s.n, n2 = a.s.n_c * a.s.n_c;
  const int ell = warp + a.t_lo;
  if (ell >= a.t_hi || lane >= 28) return;
  const bool is_s = lane < 16;
  const int o = is_s ? lane : lane - 16;          // (c * 2 + k)
  const int c = o >> 1, k = o & 1;
  const int kind = is_s ? k : 2 + k;               // bs0, bs1, bd0, bd1
  double2 acc = make_double2(0.0, 0.0);
  for (int q = a.mom_off[ell]; q < a.mom_off[ell + 1]; ++q) {
    const int p = a.mom_patch[q];
    IFGFB_DCHECK(p >= 0 && p < a.s.n_patches);
    const double2* beta = a.moments + ((size_t)q * 4 + kind) * n2;
    const double2* co = a.pcoef + ((size_t)c * a.s.n_patches + p) * n2;
#pragma unroll 4
    for (int mn = 0; mn < n2; ++mn) {
      const double2 b = __ldg(beta + mn), v = __ldg(co + mn);
      acc.x += b.x * v.x - b.y * v.y;
      acc.y += b.x * v.y + b.y * v.x;
    }
  }
  if (is_s) a.s_val[(size_t)o * n + ell] = acc;
  else a.d_val[(size_t)o * n + ell] = acc;
}

#ifndef IFGFB_NEAR_DIRECT_MINB   // 3 CTAs/SM -> <= 168 registers, no spills
#define IFGFB_NEAR_DIRECT_MINB 3
#endif
// K6b: neighbour-box direct sums (+ entries, phi * w; operators.py:279-319)
// and local corrections (- entries, (G * jw) * phi; quadrature.py:457-487)
// in ONE signed pass (one warp reduction instead of two), then the far-field
// combination (operators.py:341-350) on top of K6a's moment terms.
__global__ void __launch_bounds__(128, IFGFB_NEAR_DIRECT_MINB) near_direct_kernel(NearArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int n = a.s.n;
  const int ell = warp + a.t_lo;
  if (ell >= a.t_hi) return;
  double2 S[8][2], D[6][2];
#pragma unroll
  for (int c = 0; c < 8; ++c) S[c][0] = S[c][1] = make_double2(0, 0);
#pragma unroll
  for (int c = 0; c < 6; ++c) D[c][0] = D[c][1] = make_double2(0, 0);
  const double x0 = a.s.pts[3 * ell], x1 = a.s.pts[3 * ell + 1], x2 = a.s.pts[3 * ell + 2];
  const double n0 = a.s.nrm[3 * ell], n1 = a.s.nrm[3 * ell + 1], n2v = a.s.nrm[3 * ell + 2];
  const int e0 = a.dir_off[ell], e1 = a.dir_off[ell + 1];
  for (int e = e0 + lane; e < e1; e += 32) {
    const int code = a.dir_src[e];
    const bool neg = code < 0;
    const int src = neg ? -code - 1 : code;
    IFGFB_DCHECK(src >= 0 && src < n && src != ell);
    const double dx = x0 - a.s.pts[3 * src], dy = x1 - a.s.pts[3 * src + 1],
                 dz = x2 - a.s.pts[3 * src + 2];
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    const double ndx = dx * n0 + dy * n1 + dz * n2v;
    double2 gk[2], qk[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) kernel_pair(a.kr[k], a.ki[k], r, ndx, gk[k], qk[k]);
    const double jw = neg ? -a.s.wq[src] : 1.0;      // corrections subtract
    const double2* wrow = a.phi_pm + (size_t)src * 16 + (neg ? 0 : 8);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      gk[k] = cscale(jw, gk[k]);
      qk[k] = cscale(jw, qk[k]);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double2 w = wrow[c];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        S[c][k] = cadd(S[c][k], cmul(gk[k], w));
        if (c < 6) D[c][k] = cadd(D[c][k], cmul(qk[k], w));
      }
    }
  }
  double2 dir_s = make_double2(0, 0), dir_d = make_double2(0, 0);
  warp_reduce_owned(S, D, lane, dir_s, dir_d);
  if (lane < 16) {
    const int c = lane >> 1;
    const size_t o = (size_t)lane * n + ell;   // (c*2+k)*N + ell
    const size_t of = a.far_pm ? (size_t)(ell - a.t_lo) * 32 + lane : o;
    const double2 s_if = a.far[of];
    a.s_val[o] = cadd(a.s_val[o], cadd(s_if, dir_s));
    if (c < 6) {
      const double2 sd = a.far_pm ? a.far[of + 16] : a.far_disp[o];
      // numpy's complex / real: multiply by the reciprocal (Smith, rat = 0)
      const double scl = 1.0 / a.fd_step;
      const double2 d_if = make_double2(mul_rn(sd.x - s_if.x, scl),
                                        mul_rn(sd.y - s_if.y, scl));
      a.d_val[o] = cadd(a.d_val[o], cadd(d_if, dir_d));
    }
  }
}

// K6b, thread per target: the same signed pass with one THREAD per target
// and its 28 complex sums in registers -- no warp reductions (the warp form
// spends ~40% of its instructions in 3 x 28 shuffle trees).  Consecutive
// targets lie on one patch and walk overlapping, ascending source lists, so
// the per-lane gathers of source positions and phi rows hit L1.
#ifndef IFGFB_NEAR_THREAD_MINB
#define IFGFB_NEAR_THREAD_MINB 3
#endif
__global__ void __launch_bounds__(128, IFGFB_NEAR_THREAD_MINB)
near_direct_thread_kernel(NearArgs a) {
  const int ell = blockIdx.x * blockDim.x + threadIdx.x + a.t_lo;
  if (ell >= a.t_hi) return;
  const int n = a.s.n;
  double2 S[8][2], D[6][2];
#pragma unroll
  for (int c = 0; c < 8; ++c) S[c][0] = S[c][1] = make_double2(0, 0);
#pragma unroll
  for (int c = 0; c < 6; ++c) D[c][0] = D[c][1] = make_double2(0, 0);
  const double x0 = a.s.pts[3 * ell], x1 = a.s.pts[3 * ell + 1], x2 = a.s.pts[3 * ell + 2];
  const double n0 = a.s.nrm[3 * ell], n1 = a.s.nrm[3 * ell + 1], n2v = a.s.nrm[3 * ell + 2];
  const int e0 = a.dir_off[ell], e1 = a.dir_off[ell + 1];
#pragma unroll 1
  for (int e = e0; e < e1; ++e) {
    const int code = __ldg(a.dir_src + e);
    const bool neg = code < 0;
    const int src = neg ? -code - 1 : code;
    IFGFB_DCHECK(src >= 0 && src < n && src != ell);
    const double dx = x0 - __ldg(a.s.pts + 3 * src), dy = x1 - __ldg(a.s.pts + 3 * src + 1),
                 dz = x2 - __ldg(a.s.pts + 3 * src + 2);
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    const double ndx = dx * n0 + dy * n1 + dz * n2v;
    double2 gk[2], qk[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) kernel_pair(a.kr[k], a.ki[k], r, ndx, gk[k], qk[k]);
    const double jw = neg ? -__ldg(a.s.wq + src) : 1.0;      // corrections subtract
    const double2* wrow = a.phi_pm + (size_t)src * 16 + (neg ? 0 : 8);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      gk[k] = cscale(jw, gk[k]);
      qk[k] = cscale(jw, qk[k]);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double2 w = __ldg(wrow + c);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        S[c][k] = cadd(S[c][k], cmul(gk[k], w));
        if (c < 6) D[c][k] = cadd(D[c][k], cmul(qk[k], w));
      }
    }
  }
  const double scl = 1.0 / a.fd_step;
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int lane = c * 2 + k;
      const size_t o = (size_t)lane * n + ell;
      const size_t of = a.far_pm ? (size_t)(ell - a.t_lo) * 32 + lane : o;
      const double2 s_if = a.far[of];
      a.s_val[o] = cadd(a.s_val[o], cadd(s_if, S[c][k]));
      if (c < 6) {
        const double2 sd = a.far_pm ? a.far[of + 16] : a.far_disp[o];
        // numpy's complex / real: multiply by the reciprocal (Smith, rat = 0)
        const double2 d_if = make_double2(mul_rn(sd.x - s_if.x, scl),
                                          mul_rn(sd.y - s_if.y, scl));
        a.d_val[o] = cadd(a.d_val[o], cadd(d_if, D[c][k]));
      }
    }
}

// ---------------------------------------------------------------- K7 ----
struct AsmArgs {
  SurfPtrs s;
  const double2* s_val; const double2* d_val; const double2* y;
  double2 eps_e, mu_e, eps_i, mu_i, kap[2];
  double omega;
  double2* out;
  int p0;                // first patch handled (partition)
  int out_pm;            // rank mode: out = xout_mine, row (ell - t_lo) x 4
  int t_lo;
};

__device__ __forceinline__ void cross3(const double* n, const double2* v, double2* o) {
  o[0] = csub(cscale(n[1], v[2]), cscale(n[2], v[1]));
  o[1] = csub(cscale(n[2], v[0]), cscale(n[0], v[2]));
  o[2] = csub(cscale(n[0], v[1]), cscale(n[1], v[0]));
}

// One CTA per patch: tangential gradients of the 16 S fields (per-patch
// spectral differentiation), n x curl and R+T terms, the N-Muller rows and
// the tangent-frame encoding (operators.py:354-403).
__global__ void assemble_kernel(AsmArgs a) {
  extern __shared__ double2 sh[];   // 16 x n2
  const int nc = a.s.n_c, n2 = nc * nc, n = a.s.n;
  const int p = blockIdx.x + a.p0, loc = threadIdx.x;
  const bool act = loc < n2;
  const int ell = p * n2 + loc;
  if (act)
    for (int f = 0; f < 16; ++f) sh[f * n2 + loc] = a.s_val[(size_t)f * n + ell];
  __syncthreads();
  if (!act) return;
  const int i = loc / nc, jj = loc % nc;
  const double* eu = a.s.eu + 3 * ell;
  const double* ev = a.s.ev + 3 * ell;
  const double e = eu[0] * eu[0] + eu[1] * eu[1] + eu[2] * eu[2];
  const double f = eu[0] * ev[0] + eu[1] * ev[1] + eu[2] * ev[2];
  const double g = ev[0] * ev[0] + ev[1] * ev[1] + ev[2] * ev[2];
  const double det = e * g - f * f;
  const double nr[3] = {a.s.nrm[3 * ell], a.s.nrm[3 * ell + 1], a.s.nrm[3 * ell + 2]};
  // grad[field][3]
  double2 grad[16][3];
#pragma unroll
  for (int fld = 0; fld < 16; ++fld) {
    double2 du = make_double2(0, 0), dv = make_double2(0, 0);
    for (int k = 0; k < nc; ++k) {
      du = cadd(du, cscale(a.s.dmat[i * nc + k], sh[fld * n2 + k * nc + jj]));
      dv = cadd(dv, cscale(a.s.dmat[jj * nc + k], sh[fld * n2 + i * nc + k]));
    }
    const double2 ca = cscale(1.0 / det, csub(cscale(g, du), cscale(f, dv)));
    const double2 cb = cscale(1.0 / det, csub(cscale(e, dv), cscale(f, du)));
#pragma unroll
    for (int c = 0; c < 3; ++c) grad[fld][c] = cadd(cscale(eu[c], ca), cscale(ev[c], cb));
  }
  // field index fld = channel*2 + k
  auto curl_trace = [&](int k, int c0, double2* res) {
    double2 w[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) w[c] = a.d_val[((size_t)(c0 + c) * 2 + k) * n + ell];
    double2 nw = make_double2(0, 0);
#pragma unroll
    for (int c = 0; c < 3; ++c) nw = cadd(nw, cscale(nr[c], w[c]));
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double2 wt = csub(w[c], cscale(nr[c], nw));
      double2 gg = make_double2(0, 0);
#pragma unroll
      for (int q = 0; q < 3; ++q) gg = cadd(gg, cscale(nr[q], grad[(c0 + q) * 2 + k][c]));
      res[c] = csub(gg, wt);
    }
  };
  auto rt_terms = [&](int c0, int cdiv, double2* res) {
#pragma unroll
    for (int c = 0; c < 3; ++c) res[c] = make_double2(0, 0);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double sign = k == 0 ? 1.0 : -1.0;
      double2 sv[3], c1[3], c2[3], gd[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        sv[c] = sh[((c0 + c) * 2 + k) * n2 + loc];
        gd[c] = grad[cdiv * 2 + k][c];
      }
      cross3(nr, sv, c1);
      cross3(nr, gd, c2);
      const double2 k2 = cmul(a.kap[k], a.kap[k]);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double2 term = cadd(cmul(k2, c1[c]), c2[c]);
        res[c] = cadd(res[c], cscale(sign, term));
      }
    }
    const double2 fac = make_double2(0.0, -1.0 / a.omega);
#pragma unroll
    for (int c = 0; c < 3; ++c) res[c] = cmul(fac, res[c]);
  };
  double2 ctm0[3], ctm1[3], ctj0[3], ctj1[3], rtj[3], rtm[3];
  curl_trace(0, 3, ctm0);
  curl_trace(1, 3, ctm1);
  curl_trace(0, 0, ctj0);
  curl_trace(1, 0, ctj1);
  rt_terms(0, 6, rtj);
  rt_terms(3, 7, rtm);
  // decoded currents
  const double2 y1 = a.y[ell], y2 = a.y[n + ell], y3 = a.y[2 * n + ell], y4 = a.y[3 * n + ell];
  const double* t1 = a.s.t1 + 3 * ell;
  const double* t2 = a.s.t2 + 3 * ell;
  const double2 hmu = cscale(0.5, cadd(a.mu_e, a.mu_i));
  const double2 heps = cscale(0.5, cadd(a.eps_e, a.eps_i));
  double2 rm[3], rj[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double2 mc = cadd(cscale(t1[c], y1), cscale(t2[c], y2));
    const double2 jc = cadd(cscale(t1[c], y3), cscale(t2[c], y4));
    const double2 km = csub(cmul(a.mu_e, ctm0[c]), cmul(a.mu_i, ctm1[c]));
    const double2 kj = csub(cmul(a.eps_e, ctj0[c]), cmul(a.eps_i, ctj1[c]));
    rm[c] = csub(cadd(cmul(hmu, mc), km), rtj[c]);
    rj[c] = cadd(cadd(rtm[c], cmul(heps, jc)), kj);
  }
  double2 o[4] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0),
                  make_double2(0, 0)};
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    o[0] = cadd(o[0], cscale(t1[c], rm[c]));
    o[1] = cadd(o[1], cscale(t2[c], rm[c]));
    o[2] = cadd(o[2], cscale(t1[c], rj[c]));
    o[3] = cadd(o[3], cscale(t2[c], rj[c]));
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const size_t oi = a.out_pm ? (size_t)(ell - a.t_lo) * 4 + q : (size_t)q * n + ell;
    a.out[oi] = o[q];
  }
}

// rank mode: y-layout out[q*N + ell] = gathered point-major rows xout[ell*4 + q]
__global__ void rank_unpack_kernel(int n, const double2* __restrict__ xout,
                                   double2* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= 4 * n) return;
  const int ell = idx >> 2, q = idx & 3;
  out[(size_t)q * n + ell] = xout[idx];
}

// ------------------------------------------------------------ drivers ----
static SurfPtrs surf(const Plan& p) {
  return SurfPtrs{p.n, p.n_c, p.n_patches, p.pts, p.nrm, p.wq, p.jac,
                  p.eu, p.ev, p.t1, p.t2, p.dmat, p.cmat};
}

// near field of the owned targets combined with the (complete) far field
static int near_launch(Plan& p, cudaStream_t st) {
  NearArgs na{surf(p), p.mom_off, p.mom_patch,
              reinterpret_cast<const double2*>(p.moments), p.dir_off, p.dir_src,
              reinterpret_cast<const double2*>(p.phi),
              reinterpret_cast<const double2*>(p.phiw),
              reinterpret_cast<const double2*>(p.pcoef),
              reinterpret_cast<const double2*>(p.phi_pm),
              reinterpret_cast<const double2*>(p.far_out),
              reinterpret_cast<const double2*>(p.far_disp),
              {p.kappa[0], p.kappa[2]}, {p.kappa[1], p.kappa[3]}, p.fd_step,
              reinterpret_cast<double2*>(p.s_val), reinterpret_cast<double2*>(p.d_val),
              p.t_lo(), p.t_hi(), 0};
  if (p.rank_mode) {
    na.far = reinterpret_cast<const double2*>(p.xfar_mine);
    na.far_disp = nullptr;
    na.far_pm = 1;
  }
  const int warps_per_block = 4;
  const int nt = p.t_hi() - p.t_lo();
  if (nt <= 0) return IFGFB_OK;
  // fused single kernel (default); IFGFB_NEAR=split: moments kernel + direct
  // kernel (measured slower: 1.26 vs 1.12 ms at sphere(8,10), 5.63 vs 4.12 ms
  // on the r=2 slab; DESIGN 4)
  // IFGFB_NEAR=thread: moments kernel + thread-per-target direct kernel
  static const int mode = [] {
    const char* v = std::getenv("IFGFB_NEAR");
    return (v && v[0] == 's') ? 1 : (v && v[0] == 't') ? 2 : 0;
  }();
  const int grid = (nt + warps_per_block - 1) / warps_per_block;
  const int tk = p.timer.begin(K_NEAR, st);
  if (mode == 0) {
    near_kernel<<<grid, 32 * warps_per_block, 0, st>>>(na);
    p.launches += 1;
  } else if (mode == 2) {
    near_moments_kernel<<<grid, 32 * warps_per_block, 0, st>>>(na);
    near_direct_thread_kernel<<<(nt + 127) / 128, 128, 0, st>>>(na);
    p.launches += 2;
  } else {
    near_moments_kernel<<<grid, 32 * warps_per_block, 0, st>>>(na);
    near_direct_kernel<<<grid, 32 * warps_per_block, 0, st>>>(na);
    p.launches += 2;
  }
  p.timer.end(tk, st);
  IFGFB_CUDA(cudaGetLastError());
  return IFGFB_OK;
}

// far field on phi * weights (operators.py:336-340); rank mode: the partial
// sums of the window's sources into the point-major exchange rows
static int far_launch(Plan& p, cudaStream_t st) {
  if (p.rank_mode)
    return far_apply(p, p.phiw, 8, p.kappa, 2, p.xfar, p.xfar + 2 * 16, st, 32);
  return far_apply(p, p.phiw, 8, p.kappa, 2, p.far_out, p.far_disp, st);
}

int potentials_from_phi(Plan& p, cudaStream_t st) {
  int rc = far_launch(p, st);
  if (rc) return rc;
  return near_launch(p, st);
}

static int pack_launch(Plan& p, const double* y, const double* phi_in,
                       cudaStream_t st) {
  const int n2 = p.n_c * p.n_c;
  const int threads = ((n2 + 31) / 32) * 32;
  const size_t sm = sizeof(double2) * 20 * n2;
  const int tk = p.timer.begin(K_PACK, st);
  pack_kernel<<<p.n_patches, threads, sm, st>>>(
      surf(p), reinterpret_cast<const double2*>(y),
      reinterpret_cast<const double2*>(phi_in), reinterpret_cast<double2*>(p.phi),
      reinterpret_cast<double2*>(p.phiw), reinterpret_cast<double2*>(p.pcoef),
      reinterpret_cast<double2*>(p.phi_pm));
  p.timer.end(tk, st);
  p.launches += 1;
  IFGFB_CUDA(cudaGetLastError());
  return IFGFB_OK;
}

static int assemble_launch(Plan& p, const double* y, double* out, cudaStream_t st) {
  const int n2 = p.n_c * p.n_c;
  const int threads = ((n2 + 31) / 32) * 32;
  const int p0 = p.t_lo() / n2, p1 = p.t_hi() / n2;
  if (p1 <= p0) return IFGFB_OK;
  AsmArgs aa{surf(p), reinterpret_cast<const double2*>(p.s_val),
             reinterpret_cast<const double2*>(p.d_val),
             reinterpret_cast<const double2*>(y),
             make_double2(p.eps_e[0], p.eps_e[1]), make_double2(p.mu_e[0], p.mu_e[1]),
             make_double2(p.eps_i[0], p.eps_i[1]), make_double2(p.mu_i[0], p.mu_i[1]),
             {make_double2(p.kappa[0], p.kappa[1]), make_double2(p.kappa[2], p.kappa[3])},
             p.omega, reinterpret_cast<double2*>(out), p0, 0, p.t_lo()};
  if (p.rank_mode) {
    aa.out = reinterpret_cast<double2*>(p.xout_mine);
    aa.out_pm = 1;
  }
  const int tk = p.timer.begin(K_ASSEMBLE, st);
  assemble_kernel<<<p1 - p0, threads, sizeof(double2) * 16 * n2, st>>>(aa);
  p.timer.end(tk, st);
  p.launches += 1;
  IFGFB_CUDA(cudaGetLastError());
  return IFGFB_OK;
}

int muller_far_phase(Plan& p, const double* y, cudaStream_t st) {
  p.launches = 0;
  IFGFB_RC(pack_launch(p, y, nullptr, st));
  return far_launch(p, st);
}

int muller_near_phase(Plan& p, const double* y, double* out, cudaStream_t st) {
  IFGFB_RC(near_launch(p, st));
  return assemble_launch(p, y, out, st);
}

int muller_apply(Plan& p, const double* y, double* out, cudaStream_t st) {
  IFGFB_RC(muller_far_phase(p, y, st));
  return muller_near_phase(p, y, out, st);
}

}  // namespace ifgfb

using namespace ifgfb;
#define CHECK_ARG IFGFB_CHECK_ARG
#define RC IFGFB_RC

extern "C" {

int ifgfb_plan_set_surface(ifgfb_plan* h, const ifgfb_surface_desc* d) {
  CHECK_ARG(h && d, "null argument");
  Plan& p = h->p;
  CHECK_ARG(!p.finalized, "plan already finalized");
  CHECK_ARG(d->n_c >= 2 && d->n_c <= MAXNC, "n_c out of supported range [2,16]");
  CHECK_ARG((int64_t)d->n_patches * d->n_c * d->n_c == p.n,
            "n_patches * n_c^2 != number of points");
  p.n_patches = d->n_patches;
  p.n_c = d->n_c;
  const size_t n = p.n, n2 = (size_t)d->n_c * d->n_c;
  // pack / assemble stage 20 resp. 16 complex n_c x n_c tiles in dynamic
  // shared memory: 54 KB at n_c = 13, 80 KB at n_c = 16 (above the 48 KB
  // default from n_c = 13)
  IFGFB_CUDA(cudaFuncSetAttribute(pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double2) * 20 * n2)));
  IFGFB_CUDA(cudaFuncSetAttribute(assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double2) * 16 * n2)));
  RC(dev_upload(p, &p.pts, d->points, 3 * n));
  RC(dev_upload(p, &p.nrm, d->normals, 3 * n));
  RC(dev_upload(p, &p.wq, d->weights, n));
  RC(dev_upload(p, &p.jac, d->jacobians, n));
  RC(dev_upload(p, &p.eu, d->e_u, 3 * n));
  RC(dev_upload(p, &p.ev, d->e_v, 3 * n));
  RC(dev_upload(p, &p.t1, d->tangent1, 3 * n));
  RC(dev_upload(p, &p.t2, d->tangent2, 3 * n));
  RC(dev_upload(p, &p.dmat, d->diff_matrix, n2));
  RC(dev_upload(p, &p.cmat, d->coeff_matrix, n2));
  for (int i = 0; i < 2; ++i) {
    p.eps_e[i] = d->eps_e[i];
    p.mu_e[i] = d->mu_e[i];
    p.eps_i[i] = d->eps_i[i];
    p.mu_i[i] = d->mu_i[i];
  }
  for (int i = 0; i < 4; ++i) p.kappa[i] = d->kappas[i];
  p.omega = d->omega;
  p.fd_step = d->fd_step;
  RC(dev_upload<double>(p, &p.phi, nullptr, 16 * n));
  RC(dev_upload<double>(p, &p.phiw, nullptr, 16 * n));
  RC(dev_upload<double>(p, &p.pcoef, nullptr, 16 * n));
  RC(dev_upload<double>(p, &p.phi_pm, nullptr, 32 * n));
  RC(dev_upload<double>(p, &p.far_out, nullptr, 32 * n));
  RC(dev_upload<double>(p, &p.far_disp, nullptr, 32 * n));
  RC(dev_upload<double>(p, &p.s_val, nullptr, 32 * n));
  RC(dev_upload<double>(p, &p.d_val, nullptr, 24 * n));
  RC(dev_upload<double>(p, &p.dev_y, nullptr, 8 * n));
  RC(dev_upload<double>(p, &p.dev_out, nullptr, 8 * n));
  IFGFB_CUDA(cudaMallocHost(&p.host_stage, sizeof(double) * 16 * n));
  p.has_surface = true;
  return IFGFB_OK;
}

int ifgfb_plan_set_near(ifgfb_plan* h, const ifgfb_near_desc* d) {
  CHECK_ARG(h && d, "null argument");
  Plan& p = h->p;
  CHECK_ARG(p.has_surface, "set_surface must precede set_near");
  const int n = p.n, n2 = p.n_c * p.n_c;
  std::vector<int> tmp(n + 1);
  for (int i = 0; i <= n; ++i) tmp[i] = (int)d->mom_off[i];
  CHECK_ARG(d->mom_off[n] == d->n_mom, "mom_off end != n_mom");
  RC(dev_upload(p, &p.mom_off, tmp.data(), tmp.size()));
  std::vector<int> pt(d->n_mom);
  for (int64_t i = 0; i < d->n_mom; ++i) {
    CHECK_ARG(d->mom_patch[i] >= 0 && d->mom_patch[i] < p.n_patches, "moment patch out of range");
    pt[i] = (int)d->mom_patch[i];
  }
  RC(dev_upload(p, &p.mom_patch, pt.data(), pt.size()));
  RC(dev_upload(p, &p.moments, d->moments, (size_t)d->n_mom * 4 * n2 * 2));
  for (int i = 0; i <= n; ++i) tmp[i] = (int)d->dir_off[i];
  CHECK_ARG(d->dir_off[n] == d->n_direct, "dir_off end != n_direct");
  RC(dev_upload(p, &p.dir_off, tmp.data(), tmp.size()));
  std::vector<int> ds(d->n_direct);
  for (int64_t i = 0; i < d->n_direct; ++i) {
    const int64_t c = d->dir_src[i];
    CHECK_ARG(c >= -(int64_t)n && c < n, "direct source out of range");
    ds[i] = (int)c;
  }
  RC(dev_upload(p, &p.dir_src, ds.data(), ds.size()));
  p.n_mom = d->n_mom;
  p.n_direct = d->n_direct;
  p.has_near = true;
  return IFGFB_OK;
}

// a partitioned plan computes rank-local partial sums: only the phase entry
// points (ifgfb_muller_far_phase / _near_phase, driven by the collective
// layer) may run it
static int whole_plan_state(const Plan& p) {
  if (!p.finalized || !p.has_near) {
    set_error("plan has no surface/near-field data");
    return IFGFB_ERR_STATE;
  }
  if (p.rank_mode) {
    set_error("plan is one rank's share (partitioned across ranks): use the far/near "
              "phase entry points with the rank exchange (DistributedMullerOperator)");
    return IFGFB_ERR_STATE;
  }
  return IFGFB_OK;
}

int ifgfb_potentials(ifgfb_plan* h, const double* phi, double* s_val,
                     double* d_val, void* stream) {
  CHECK_ARG(h && phi && s_val && d_val, "null argument");
  Plan& p = h->p;
  RC(whole_plan_state(p));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  p.launches = 0;
  RC(pack_launch(p, nullptr, phi, st));
  RC(potentials_from_phi(p, st));
  IFGFB_CUDA(cudaMemcpyAsync(s_val, p.s_val, sizeof(double2) * 16 * (size_t)p.n,
                             cudaMemcpyDeviceToDevice, st));
  IFGFB_CUDA(cudaMemcpyAsync(d_val, p.d_val, sizeof(double2) * 12 * (size_t)p.n,
                             cudaMemcpyDeviceToDevice, st));
  return IFGFB_OK;
}

int ifgfb_muller_apply(ifgfb_plan* h, const double* y, double* out, void* stream) {
  CHECK_ARG(h && y && out, "null argument");
  Plan& p = h->p;
  RC(whole_plan_state(p));
  return muller_apply(p, y, out, static_cast<cudaStream_t>(stream));
}

int ifgfb_muller_far_phase(ifgfb_plan* h, const double* y, void* stream) {
  CHECK_ARG(h && y, "null argument");
  Plan& p = h->p;
  if (!p.finalized || !p.has_near) {
    set_error("plan has no surface/near-field data");
    return IFGFB_ERR_STATE;
  }
  return muller_far_phase(p, y, static_cast<cudaStream_t>(stream));
}

int ifgfb_muller_near_phase(ifgfb_plan* h, const double* y, double* out, void* stream) {
  CHECK_ARG(h && y && (out || h->p.rank_mode), "null argument");
  Plan& p = h->p;
  if (!p.finalized || !p.has_near) {
    set_error("plan has no surface/near-field data");
    return IFGFB_ERR_STATE;
  }
  return muller_near_phase(p, y, out, static_cast<cudaStream_t>(stream));
}

int ifgfb_plan_set_rank(ifgfb_plan* h, const ifgfb_rank_desc* d) {
  CHECK_ARG(h && d, "null argument");
  Plan& p = h->p;
  CHECK_ARG(p.finalized && p.has_near, "finalize the plan (with surface and near field) first");
  CHECK_ARG(!p.rank_mode, "rank already set");
  CHECK_ARG(d->n_ranks >= 1 && 0 <= d->rank && d->rank < d->n_ranks, "bad rank");
  const int n2 = p.n_c * p.n_c;
  CHECK_ARG(0 <= d->target_lo && d->target_lo <= d->target_hi && d->target_hi <= p.n,
            "target range out of bounds");
  CHECK_ARG(d->target_lo % n2 == 0 && d->target_hi % n2 == 0,
            "target range must be patch aligned");
  CHECK_ARG(d->target_lo == (int64_t)d->rank * d->chunk &&
                d->target_hi - d->target_lo <= d->chunk,
            "targets must be rank * chunk .. (rank + 1) * chunk (clipped to N)");
  CHECK_ARG((int64_t)d->n_ranks * d->chunk >= p.n, "n_ranks * chunk must cover N");
  const size_t rows = (size_t)d->n_ranks * d->chunk;
  RC(dev_alloc(p, &p.xfar, rows * 32 * 2));
  RC(dev_alloc(p, &p.xfar_mine, (size_t)d->chunk * 32 * 2));
  RC(dev_alloc(p, &p.xout_mine, (size_t)d->chunk * 4 * 2));
  RC(dev_alloc(p, &p.xout, rows * 4 * 2));
  // padding rows (>= N) are never written: zero once
  IFGFB_CUDA(cudaMemset(p.xfar, 0, rows * 32 * 2 * sizeof(double)));
  IFGFB_CUDA(cudaMemset(p.xout_mine, 0, (size_t)d->chunk * 4 * 2 * sizeof(double)));
  p.rank = d->rank;
  p.n_ranks = d->n_ranks;
  p.chunk = d->chunk;
  p.part_t_lo = (int)d->target_lo;
  p.part_t_hi = (int)d->target_hi;
  p.rank_mode = true;
  return IFGFB_OK;
}

int ifgfb_plan_rank_buffers(ifgfb_plan* h, double** xfar, double** xfar_mine,
                            double** xout_mine, double** xout, int64_t* chunk) {
  CHECK_ARG(h && xfar && xfar_mine && xout_mine && xout && chunk, "null argument");
  Plan& p = h->p;
  if (!p.rank_mode) {
    set_error("plan has no rank (ifgfb_plan_set_rank)");
    return IFGFB_ERR_STATE;
  }
  *xfar = p.xfar;
  *xfar_mine = p.xfar_mine;
  *xout_mine = p.xout_mine;
  *xout = p.xout;
  *chunk = p.chunk;
  return IFGFB_OK;
}

int ifgfb_rank_unpack(ifgfb_plan* h, double* out, void* stream) {
  CHECK_ARG(h && out, "null argument");
  Plan& p = h->p;
  if (!p.rank_mode) {
    set_error("plan has no rank (ifgfb_plan_set_rank)");
    return IFGFB_ERR_STATE;
  }
  const int threads = 256;
  rank_unpack_kernel<<<(4 * p.n + threads - 1) / threads, threads, 0,
                       static_cast<cudaStream_t>(stream)>>>(
      p.n, reinterpret_cast<const double2*>(p.xout), reinterpret_cast<double2*>(out));
  p.launches += 1;
  IFGFB_CUDA(cudaGetLastError());
  return IFGFB_OK;
}

int ifgfb_muller_apply_host(ifgfb_plan* h, const double* y_host, double* out_host,
                            void* stream) {
  CHECK_ARG(h && y_host && out_host, "null argument");
  Plan& p = h->p;
  RC(whole_plan_state(p));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t bytes = sizeof(double) * 8 * (size_t)p.n;
  memcpy(p.host_stage, y_host, bytes);
  IFGFB_CUDA(cudaMemcpyAsync(p.dev_y, p.host_stage, bytes, cudaMemcpyHostToDevice, st));
  RC(muller_apply(p, p.dev_y, p.dev_out, st));
  IFGFB_CUDA(cudaMemcpyAsync(p.host_stage + 8 * (size_t)p.n, p.dev_out, bytes,
                             cudaMemcpyDeviceToHost, st));
  IFGFB_CUDA(cudaStreamSynchronize(st));
  memcpy(out_host, p.host_stage + 8 * (size_t)p.n, bytes);
  return IFGFB_OK;
}

}  // extern "C"
