// Plan-time singular moments on the device: for every
// (target, singular patch) pair the integrals
//   beta_s[k][m][n] = sum_ij put[m][i] G_k(x, y_ij) J_ij pvw[j][n]
//   beta_d[k][m][n] = same with dG_k/dn_x
// on the 48 x 48 graded grid clustered at the pair's closest point (u0, v0).
// Reference: quadrature.py:271-331 (compute_moments), :163-228 (graded_map,
// clustered_nodes); host restatement nearfield.compute_moments.
//
// One CTA per pair.  The grid is walked in chunks of RC rows: kernel values
// of a chunk (4 kinds: S/D x 2 wavenumbers) go to shared memory, are
// contracted over j with pvw, then over the chunk's i with put into
// per-thread accumulators.  FP64 throughout; the contraction order differs
// from numpy's ((put @ K) @ pvw) by rounding only.
#include "common.cuh"

namespace ifgfb {

namespace {

constexpr int MOM_THREADS = 256;
constexpr int RC = 16;          // grid rows per chunk

struct MomArgs {
  const double* txyz; const double* tnrm; const int* patch; const double* uv;
  const double* cf;             // n_patches x 9 x np x np
  const double* base; const double* wb;
  int np_, nc, nb, d;
  double kr[2], ki[2];
  double2* out;                 // pair x 4 x nc x nc
  int64_t pair0;
  const double* nodes;          // optional: pair x 4 x nb (xi_u, dxi_u, xi_v, dxi_v)
  int tail_u, tail_v;           // first column of the 8-lane gemm order (exact mode)
};

// Exact mode (nodes given): the geometry at the clustered grid reproduces the
// reference's float64 values bit for bit.  The graded map (np.power) comes
// from the host; the device replays numpy's elementwise operation order
// without contraction (chebyshev_basis, np.cross, norm, sum over axis 0,
// einsum "cbij,bc->bij") and OpenBLAS's dgemm order for the two position
// products (tu @ coeff, (.) @ tv^T): a sequential FMA chain over k per
// column, except the columns of an N-tail (>= tail) which OpenBLAS 0.3.30
// (SkylakeX) reduces as 8 k-interleaved FMA lanes + a pairwise tree
// (verified for n_p = 8, 10, 20 in this build's tests).  This matters because
// (x - y(u, v)).n_x loses ~8 digits at the clustered nodes: any other
// rounding of y moves beta_d by ~1e-7.
__device__ __forceinline__ double dot_exact(const double* a, int sa, const double* b, int sb,
                                            int k, bool tail) {
  if (!tail) {
    double s = 0.0;
    for (int m = 0; m < k; ++m) s = __fma_rn(a[m * sa], b[m * sb], s);
    return s;
  }
  double q[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int m = 0; m < k; ++m) q[m & 7] = __fma_rn(a[m * sa], b[m * sb], q[m & 7]);
  return __dadd_rn(__dadd_rn(__dadd_rn(q[0], q[1]), __dadd_rn(q[2], q[3])),
                   __dadd_rn(__dadd_rn(q[4], q[5]), __dadd_rn(q[6], q[7])));
}

__device__ __forceinline__ double nu(double tau, double d) {
  const double q = (M_PI - tau) / M_PI;
  return (1.0 / d - 0.5) * (q * q * q) + (tau - M_PI) / (d * M_PI) + 0.5;
}
__device__ __forceinline__ double nu_prime(double tau, double d) {
  const double q = M_PI - tau;
  return 3.0 * (0.5 - 1.0 / d) * (q * q) / (M_PI * M_PI * M_PI) + 1.0 / (d * M_PI);
}
__device__ __forceinline__ double ipow(double x, int d) {
  double r = 1.0;
  for (int i = 0; i < d; ++i) r *= x;
  return r;
}
// graded_map and its derivative (reference quadrature.py:163-200)
__device__ __forceinline__ void graded(double tau, int d, double& w, double& dw) {
  tau = fmin(fmax(tau, 0.0), 2.0 * M_PI);
  const double dd = (double)d;
  const double n1 = nu(tau, dd), n2 = nu(2.0 * M_PI - tau, dd);
  const double a = ipow(n1, d), b = ipow(n2, d);
  w = 2.0 * M_PI * a / (a + b);
  const double dn1 = nu_prime(tau, dd), dn2 = -nu_prime(2.0 * M_PI - tau, dd);
  const double da = dd * ipow(n1, d - 1) * dn1, db = dd * ipow(n2, d - 1) * dn2;
  dw = 2.0 * M_PI * (da * b - a * db) / ((a + b) * (a + b));
}
// clustered_nodes (reference quadrature.py:203-228): base node t remapped to
// accumulate at alpha, and its derivative
__device__ __forceinline__ void clustered(double alpha, double t, int d, double& xi,
                                          double& dxi) {
  double w, dw;
  if (alpha >= 1.0 - 1e-12) {
    graded(M_PI * fabs(t - 1.0) / 2.0, d, w, dw);
    xi = 1.0 - (2.0 / M_PI) * w;
    dxi = dw;
  } else if (alpha <= -1.0 + 1e-12) {
    graded(M_PI * fabs(t + 1.0) / 2.0, d, w, dw);
    xi = -1.0 + (2.0 / M_PI) * w;
    dxi = dw;
  } else {
    const double sg = (t > 0.0) ? 1.0 : (t < 0.0 ? -1.0 : 0.0);
    graded(M_PI * fabs(t), d, w, dw);
    xi = alpha + (sg - alpha) / M_PI * w;
    dxi = (1.0 - alpha * sg) * dw;
  }
}

__global__ void __launch_bounds__(MOM_THREADS) moments_kernel(MomArgs a) {
  extern __shared__ double sm[];
  const int np_ = a.np_, nc = a.nc, nb = a.nb, tid = threadIdx.x;
  const int64_t pair = a.pair0 + blockIdx.x;
  // shared layout
  double* tu = sm;                         // nb x np
  double* tv = tu + nb * np_;              // nb x np
  double* put = tv + nb * np_;             // nc x nb  (T_m(xu_i) dxu_i wb_i)
  double* pvw = put + nc * nb;             // nb x nc
  double* cf = pvw + nb * nc;              // 9 x np x np
  double* A = cf + 9 * np_ * np_;          // 9 x nb x np
  double2* K = reinterpret_cast<double2*>(A + 9 * nb * np_);   // 4 x RC x nb
  double2* Y = K + 4 * RC * nb;            // 4 x RC x nc
  const int p = a.patch[pair];
  const double u0 = a.uv[2 * pair], v0 = a.uv[2 * pair + 1];
  for (int e = tid; e < 9 * np_ * np_; e += blockDim.x)
    cf[e] = a.cf[(size_t)p * 9 * np_ * np_ + e];
  for (int e = tid; e < 2 * nb; e += blockDim.x) {
    const int i = e % nb;
    const bool isv = e >= nb;
    double xi, dxi;
    if (a.nodes) {
      const double* nd = a.nodes + ((size_t)blockIdx.x * 4 + (isv ? 2 : 0)) * nb;
      xi = nd[i];
      dxi = nd[nb + i];
    } else {
      clustered(isv ? v0 : u0, a.base[i], a.d, xi, dxi);
    }
    // reference chebyshev_basis: out[i] = 2.0 * x * out[i-1] - out[i-2]
    const double x2 = 2.0 * xi;   // exact
    double* T = (isv ? tv : tu) + i * np_;
    T[0] = 1.0;
    if (np_ > 1) T[1] = xi;
    for (int m = 2; m < np_; ++m) T[m] = __dsub_rn(__dmul_rn(x2, T[m - 1]), T[m - 2]);
    const double sc = __dmul_rn(dxi, a.wb[i]);
    double t0 = 1.0, t1 = xi;
    for (int m = 0; m < nc; ++m) {
      double tm;
      if (m == 0) tm = 1.0;
      else if (m == 1) tm = xi;
      else { tm = __dsub_rn(__dmul_rn(x2, t1), t0); t0 = t1; t1 = tm; }
      if (isv) pvw[i * nc + m] = __dmul_rn(tm, sc);
      else put[m * nb + i] = __dmul_rn(tm, sc);
    }
  }
  __syncthreads();
  // A[c][i][n] = sum_m tu[i][m] cf[c][m][n]  (numpy: tu @ cf[c])
  for (int e = tid; e < 9 * nb * np_; e += blockDim.x) {
    const int n = e % np_, i = (e / np_) % nb, c = e / (np_ * nb);
    A[e] = dot_exact(tu + i * np_, 1, cf + c * np_ * np_ + n, np_, np_, n >= a.tail_u);
  }
  __syncthreads();
  const double x0 = a.txyz[3 * pair], x1 = a.txyz[3 * pair + 1], x2 = a.txyz[3 * pair + 2];
  const double n0 = a.tnrm[3 * pair], n1 = a.tnrm[3 * pair + 1], n2 = a.tnrm[3 * pair + 2];
  const int nout = 4 * nc * nc;
  double2 acc[2] = {make_double2(0, 0), make_double2(0, 0)};
  for (int i0 = 0; i0 < nb; i0 += RC) {
    const int rc = min(RC, nb - i0);
    for (int e = tid; e < rc * nb; e += blockDim.x) {
      const int ii = e / nb, j = e % nb, i = i0 + ii;
      double g[9];
      const bool tl = j >= a.tail_v;
#pragma unroll
      for (int c = 0; c < 9; ++c)
        g[c] = dot_exact(A + (c * nb + i) * np_, 1, tv + j * np_, 1, np_, tl);
      // g[0..2] position, g[3..5] e_u, g[6..8] e_v; numpy's np.cross and
      // norm / sum orders, no contraction (reference quadrature.py:310-317)
      const double cx = __dsub_rn(__dmul_rn(g[4], g[8]), __dmul_rn(g[5], g[7]));
      const double cy = __dsub_rn(__dmul_rn(g[5], g[6]), __dmul_rn(g[3], g[8]));
      const double cz = __dsub_rn(__dmul_rn(g[3], g[7]), __dmul_rn(g[4], g[6]));
      const double jac = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)),
                                        __dmul_rn(cz, cz)));
      const double dx = __dsub_rn(x0, g[0]), dy = __dsub_rn(x1, g[1]), dz = __dsub_rn(x2, g[2]);
      const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                  __dmul_rn(dz, dz));
      const double r = sqrt(r2);
      const double ndx = __dadd_rn(__dadd_rn(__dmul_rn(dx, n0), __dmul_rn(dy, n1)),
                                   __dmul_rn(dz, n2));
      // phase = exp(1j kappa r) / (4 pi r); numpy divides a complex by a real
      // as a multiply by the reciprocal (Smith's rule with a zero imaginary part)
      const double inv4pr = __ddiv_rn(1.0, __dmul_rn(4.0 * M_PI, r));
      const double rr = __dmul_rn(r, r);
      const double inv_rr = __ddiv_rn(1.0, rr);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double tre = -__dmul_rn(a.ki[k], r), tim = __dmul_rn(a.kr[k], r);   // 1j kappa r
        double s, c;
        sincos(tim, &s, &c);
        const double damp = a.ki[k] != 0.0 ? exp(tre) : 1.0;
        const double2 ph = make_double2(__dmul_rn(__dmul_rn(damp, c), inv4pr),
                                        __dmul_rn(__dmul_rn(damp, s), inv4pr));
        const double2 ks = make_double2(__dmul_rn(ph.x, jac), __dmul_rn(ph.y, jac));
        // ndx * (1j kappa r - 1) / r**2
        const double2 fac = make_double2(__dmul_rn(__dmul_rn(ndx, __dsub_rn(tre, 1.0)), inv_rr),
                                         __dmul_rn(__dmul_rn(ndx, tim), inv_rr));
        K[(k * RC + ii) * nb + j] = ks;
        K[((2 + k) * RC + ii) * nb + j] =
            make_double2(__fma_rn(ks.x, fac.x, -__dmul_rn(ks.y, fac.y)),
                         __fma_rn(ks.x, fac.y, __dmul_rn(ks.y, fac.x)));
      }
    }
    __syncthreads();
    // Y[q][ii][n] = sum_j K[q][ii][j] pvw[j][n]
    for (int e = tid; e < 4 * rc * nc; e += blockDim.x) {
      const int n = e % nc, ii = (e / nc) % rc, q = e / (nc * rc);
      const double2* Kr = K + (q * RC + ii) * nb;
      double2 s = make_double2(0.0, 0.0);
      for (int j = 0; j < nb; ++j) {
        const double w = pvw[j * nc + n];
        s.x += Kr[j].x * w;
        s.y += Kr[j].y * w;
      }
      Y[(q * RC + ii) * nc + n] = s;
    }
    __syncthreads();
    // acc[q][m][n] += sum_ii put[m][i0+ii] Y[q][ii][n]
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = tid + h * MOM_THREADS;
      if (e < nout) {
        const int n = e % nc, m = (e / nc) % nc, q = e / (nc * nc);
        for (int ii = 0; ii < rc; ++ii) {
          const double w = put[m * nb + i0 + ii];
          const double2 y = Y[(q * RC + ii) * nc + n];
          acc[h].x += w * y.x;
          acc[h].y += w * y.y;
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int e = tid + h * MOM_THREADS;
    if (e < nout) a.out[(size_t)blockIdx.x * nout + e] = acc[h];
  }
}

size_t moments_smem(int np_, int nc, int nb) {
  return sizeof(double) * (2 * nb * np_ + 2 * nc * nb + 9 * np_ * np_ + 9 * nb * np_) +
         sizeof(double2) * (4 * RC * nb + 4 * RC * nc);
}

}  // namespace

}  // namespace ifgfb

extern "C" {

int ifgfb_singular_moments(const ifgfb_moment_desc* m, double* out) {
  using namespace ifgfb;
  if (!m || !out) { set_error("ifgfb_singular_moments: null argument"); return IFGFB_ERR_ARG; }
  if (m->gemm_tail_u < 0 || m->gemm_tail_v < 0) {
    set_error("ifgfb_singular_moments: negative gemm tail");
    return IFGFB_ERR_ARG;
  }
  if (m->n_pairs < 0 || m->n_p < 1 || m->n_p > 32 || m->n_c < 1 || m->n_c > 16 ||
      m->n_beta < 1 || m->n_beta > 128 || m->grading < 2 || m->n_patches < 1) {
    set_error("ifgfb_singular_moments: sizes out of range (n_p <= 32, n_c <= 16, "
              "n_beta <= 128, grading >= 2)");
    return IFGFB_ERR_ARG;
  }
  if (m->n_pairs == 0) return IFGFB_OK;
  for (int64_t i = 0; i < m->n_pairs; ++i)
    if (m->patch[i] < 0 || m->patch[i] >= m->n_patches) {
      set_error("ifgfb_singular_moments: patch index out of range");
      return IFGFB_ERR_ARG;
    }
  const int np_ = m->n_p, nc = m->n_c, nb = m->n_beta;
  const size_t smem = moments_smem(np_, nc, nb);
  if (smem > 227 * 1024) { set_error("ifgfb_singular_moments: shared memory"); return IFGFB_ERR_ARG; }
  IFGFB_CUDA(cudaFuncSetAttribute(moments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  const int64_t chunk = 1 << 16;
  const int64_t n = m->n_pairs;
  const size_t out_per = (size_t)4 * nc * nc;   // complex per pair
  const size_t cf_n = (size_t)m->n_patches * 9 * np_ * np_;
  // device copies (whole inputs; outputs chunked)
  double *d_x = nullptr, *d_n = nullptr, *d_uv = nullptr, *d_cf = nullptr, *d_b = nullptr,
         *d_w = nullptr;
  int* d_p = nullptr;
  double2* d_out = nullptr;
  int rc = IFGFB_OK;
  auto fail = [&](cudaError_t e, const char* what) {
    set_error(std::string("ifgfb_singular_moments: ") + what + ": " + cudaGetErrorString(e));
    rc = IFGFB_ERR_CUDA;
  };
  cudaError_t e;
  std::vector<int> pidx(m->patch, m->patch + n);
  if ((e = cudaMalloc(&d_x, n * 3 * sizeof(double))) ||
      (e = cudaMalloc(&d_n, n * 3 * sizeof(double))) ||
      (e = cudaMalloc(&d_uv, n * 2 * sizeof(double))) ||
      (e = cudaMalloc(&d_p, n * sizeof(int))) ||
      (e = cudaMalloc(&d_cf, cf_n * sizeof(double))) ||
      (e = cudaMalloc(&d_b, nb * sizeof(double))) ||
      (e = cudaMalloc(&d_w, nb * sizeof(double))) ||
      (e = cudaMalloc(&d_out, std::min<int64_t>(n, chunk) * out_per * sizeof(double2)))) {
    fail(e, "cudaMalloc");
  } else if ((e = cudaMemcpy(d_x, m->target_xyz, n * 3 * sizeof(double), cudaMemcpyHostToDevice)) ||
             (e = cudaMemcpy(d_n, m->target_nrm, n * 3 * sizeof(double), cudaMemcpyHostToDevice)) ||
             (e = cudaMemcpy(d_uv, m->uv, n * 2 * sizeof(double), cudaMemcpyHostToDevice)) ||
             (e = cudaMemcpy(d_p, pidx.data(), n * sizeof(int), cudaMemcpyHostToDevice)) ||
             (e = cudaMemcpy(d_cf, m->patch_coeffs, cf_n * sizeof(double), cudaMemcpyHostToDevice)) ||
             (e = cudaMemcpy(d_b, m->base, nb * sizeof(double), cudaMemcpyHostToDevice)) ||
             (e = cudaMemcpy(d_w, m->weights, nb * sizeof(double), cudaMemcpyHostToDevice))) {
    fail(e, "cudaMemcpy");
  } else {
    MomArgs a{d_x, d_n, d_p, d_uv, d_cf, d_b, d_w, np_, nc, nb, m->grading,
              {m->kappas[0], m->kappas[2]}, {m->kappas[1], m->kappas[3]}, d_out, 0,
              nullptr, m->gemm_tail_u > 0 ? m->gemm_tail_u : np_,
              m->gemm_tail_v > 0 ? m->gemm_tail_v : nb};
    double* d_nodes = nullptr;
    if (m->nodes &&
        (e = cudaMalloc(&d_nodes, std::min<int64_t>(n, chunk) * 4 * nb * sizeof(double))))
      fail(e, "cudaMalloc");
    for (int64_t c0 = 0; c0 < n && rc == IFGFB_OK; c0 += chunk) {
      const int64_t cn = std::min(chunk, n - c0);
      a.pair0 = c0;
      if (m->nodes) {
        if ((e = cudaMemcpy(d_nodes, m->nodes + (size_t)c0 * 4 * nb,
                            cn * 4 * nb * sizeof(double), cudaMemcpyHostToDevice))) {
          fail(e, "cudaMemcpy");
          break;
        }
        a.nodes = d_nodes;
      }
      moments_kernel<<<(unsigned)cn, MOM_THREADS, smem>>>(a);
      if ((e = cudaGetLastError()) ||
          (e = cudaMemcpy(out + (size_t)c0 * out_per * 2, d_out, cn * out_per * sizeof(double2),
                          cudaMemcpyDeviceToHost)))
        fail(e, "moments_kernel");
    }
    cudaFree(d_nodes);
  }
  cudaFree(d_x); cudaFree(d_n); cudaFree(d_uv); cudaFree(d_p); cudaFree(d_cf);
  cudaFree(d_b); cudaFree(d_w); cudaFree(d_out);
  return rc;
}

}  // extern "C"
