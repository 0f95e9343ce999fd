// Off-surface field evaluation from solved surface currents (reference
// reference.py:285-312 _layer_fields, used by evaluate_fields :315-347):
//   curl S[m], curl S[j], curlcurl S[m], curlcurl S[j]
// at M targets from N quadrature sources with the Helmholtz kernel
// G = exp(i kappa r) / (4 pi r), densities pre-multiplied by the quadrature
// weights.  A dense O(M N) reduction: FP64 ALU bound (one sincos, one sqrt,
// one division and ~200 FLOP per (target, source) pair).
//
// Layout: grid (target blocks of FLD_THREADS, source chunks).  Each CTA stages
// its chunk's sources (position, m w, j w = 15 doubles) through shared memory
// in tiles of FLD_THREADS; each thread owns one target and keeps the 4 x 3
// complex sums plus the minimum distance in registers.  Chunk partials are
// reduced over chunks in a fixed order (deterministic, run-to-run bitwise).
#include "common.cuh"

#include <algorithm>
#include <cmath>

namespace ifgfb {

constexpr int FLD_THREADS = 128;
constexpr int FLD_VALS = 24;        // 4 fields x 3 components x (re, im)
constexpr int FLD_PART = FLD_VALS + 1;   // + minimum source distance

struct FieldArgs {
  const double* tgt;     // M x 3
  const double* src;     // N x 15: x y z, m_w (3 complex), j_w (3 complex)
  int64_t n_tgt, n_src, chunk;
  double kr, ki;         // kappa
  double* part;          // [n_chunks][FLD_PART][M]
};

__global__ void __launch_bounds__(FLD_THREADS) layer_fields_kernel(FieldArgs a) {
  __shared__ double s[FLD_THREADS * 15];
  const int64_t t = blockIdx.x * (int64_t)FLD_THREADS + threadIdx.x;
  const bool live = t < a.n_tgt;
  double x0 = 0.0, x1 = 0.0, x2 = 0.0;
  if (live) { x0 = a.tgt[3 * t]; x1 = a.tgt[3 * t + 1]; x2 = a.tgt[3 * t + 2]; }
  double2 cm[3], cj[3], qm[3], qj[3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
    cm[c] = cj[c] = qm[c] = qj[c] = make_double2(0.0, 0.0);
  double dmin = INFINITY;
  const double k2r = a.kr * a.kr - a.ki * a.ki, k2i = 2.0 * a.kr * a.ki;   // kappa^2
  const int64_t s0 = blockIdx.y * a.chunk;
  const int64_t s1 = min(s0 + a.chunk, a.n_src);
  for (int64_t b = s0; b < s1; b += FLD_THREADS) {
    const int nb = (int)min((int64_t)FLD_THREADS, s1 - b);
    __syncthreads();
    for (int e = threadIdx.x; e < nb * 15; e += FLD_THREADS) s[e] = a.src[b * 15 + e];
    __syncthreads();
    if (!live) continue;
    for (int q = 0; q < nb; ++q) {
      const double* p = s + 15 * q;
      const double d0 = x0 - p[0], d1 = x1 - p[1], d2 = x2 - p[2];
      const double r2 = d0 * d0 + d1 * d1 + d2 * d2;
      const double r = sqrt(r2);
      dmin = fmin(dmin, r);
      const double ir = 1.0 / r, ir2 = ir * ir;
      // g = exp(i kappa r) / (4 pi r)
      double sn, cs;
      sincos(a.kr * r, &sn, &cs);
      const double damp = a.ki != 0.0 ? exp(-a.ki * r) : 1.0;
      const double gs = damp * ir * 0.07957747154594767;   // 1 / (4 pi)
      const double2 g = make_double2(gs * cs, gs * sn);
      // a = (i kappa r - 1) / r^2, bb = (-kappa^2 r^2 - 3 i kappa r + 3) / r^2
      const double2 ikr = make_double2(-a.ki * r, a.kr * r);
      const double2 av = make_double2((ikr.x - 1.0) * ir2, ikr.y * ir2);
      const double2 bb = make_double2((-k2r * r2 - 3.0 * ikr.x + 3.0) * ir2,
                                      (-k2i * r2 - 3.0 * ikr.y) * ir2);
      const double2 ga = cmul(g, av);                                  // grad G = ga * dx
      const double2 c1 = cmul(g, make_double2(av.x + k2r, av.y + k2i));  // G (a + kappa^2)
      const double2 c2 = cmul(g, make_double2(bb.x * ir2, bb.y * ir2));  // G bb / r^2
      const double dx[3] = {d0, d1, d2};
#pragma unroll
      for (int f = 0; f < 2; ++f) {   // f = 0: m, f = 1: j
        const double2 w[3] = {make_double2(p[3 + 6 * f], p[4 + 6 * f]),
                              make_double2(p[5 + 6 * f], p[6 + 6 * f]),
                              make_double2(p[7 + 6 * f], p[8 + 6 * f])};
        double2* cu = f ? cj : cm;
        double2* cc = f ? qj : qm;
        // (ga dx) x w
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int i1 = (c + 1) % 3, i2 = (c + 2) % 3;
          const double2 v = make_double2(dx[i1] * w[i2].x - dx[i2] * w[i1].x,
                                         dx[i1] * w[i2].y - dx[i2] * w[i1].y);
          const double2 u = cmul(ga, v);
          cu[c].x += u.x; cu[c].y += u.y;
        }
        // c1 w + c2 (dx . w) dx
        const double2 dw = make_double2(d0 * w[0].x + d1 * w[1].x + d2 * w[2].x,
                                        d0 * w[0].y + d1 * w[1].y + d2 * w[2].y);
        const double2 c2dw = cmul(c2, dw);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double2 u = cmul(c1, w[c]);
          cc[c].x += u.x + c2dw.x * dx[c];
          cc[c].y += u.y + c2dw.y * dx[c];
        }
      }
    }
  }
  if (!live) return;
  double* out = a.part + (size_t)blockIdx.y * FLD_PART * a.n_tgt + t;
  const double2* rows[4] = {cm, cj, qm, qj};
#pragma unroll
  for (int f = 0; f < 4; ++f)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      out[(size_t)(6 * f + 2 * c) * a.n_tgt] = rows[f][c].x;
      out[(size_t)(6 * f + 2 * c + 1) * a.n_tgt] = rows[f][c].y;
    }
  out[(size_t)FLD_VALS * a.n_tgt] = dmin;
}

// out[f][t][c] (complex) = sum over chunks in order; dmin = min over chunks
__global__ void layer_fields_reduce(const double* __restrict__ part, int n_chunks,
                                    int64_t n_tgt, double* __restrict__ out,
                                    double* __restrict__ dmin) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n_tgt * FLD_PART) return;
  const int v = (int)(idx / n_tgt);
  const int64_t t = idx - (int64_t)v * n_tgt;
  const size_t stride = (size_t)FLD_PART * n_tgt;
  if (v == FLD_VALS) {
    double m = INFINITY;
    for (int c = 0; c < n_chunks; ++c) m = fmin(m, part[c * stride + idx]);
    dmin[t] = m;
    return;
  }
  double acc = 0.0;
  for (int c = 0; c < n_chunks; ++c) acc += part[c * stride + idx];
  const int f = v / 6, rem = v % 6;   // rem = 2 * component + (re|im)
  out[((size_t)f * n_tgt + t) * 6 + rem] = acc;
}

}  // namespace ifgfb

extern "C" int ifgfb_layer_fields(int64_t n_src, const double* src, int64_t n_tgt,
                                  const double* tgt, const double* kappa, double* out,
                                  double* min_dist) {
  using namespace ifgfb;
  if (!src || !tgt || !kappa || !out) {
    set_error("ifgfb_layer_fields: null argument");
    return IFGFB_ERR_ARG;
  }
  if (n_src < 0 || n_tgt < 0) {
    set_error("ifgfb_layer_fields: negative size");
    return IFGFB_ERR_ARG;
  }
  if (n_tgt == 0) return IFGFB_OK;
  if (n_src == 0) {
    std::fill(out, out + (size_t)n_tgt * FLD_VALS, 0.0);
    if (min_dist) std::fill(min_dist, min_dist + n_tgt, INFINITY);
    return IFGFB_OK;
  }
  int dev = 0, n_sm = 148;
  IFGFB_CUDA(cudaGetDevice(&dev));
  IFGFB_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  const int64_t tb = (n_tgt + FLD_THREADS - 1) / FLD_THREADS;
  // about 4 resident CTAs per SM in total; chunks of >= FLD_THREADS sources
  int64_t n_chunks = std::max<int64_t>(1, (4 * (int64_t)n_sm + tb - 1) / tb);
  n_chunks = std::min<int64_t>(n_chunks, (n_src + FLD_THREADS - 1) / FLD_THREADS);
  n_chunks = std::min<int64_t>(n_chunks, 65535);
  const int64_t chunk = (n_src + n_chunks - 1) / n_chunks;
  n_chunks = (n_src + chunk - 1) / chunk;
  double *d_src = nullptr, *d_tgt = nullptr, *d_part = nullptr, *d_out = nullptr,
         *d_min = nullptr;
  int rc = IFGFB_OK;
  cudaError_t e;
  if ((e = cudaMalloc(&d_src, n_src * 15 * sizeof(double))) ||
      (e = cudaMalloc(&d_tgt, n_tgt * 3 * sizeof(double))) ||
      (e = cudaMalloc(&d_part, n_chunks * FLD_PART * n_tgt * sizeof(double))) ||
      (e = cudaMalloc(&d_out, n_tgt * FLD_VALS * sizeof(double))) ||
      (e = cudaMalloc(&d_min, n_tgt * sizeof(double))) ||
      (e = cudaMemcpy(d_src, src, n_src * 15 * sizeof(double), cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(d_tgt, tgt, n_tgt * 3 * sizeof(double), cudaMemcpyHostToDevice))) {
    set_error(std::string("ifgfb_layer_fields: ") + cudaGetErrorString(e));
    rc = IFGFB_ERR_CUDA;
  } else {
    FieldArgs a{d_tgt, d_src, n_tgt, n_src, chunk, kappa[0], kappa[1], d_part};
    layer_fields_kernel<<<dim3((unsigned)tb, (unsigned)n_chunks), FLD_THREADS>>>(a);
    const int64_t nr = n_tgt * FLD_PART;
    layer_fields_reduce<<<(unsigned)((nr + 255) / 256), 256>>>(d_part, (int)n_chunks, n_tgt,
                                                             d_out, d_min);
    if ((e = cudaGetLastError()) ||
        (e = cudaMemcpy(out, d_out, n_tgt * FLD_VALS * sizeof(double), cudaMemcpyDeviceToHost)) ||
        (min_dist && (e = cudaMemcpy(min_dist, d_min, n_tgt * sizeof(double),
                                     cudaMemcpyDeviceToHost)))) {
      set_error(std::string("ifgfb_layer_fields: ") + cudaGetErrorString(e));
      rc = IFGFB_ERR_CUDA;
    }
  }
  cudaFree(d_src); cudaFree(d_tgt); cudaFree(d_part); cudaFree(d_out); cudaFree(d_min);
  return rc;
}
