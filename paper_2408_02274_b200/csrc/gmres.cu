// GMRES vector work on device (K8): modified Gram-Schmidt Arnoldi step with
// device-resident Hessenberg column (one host sync per iteration, for the
// Givens rotations that stay on the host exactly as the reference does),
// basis combination x = V^T y, and plain BLAS-1 primitives.
//
// Reference: solver.py:58-66 (MGS), :91-92 (x = basis[:k].T @ y).
// All reductions use a fixed grid and fixed order: bitwise deterministic.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace ifgfb {

constexpr int RED_BLOCKS = 296;   // 2 x 148 SMs
constexpr int RED_THREADS = 256;

__device__ __forceinline__ double2 block_sum2(double re, double im) {
  __shared__ double sr[RED_THREADS / 32], si[RED_THREADS / 32];
  re = warp_sum(re);
  im = warp_sum(im);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sr[w] = re; si[w] = im; }
  __syncthreads();
  double2 r = make_double2(0, 0);
  if (w == 0) {
    re = l < RED_THREADS / 32 ? sr[l] : 0.0;
    im = l < RED_THREADS / 32 ? si[l] : 0.0;
    r = make_double2(warp_sum(re), warp_sum(im));
  }
  __syncthreads();
  return r;
}

// w -= h[prev] * vp (if vp), then partial[b] = sum conj(vc) w (vc == null:
// partial = sum |w|^2).  Basis rows are plain pointers: device memory or
// pinned host memory (directly addressable under UVA) for spilled rows.
__global__ void __launch_bounds__(RED_THREADS) axpy_dot_kernel(
    const double2* __restrict__ vp, const double2* __restrict__ vc, int64_t n,
    double2* __restrict__ w, const double2* __restrict__ h, int prev,
    double2* __restrict__ partial) {
  double re = 0, im = 0;
  const double2 hp = vp ? h[prev] : make_double2(0, 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 x = w[i];
    if (vp) {
      const double2 v = vp[i];
      x.x -= hp.x * v.x - hp.y * v.y;
      x.y -= hp.x * v.y + hp.y * v.x;
      w[i] = x;
    }
    if (vc) {
      const double2 v = vc[i];
      re += v.x * x.x + v.y * x.y;
      im += v.x * x.y - v.y * x.x;
    } else {
      re += x.x * x.x + x.y * x.y;
    }
  }
  const double2 s = block_sum2(re, im);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// h[slot] = sum of partials (or sqrt of it for the norm)
__global__ void finish_kernel(const double2* __restrict__ partial, int nb,
                              double2* __restrict__ h, int slot, int is_norm) {
  double re = 0, im = 0;
  for (int i = threadIdx.x; i < nb; i += 32) { re += partial[i].x; im += partial[i].y; }
  re = warp_sum(re);
  im = warp_sum(im);
  if (threadIdx.x == 0) h[slot] = is_norm ? make_double2(sqrt(re), 0.0) : make_double2(re, im);
}

// V[k+1] = w / h[k+1] when h[k+1] != 0 (reference solver.py:66-67)
__global__ void normalize_kernel(const double2* __restrict__ w, int64_t n,
                                 const double2* __restrict__ h, int slot,
                                 double2* __restrict__ dst) {
  const double nrm = h[slot].x;
  if (nrm == 0.0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = make_double2(w[i].x / nrm, w[i].y / nrm);
}

__global__ void combine_kernel(const double2* const* __restrict__ rows, int k,
                               int64_t n, const double2* __restrict__ y,
                               double2* __restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double re = 0, im = 0;
    for (int j = 0; j < k; ++j) {
      const double2 v = rows[j][i], c = y[j];
      re += v.x * c.x - v.y * c.y;
      im += v.x * c.y + v.y * c.x;
    }
    x[i] = make_double2(re, im);
  }
}

__global__ void zaxpy_kernel(double2 alpha, const double2* __restrict__ x,
                             double2* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = x[i];
    y[i] = make_double2(y[i].x + alpha.x * v.x - alpha.y * v.y,
                        y[i].y + alpha.x * v.y + alpha.y * v.x);
  }
}

__global__ void zdiv_kernel(double2* __restrict__ y, const double2* __restrict__ x,
                            double denom, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = make_double2(x[i].x / denom, x[i].y / denom);
}

struct Scratch {
  double2* partial = nullptr;
  double2* scal = nullptr;
  double2* host = nullptr;
  const double2** rows = nullptr;   // device copy of a basis row table
  int rows_cap = 0;
};
static Scratch g_s;

static int scratch() {
  if (!g_s.partial) {
    IFGFB_CUDA(cudaMalloc(&g_s.partial, sizeof(double2) * RED_BLOCKS));
    IFGFB_CUDA(cudaMalloc(&g_s.scal, sizeof(double2) * 2));
    IFGFB_CUDA(cudaMallocHost(&g_s.host, sizeof(double2) * 2));
  }
  return IFGFB_OK;
}

static int grid_for(int64_t n) {
  return (int)std::min<int64_t>(RED_BLOCKS, std::max<int64_t>(1, (n + RED_THREADS - 1) / RED_THREADS));
}

}  // namespace ifgfb

using namespace ifgfb;
#define CHECK_ARG IFGFB_CHECK_ARG
#define RC IFGFB_RC

extern "C" {

// one MGS Arnoldi step over basis rows given as pointers (host array of
// k+1 device-addressable pointers); v_next receives w / h[k+1]
static int arnoldi_rows(const double2* const* V, int k, int64_t n, double2* W,
                        double2* H, double2* v_next, cudaStream_t st) {
  RC(scratch());
  const int nb = RED_BLOCKS;   // fixed grid: reduction order independent of n
  for (int i = 0; i <= k; ++i) {
    axpy_dot_kernel<<<nb, RED_THREADS, 0, st>>>(i > 0 ? V[i - 1] : nullptr, V[i], n, W,
                                                H, i - 1, g_s.partial);
    finish_kernel<<<1, 32, 0, st>>>(g_s.partial, nb, H, i, 0);
  }
  axpy_dot_kernel<<<nb, RED_THREADS, 0, st>>>(V[k], nullptr, n, W, H, k, g_s.partial);
  finish_kernel<<<1, 32, 0, st>>>(g_s.partial, nb, H, k + 1, 1);
  normalize_kernel<<<grid_for(n), RED_THREADS, 0, st>>>(W, n, H, k + 1, v_next);
  IFGFB_CUDA(cudaGetLastError());
  return IFGFB_OK;
}

static int combine_rows(const double2* const* rows, int k, int64_t n, const double2* y,
                        double2* x, cudaStream_t st) {
  RC(scratch());
  if (k > g_s.rows_cap) {
    if (g_s.rows) IFGFB_CUDA(cudaFree(g_s.rows));
    g_s.rows = nullptr;
    IFGFB_CUDA(cudaMalloc(&g_s.rows, sizeof(double2*) * k));
    g_s.rows_cap = k;
  }
  if (k > 0)
    IFGFB_CUDA(cudaMemcpyAsync(g_s.rows, rows, sizeof(double2*) * k,
                               cudaMemcpyHostToDevice, st));
  combine_kernel<<<grid_for(n) * 4, RED_THREADS, 0, st>>>(g_s.rows, k, n, y, x);
  IFGFB_CUDA(cudaGetLastError());
  // the row table is pageable host memory owned by the caller
  IFGFB_CUDA(cudaStreamSynchronize(st));
  return IFGFB_OK;
}

}  // namespace ifgfb

using namespace ifgfb;
#define CHECK_ARG IFGFB_CHECK_ARG
#define RC IFGFB_RC

extern "C" {

int ifgfb_arnoldi_mgs(double* basis, int64_t ld, int k, int64_t n, double* w,
                      double* h, void* stream) {
  CHECK_ARG(basis && w && h && k >= 0 && n > 0 && ld >= n, "bad argument");
  auto* V = reinterpret_cast<double2*>(basis);
  std::vector<const double2*> rows(k + 1);
  for (int i = 0; i <= k; ++i) rows[i] = V + (size_t)i * ld;
  return arnoldi_rows(rows.data(), k, n, reinterpret_cast<double2*>(w),
                      reinterpret_cast<double2*>(h), V + (size_t)(k + 1) * ld,
                      static_cast<cudaStream_t>(stream));
}

int ifgfb_arnoldi_mgs_rows(const double* const* rows, int k, int64_t n, double* w,
                           double* h, double* v_next, void* stream) {
  CHECK_ARG(rows && w && h && v_next && k >= 0 && n > 0, "bad argument");
  for (int i = 0; i <= k; ++i) CHECK_ARG(rows[i] != nullptr, "null basis row");
  return arnoldi_rows(reinterpret_cast<const double2* const*>(rows), k, n,
                      reinterpret_cast<double2*>(w), reinterpret_cast<double2*>(h),
                      reinterpret_cast<double2*>(v_next), static_cast<cudaStream_t>(stream));
}

int ifgfb_basis_combine(const double* basis, int64_t ld, int k, int64_t n,
                        const double* y, double* x, void* stream) {
  CHECK_ARG(basis && y && x && k >= 0 && n > 0, "bad argument");
  auto* V = reinterpret_cast<const double2*>(basis);
  std::vector<const double2*> rows(std::max(k, 1));
  for (int i = 0; i < k; ++i) rows[i] = V + (size_t)i * ld;
  return combine_rows(rows.data(), k, n, reinterpret_cast<const double2*>(y),
                      reinterpret_cast<double2*>(x), static_cast<cudaStream_t>(stream));
}

int ifgfb_basis_combine_rows(const double* const* rows, int k, int64_t n,
                             const double* y, double* x, void* stream) {
  CHECK_ARG(rows && y && x && k >= 0 && n > 0, "bad argument");
  return combine_rows(reinterpret_cast<const double2* const*>(rows), k, n,
                      reinterpret_cast<const double2*>(y), reinterpret_cast<double2*>(x),
                      static_cast<cudaStream_t>(stream));
}

int ifgfb_zdotc(const double* x, const double* y, int64_t n, double* result,
                void* stream) {
  CHECK_ARG(x && y && result && n >= 0, "bad argument");
  RC(scratch());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // partial = sum conj(x) y via the fused kernel with prev = -1
  axpy_dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(
      nullptr, reinterpret_cast<const double2*>(x), n,
      const_cast<double2*>(reinterpret_cast<const double2*>(y)), g_s.scal, -1,
      g_s.partial);
  finish_kernel<<<1, 32, 0, st>>>(g_s.partial, RED_BLOCKS, g_s.scal, 0, 0);
  IFGFB_CUDA(cudaMemcpyAsync(g_s.host, g_s.scal, sizeof(double2), cudaMemcpyDeviceToHost, st));
  IFGFB_CUDA(cudaStreamSynchronize(st));
  result[0] = g_s.host->x;
  result[1] = g_s.host->y;
  return IFGFB_OK;
}

int ifgfb_dznrm2(const double* x, int64_t n, double* result, void* stream) {
  CHECK_ARG(x && result && n >= 0, "bad argument");
  RC(scratch());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  axpy_dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(
      nullptr, nullptr, n, const_cast<double2*>(reinterpret_cast<const double2*>(x)),
      g_s.scal, -1, g_s.partial);
  finish_kernel<<<1, 32, 0, st>>>(g_s.partial, RED_BLOCKS, g_s.scal, 0, 1);
  IFGFB_CUDA(cudaMemcpyAsync(g_s.host, g_s.scal, sizeof(double2), cudaMemcpyDeviceToHost, st));
  IFGFB_CUDA(cudaStreamSynchronize(st));
  *result = g_s.host->x;
  return IFGFB_OK;
}

int ifgfb_zaxpy(const double* alpha, const double* x, double* y, int64_t n,
                void* stream) {
  CHECK_ARG(alpha && x && y && n >= 0, "bad argument");
  zaxpy_kernel<<<grid_for(n), RED_THREADS, 0, static_cast<cudaStream_t>(stream)>>>(
      make_double2(alpha[0], alpha[1]), reinterpret_cast<const double2*>(x),
      reinterpret_cast<double2*>(y), n);
  IFGFB_CUDA(cudaGetLastError());
  return IFGFB_OK;
}

int ifgfb_zscal_div(double* y, const double* x, double denom, int64_t n,
                    void* stream) {
  CHECK_ARG(x && y && n >= 0, "bad argument");
  zdiv_kernel<<<grid_for(n), RED_THREADS, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<double2*>(y), reinterpret_cast<const double2*>(x), denom, n);
  IFGFB_CUDA(cudaGetLastError());
  return IFGFB_OK;
}

}  // extern "C"
