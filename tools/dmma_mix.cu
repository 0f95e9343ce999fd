// Does scalar FP64 work interleaved with DMMA (the per-k-step A-value multiply
// of K4) cost more than its own issue slots on the shared FP64 pipe?
// Per k-step and row tile: 4 DMMAs + MULS scalar multiplies (0, 1, 2) feeding
// the next k-step's A operand.  Prints TFLOP/s (DMMA flops only).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ double vmul(double a, double b) {
  double r;
  asm volatile("mul.rn.f64 %0, %1, %2;\n" : "=d"(r) : "d"(a), "d"(b));
  return r;
}

template <int NT, int MULS>
__global__ void k(double* out, int iters, double s) {
  double c0[NT][4], c1[NT][4], a[NT];
  const double b0 = 0.5 + 1e-3 * (threadIdx.x & 31);
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    a[i] = 1.0 + 1e-3 * threadIdx.x + i;
#pragma unroll
    for (int n = 0; n < 4; ++n) c0[i][n] = c1[i][n] = 0.0;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ks = 0; ks < 19; ++ks) {
#pragma unroll
      for (int i = 0; i < NT; ++i) {
#pragma unroll
        for (int n = 0; n < 4; ++n) dmma(c0[i][n], c1[i][n], a[i], b0 + n);
#pragma unroll
        for (int m = 0; m < MULS; ++m) a[i] = vmul(a[i], s);
      }
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int n = 0; n < 4; ++n) t += c0[i][n] + c1[i][n];
  if (t == 1.2345e300) out[0] = t;
}

template <int NT, int MULS>
void run(double* out, int warps_per_sm) {
  const int iters = 400 / NT;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = 148 * warps_per_sm;
  k<NT, MULS><<<grid, 32>>>(out, 2, 1.0000001);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<NT, MULS><<<grid, 32>>>(out, iters, 1.0000001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 5.0 * grid * iters * 19.0 * NT * 4 * 512.0;
  printf("warps/SM %2d tiles %d muls/tile/k-step %d: %6.2f TFLOP/s\n", warps_per_sm, NT, MULS,
         flop / ms * 1e-9);
}

int main() {
  double* out; cudaMalloc(&out, 8);
  for (int w : {4, 8, 16, 24}) {
    run<1, 0>(out, w); run<1, 1>(out, w); run<1, 2>(out, w);
    run<2, 0>(out, w); run<2, 1>(out, w); run<2, 2>(out, w);
    run<4, 0>(out, w); run<4, 1>(out, w); run<4, 2>(out, w);
  }
  return 0;
}
