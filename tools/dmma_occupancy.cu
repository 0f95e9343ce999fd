// FP64 DMMA (m8n8k4) throughput against resident warps per SM and independent
// accumulator chains per warp: how many warps the K4 inner loop needs in its
// DMMA phase to keep the pipe busy.  nvcc -arch=sm_100a -O3 -o dmma_occupancy
// tools/dmma_occupancy.cu; prints TFLOP/s per (warps per SM, chains per warp).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k(double* out, int iters) {
  double c0[CH], c1[CH];
  const double a0 = 1.0 + 1e-3 * threadIdx.x, b0 = 0.5 + 1e-3 * (threadIdx.x & 31);
#pragma unroll
  for (int i = 0; i < CH; ++i) c0[i] = c1[i] = 0.0;
  double a = a0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < CH; ++i) dmma(c0[i], c1[i], a, b0 + i);
      a = a * 1.0000001;   // one FP64 multiply per group, as the A value of a k-step
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c0[i] + c1[i];
  if (s == 1.2345e300) out[0] = s;
}

template <int CH>
void run(double* out, int warps_per_sm) {
  // warps_per_sm resident warps: CTAs of 32 threads (1 warp), one CTA per warp
  const int iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = 148 * warps_per_sm;
  k<CH><<<grid, 32>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<CH><<<grid, 32>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flop = (double)grid * iters * 8.0 * CH * 512.0;
  printf("warps/SM %2d chains %2d: %7.2f TFLOP/s (%.3f ms)\n", warps_per_sm, CH, flop / ms * 1e-9, ms);
}

int main() {
  double* out; cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16, 20, 24, 32}) {
    run<1>(out, w); run<2>(out, w); run<4>(out, w); run<8>(out, w); run<16>(out, w);
  }
  return 0;
}
