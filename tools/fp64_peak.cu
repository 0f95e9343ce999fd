// Microbenchmark: FP64 peak on B200 via DFMA (CUDA cores) and DMMA (mma.sync m8n8k4 f64).
// Used to set the FP64 roofline denominator (MEASURED_PEAKS.json has no FP64 figure).
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c0[CHAINS], c1[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { c0[c] = c; c1[c] = -c; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[c]), "+d"(c1[c]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int blocksPerSM : {1, 2, 4, 8}) {
    for (int threads : {128, 256, 512}) {
      int grid = sms * blocksPerSM;
      dfma_kernel<8><<<grid, threads>>>(d, 100, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_kernel<8><<<grid, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = 2.0 * 8 * iters * (double)grid * threads;
      printf("DFMA grid=%d thr=%d : %.2f TFLOP/s\n", grid, threads, flop / ms / 1e9);
    }
  }
  for (int blocksPerSM : {1, 2, 4, 8}) {
    for (int threads : {128, 256, 512}) {
      int grid = sms * blocksPerSM;
      dmma_kernel<4><<<grid, threads>>>(d, 100);
      cudaEventRecord(e0);
      dmma_kernel<4><<<grid, threads>>>(d, iters / 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = 2.0 * 256 * 4 * (iters / 4) * (double)grid * (threads / 32);
      printf("DMMA grid=%d thr=%d : %.2f TFLOP/s\n", grid, threads, flop / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s sms=%d\n", cudaGetErrorString(err), sms);
  return 0;
}
