// Microbenchmark: FP64 tensor-core throughput on B200 per mma.sync shape
// (m8n8k4, m16n8k4, m16n8k8, m16n8k16), independent accumulator chains.
// Decides the DMMA shape of the propagation kernel (K4) and the FP64 peak
// denominator of its roofline.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void m16n8k4(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 0.5, b = 0.999999;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(b));
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void m16n8k8(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 0.5, a2 = 0.25, a3 = 0.125, b0 = 0.999999, b1 = 0.3;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 0.999 - i * 1e-3;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]),
                     "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
static void run(const char* name, K kern, double flop_per_mma, int chains, double* d, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  for (int bps : {1, 2, 4, 8})
    for (int thr : {128, 256, 512}) {
      const int grid = sms * bps;
      kern<<<grid, thr>>>(d, 50);
      cudaEventRecord(e0);
      kern<<<grid, thr>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flop = flop_per_mma * chains * iters * (double)grid * (thr / 32);
      printf("%-9s chains=%d grid=%5d thr=%3d : %6.2f TFLOP/s\n", name, chains, grid, thr,
             flop / ms / 1e9);
    }
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run("m8n8k4", m8n8k4<4>, 2.0 * 8 * 8 * 4, 4, d, sms);
  run("m16n8k4", m16n8k4<4>, 2.0 * 16 * 8 * 4, 4, d, sms);
  run("m16n8k8", m16n8k8<2>, 2.0 * 16 * 8 * 8, 2, d, sms);
  run("m16n8k8", m16n8k8<4>, 2.0 * 16 * 8 * 8, 4, d, sms);
  run("m16n8k16", m16n8k16<2>, 2.0 * 16 * 8 * 16, 2, d, sms);
  run("m16n8k16", m16n8k16<4>, 2.0 * 16 * 8 * 16, 4, d, sms);
  printf("err=%s sms=%d\n", cudaGetErrorString(cudaGetLastError()), sms);
  return 0;
}
