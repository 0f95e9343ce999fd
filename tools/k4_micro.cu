// Microbenchmark of the K4 inner loop (20 k-steps x 4 column tiles of
// m8n8k4 f64 DMMA per 8-row tile) with the B fragments fed from
//   0: registers (upper bound), 1: shared memory, 2: global (L1-resident),
// and the per-tile epilogue (complex scale + shared-memory accumulate).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int MODE, bool EPI, int NT = 1, int MINB = 6>
__global__ void __launch_bounds__(160, MINB) k(const double* __restrict__ gB, double* out,
                                          int tiles) {
  __shared__ double sB[20 * 32 * 4];
  __shared__ double2 acc[5 * 15 * 16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 20 * 128; i += blockDim.x) sB[i] = gB[i];
  for (int i = threadIdx.x; i < 5 * 15 * 16; i += blockDim.x) acc[i] = make_double2(0, 0);
  __syncthreads();
  double tst[4], tp[5];
  for (int q = 0; q < 4; ++q) tst[q] = 1.0 + 1e-3 * (lane + q);
  for (int c = 0; c < 5; ++c) tp[c] = 1.0 - 1e-3 * c;
  double rb = 0.5 + lane * 1e-3;
  double tst2[4];
  for (int q = 0; q < 4; ++q) tst2[q] = 1.0 + 2e-3 * (lane + q);
  for (int t = 0; t < tiles; t += NT) {
    double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
    double d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
    const double4* F = reinterpret_cast<const double4*>(gB + (size_t)(((t * 7 + blockIdx.x) & 3) * 2560)) + lane;
    const double4* S = reinterpret_cast<const double4*>(sB) + lane;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        double4 b;
        if (MODE == 0) b = make_double4(rb, rb + 1, rb + 2, rb + 3);
        else if (MODE == 1) b = S[(5 * q + c) * 32];
        else b = F[(5 * q + c) * 32];
        const double a = tst[q] * tp[c];
        dmma(c0[0], c1[0], a, b.x);
        dmma(c0[1], c1[1], a, b.y);
        dmma(c0[2], c1[2], a, b.z);
        dmma(c0[3], c1[3], a, b.w);
        if (NT == 2) {
          const double a2 = tst2[q] * tp[c];
          dmma(d0[0], d1[0], a2, b.x);
          dmma(d0[1], d1[1], a2, b.y);
          dmma(d0[2], d1[2], a2, b.z);
          dmma(d0[3], d1[3], a2, b.w);
        }
      }
    if (EPI) {
      double2* dst = acc + (warp * 15 + (lane >> 2) % 15) * 16;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int m = 4 * nt + (lane & 3);
        dst[m].x += c0[nt] * 0.5 - c1[nt] * 0.25;
        dst[m].y += c0[nt] * 0.25 + c1[nt] * 0.5;
      }
      if (NT == 2) {
        double2* dst2 = acc + (warp * 15 + ((lane >> 2) + 7) % 15) * 16;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const int m = 4 * nt + (lane & 3);
          dst2[m].x += d0[nt] * 0.5 - d1[nt] * 0.25;
          dst2[m].y += d0[nt] * 0.25 + d1[nt] * 0.5;
        }
      }
      __syncwarp();
    } else {
      rb += c0[0] + c0[1] + c0[2] + c0[3] + c1[0] + c1[1] + c1[2] + c1[3];
      if (NT == 2) rb += d0[0] + d0[1] + d0[2] + d0[3] + d1[0] + d1[1] + d1[2] + d1[3];
    }
    tst[t & 3] += 1e-9;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = acc[7].x + rb;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *gB, *out;
  cudaMalloc(&gB, 4 * 20 * 128 * 8);
  cudaMalloc(&out, 1 << 20);
  cudaMemset(gB, 0, 4 * 20 * 128 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int tiles = 400, grid = sms * 6 * 4;
  auto run = [&](auto kern, const char* name) {
    kern<<<grid, 160>>>(gB, out, 10);
    cudaEventRecord(e0);
    kern<<<grid, 160>>>(gB, out, tiles);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 2.0 * 256 * 80 * (double)tiles * grid * 5;
    printf("%-32s %.2f TFLOP/s\n", name, flop / ms / 1e9);
  };
  run(k<0, false>, "B regs, no epilogue");
  run(k<1, false>, "B smem, no epilogue");
  run(k<2, false>, "B global(L1), no epilogue");
  run(k<0, true>, "B regs, epilogue");
  run(k<1, true>, "B smem, epilogue");
  run(k<2, true>, "B global(L1), epilogue");
  run(k<2, true, 2, 6>, "2 tiles/B global, epi, minb6");
  run(k<2, true, 2, 4>, "2 tiles/B global, epi, minb4");
  run(k<1, true, 2, 6>, "2 tiles/B smem, epi, minb6");
  run(k<2, false, 2, 6>, "2 tiles/B global, no epi");
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
