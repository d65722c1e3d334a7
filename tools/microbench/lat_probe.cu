// Dependent-chain latency of DADD / DMUL / SHFL (64-bit as two 32-bit shuffles) on B200, one warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double a, double m) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    x = x + a; x = x + a; x = x + a; x = x + a;
  }
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    x = x * m; x = x * m; x = x * m; x = x * m;
  }
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    x = __shfl_down_sync(0xffffffffu, x, 1); x = __shfl_down_sync(0xffffffffu, x, 1);
    x = __shfl_down_sync(0xffffffffu, x, 1); x = __shfl_down_sync(0xffffffffu, x, 1);
  }
  long long t3 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}

int main() {
  double* o; long long* c; long long h[3];
  cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 3 * 8);
  for (int r = 0; r < 2; ++r) lat<<<1, 32>>>(o, c, 1e-9, 1.0000001);
  cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency %.1f cycles\nDMUL dependent latency %.1f cycles\nSHFL.64 (2x32) dependent latency %.1f cycles\n",
         h[0] / 4096.0, h[1] / 4096.0, h[2] / 4096.0);
  return 0;
}
