// Throughput probes for the sm_100a design decisions of DESIGN.md:
//   * fp64 DMMA (mma.sync .f64) per shape vs plain DFMA  -> which unit MATMUL targets
//   * HBM read / copy / triad with 256-bit (v4.f64) and 128-bit accesses
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe probe.cu
// Output: one line per probe, "name value unit".
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

template <int NACC>
__global__ void dfma_kernel(double* out, double s) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], s, 1e-9);
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) t += acc[i];
  if (t == 123.0) out[0] = t;
}

// ---- DMMA shapes ----
struct M8N8K4 {
  static constexpr int M = 8, N = 8, K = 4, NA = 1, NB = 1, NC = 2;
  __device__ static void mma(double* d, const double* a, const double* b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a[0]), "d"(b[0]));
  }
};
struct M16N8K4 {
  static constexpr int M = 16, N = 8, K = 4, NA = 2, NB = 1, NC = 4;
  __device__ static void mma(double* d, const double* a, const double* b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  }
};
struct M16N8K8 {
  static constexpr int M = 16, N = 8, K = 8, NA = 4, NB = 2, NC = 4;
  __device__ static void mma(double* d, const double* a, const double* b) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
};
struct M16N8K16 {
  static constexpr int M = 16, N = 8, K = 16, NA = 8, NB = 4, NC = 4;
  __device__ static void mma(double* d, const double* a, const double* b) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
};

template <class S, int NACC>
__global__ void dmma_kernel(double* out, double s) {
  double a[S::NA], b[S::NB], c[NACC][S::NC];
#pragma unroll
  for (int i = 0; i < S::NA; ++i) a[i] = s * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < S::NB; ++i) b[i] = s * (threadIdx.x - i);
#pragma unroll
  for (int j = 0; j < NACC; ++j)
#pragma unroll
    for (int i = 0; i < S::NC; ++i) c[j][i] = 0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) S::mma(c[j], a, b);
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j)
#pragma unroll
    for (int i = 0; i < S::NC; ++i) t += c[j][i];
  if (t == 123.0) out[0] = t;
}

// ---- HBM ----
__global__ void read_v4(const double* __restrict__ x, size_t n4, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    double a0, a1, a2, a3;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a0), "=d"(a1), "=d"(a2), "=d"(a3) : "l"(x + 4 * i));
    s += (a0 + a1) + (a2 + a3);
  }
  if (s == 123.0) out[0] = s;
}
template <int U>
__global__ void read_v4_unroll(const double* __restrict__ x, size_t n4, double* out) {
  double s = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    double v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(v[u][0]), "=d"(v[u][1]), "=d"(v[u][2]), "=d"(v[u][3]) : "l"(x + 4 * (i + u * stride)));
#pragma unroll
    for (int u = 0; u < U; ++u) s += (v[u][0] + v[u][1]) + (v[u][2] + v[u][3]);
  }
  for (; i < n4; i += stride) s += x[4 * i];
  if (s == 123.0) out[0] = s;
}
__global__ void copy_v4(const double* __restrict__ x, double* __restrict__ y, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    double a0, a1, a2, a3;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a0), "=d"(a1), "=d"(a2), "=d"(a3) : "l"(x + 4 * i));
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(y + 4 * i), "d"(a0), "d"(a1), "d"(a2), "d"(a3) : "memory");
  }
}
__global__ void copy_v2(const double2* __restrict__ x, double2* __restrict__ y, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) y[i] = x[i];
}
__global__ void triad4_v4(const double* __restrict__ b, const double* __restrict__ c, const double* __restrict__ d,
                          double* __restrict__ r, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    double b0, b1, b2, b3, c0, c1, c2, c3, d0, d1, d2, d3;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(b0), "=d"(b1), "=d"(b2), "=d"(b3) : "l"(b + 4 * i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(c0), "=d"(c1), "=d"(c2), "=d"(c3) : "l"(c + 4 * i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(d0), "=d"(d1), "=d"(d2), "=d"(d3) : "l"(d + 4 * i));
    double r0 = __dadd_rn(__dmul_rn(b0, c0), d0), r1 = __dadd_rn(__dmul_rn(b1, c1), d1);
    double r2 = __dadd_rn(__dmul_rn(b2, c2), d2), r3 = __dadd_rn(__dmul_rn(b3, c3), d3);
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(r + 4 * i), "d"(r0), "d"(r1), "d"(r2), "d"(r3) : "memory");
  }
}

template <class F>
float time_ms(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();  // warm
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

template <class S, int NACC, int WARPS>
void run_dmma(const char* name, double* out, int sms) {
  int blocks = sms * 4;
  float ms = time_ms([&] { dmma_kernel<S, NACC><<<blocks, 32 * WARPS>>>(out, 1.0000001); }, 5);
  double flops = 2.0 * S::M * S::N * S::K * NACC * (double)ITERS * blocks * WARPS;
  printf("%s_nacc%d_w%d %.2f TFLOP/s\n", name, NACC, WARPS * 4, flops / ms / 1e9);
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("device %s sms %d l2 %d MB\n", p.name, sms, p.l2CacheSize >> 20);
  double* out; CK(cudaMalloc(&out, 64));
  {
    int blocks = sms * 8;
    float ms = time_ms([&] { dfma_kernel<8><<<blocks, 256>>>(out, 1.0000001); }, 5);
    printf("dfma_nacc8 %.2f TFLOP/s\n", 2.0 * 8 * ITERS * (double)blocks * 256 / ms / 1e9);
    ms = time_ms([&] { dfma_kernel<16><<<blocks, 256>>>(out, 1.0000001); }, 5);
    printf("dfma_nacc16 %.2f TFLOP/s\n", 2.0 * 16 * ITERS * (double)blocks * 256 / ms / 1e9);
  }
  run_dmma<M8N8K4, 4, 4>("dmma_m8n8k4", out, sms);
  run_dmma<M8N8K4, 8, 4>("dmma_m8n8k4", out, sms);
  run_dmma<M16N8K4, 4, 4>("dmma_m16n8k4", out, sms);
  run_dmma<M16N8K4, 8, 4>("dmma_m16n8k4", out, sms);
  run_dmma<M16N8K4, 8, 8>("dmma_m16n8k4", out, sms);
  run_dmma<M16N8K8, 4, 4>("dmma_m16n8k8", out, sms);
  run_dmma<M16N8K8, 8, 4>("dmma_m16n8k8", out, sms);
  run_dmma<M16N8K16, 4, 4>("dmma_m16n8k16", out, sms);
  run_dmma<M16N8K16, 8, 4>("dmma_m16n8k16", out, sms);
  run_dmma<M16N8K16, 8, 8>("dmma_m16n8k16", out, sms);
  run_dmma<M16N8K16, 2, 16>("dmma_m16n8k16", out, sms);

  size_t n = (size_t)1 << 30;  // 8 GiB per array
  double *x, *y, *z, *w;
  CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&y, n * 8)); CK(cudaMalloc(&z, n * 8)); CK(cudaMalloc(&w, n * 8));
  CK(cudaMemset(x, 0, n * 8)); CK(cudaMemset(y, 0, n * 8)); CK(cudaMemset(z, 0, n * 8)); CK(cudaMemset(w, 0, n * 8));
  for (int bpsm : {4, 8, 16}) {
    int blocks = sms * bpsm;
    float ms = time_ms([&] { read_v4<<<blocks, 256>>>(x, n / 4, out); }, 5);
    printf("read_v4_b%d %.1f GB/s\n", bpsm, n * 8.0 / ms / 1e6);
    ms = time_ms([&] { read_v4_unroll<4><<<blocks, 256>>>(x, n / 4, out); }, 5);
    printf("read_v4u4_b%d %.1f GB/s\n", bpsm, n * 8.0 / ms / 1e6);
    ms = time_ms([&] { copy_v4<<<blocks, 256>>>(x, y, n / 4); }, 5);
    printf("copy_v4_b%d %.1f GB/s\n", bpsm, n * 16.0 / ms / 1e6);
    ms = time_ms([&] { copy_v2<<<blocks, 256>>>((const double2*)x, (double2*)y, n / 2); }, 5);
    printf("copy_v2_b%d %.1f GB/s\n", bpsm, n * 16.0 / ms / 1e6);
    ms = time_ms([&] { triad4_v4<<<blocks, 256>>>(x, y, z, w, n / 4); }, 5);
    printf("triad_v4_b%d %.1f GB/s\n", bpsm, n * 32.0 / ms / 1e6);
  }
  float ms = time_ms([&] { cudaMemcpyAsync(y, x, n * 8, cudaMemcpyDeviceToDevice); }, 5);
  printf("memcpy_d2d %.1f GB/s\n", n * 16.0 / ms / 1e6);
  CK(cudaDeviceSynchronize());
  return 0;
}
