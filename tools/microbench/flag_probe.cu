// Neighbour-flag handshake latency on B200: G co-resident CTAs, each epoch a
// CTA publishes its flag and waits for the flags of CTAs b-1 and b+1 (the resident Jacobi's
// exchange without data).  Prints microseconds per epoch for several publish / poll variants.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o flag_probe flag_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

template <int V>
__global__ void probe(uint32_t* flags, int epochs, int with_barrier) {
  const int b = blockIdx.x, G = gridDim.x;
  for (uint32_t e = 1; e <= (uint32_t)epochs; ++e) {
    if (with_barrier) __syncthreads();
    if (threadIdx.x == 0) {
      if (V == 0) {
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + b), "r"(e) : "memory");
      } else if (V == 1) {
        __threadfence();
        atomicExch(flags + b, e);
      } else {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(flags + b) : "memory");
      }
      for (int nb = b - 1; nb <= b + 1; nb += 2) {
        if (nb < 0 || nb >= G) continue;
        uint32_t v;
        do {
          if (V == 2)
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + nb) : "memory");
          else
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + nb) : "memory");
        } while (v < e);
      }
      if (V != 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    if (with_barrier) __syncthreads();
  }
}

template <int V>
int run(const char* name, int G, int threads, int barrier) {
  uint32_t* flags;
  CK(cudaMalloc(&flags, G * 4));
  const int epochs = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemset(flags, 0, G * 4));
    int ep = epochs, wb = barrier;
    void* args[] = {&flags, &ep, &wb};
    cudaEventRecord(a);
    CK(cudaLaunchCooperativeKernel((const void*)probe<V>, dim3(G), dim3(threads), args, 0, 0));
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-28s G=%3d threads=%4d barrier=%d: %.3f us per epoch\n", name, G, threads, barrier, ms * 1e3 / epochs);
  cudaFree(flags);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int G : {2, 16, sms}) {
    run<0>("st.release / ld.relaxed", G, 32, 0);
    run<1>("threadfence+atomicExch", G, 32, 0);
    run<2>("red.release / ld.acquire", G, 32, 0);
    run<0>("st.release / ld.relaxed", G, 512, 1);
  }
  return 0;
}
