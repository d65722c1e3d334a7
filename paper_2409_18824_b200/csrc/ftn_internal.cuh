// Internal helpers shared by the libftn translation units (host + device).
// Nothing here is part of the C ABI (include/ftn.h).
#pragma once

#include <cuda_runtime.h>
#include <cuda.h>
#include <stdint.h>
#include <stddef.h>
#include <string>
#include <atomic>

#include "ftn.h"

#include <nvtx3/nvToolsExt.h>

namespace ftn {

// NVTX range for profilers (nsys / ncu --nvtx); header-only NVTX3, free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
ftn_status_t fail(ftn_status_t s, const std::string& msg);
ftn_status_t cuda_fail(cudaError_t e, const char* what);

#define FTN_CHECK(expr)                    \
  do {                                     \
    ftn_status_t s__ = (expr);             \
    if (s__ != FTN_OK) return s__;         \
  } while (0)

#define FTN_CUDA(expr)                                        \
  do {                                                        \
    cudaError_t e__ = (expr);                                 \
    if (e__ != cudaSuccess) return ftn::cuda_fail(e__, #expr); \
  } while (0)

// Called after every kernel launch: counts it and turns a launch error into a status.
ftn_status_t after_launch(const char* what, uint64_t n = 1);
extern std::atomic<uint64_t> g_launches;

// FTN_ERR_DEVICE unless the current device is sm_100.
ftn_status_t require_sm100();
// SM count of the current device, minus the calling thread's reserve (ScopedSmReserve):
// persistent grids are sized from it.
int num_sms();
// While alive, kernels this thread sizes by num_sms() leave n SMs free (e.g. for the NCCL
// kernels of a halo exchange that runs concurrently on another stream).
struct ScopedSmReserve {
  explicit ScopedSmReserve(int n);
  ~ScopedSmReserve();
  ScopedSmReserve(const ScopedSmReserve&) = delete;
  ScopedSmReserve& operator=(const ScopedSmReserve&) = delete;
  int saved;
};

// ---------------------------------------------------------------- descriptors
int64_t type_len(int32_t type);
bool type_ok(int32_t type);
ftn_status_t check_desc(const ftn_desc_t* d, const char* name, int min_rank, int max_rank);
int64_t desc_size(const ftn_desc_t* d);
bool same_shape(const ftn_desc_t* a, const ftn_desc_t* b);
// Lowest and one-past-highest byte touched by the described elements.
void desc_byte_range(const ftn_desc_t* d, uintptr_t* lo, uintptr_t* hi);
bool desc_overlap(const ftn_desc_t* a, const ftn_desc_t* b);
bool desc_identical(const ftn_desc_t* a, const ftn_desc_t* b);
bool desc_contiguous(const ftn_desc_t* d);  // packed column-major

// Kernel-side view: 0-based positions, rank padded to 3 (ext 1, sm 0).
struct KDesc {
  char* base;
  int64_t ext[3];
  int64_t sm[3];
};
KDesc to_kdesc(const ftn_desc_t* d);

// Merge adjacent dimensions that are contiguous with each other in EVERY array of
// `arrays` (all with dst's extents; rank-0 entries are scalars and are skipped)
// and drop extent-1 dimensions.  Writes the merged kernel views.  Returns the
// number of merged dims (>= 1).
int collapse(const ftn_desc_t* const* arrays, int n, KDesc* out);

// Temporary device buffer on a stream (cudaMallocAsync / cudaFreeAsync).
struct StreamTemp {
  void* ptr = nullptr;
  cudaStream_t stream = nullptr;
  ~StreamTemp();
  ftn_status_t alloc(size_t bytes, cudaStream_t s);
};
ftn_status_t make_packed(ftn_desc_t* out, void* base, const ftn_desc_t* like);

// element-wise engine shared by assign / fill / elemental / matmul packing
ftn_status_t launch_elementwise(int32_t op, const ftn_desc_t* dst, const ftn_desc_t* a,
                                const ftn_desc_t* b, const ftn_desc_t* c, uint32_t flags,
                                cudaStream_t stream);
ftn_status_t launch_copy(const ftn_desc_t* dst, const ftn_desc_t* src, cudaStream_t stream);

// reductions shared with the distributed layer
ftn_status_t reduce_local(int kind, const ftn_desc_t* x, const ftn_desc_t* y, void* result_dev,
                          void* ws, size_t ws_bytes, cudaStream_t stream);
size_t reduce_ws_bytes(int64_t n);
enum { RK_SUM = 0, RK_MAX = 1, RK_MIN = 2, RK_DOT = 3, RK_PROD = 4, RK_MAXABSDIFF = 5 };
ftn_status_t tree_combine_launch(int kind, int32_t type, const void* partials, int64_t n,
                                 void* result, cudaStream_t stream);

// Jacobi sweep on explicit plane ranges (used by the distributed layer).
ftn_status_t jacobi_sweep(const ftn_desc_t* src, const ftn_desc_t* dst, double coeff,
                          int64_t last_lo, int64_t last_hi, cudaStream_t stream);

// TMA descriptor encoding through the driver entry point (no -lcuda needed).
ftn_status_t encode_tma(CUtensorMap* map, CUtensorMapDataType dt, int rank, void* base,
                        const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                        CUtensorMapSwizzle swizzle);

}  // namespace ftn

// ---------------------------------------------------------------- device PTX helpers
#ifdef __CUDACC__
namespace ftn {
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}
// Producer-side wait: the thread is suspended in hardware until the phase completes (or
// the time hint, in ns, expires) instead of spinning on try_wait, which would take issue
// slots from the compute warps of its SM sub-partition.
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t* bar, uint32_t phase, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase), "r"(ns)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_idle(uint64_t* bar, uint32_t phase) {
  while (!mbar_try_wait_hint(bar, phase, 1000000u)) {
  }
}
__device__ __forceinline__ void prefetch_tma(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// TMA store of a box from shared memory (bulk-group completion; the writing threads must have
// executed fence_proxy_async and a barrier before the issuing thread calls this).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N committed bulk groups still reading their shared-memory source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// at most N committed bulk groups not yet complete
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// *slot = fmax(*slot, v) atomically (maxNum: a NaN v leaves the slot, a NaN slot takes v), for
// the Jacobi residual MAXVAL(ABS(u_s - u_{s-1})) accumulated by the sweep kernels themselves.
// fmax over non-negative values is exact and order-independent, so any accumulation order
// gives the bits of the sequential fold.
__device__ __forceinline__ void atomic_fmax_slot(double* slot, double v) {
  if (v != v) return;
  unsigned long long* a = reinterpret_cast<unsigned long long*>(slot);
  unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(a);
  for (;;) {
    const double o = __longlong_as_double(old);
    if (o == o && o >= v) return;
    const unsigned long long prev = atomicCAS(a, old, __double_as_longlong(v));
    if (prev == old) return;
    old = prev;
  }
}
// fmax over the 32 lanes of a warp (every lane gets the result)
__device__ __forceinline__ double warp_fmax(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}

// 256-bit global accesses (sm_100a, PTX 8.8)
__device__ __forceinline__ void ld_v4(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}
// read-only (non-coherent) 256-bit load that may allocate in L1 (operands re-read by many warps)
__device__ __forceinline__ void ldg_v4(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void st_v4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

}  // namespace dev
}  // namespace ftn
#endif
