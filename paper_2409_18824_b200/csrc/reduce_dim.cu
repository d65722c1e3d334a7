// DIM= reductions: SUM / PRODUCT / MAXVAL / MINVAL (x, DIM=d).
//
// the intrinsic lowers to linalg.reduce whose `dimensions` attribute names the
// reduced dimension(s); MAXVAL and PRODUCT "are also implemented" the same way.  Every
// result element is the sequential fold over the reduced subscript in ascending order
// from the neutral element (R#24) -- the literal linalg.reduce loop -- so results are
// bit-identical to the oracle.  Parallelism comes from the result elements:
//   * reduced dim is not the first (dim-1) dimension: one thread per result element;
//     consecutive threads take consecutive elements of the first kept dimension, so
//     each step of the fold is a coalesced load across the warp (4 loads in flight);
//   * reduced dim is dimension 1 (contiguous): each warp stages 32 result rows x 32
//     reduced elements through shared memory (coalesced row loads), then lane l folds
//     row l in order.
// HBM-bound: elem_len bytes per reduced element.
#include "ftn_internal.cuh"

#include <cstring>
#include <type_traits>
#include <cmath>

namespace ftn {
namespace {

struct RDParams {
  char* x;
  int64_t n;          // extent of the reduced dimension
  int64_t step;       // its byte stride
  int64_t ke[2];      // kept extents (dim order), padded with 1
  int64_t ks[2];      // kept byte strides of x
  char* r;
  int64_t rs[2];      // result byte strides
  int64_t nout;
};

template <typename T> struct U_ { typedef T type; };
template <> struct U_<int32_t> { typedef uint32_t type; };
template <> struct U_<int64_t> { typedef uint64_t type; };

template <typename T, int KIND>
__device__ __forceinline__ T init_val() {
  if constexpr (KIND == RK_SUM) return T(0);
  if constexpr (KIND == RK_PROD) return T(1);
  if constexpr (std::is_floating_point<T>::value) return (T)NAN;   // maxNum/minNum start
  if constexpr (sizeof(T) == 4) return (T)(KIND == RK_MAX ? INT32_MIN : INT32_MAX);
  return (T)(KIND == RK_MAX ? INT64_MIN : INT64_MAX);
}

template <typename T, int KIND>
__device__ __forceinline__ T fold(T acc, T v) {
  typedef typename U_<T>::type Uu;
  if constexpr (KIND == RK_SUM) {
    if constexpr (std::is_floating_point<T>::value) return acc + v;
    else return (T)((Uu)acc + (Uu)v);
  } else if constexpr (KIND == RK_PROD) {
    if constexpr (std::is_floating_point<T>::value) return acc * v;
    else return (T)((Uu)acc * (Uu)v);
  } else if constexpr (std::is_floating_point<T>::value) {
    return KIND == RK_MAX ? fmax(acc, v) : fmin(acc, v);
  } else {
    return KIND == RK_MAX ? (v > acc ? v : acc) : (v < acc ? v : acc);
  }
}

template <typename T, int KIND>
__device__ __forceinline__ T finish(T acc, int64_t n) {
  if constexpr (std::is_floating_point<T>::value && (KIND == RK_MAX || KIND == RK_MIN))
    if (n == 0) return KIND == RK_MAX ? (T)-INFINITY : (T)INFINITY;
  return acc;
}

// Case A: one thread per result element, sequential fold along a non-leading dimension.
template <typename T, int KIND>
__global__ void __launch_bounds__(256) reduce_dim_strided(const __grid_constant__ RDParams p) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < p.nout; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k0 = o % p.ke[0], k1 = o / p.ke[0];
    const char* xp = p.x + k0 * p.ks[0] + k1 * p.ks[1];
    T acc = init_val<T, KIND>();
    int64_t j = 0;
    for (; j + 4 <= p.n; j += 4) {
      const T a = *reinterpret_cast<const T*>(xp + (j + 0) * p.step);
      const T b = *reinterpret_cast<const T*>(xp + (j + 1) * p.step);
      const T c = *reinterpret_cast<const T*>(xp + (j + 2) * p.step);
      const T d = *reinterpret_cast<const T*>(xp + (j + 3) * p.step);
      acc = fold<T, KIND>(acc, a);
      acc = fold<T, KIND>(acc, b);
      acc = fold<T, KIND>(acc, c);
      acc = fold<T, KIND>(acc, d);
    }
    for (; j < p.n; ++j) acc = fold<T, KIND>(acc, *reinterpret_cast<const T*>(xp + j * p.step));
    *reinterpret_cast<T*>(p.r + k0 * p.rs[0] + k1 * p.rs[1]) = finish<T, KIND>(acc, p.n);
  }
}

// Case B: the reduced dimension is the leading one.  Warp w of the block owns result
// elements [o0, o0 + 32); tiles of 32 reduced elements are staged through shared memory.
constexpr int RB_WARPS = 4;  // 4 x 32 x 33 x 8 B = 33.8 KB static shared memory
template <typename T, int KIND>
__global__ void __launch_bounds__(RB_WARPS * 32) reduce_dim_leading(const __grid_constant__ RDParams p) {
  __shared__ T tile[RB_WARPS][32][33];
  __shared__ const char* rowbase[RB_WARPS][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ngroups = (p.nout + 31) / 32;
  for (int64_t g = blockIdx.x * (int64_t)RB_WARPS + warp; g < ngroups; g += (int64_t)gridDim.x * RB_WARPS) {
    const int64_t o0 = g * 32;
    const int64_t my = o0 + lane;  // this lane's result element
    const int64_t mk0 = my % p.ke[0], mk1 = my / p.ke[0];
    const int rows = (int)min((int64_t)32, p.nout - o0);
    __syncwarp();
    rowbase[warp][lane] = p.x + mk0 * p.ks[0] + mk1 * p.ks[1];
    __syncwarp();
    T acc = init_val<T, KIND>();
    // software pipeline: the 32 row loads of tile j0 + 32 are in flight while tile j0 is
    // transposed through shared memory and folded (the fold order is unchanged)
    T v[32];
    {
      const bool jok = lane < p.n;
#pragma unroll
      for (int rr = 0; rr < 32; ++rr)
        v[rr] = (rr < rows && jok) ? *reinterpret_cast<const T*>(rowbase[warp][rr] + (int64_t)lane * p.step) : T(0);
    }
    for (int64_t j0 = 0; j0 < p.n; j0 += 32) {
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) tile[warp][rr][lane] = v[rr];
      {
        const int64_t jn = j0 + 32 + lane;
        const bool jok = jn < p.n;
#pragma unroll
        for (int rr = 0; rr < 32; ++rr)  // 32 independent coalesced row loads in flight
          v[rr] = (rr < rows && jok) ? *reinterpret_cast<const T*>(rowbase[warp][rr] + jn * p.step) : T(0);
      }
      __syncwarp();
      const int cnt = (int)min((int64_t)32, p.n - j0);
      if (cnt == 32) {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) acc = fold<T, KIND>(acc, tile[warp][lane][jj]);
      } else {
        for (int jj = 0; jj < cnt; ++jj) acc = fold<T, KIND>(acc, tile[warp][lane][jj]);
      }
      __syncwarp();
    }
    if (my < p.nout) *reinterpret_cast<T*>(p.r + mk0 * p.rs[0] + mk1 * p.rs[1]) = finish<T, KIND>(acc, p.n);
  }
}

template <typename T, int KIND>
ftn_status_t launch_rd(const RDParams& p, bool leading, cudaStream_t s) {
  if (p.nout == 0) return FTN_OK;
  const int sms = num_sms();
  if (leading) {
    const int64_t groups = (p.nout + 31) / 32;
    int64_t blocks = (groups + RB_WARPS - 1) / RB_WARPS;
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    reduce_dim_leading<T, KIND><<<(unsigned)blocks, RB_WARPS * 32, 0, s>>>(p);
  } else {
    int64_t blocks = (p.nout + 255) / 256;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    reduce_dim_strided<T, KIND><<<(unsigned)blocks, 256, 0, s>>>(p);
  }
  return after_launch("reduce_dim");
}

template <typename T>
ftn_status_t by_kind(int kind, const RDParams& p, bool leading, cudaStream_t s) {
  switch (kind) {
    case RK_SUM: return launch_rd<T, RK_SUM>(p, leading, s);
    case RK_MAX: return launch_rd<T, RK_MAX>(p, leading, s);
    case RK_MIN: return launch_rd<T, RK_MIN>(p, leading, s);
    case RK_PROD: return launch_rd<T, RK_PROD>(p, leading, s);
  }
  return fail(FTN_ERR_UNSUPPORTED, "reduce_dim: kind");
}

ftn_status_t reduce_dim(int kind, const char* name, const ftn_desc_t* x, int32_t dim, const ftn_desc_t* result,
                        ftn_stream_t stream) {
  FTN_CHECK(check_desc(x, name, 1, FTN_MAX_RANK));
  if (!result) return fail(FTN_ERR_NULL, std::string(name) + ": result NULL");
  if (dim < 1 || dim > x->rank) return fail(FTN_ERR_DIM, std::string(name) + ": DIM out of range");
  if (result->rank != x->rank - 1) return fail(FTN_ERR_RANK, std::string(name) + ": result rank must be rank(x)-1");
  if (result->type != x->type) return fail(FTN_ERR_TYPE, std::string(name) + ": result type differs from x");
  if (x->type == FTN_F32) return fail(FTN_ERR_TYPE, std::string(name) + ": real(4) reductions are not offered");
  if (result->rank > 0) FTN_CHECK(check_desc(result, name, 1, FTN_MAX_RANK));
  else if (!result->base_addr) return fail(FTN_ERR_NULL, std::string(name) + ": result base NULL");
  RDParams p;
  memset(&p, 0, sizeof(p));
  p.x = (char*)x->base_addr;
  p.n = x->dim[dim - 1].extent;
  p.step = x->dim[dim - 1].sm;
  p.r = (char*)result->base_addr;
  p.ke[0] = p.ke[1] = 1;
  int nk = 0;
  for (int d = 0; d < x->rank; ++d) {
    if (d == dim - 1) continue;
    if (result->dim[nk].extent != x->dim[d].extent)
      return fail(FTN_ERR_SHAPE, std::string(name) + ": result shape must be x's shape without DIM");
    p.ke[nk] = x->dim[d].extent;
    p.ks[nk] = x->dim[d].sm;
    p.rs[nk] = result->dim[nk].sm;
    ++nk;
  }
  p.nout = p.ke[0] * p.ke[1];
  if (desc_overlap(x, result)) return fail(FTN_ERR_SHAPE, std::string(name) + ": result overlaps x");
  FTN_CHECK(require_sm100());
  // the leading-dimension kernel when the reduced elements are the contiguous ones
  const bool leading = (dim == 1) && p.n > 1 && (p.ke[0] == 1 || (p.step < (p.ks[0] < 0 ? -p.ks[0] : p.ks[0])));
  cudaStream_t s = (cudaStream_t)stream;
  switch (x->type) {
    case FTN_F64: return by_kind<double>(kind, p, leading, s);
    case FTN_I32: return by_kind<int32_t>(kind, p, leading, s);
    case FTN_I64: return by_kind<int64_t>(kind, p, leading, s);
  }
  return fail(FTN_ERR_TYPE, std::string(name) + ": type");
}

}  // namespace
}  // namespace ftn

using namespace ftn;

extern "C" {

ftn_status_t ftn_sum_dim(const ftn_desc_t* x, int32_t dim, const ftn_desc_t* result, ftn_stream_t stream) {
  return reduce_dim(RK_SUM, "ftn_sum_dim", x, dim, result, stream);
}
ftn_status_t ftn_product_dim(const ftn_desc_t* x, int32_t dim, const ftn_desc_t* result, ftn_stream_t stream) {
  return reduce_dim(RK_PROD, "ftn_product_dim", x, dim, result, stream);
}
ftn_status_t ftn_maxval_dim(const ftn_desc_t* x, int32_t dim, const ftn_desc_t* result, ftn_stream_t stream) {
  return reduce_dim(RK_MAX, "ftn_maxval_dim", x, dim, result, stream);
}
ftn_status_t ftn_minval_dim(const ftn_desc_t* x, int32_t dim, const ftn_desc_t* result, ftn_stream_t stream) {
  return reduce_dim(RK_MIN, "ftn_minval_dim", x, dim, result, stream);
}

}  // extern "C"
