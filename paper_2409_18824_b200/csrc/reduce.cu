// Reductions to a scalar: SUM, MAXVAL, MINVAL, DOT_PRODUCT.
//
// SUM lowers to a zero-initialised rank-0 output plus a linalg.reduce over
// the array ("maxval ... also implemented" the same way).  P:317: the paper's
// OpenMP lowering could not parallelise reductions at all; here they are fully
// parallel in the documented combine order R, which makes the
// fp64 result deterministic, path-independent (section == packed copy) and
// reproducible across GPU counts:
//   chunk kernel : one 256-thread block per 65536-element chunk; thread tau owns
//                  the 4-groups at chunk + 1024 m + 4 tau (one 256-bit load each
//                  on the contiguous path), 4 accumulators, then a shfl.xor
//                  butterfly and a fixed 8-warp tree -> P[c]
//   tree kernel  : balanced adjacent-pair tree over P[0..nc) (one block)
// HBM-bound: 8 B/element (16 B for DOT).
#include "ftn_internal.cuh"

#include <cstring>
#include <type_traits>
#include <cmath>

namespace ftn {
namespace {

constexpr int R_THREADS = 256;
constexpr int R_GROUP = 4;
constexpr int64_t R_CHUNK = 65536;
constexpr int R_STEPS = (int)(R_CHUNK / (R_THREADS * R_GROUP));  // 64
constexpr int TREE_THREADS = 1024;

struct RParams {
  KDesc x, y;   // y used by DOT only
  int64_t n;    // number of elements
  int64_t nc;   // number of chunks
};

// accumulator type and combine ops per element type
template <typename T> struct Acc { typedef T type; };
template <> struct Acc<int32_t> { typedef uint32_t type; };
template <> struct Acc<int64_t> { typedef uint64_t type; };

template <typename T, int KIND>
__device__ __forceinline__ typename Acc<T>::type neutral() {
  typedef typename Acc<T>::type A;
  if constexpr (KIND == RK_SUM || KIND == RK_DOT) {
    return A(0);
  } else if constexpr (KIND == RK_PROD) {
    return A(1);
  } else if constexpr (std::is_floating_point<T>::value) {
    return NAN;  // maxNum/minNum ignore NaN (MAXABSDIFF too): an all-NaN (or empty) combine stays NaN (R#11)
  } else {
    if constexpr (sizeof(T) == 4) return (A)(KIND == RK_MAX ? INT32_MIN : INT32_MAX);
    else return (A)(KIND == RK_MAX ? INT64_MIN : INT64_MAX);
  }
}

// MAXVAL / MINVAL of an empty array: -inf / +inf (R#10)
template <typename T, int KIND>
__device__ __forceinline__ typename Acc<T>::type empty_value() {
  if constexpr (std::is_floating_point<T>::value && (KIND == RK_MAX || KIND == RK_MIN || KIND == RK_MAXABSDIFF))
    return KIND == RK_MIN ? INFINITY : -INFINITY;
  return neutral<T, KIND>();
}

template <typename T, int KIND>
__device__ __forceinline__ typename Acc<T>::type combine(typename Acc<T>::type a, typename Acc<T>::type b) {
  if constexpr (KIND == RK_SUM || KIND == RK_DOT) {
    return a + b;  // fp: one IEEE add (RN); ints: modulo 2^w
  } else if constexpr (KIND == RK_PROD) {
    return a * b;  // fp: one IEEE multiply (RN); ints: modulo 2^w
  } else if constexpr (std::is_floating_point<T>::value) {
    return (KIND == RK_MAX || KIND == RK_MAXABSDIFF) ? fmax(a, b) : fmin(a, b);  // maxNum: NaN ignored (R#11)
  } else {
    T x = (T)a, y = (T)b;
    return (typename Acc<T>::type)(KIND == RK_MAX ? (x > y ? x : y) : (x < y ? x : y));
  }
}

template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int mask) {
  return __shfl_xor_sync(0xffffffffu, v, mask);
}

template <typename T>
__device__ __forceinline__ void ld_group(const char* p, T* v) {
  if constexpr (sizeof(T) == 8) {
    unsigned long long a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.v4.b64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
    unsigned long long t[4] = {a, b, c, d};
    memcpy(v, t, 32);
  } else {
    unsigned int a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "l"(p));
    unsigned int t[4] = {a, b, c, d};
    memcpy(v, t, 16);
  }
}

// position (i0, i1, i2) advanced by `delta` elements of array element order
__device__ __forceinline__ void advance(const KDesc& k, int64_t& i0, int64_t& i1, int64_t& i2, int64_t delta) {
  i0 += delta;
  if (i0 >= k.ext[0]) {
    const int64_t q = i0 / k.ext[0];
    i0 -= q * k.ext[0];
    i1 += q;
    if (i1 >= k.ext[1]) {
      const int64_t q2 = i1 / k.ext[1];
      i1 -= q2 * k.ext[1];
      i2 += q2;
    }
  }
}

__device__ __forceinline__ const char* addr(const KDesc& k, int64_t i0, int64_t i1, int64_t i2) {
  return k.base + i0 * k.sm[0] + i1 * k.sm[1] + i2 * k.sm[2];
}

// Steps 1-5 of order R for chunk blockIdx.x.  FLAT: every chunk is one contiguous, 32-byte
// aligned run -- the array is one contiguous run after collapsing, or its (collapsed) rows are
// unit-stride, a whole number of chunks long and aligned, as for a section of whole planes.
// VEC: groups never straddle a row and rows are aligned, so each group is one vector load.
template <typename T, int KIND, bool FLAT, bool VEC>
__global__ void __launch_bounds__(R_THREADS) reduce_chunks(const __grid_constant__ RParams p, void* out) {
  typedef typename Acc<T>::type A;
  const int64_t c = blockIdx.x;
  const int64_t start = c * R_CHUNK;
  const int64_t end = min(start + R_CHUNK, p.n);
  const int tau = threadIdx.x;

  A acc[R_GROUP];
#pragma unroll
  for (int v = 0; v < R_GROUP; ++v) acc[v] = neutral<T, KIND>();

  const int64_t g0 = start + R_GROUP * tau;
  if constexpr (FLAT) {
    // chunk base pointers: element g of the chunk is xp[g - start]
    const int64_t r0 = start % p.x.ext[0], rr = start / p.x.ext[0];
    const int64_t r1 = rr % p.x.ext[1], r2 = rr / p.x.ext[1];
    const T* xp = reinterpret_cast<const T*>(addr(p.x, r0, r1, r2));
    const T* yp = KIND == RK_DOT || KIND == RK_MAXABSDIFF ? reinterpret_cast<const T*>(addr(p.y, r0, r1, r2))
                                                          : nullptr;
    const int64_t l0 = g0 - start;  // this thread's first group, relative to the chunk
    if (end - start == R_CHUNK) {
      constexpr int U = 8;
#pragma unroll 1
      for (int m0 = 0; m0 < R_STEPS; m0 += U) {
        T xv[U][R_GROUP], yv[U][R_GROUP];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          ld_group<T>(reinterpret_cast<const char*>(xp + l0 + 1024 * (m0 + u)), xv[u]);
          if constexpr (KIND == RK_DOT || KIND == RK_MAXABSDIFF)
            ld_group<T>(reinterpret_cast<const char*>(yp + l0 + 1024 * (m0 + u)), yv[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int v = 0; v < R_GROUP; ++v) {
            A e;
            if constexpr (KIND == RK_DOT) e = __dmul_rn(xv[u][v], yv[u][v]);
            else if constexpr (KIND == RK_MAXABSDIFF) e = fabs(__dsub_rn(xv[u][v], yv[u][v]));
            else e = (A)xv[u][v];
            acc[v] = combine<T, KIND>(acc[v], e);
          }
      }
    } else {
      for (int m = 0; m < R_STEPS; ++m) {
        const int64_t g = g0 + 1024 * m;
#pragma unroll
        for (int v = 0; v < R_GROUP; ++v)
          if (g + v < end) {
            A e;
            const int64_t l = g + v - start;
            if constexpr (KIND == RK_DOT) e = __dmul_rn(xp[l], yp[l]);
            else if constexpr (KIND == RK_MAXABSDIFF) e = fabs(__dsub_rn(xp[l], yp[l]));
            else e = (A)xp[l];
            acc[v] = combine<T, KIND>(acc[v], e);
          }
      }
    }
  } else {
    // general descriptor: walk positions incrementally (one division per row crossing)
    int64_t i0 = 0, i1 = 0, i2 = 0;
    if (g0 < end) {
      int64_t t = g0;
      i0 = t % p.x.ext[0];
      t /= p.x.ext[0];
      i1 = t % p.x.ext[1];
      i2 = t / p.x.ext[1];

    }
    for (int m = 0; m < R_STEPS; ++m) {
      const int64_t g = g0 + 1024 * m;
      if (g >= end) break;
      if (VEC && g + R_GROUP <= end) {
        T xv[R_GROUP];
        ld_group<T>(addr(p.x, i0, i1, i2), xv);
#pragma unroll
        for (int v = 0; v < R_GROUP; ++v) acc[v] = combine<T, KIND>(acc[v], (A)xv[v]);
      } else {
        int64_t a0 = i0, a1 = i1, a2 = i2;
#pragma unroll
        for (int v = 0; v < R_GROUP; ++v) {
          if (g + v < end) {
            A e;
            if constexpr (KIND == RK_DOT || KIND == RK_MAXABSDIFF) {
              // the second operand has the same (collapsed) shape: same position, own strides
              const T xv = *reinterpret_cast<const T*>(addr(p.x, a0, a1, a2));
              const T yv = *reinterpret_cast<const T*>(addr(p.y, a0, a1, a2));
              if constexpr (KIND == RK_DOT) e = __dmul_rn(xv, yv);
              else e = fabs(__dsub_rn(xv, yv));
            } else {
              e = (A)*reinterpret_cast<const T*>(addr(p.x, a0, a1, a2));
            }
            acc[v] = combine<T, KIND>(acc[v], e);
          }
          advance(p.x, a0, a1, a2, 1);
        }
      }
      advance(p.x, i0, i1, i2, 1024);
    }
  }

  // step 3: thread value; step 4: butterfly; step 5: fixed 8-warp tree
  A tv = combine<T, KIND>(combine<T, KIND>(acc[0], acc[1]), combine<T, KIND>(acc[2], acc[3]));
#pragma unroll
  for (int mask = 16; mask >= 1; mask >>= 1) tv = combine<T, KIND>(tv, shfl_xor(tv, mask));
  __shared__ A wv[R_THREADS / 32];
  if ((tau & 31) == 0) wv[tau >> 5] = tv;
  __syncthreads();
  if (tau == 0) {
    const A b01 = combine<T, KIND>(wv[0], wv[1]), b23 = combine<T, KIND>(wv[2], wv[3]);
    const A b45 = combine<T, KIND>(wv[4], wv[5]), b67 = combine<T, KIND>(wv[6], wv[7]);
    A r = combine<T, KIND>(combine<T, KIND>(b01, b23), combine<T, KIND>(b45, b67));
    if (p.n == 0) r = empty_value<T, KIND>();
    reinterpret_cast<A*>(out)[c] = r;
  }
}

// Step 6: balanced adjacent-pair tree over part[0..n), padded with the neutral
// element (padding beyond the next power of two changes nothing).
template <typename T, int KIND>
__global__ void __launch_bounds__(TREE_THREADS) tree_kernel(const void* part_v, int64_t n, void* out) {
  typedef typename Acc<T>::type A;
  const A* part = reinterpret_cast<const A*>(part_v);
  int64_t m = 1;
  while (m < n) m <<= 1;
  const int64_t seg = m > TREE_THREADS ? m / TREE_THREADS : 1;  // power of two
  const int t = threadIdx.x;
  A v;
  {
    // this thread's aligned subtree [t*seg, (t+1)*seg) by a binary counter:
    // merging equal-level neighbours left to right builds the balanced tree
    A stk[40];
    int lvl[40];
    int sp = 0;
    for (int64_t i = 0; i < seg; ++i) {
      const int64_t k = (int64_t)t * seg + i;
      A x = k < n ? part[k] : neutral<T, KIND>();
      int l = 0;
      while (sp > 0 && lvl[sp - 1] == l) {
        x = combine<T, KIND>(stk[--sp], x);
        ++l;
      }
      stk[sp] = x;
      lvl[sp++] = l;
    }
    v = stk[0];
  }
  __shared__ A buf[TREE_THREADS];
  buf[t] = v;
  __syncthreads();
  for (int s = 1; s < TREE_THREADS; s <<= 1) {
    if ((t % (2 * s)) == 0) buf[t] = combine<T, KIND>(buf[t], buf[t + s]);
    __syncthreads();
  }
  if (t == 0) *reinterpret_cast<A*>(out) = buf[0];
}

template <typename T, int KIND>
ftn_status_t launch_reduce(const RParams& p, bool flat, bool vec, void* result, void* ws, cudaStream_t s) {
  const int64_t nc = p.nc;
  void* out = nc > 1 ? ws : result;
  const unsigned blocks = (unsigned)(nc > 0 ? nc : 1);
  if (flat)
    reduce_chunks<T, KIND, true, true><<<blocks, R_THREADS, 0, s>>>(p, out);
  else if (vec)
    reduce_chunks<T, KIND, false, true><<<blocks, R_THREADS, 0, s>>>(p, out);
  else
    reduce_chunks<T, KIND, false, false><<<blocks, R_THREADS, 0, s>>>(p, out);
  FTN_CHECK(after_launch("reduce_chunks"));
  if (nc > 1) {
    tree_kernel<T, KIND><<<1, TREE_THREADS, 0, s>>>(ws, nc, result);
    FTN_CHECK(after_launch("reduce_tree"));
  }
  return FTN_OK;
}

template <typename T>
ftn_status_t by_kind(int kind, const RParams& p, bool flat, bool vec, void* result, void* ws, cudaStream_t s) {
  switch (kind) {
    case RK_SUM: return launch_reduce<T, RK_SUM>(p, flat, vec, result, ws, s);
    case RK_MAX: return launch_reduce<T, RK_MAX>(p, flat, vec, result, ws, s);
    case RK_MIN: return launch_reduce<T, RK_MIN>(p, flat, vec, result, ws, s);
    case RK_PROD: return launch_reduce<T, RK_PROD>(p, flat, vec, result, ws, s);
  }
  return fail(FTN_ERR_UNSUPPORTED, "reduce kind");
}

}  // namespace

size_t reduce_ws_bytes(int64_t n) {
  const int64_t nc = (n + R_CHUNK - 1) / R_CHUNK;
  return (size_t)(nc > 1 ? nc : 1) * 8;
}

ftn_status_t reduce_local(int kind, const ftn_desc_t* x, const ftn_desc_t* y, void* result, void* ws,
                          size_t ws_bytes, cudaStream_t stream) {
  RParams p;
  memset(&p, 0, sizeof(p));
  p.n = desc_size(x);
  p.nc = (p.n + R_CHUNK - 1) / R_CHUNK;
  if (p.nc > 1 && (!ws || ws_bytes < reduce_ws_bytes(p.n)))
    return fail(FTN_ERR_WORKSPACE, "reduction workspace too small (need " + std::to_string(reduce_ws_bytes(p.n)) + " bytes)");
  if (p.nc > 1 && ((uintptr_t)ws % 8)) return fail(FTN_ERR_ALIGN, "reduction workspace must be 8-byte aligned");
  const int64_t el = x->elem_len;
  if (kind == RK_DOT || kind == RK_MAXABSDIFF) {
    const ftn_desc_t* arr2[2] = {x, y};
    KDesc kd[2];
    const int r2 = collapse(arr2, 2, kd);
    p.x = kd[0];
    p.y = kd[1];
    auto chunks_flat = [&](const KDesc& k) {
      return k.sm[0] == el && ((uintptr_t)k.base % 32) == 0 &&
             (r2 == 1 || ((k.ext[0] % R_CHUNK) == 0 && (k.sm[1] % 32) == 0 && (k.sm[2] % 32) == 0));
    };
    const bool flat = chunks_flat(p.x) && chunks_flat(p.y);
    const unsigned blocks = (unsigned)(p.nc > 0 ? p.nc : 1);
    void* out = p.nc > 1 ? ws : result;
    if (kind == RK_DOT) {
      if (flat) reduce_chunks<double, RK_DOT, true, true><<<blocks, R_THREADS, 0, stream>>>(p, out);
      else reduce_chunks<double, RK_DOT, false, false><<<blocks, R_THREADS, 0, stream>>>(p, out);
    } else {
      if (flat) reduce_chunks<double, RK_MAXABSDIFF, true, true><<<blocks, R_THREADS, 0, stream>>>(p, out);
      else reduce_chunks<double, RK_MAXABSDIFF, false, false><<<blocks, R_THREADS, 0, stream>>>(p, out);
    }
    FTN_CHECK(after_launch("reduce_chunks(2 operands)"));
    if (p.nc > 1) {
      if (kind == RK_DOT) tree_kernel<double, RK_SUM><<<1, TREE_THREADS, 0, stream>>>(ws, p.nc, result);
      else tree_kernel<double, RK_MAXABSDIFF><<<1, TREE_THREADS, 0, stream>>>(ws, p.nc, result);
      FTN_CHECK(after_launch("reduce_tree"));
    }
    return FTN_OK;
  }
  const ftn_desc_t* arr[1] = {x};
  KDesc k;
  const int r = collapse(arr, 1, &k);
  p.x = k;
  const int64_t va = R_GROUP * el;
  // every chunk one aligned contiguous run (see reduce_chunks)
  const bool flat = k.sm[0] == el && ((uintptr_t)k.base % 32) == 0 &&
                    (r == 1 || ((k.ext[0] % R_CHUNK) == 0 && (k.sm[1] % 32) == 0 && (k.sm[2] % 32) == 0));
  const bool vec = k.sm[0] == el && (k.ext[0] % R_GROUP) == 0 && ((uintptr_t)k.base % va) == 0 &&
                   (k.sm[1] % va) == 0 && (k.sm[2] % va) == 0;
  switch (x->type) {
    case FTN_F64: return by_kind<double>(kind, p, flat, vec, result, ws, stream);
    case FTN_I32: return by_kind<int32_t>(kind, p, flat, vec, result, ws, stream);
    case FTN_I64: return by_kind<int64_t>(kind, p, flat, vec, result, ws, stream);
  }
  return fail(FTN_ERR_TYPE, "reductions accept real(8), integer(4), integer(8)");
}

ftn_status_t tree_combine_launch(int kind, int32_t type, const void* partials, int64_t n, void* result,
                                 cudaStream_t s) {
  if (type == FTN_F64) {
    if (kind == RK_SUM || kind == RK_DOT) tree_kernel<double, RK_SUM><<<1, TREE_THREADS, 0, s>>>(partials, n, result);
    else if (kind == RK_MAX || kind == RK_MAXABSDIFF) tree_kernel<double, RK_MAX><<<1, TREE_THREADS, 0, s>>>(partials, n, result);
    else if (kind == RK_PROD) tree_kernel<double, RK_PROD><<<1, TREE_THREADS, 0, s>>>(partials, n, result);
    else tree_kernel<double, RK_MIN><<<1, TREE_THREADS, 0, s>>>(partials, n, result);
  } else if (type == FTN_I64) {
    if (kind == RK_SUM) tree_kernel<int64_t, RK_SUM><<<1, TREE_THREADS, 0, s>>>(partials, n, result);
    else if (kind == RK_MAX) tree_kernel<int64_t, RK_MAX><<<1, TREE_THREADS, 0, s>>>(partials, n, result);
    else tree_kernel<int64_t, RK_MIN><<<1, TREE_THREADS, 0, s>>>(partials, n, result);
  } else {
    return fail(FTN_ERR_TYPE, "tree_combine: type");
  }
  return after_launch("reduce_tree");
}

}  // namespace ftn

using namespace ftn;

static ftn_status_t reduce_entry(int kind, const char* name, const ftn_desc_t* x, void* result, void* ws,
                                 size_t ws_bytes, ftn_stream_t stream) {
  FTN_CHECK(check_desc(x, name, 1, FTN_MAX_RANK));
  if (!result) return fail(FTN_ERR_NULL, std::string(name) + ": result_dev NULL");
  if (x->type == FTN_F32) return fail(FTN_ERR_TYPE, std::string(name) + ": real(4) reductions are not offered");
  FTN_CHECK(require_sm100());
  return reduce_local(kind, x, nullptr, result, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" {

ftn_status_t ftn_product(const ftn_desc_t* x, void* result_dev, void* ws, size_t ws_bytes, ftn_stream_t stream) {
  return reduce_entry(RK_PROD, "ftn_product", x, result_dev, ws, ws_bytes, stream);
}

ftn_status_t ftn_reduce_workspace_size(const ftn_desc_t* x, size_t* bytes) {
  FTN_CHECK(check_desc(x, "ftn_reduce_workspace_size", 1, FTN_MAX_RANK));
  if (!bytes) return fail(FTN_ERR_NULL, "ftn_reduce_workspace_size: bytes NULL");
  *bytes = reduce_ws_bytes(desc_size(x));
  return FTN_OK;
}

ftn_status_t ftn_sum(const ftn_desc_t* x, void* result_dev, void* ws, size_t ws_bytes, ftn_stream_t stream) {
  return reduce_entry(RK_SUM, "ftn_sum", x, result_dev, ws, ws_bytes, stream);
}
ftn_status_t ftn_maxval(const ftn_desc_t* x, void* result_dev, void* ws, size_t ws_bytes, ftn_stream_t stream) {
  return reduce_entry(RK_MAX, "ftn_maxval", x, result_dev, ws, ws_bytes, stream);
}
ftn_status_t ftn_minval(const ftn_desc_t* x, void* result_dev, void* ws, size_t ws_bytes, ftn_stream_t stream) {
  return reduce_entry(RK_MIN, "ftn_minval", x, result_dev, ws, ws_bytes, stream);
}

ftn_status_t ftn_maxval_absdiff(const ftn_desc_t* x, const ftn_desc_t* y, void* result_dev, void* ws,
                                size_t ws_bytes, ftn_stream_t stream) {
  FTN_CHECK(check_desc(x, "ftn_maxval_absdiff(x)", 1, FTN_MAX_RANK));
  FTN_CHECK(check_desc(y, "ftn_maxval_absdiff(y)", 1, FTN_MAX_RANK));
  if (x->type != FTN_F64 || y->type != FTN_F64) return fail(FTN_ERR_TYPE, "ftn_maxval_absdiff: real(8) only");
  if (!same_shape(x, y)) return fail(FTN_ERR_SHAPE, "ftn_maxval_absdiff: x and y are not conformable");
  if (!result_dev) return fail(FTN_ERR_NULL, "ftn_maxval_absdiff: result_dev NULL");
  FTN_CHECK(require_sm100());
  return reduce_local(RK_MAXABSDIFF, x, y, result_dev, ws, ws_bytes, (cudaStream_t)stream);
}

ftn_status_t ftn_dot_product(const ftn_desc_t* x, const ftn_desc_t* y, void* result_dev, void* ws, size_t ws_bytes,
                             ftn_stream_t stream) {
  FTN_CHECK(check_desc(x, "ftn_dot_product(x)", 1, 1));
  FTN_CHECK(check_desc(y, "ftn_dot_product(y)", 1, 1));
  if (x->type != FTN_F64 || y->type != FTN_F64)
    return fail(FTN_ERR_TYPE, "ftn_dot_product: real(8) vectors only");
  if (x->dim[0].extent != y->dim[0].extent) return fail(FTN_ERR_SHAPE, "ftn_dot_product: sizes differ");
  if (!result_dev) return fail(FTN_ERR_NULL, "ftn_dot_product: result_dev NULL");
  FTN_CHECK(require_sm100());
  return reduce_local(RK_DOT, x, y, result_dev, ws, ws_bytes, (cudaStream_t)stream);
}

}  // extern "C"
