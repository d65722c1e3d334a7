// TRANSPOSE: dst(j, i) = src(i, j), P:298 / P:309.
//
// The paper's slowest intrinsic (Table III: 214 s serial, 40.8 s on 64 cores for
// int32 32768^2): the strided side of the access kills locality.  Here a
// 64x64 tile is read with dim-1-contiguous (coalesced) loads into padded shared
// memory and written back with dim-1-contiguous stores of the result, so both
// HBM streams are sector-efficient.  On full tiles of unit-stride, 16-byte
// aligned operands every thread moves 16 bytes per global access (4 int32 or
// 2 fp64); ragged edge tiles and strided sections take the element-wise path.
// Pure data movement: 2 * elem_len bytes per element.
#include "ftn_internal.cuh"

namespace ftn {
namespace {

constexpr int TT = 64;           // tile edge
constexpr int T_THREADS = 256;

struct TParams {
  KDesc dst, src;
  int64_t n1, n2;      // src extents
  int64_t tiles1, tiles;
  int vec;             // operands allow 16-byte accesses
};

template <typename T>
__global__ void __launch_bounds__(T_THREADS) transpose_kernel(const __grid_constant__ TParams p) {
  constexpr int V = 16 / sizeof(T);       // elements per 16-byte vector
  constexpr int GPR = TT / V;             // vector groups per tile row
  __shared__ T tile[TT][TT + 1];
  const int tid = threadIdx.x;
  for (int64_t w = blockIdx.x; w < p.tiles; w += gridDim.x) {
    const int64_t i0 = (w % p.tiles1) * TT;
    const int64_t j0 = (w / p.tiles1) * TT;
    const bool full = p.vec && i0 + TT <= p.n1 && j0 + TT <= p.n2;
    if (full) {
      // load: tile[jj][ii..ii+V) = src(i0+ii.., j0+jj) with one 16-byte load
#pragma unroll
      for (int q = 0; q < TT * GPR / T_THREADS; ++q) {
        const int g = tid + q * T_THREADS;
        const int jj = g / GPR, ii = (g % GPR) * V;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.src.base + (i0 + ii) * (int64_t)sizeof(T) +
                                                             (j0 + jj) * p.src.sm[1]));
        const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
        for (int k = 0; k < V; ++k) tile[jj][ii + k] = e[k];
      }
      __syncthreads();
      // store: dst(j0+jj.., i0+ii) = tile[jj..jj+V)[ii] with one 16-byte store
#pragma unroll
      for (int q = 0; q < TT * GPR / T_THREADS; ++q) {
        const int g = tid + q * T_THREADS;
        const int ii = g / GPR, jj = (g % GPR) * V;
        uint4 v;
        T* e = reinterpret_cast<T*>(&v);
#pragma unroll
        for (int k = 0; k < V; ++k) e[k] = tile[jj + k][ii];
        *reinterpret_cast<uint4*>(p.dst.base + (j0 + jj) * (int64_t)sizeof(T) + (i0 + ii) * p.dst.sm[1]) = v;
      }
      __syncthreads();
      continue;
    }
    const int tx = tid & (TT - 1);
    const int ty = tid / TT;  // 0..3
    const int64_t i = i0 + tx;
#pragma unroll 4
    for (int jj = ty; jj < TT; jj += T_THREADS / TT) {
      const int64_t j = j0 + jj;
      if (i < p.n1 && j < p.n2)
        tile[jj][tx] = *reinterpret_cast<const T*>(p.src.base + i * p.src.sm[0] + j * p.src.sm[1]);
    }
    __syncthreads();
    const int64_t j = j0 + tx;
#pragma unroll 4
    for (int ii = ty; ii < TT; ii += T_THREADS / TT) {
      const int64_t i2 = i0 + ii;
      if (j < p.n2 && i2 < p.n1)
        *reinterpret_cast<T*>(p.dst.base + j * p.dst.sm[0] + i2 * p.dst.sm[1]) = tile[tx][ii];
    }
    __syncthreads();
  }
}

ftn_status_t launch(const ftn_desc_t* dst, const ftn_desc_t* src, cudaStream_t s) {
  TParams p;
  p.dst = to_kdesc(dst);
  p.src = to_kdesc(src);
  p.n1 = src->dim[0].extent;
  p.n2 = src->dim[1].extent;
  p.tiles1 = (p.n1 + TT - 1) / TT;
  p.tiles = p.tiles1 * ((p.n2 + TT - 1) / TT);
  const int64_t el = src->elem_len;
  p.vec = p.src.sm[0] == el && p.dst.sm[0] == el && ((uintptr_t)p.src.base % 16) == 0 &&
          ((uintptr_t)p.dst.base % 16) == 0 && (p.src.sm[1] % 16) == 0 && (p.dst.sm[1] % 16) == 0;
  if (p.tiles == 0) return FTN_OK;
  const int64_t maxb = (int64_t)num_sms() * 8 * 16;
  const unsigned blocks = (unsigned)(p.tiles < maxb ? p.tiles : maxb);
  switch (src->elem_len) {
    case 4: transpose_kernel<uint32_t><<<blocks, T_THREADS, 0, s>>>(p); break;
    case 8: transpose_kernel<uint64_t><<<blocks, T_THREADS, 0, s>>>(p); break;
    default: return fail(FTN_ERR_TYPE, "transpose: element size");
  }
  return after_launch("transpose_kernel");
}

}  // namespace
}  // namespace ftn

using namespace ftn;

extern "C" ftn_status_t ftn_transpose(const ftn_desc_t* dst, const ftn_desc_t* src, ftn_stream_t stream) {
  FTN_CHECK(check_desc(dst, "ftn_transpose(dst)", 2, 2));
  FTN_CHECK(check_desc(src, "ftn_transpose(src)", 2, 2));
  if (dst->type != src->type) return fail(FTN_ERR_TYPE, "ftn_transpose: types differ");
  if (dst->dim[0].extent != src->dim[1].extent || dst->dim[1].extent != src->dim[0].extent)
    return fail(FTN_ERR_SHAPE, "ftn_transpose: dst shape must be (n2, n1)");
  FTN_CHECK(require_sm100());
  cudaStream_t s = (cudaStream_t)stream;
  if (!desc_overlap(dst, src)) return launch(dst, src, s);
  StreamTemp tmp;  // R#5: overlapping dst -> through a temporary
  FTN_CHECK(tmp.alloc((size_t)desc_size(dst) * dst->elem_len, s));
  ftn_desc_t t;
  FTN_CHECK(make_packed(&t, tmp.ptr, dst));
  FTN_CHECK(launch(&t, src, s));
  return launch_copy(dst, &t, s);
}
