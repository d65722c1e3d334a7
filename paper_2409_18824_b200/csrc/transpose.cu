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
//
// TMA path (8-byte elements; both operands unit-stride in dim 1 with 16-byte aligned bases and
// columns): a persistent CTA moves tiles of TI x TJ elements (32 x 32 for 8-byte types; the
// kernel also handles 4-byte types with 64 x 64 tiles, slower than the path above for them)
// as 128-byte-wide boxes.  Two
// boxes {E, TJ} of src arrive by TMA (cp.async.bulk.tensor, 128-byte swizzle) into one of
// two stages; each thread transposes one V x V block (V = 16 / elem_len) in registers -- V
// 16-byte shared loads, V 16-byte shared stores -- into the two swizzled output boxes
// {E, TI} of dst, which one thread stores with TMA (bulk groups, two stages).  The
// thread -> block map (lane = 8 p + x: chunk x, row block b + ((x >> log2(8/V)) ^ p)) makes
// every quarter-warp phase of both the loads and the stores touch 8 distinct 16-byte bank
// groups under the 128-byte swizzle: no bank conflicts.  Ragged edge tiles need no separate
// path: TMA zero-fills out-of-range loads and clips out-of-range stores.
#include "ftn_internal.cuh"

#include <atomic>

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

#ifndef FTN_TT_NIN
#define FTN_TT_NIN 2  // input boxes per tile (tile extent in dim 1 = NIN * 128 bytes)
#endif
#ifndef FTN_TT_NS
#define FTN_TT_NS 2   // pipeline stages (input and output)
#endif

template <typename T>
struct TmaCfg {
  static constexpr int V = 16 / sizeof(T);   // elements per 16-byte chunk
  static constexpr int E = 128 / sizeof(T);  // elements per 128-byte box row (the swizzle span)
  static constexpr int NIN = FTN_TT_NIN, NS = FTN_TT_NS;
  static constexpr int TI = NIN * E;         // tile extent in dim 1 of src
  static constexpr int TJ = 16 * V;          // tile extent in dim 2 of src
  static constexpr int IN_BOX = TJ * 128, OUT_BOX = TI * 128;
  static constexpr int NOUT = TJ / E;        // output boxes per tile
  static constexpr int STAGE_IN = NIN * IN_BOX, STAGE_OUT = NOUT * OUT_BOX;
  static constexpr int SMEM = NS * (STAGE_IN + STAGE_OUT) + 8 * NS + 1024;  // + barriers, 1024-B alignment
  static_assert(NOUT == 2 && E / V == 8 && NIN % 2 == 0, "tile geometry");
};

template <typename T>
__global__ void __launch_bounds__(T_THREADS) transpose_tma(const __grid_constant__ CUtensorMap in_map,
                                                           const __grid_constant__ CUtensorMap out_map,
                                                           int64_t tiles_i, int64_t tiles) {
  using C = TmaCfg<T>;
  constexpr int V = C::V, E = C::E, NS = C::NS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* in = sm;
  uint8_t* out = sm + NS * C::STAGE_IN;
  uint64_t* full = reinterpret_cast<uint64_t*>(out + NS * C::STAGE_OUT);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int p = lane >> 3, x = lane & 7;
  const int cq = x;                                     // 16-byte chunk of the box row
  const int jr = 4 * (warp & 3) + ((x >> (V == 4 ? 1 : 2)) ^ p);  // block of V rows
  const int g = (V * jr) / E, dq = jr & 7;              // output box and its 16-byte chunk
  // box pair hp: input boxes 2 hp + (warp >> 2)
  uint32_t ld_off[C::NIN / 2][V], st_off[C::NIN / 2][V];
#pragma unroll
  for (int hp = 0; hp < C::NIN / 2; ++hp) {
    const int h = 2 * hp + (warp >> 2);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int jj = V * jr + k;                        // input box row (dim 2)
      ld_off[hp][k] = (uint32_t)(h * C::IN_BOX + jj * 128 + ((cq ^ (jj & 7)) << 4));
    }
#pragma unroll
    for (int m = 0; m < V; ++m) {
      const int row = h * E + V * cq + m;               // output box row (dim 1 of src)
      st_off[hp][m] = (uint32_t)(g * C::OUT_BOX + row * 128 + ((dq ^ (row & 7)) << 4));
    }
  }
  const uint32_t in_s = dev::smem_u32(in), out_s = dev::smem_u32(out);
  const int64_t G = gridDim.x;
  auto issue = [&](int64_t t, int st) {
    const int32_t i0 = (int32_t)((t % tiles_i) * C::TI), j0 = (int32_t)((t / tiles_i) * C::TJ);
    dev::mbar_arrive_expect_tx(&full[st], C::STAGE_IN);
#pragma unroll
    for (int h = 0; h < C::NIN; ++h)
      dev::tma_load_2d(in + st * C::STAGE_IN + h * C::IN_BOX, &in_map, &full[st], i0 + h * E, j0);
  };
  int64_t w = blockIdx.x;
  if (tid == 0) {
    for (int q = 0; q < NS; ++q) dev::mbar_init(&full[q], 1);
    dev::fence_barrier_init();
    dev::prefetch_tma(&in_map);
    dev::prefetch_tma(&out_map);
    for (int q = 0; q < NS; ++q)
      if (w + q * G < tiles) issue(w + q * G, q);
  }
  __syncthreads();
  int st = 0;
  uint32_t ph = 0;
  for (; w < tiles; w += G) {
    dev::mbar_wait(&full[st], ph);
    if (tid == 0) dev::bulk_wait_read<NS - 1>();        // the store NS tiles back has read this stage
    __syncthreads();
#pragma unroll
    for (int hp = 0; hp < C::NIN / 2; ++hp) {
      uint32_t v[V][4];
#pragma unroll
      for (int k = 0; k < V; ++k)
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[k][0]), "=r"(v[k][1]), "=r"(v[k][2]), "=r"(v[k][3])
                     : "r"(in_s + st * C::STAGE_IN + ld_off[hp][k]));
#pragma unroll
      for (int m = 0; m < V; ++m) {
        uint32_t o[4];
        if (V == 4) {
#pragma unroll
          for (int k = 0; k < 4; ++k) o[k] = v[k][m];
        } else {  // 8-byte elements: element m of row k is the u32 pair (2m, 2m+1)
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            o[2 * k] = v[k][2 * m];
            o[2 * k + 1] = v[k][2 * m + 1];
          }
        }
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(out_s + st * C::STAGE_OUT + st_off[hp][m]),
                     "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3])
                     : "memory");
      }
    }
    dev::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      const int32_t i0 = (int32_t)((w % tiles_i) * C::TI), j0 = (int32_t)((w / tiles_i) * C::TJ);
#pragma unroll
      for (int q = 0; q < C::NOUT; ++q)
        dev::tma_store_2d(&out_map, out + st * C::STAGE_OUT + q * C::OUT_BOX, j0 + q * E, i0);
      dev::bulk_commit();
      if (w + NS * G < tiles) issue(w + NS * G, st);    // every thread has read input stage st
    }
    if (++st == NS) {
      st = 0;
      ph ^= 1;
    }
  }
  if (tid == 0) dev::bulk_wait<0>();
}

bool tma_able_2d(const ftn_desc_t* d) {
  return d->dim[0].sm == d->elem_len && ((uintptr_t)d->base_addr % 16) == 0 && d->dim[1].sm > 0 &&
         (d->dim[1].sm % 16) == 0 && d->dim[0].extent < (int64_t(1) << 31) && d->dim[1].extent < (int64_t(1) << 31);
}

template <typename T>
ftn_status_t launch_tma(const ftn_desc_t* dst, const ftn_desc_t* src, cudaStream_t s) {
  using C = TmaCfg<T>;
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64;
  CUtensorMap in_map, out_map;
  {
    uint64_t dims[2] = {(uint64_t)src->dim[0].extent, (uint64_t)src->dim[1].extent};
    uint64_t strides[1] = {(uint64_t)src->dim[1].sm};
    uint32_t box[2] = {(uint32_t)C::E, (uint32_t)C::TJ};
    FTN_CHECK(encode_tma(&in_map, dt, 2, src->base_addr, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  {
    uint64_t dims[2] = {(uint64_t)dst->dim[0].extent, (uint64_t)dst->dim[1].extent};
    uint64_t strides[1] = {(uint64_t)dst->dim[1].sm};
    uint32_t box[2] = {(uint32_t)C::E, (uint32_t)C::TI};  // TI <= 256 (TMA box limit)
    FTN_CHECK(encode_tma(&out_map, dt, 2, dst->base_addr, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  const int64_t tiles_i = (src->dim[0].extent + C::TI - 1) / C::TI;
  const int64_t tiles = tiles_i * ((src->dim[1].extent + C::TJ - 1) / C::TJ);
  static std::atomic<int> occ[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!occ[dev & 63]) {
    FTN_CUDA(cudaFuncSetAttribute(transpose_tma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    int o = 0;
    FTN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, transpose_tma<T>, T_THREADS, C::SMEM));
    occ[dev & 63] = o > 0 ? o : 1;
  }
  const int64_t maxb = (int64_t)num_sms() * occ[dev & 63];
  const unsigned blocks = (unsigned)(tiles < maxb ? tiles : maxb);
  transpose_tma<T><<<blocks, T_THREADS, C::SMEM, s>>>(in_map, out_map, tiles_i, tiles);
  return after_launch("transpose_tma");
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
  static const bool no_tma = getenv("FTN_TRANSPOSE_NO_TMA") != nullptr;  // A/B timing of the two paths
  // 8-byte elements take the TMA path (16384^2 real(8): 5.80 vs 5.58 TB/s); 4-byte elements keep
  // the 16-byte-load path, which is faster for them (32768^2 int32: 6.31 vs 5.83 TB/s with TMA;
  // 2 or 4 input boxes per tile and 2 or 3 stages all measured 5.74-5.83)
  if (!no_tma && el == 8 && tma_able_2d(src) && tma_able_2d(dst)) return launch_tma<uint64_t>(dst, src, s);
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
