// Jacobi sweeps, P:92 ("a Jacobi iteration solving Laplace's
// equation"), Table II (249 s for 1024^2 x 10^5 on one EPYC core), Table IV.
//
//   unew(i,j)   = c * (((u(i-1,j) + u(i+1,j)) + u(i,j-1)) + u(i,j+1))            (2-D)
//   unew(i,j,k) = c * (((((u(i-1)+u(i+1)) + u(j-1)) + u(j+1)) + u(k-1)) + u(k+1))  (3-D)
//
// Same neighbour order and the same single rounding per add as the oracle
// (compiled with -fmad=false), so results are bit-exact.
//
// HBM-bound at 16 B per lattice update (read u once, write unew once).  The
// paper's stencil problems were missing vectorisation and dynamic shapes (P:281-
// 286); here each CTA streams a strip of the grid through shared memory with TMA
// (cp.async.bulk.tensor + mbarrier pipeline, one producer warp), so every u value
// is read from HBM once per sweep and reused from shared memory by its 4 (6)
// neighbours.
//   2-D: strips 128 columns wide; stages of {132 x 32} rows (30 output rows, 1-row
//        halo each side), 3 stages.
//   3-D: columns of 128 x 16 points streamed along k; a ring of 5 planes
//        {132 x 18}, outputs for plane k once plane k+1 has landed.
// Work is split evenly over a persistent grid (2 CTAs per SM) in row (plane)
// units, so every CTA moves the same number of bytes.
#include "ftn_internal.cuh"

#include <cstring>
#include <cstdlib>
#include <vector>

namespace ftn {

// Split `len` rows (planes) of each of `tiles` strips (columns) into segments so that the
// units (tiles x segments) fill whole waves of `grid` CTAs: minimise
//   wave-quantisation loss x re-read halo rows (`halo_rows` per segment, they miss L2).
void plan_units_halo(int64_t tiles, int64_t len, int64_t grid, int64_t halo_rows, int64_t* seg, int64_t* units) {
  double best = 1e30;
  int64_t best_n = 1;
  for (int64_t nseg = 1; nseg <= 512 && nseg <= len; ++nseg) {
    const int64_t sl = (len + nseg - 1) / nseg;
    const int64_t nseg_eff = (len + sl - 1) / sl;
    const int64_t U = tiles * nseg_eff;
    const int64_t waves = (U + grid - 1) / grid;
    const double cost = (double)waves * grid / (double)U * (1.0 + (double)halo_rows / (double)(sl + halo_rows));
    if (cost < best - 1e-9) {
      best = cost;
      best_n = nseg;
    }
  }
  *seg = (len + best_n - 1) / best_n;
  *units = tiles * ((len + *seg - 1) / *seg);
}

ftn_status_t jacobi2d_fused(const ftn_desc_t* src, const ftn_desc_t* dst, int T, double coeff, cudaStream_t s);
ftn_status_t jacobi3d_fused2(const ftn_desc_t* src, const ftn_desc_t* dst, double coeff, cudaStream_t s);
ftn_status_t jacobi3d_wr_planes(const ftn_desc_t* src, const ftn_desc_t* dst, int T, double coeff, int64_t plane_lo,
                                int64_t plane_hi, int64_t fix_lo, int64_t fix_hi, cudaStream_t s);
ftn_status_t jacobi3d_fused2_planes(const ftn_desc_t* src, const ftn_desc_t* dst, double coeff, int64_t plane_lo,
                                    int64_t plane_hi, int64_t fix_lo, int64_t fix_hi, cudaStream_t s);
ftn_status_t jacobi2d_fused_rows(const ftn_desc_t* src, const ftn_desc_t* dst, int T, double coeff, int64_t row_lo,
                                 int64_t row_hi, int64_t fix_lo, int64_t fix_hi, cudaStream_t s, double* res);

bool stencil_tma_able(const ftn_desc_t* d) {
  if (d->type != FTN_F64 || d->dim[0].sm != 8 || ((uintptr_t)d->base_addr % 16) != 0) return false;
  for (int k = 1; k < d->rank; ++k)
    if (d->dim[k].sm <= 0 || (d->dim[k].sm % 16) != 0 || d->dim[k].sm >= (1ll << 40)) return false;
  for (int k = 0; k < d->rank; ++k)
    if (d->dim[k].extent >= (1ll << 31)) return false;
  return true;
}

namespace {

// ---------------------------------------------------------------- 2-D
constexpr int S2_W = 128;              // interior columns per strip
// The box starts 2 columns left of the strip: TMA needs the dim-0 start of a box
// 16-byte aligned (an odd fp64 coordinate such as -1 raises "illegal instruction",
// tools/microbench/tma_probe.cu), so the halo column i0-1 comes with i0-2.
constexpr int S2_BOXW = S2_W + 4;      // 132: columns i0-2 .. i0+129
constexpr int S2_X0 = 2;               // smem column of i0
constexpr int S2_R = 30;               // output rows per stage
constexpr int S2_BOXH = S2_R + 2;      // 32
constexpr int S2_STAGES = 3;
constexpr int S2_STAGE_BYTES = S2_BOXW * S2_BOXH * 8;  // 33792
constexpr int S2_CONS_WARPS = S2_W / 32;               // 4
constexpr int S2_THREADS = (S2_CONS_WARPS + 1) * 32;
constexpr int S2_SMEM = S2_STAGES * S2_STAGE_BYTES + 128 + 64;

struct J2Params {
  char* dst;
  int64_t d_sm1, d_sm2;
  int64_t n1, n2;
  int64_t tiles_i;  // strips
  int64_t nrows;    // rows to update
  int64_t seg;      // rows per work unit
  int64_t units;    // tiles_i * ceil(nrows / seg)
  int64_t lo;       // first output row (0-based position in dim 2)
  double coeff;
};

// Work units u = strip + tiles_i * segment (strip fastest), taken round-robin by the
// CTAs: units of one wave are neighbouring strips over the same rows, so the halo
// columns a CTA loads were just brought into L2 by its neighbours (no DRAM re-read).
// Each unit is streamed in chunks of at most S2_R rows.
struct ChunkIter2 {
  int64_t u, G, units, tiles, seg, nrows, lo;
  int64_t strip = 0, r = 0, rend = 0;
  __device__ bool next(int64_t& s_out, int64_t& j0, int& cnt) {
    while (r >= rend) {
      u += G;
      if (u >= units) return false;
      strip = u % tiles;
      r = (u / tiles) * seg;
      rend = min(r + seg, nrows);
    }
    const int64_t n = min((int64_t)S2_R, rend - r);
    s_out = strip;
    j0 = lo + r;
    cnt = (int)n;
    r += n;
    return true;
  }
};

__global__ void __launch_bounds__(S2_THREADS) jacobi2d_tma(const __grid_constant__ CUtensorMap src_map,
                                                           const __grid_constant__ J2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S2_STAGES * S2_STAGE_BYTES);
  uint64_t* empty = full + S2_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S2_STAGES; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], S2_CONS_WARPS);
    }
    dev::fence_barrier_init();
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  const ChunkIter2 it0{(int64_t)blockIdx.x - G, G, p.units, p.tiles_i, p.seg, p.nrows, p.lo};

  if (warp == S2_CONS_WARPS) {
    if (lane == 0) {
      dev::prefetch_tma(&src_map);
      ChunkIter2 it = it0;
      int64_t strip, j0;
      int cnt;
      int k = 0;
      for (; it.next(strip, j0, cnt); ++k) {
        const int s = k % S2_STAGES;
        if (k >= S2_STAGES) dev::mbar_wait_idle(&empty[s], ((k / S2_STAGES) - 1) & 1);
        dev::mbar_arrive_expect_tx(&full[s], S2_STAGE_BYTES);
        dev::tma_load_2d(smem + s * S2_STAGE_BYTES, &src_map, &full[s], (int32_t)(strip * S2_W - S2_X0),
                         (int32_t)(j0 - 1));
      }
      // producer tail: do not retire while loads are in flight / unconsumed
      for (int kk = k - S2_STAGES > 0 ? k - S2_STAGES : 0; kk < k; ++kk)
        dev::mbar_wait_idle(&empty[kk % S2_STAGES], (kk / S2_STAGES) & 1);
    }
    return;
  }

  const int x = threadIdx.x;  // column within the strip
  ChunkIter2 it = it0;
  int64_t strip, j0;
  int cnt;
  const double c = p.coeff;
  for (int k = 0; it.next(strip, j0, cnt); ++k) {
    const int s = k % S2_STAGES;
    const int64_t i = strip * S2_W + x;
    const bool active = i >= 1 && i <= p.n1 - 2;
    dev::mbar_wait(&full[s], (k / S2_STAGES) & 1);
    const double* t = reinterpret_cast<const double*>(smem + s * S2_STAGE_BYTES);
    // smem row r holds u(:, j0 - 1 + r); column x + 2 holds i
    const int xc = x + S2_X0;
    double up = t[xc], mid = t[S2_BOXW + xc];
    char* out = p.dst + i * p.d_sm1 + j0 * p.d_sm2;
    for (int r = 1; r <= cnt; ++r) {
      const double* row = t + r * S2_BOXW;
      const double down = row[S2_BOXW + xc];
      double v = row[xc - 1] + row[xc + 1];
      v = v + up;
      v = v + down;
      if (active) *reinterpret_cast<double*>(out) = c * v;
      out += p.d_sm2;
      up = mid;
      mid = down;
    }
    __syncwarp();
    if (lane == 0) dev::mbar_arrive(&empty[s]);
  }
}

// ---------------------------------------------------------------- 3-D
constexpr int S3_W = 128, S3_H = 16;
constexpr int S3_BOXW = S3_W + 4, S3_BOXH = S3_H + 2;  // 132 x 18 (dim-0 start 16-byte aligned, see S2_BOXW)
constexpr int S3_STAGES = 5;
constexpr int S3_PLANE_BYTES = S3_BOXW * S3_BOXH * 8;  // 19008 (TMA transaction bytes)
constexpr int S3_PLANE_STRIDE = (S3_PLANE_BYTES + 127) / 128 * 128;  // 128-byte aligned stages
constexpr int S3_ROWS_PER_THREAD = 8;
constexpr int S3_CONS_THREADS = S3_W * S3_H / S3_ROWS_PER_THREAD;  // 256
constexpr int S3_CONS_WARPS = S3_CONS_THREADS / 32;                // 8
constexpr int S3_THREADS = S3_CONS_THREADS + 32;
constexpr int S3_SMEM = S3_STAGES * S3_PLANE_STRIDE + 128 + 128;

struct J3Params {
  char* dst;
  int64_t d_sm1, d_sm2, d_sm3;
  int64_t n1, n2, n3;
  int64_t tiles_i, tiles_j;
  int64_t nk;      // planes to update
  int64_t seg;     // planes per work unit
  int64_t units;   // tiles_i * tiles_j * ceil(nk / seg)
  int64_t lo;      // first output plane
  double coeff;
};

// Work units u = column + ncols * segment (column = i-tile fastest, then j-tile), taken
// round-robin: one wave streams neighbouring columns through the same planes together.
struct SegIter3 {
  int64_t u, G, units, ncols, seg, nk, lo;
  __device__ bool next(int64_t& col, int64_t& k0, int64_t& n) {
    u += G;
    if (u >= units) return false;
    col = u % ncols;
    const int64_t r = (u / ncols) * seg;
    n = min(seg, nk - r);
    k0 = lo + r;
    return true;
  }
};

__global__ void __launch_bounds__(S3_THREADS) jacobi3d_tma(const __grid_constant__ CUtensorMap src_map,
                                                           const __grid_constant__ J3Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S3_STAGES * S3_PLANE_STRIDE);
  uint64_t* empty = full + S3_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S3_STAGES; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], S3_CONS_WARPS);
    }
    dev::fence_barrier_init();
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  const SegIter3 it0{(int64_t)blockIdx.x - G, G, p.units, p.tiles_i * p.tiles_j, p.seg, p.nk, p.lo};

  if (warp == S3_CONS_WARPS) {
    if (lane == 0) {
      dev::prefetch_tma(&src_map);
      SegIter3 it = it0;
      int64_t col, k0, n;
      int64_t gp = 0;  // global plane counter of this CTA
      while (it.next(col, k0, n)) {
        const int32_t ci = (int32_t)((col % p.tiles_i) * S3_W - 2);
        const int32_t cj = (int32_t)((col / p.tiles_i) * S3_H - 1);
        for (int64_t kk = k0 - 1; kk <= k0 + n; ++kk, ++gp) {
          const int s = (int)(gp % S3_STAGES);
          if (gp >= S3_STAGES) dev::mbar_wait_idle(&empty[s], (uint32_t)(((gp / S3_STAGES) - 1) & 1));
          dev::mbar_arrive_expect_tx(&full[s], S3_PLANE_BYTES);
          dev::tma_load_3d(smem + s * S3_PLANE_STRIDE, &src_map, &full[s], ci, cj, (int32_t)kk);
        }
      }
      for (int64_t q = gp - S3_STAGES > 0 ? gp - S3_STAGES : 0; q < gp; ++q)   // producer tail
        dev::mbar_wait_idle(&empty[q % S3_STAGES], (uint32_t)((q / S3_STAGES) & 1));
    }
    return;
  }

  const int x = threadIdx.x % S3_W;
  const int yb = threadIdx.x / S3_W;  // 0..1
  SegIter3 it = it0;
  int64_t col, k0, n;
  int64_t gp = 0;
  const double c = p.coeff;
  while (it.next(col, k0, n)) {
    const int64_t i = (col % p.tiles_i) * S3_W + x;
    const int64_t jbase = (col / p.tiles_i) * S3_H + yb * S3_ROWS_PER_THREAD;
    const bool iact = i >= 1 && i <= p.n1 - 2;
    // planes gp (k0-1) and gp+1 (k0) first
    dev::mbar_wait(&full[gp % S3_STAGES], (uint32_t)((gp / S3_STAGES) & 1));
    dev::mbar_wait(&full[(gp + 1) % S3_STAGES], (uint32_t)(((gp + 1) / S3_STAGES) & 1));
    for (int64_t q = 0; q < n; ++q) {
      const int64_t pn = gp + q + 2;  // plane k+1
      dev::mbar_wait(&full[pn % S3_STAGES], (uint32_t)((pn / S3_STAGES) & 1));
      const double* Pm = reinterpret_cast<const double*>(smem + ((gp + q) % S3_STAGES) * S3_PLANE_STRIDE);
      const double* P0 = reinterpret_cast<const double*>(smem + ((gp + q + 1) % S3_STAGES) * S3_PLANE_STRIDE);
      const double* Pp = reinterpret_cast<const double*>(smem + (pn % S3_STAGES) * S3_PLANE_STRIDE);
      const int64_t k = k0 + q;
      const int r0 = yb * S3_ROWS_PER_THREAD + 1;  // smem row of the first j
      const int xc = x + 2;  // smem column of i
      double jm = P0[(r0 - 1) * S3_BOXW + xc];
      double jc = P0[r0 * S3_BOXW + xc];
      char* out = p.dst + i * p.d_sm1 + jbase * p.d_sm2 + k * p.d_sm3;
#pragma unroll
      for (int jj = 0; jj < S3_ROWS_PER_THREAD; ++jj) {
        const int r = r0 + jj;
        const double jp = P0[(r + 1) * S3_BOXW + xc];
        double v = P0[r * S3_BOXW + xc - 1] + P0[r * S3_BOXW + xc + 1];
        v = v + jm;
        v = v + jp;
        v = v + Pm[r * S3_BOXW + xc];
        v = v + Pp[r * S3_BOXW + xc];
        const int64_t j = jbase + jj;
        if (iact && j >= 1 && j <= p.n2 - 2) *reinterpret_cast<double*>(out) = c * v;
        out += p.d_sm2;
        jm = jc;
        jc = jp;
      }
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&empty[(gp + q) % S3_STAGES]);  // plane k-1 is done
    }
    __syncwarp();
    if (lane == 0) {
      dev::mbar_arrive(&empty[(gp + n) % S3_STAGES]);
      dev::mbar_arrive(&empty[(gp + n + 1) % S3_STAGES]);
    }
    gp += n + 2;
  }
}

// ---------------------------------------------------------------- generic (any strides)
struct JGParams {
  KDesc src, dst;
  int rank;
  int64_t n1, n2, n3;
  int64_t k_lo, k_hi;  // planes (3-D) / rows (2-D) of the last dim to update, inclusive
  double coeff;
};

__global__ void __launch_bounds__(256) jacobi_generic(const __grid_constant__ JGParams p) {
  const int64_t m1 = p.n1 - 2;
  const int64_t m2 = p.rank == 3 ? p.n2 - 2 : 1;
  const int64_t nl = p.k_hi - p.k_lo + 1;
  const int64_t total = m1 * m2 * nl;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = 1 + t % m1;
    const int64_t rest = t / m1;
    const char* b = p.src.base;
    const int64_t s0 = p.src.sm[0], s1 = p.src.sm[1], s2 = p.src.sm[2];
    if (p.rank == 2) {
      const int64_t j = p.k_lo + rest;
      const char* c0 = b + i * s0 + j * s1;
      double v = *(const double*)(c0 - s0) + *(const double*)(c0 + s0);
      v = v + *(const double*)(c0 - s1);
      v = v + *(const double*)(c0 + s1);
      *(double*)(p.dst.base + i * p.dst.sm[0] + j * p.dst.sm[1]) = p.coeff * v;
    } else {
      const int64_t j = 1 + rest % m2;
      const int64_t k = p.k_lo + rest / m2;
      const char* c0 = b + i * s0 + j * s1 + k * s2;
      double v = *(const double*)(c0 - s0) + *(const double*)(c0 + s0);
      v = v + *(const double*)(c0 - s1);
      v = v + *(const double*)(c0 + s1);
      v = v + *(const double*)(c0 - s2);
      v = v + *(const double*)(c0 + s2);
      *(double*)(p.dst.base + i * p.dst.sm[0] + j * p.dst.sm[1] + k * p.dst.sm[2]) = p.coeff * v;
    }
  }
}


ftn_status_t make_stencil_map(CUtensorMap* m, const ftn_desc_t* d) {
  uint64_t dims[3] = {(uint64_t)d->dim[0].extent, (uint64_t)d->dim[1].extent,
                      (uint64_t)(d->rank == 3 ? d->dim[2].extent : 1)};
  uint64_t strides[2] = {(uint64_t)d->dim[1].sm, (uint64_t)(d->rank == 3 ? d->dim[2].sm : 0)};
  if (d->rank == 2) {
    uint32_t box[2] = {S2_BOXW, S2_BOXH};
    return encode_tma(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d->base_addr, dims, strides, box,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  uint32_t box[3] = {S3_BOXW, S3_BOXH, 1};
  return encode_tma(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d->base_addr, dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_NONE);
}

// One sweep src -> dst over last-dimension planes [lo, hi] (inclusive, 0-based,
// interior only).  TMA path when the whole range is the full interior and both
// descriptors are TMA-able; otherwise the generic kernel.
ftn_status_t sweep(const ftn_desc_t* src, const ftn_desc_t* dst, const CUtensorMap* map, double coeff, int64_t lo,
                   int64_t hi, cudaStream_t s) {
  const int rank = src->rank;
  const int64_t n1 = src->dim[0].extent, n2 = src->dim[1].extent, n3 = rank == 3 ? src->dim[2].extent : 1;
  const int64_t nlast = rank == 3 ? n3 : n2;
  if (n1 < 3 || n2 < 3 || (rank == 3 && n3 < 3)) return FTN_OK;  // no interior
  if (lo < 1) lo = 1;
  if (hi > nlast - 2) hi = nlast - 2;
  if (hi < lo) return FTN_OK;
  const int sms = num_sms();
  if (map) {
    if (rank == 2) {
      J2Params p;
      p.dst = (char*)dst->base_addr;
      p.d_sm1 = dst->dim[0].sm;
      p.d_sm2 = dst->dim[1].sm;
      p.n1 = n1;
      p.n2 = n2;
      p.tiles_i = (n1 + S2_W - 1) / S2_W;
      p.nrows = hi - lo + 1;
      p.coeff = coeff;
      int64_t grid = (int64_t)sms * 2;
      plan_units_halo(p.tiles_i, p.nrows, grid, 2, &p.seg, &p.units);
      if (grid > p.units) grid = p.units;
      p.lo = lo;
      jacobi2d_tma<<<(unsigned)grid, S2_THREADS, S2_SMEM, s>>>(*map, p);
      return after_launch("jacobi2d_tma");
    } else {
      J3Params p;
      p.dst = (char*)dst->base_addr;
      p.d_sm1 = dst->dim[0].sm;
      p.d_sm2 = dst->dim[1].sm;
      p.d_sm3 = dst->dim[2].sm;
      p.n1 = n1;
      p.n2 = n2;
      p.n3 = n3;
      p.tiles_i = (n1 + S3_W - 1) / S3_W;
      p.tiles_j = (n2 + S3_H - 1) / S3_H;
      p.nk = hi - lo + 1;
      p.coeff = coeff;
      int64_t grid = (int64_t)sms * 2;
      plan_units_halo(p.tiles_i * p.tiles_j, p.nk, grid, 2, &p.seg, &p.units);
      if (grid > p.units) grid = p.units;
      p.lo = lo;
      jacobi3d_tma<<<(unsigned)grid, S3_THREADS, S3_SMEM, s>>>(*map, p);
      return after_launch("jacobi3d_tma");
    }
  }
  JGParams g;
  g.src = to_kdesc(src);
  g.dst = to_kdesc(dst);
  g.rank = rank;
  g.n1 = n1;
  g.n2 = n2;
  g.n3 = n3;
  g.k_lo = lo;
  g.k_hi = hi;
  g.coeff = coeff;
  const int64_t total = (n1 - 2) * (rank == 3 ? n2 - 2 : 1) * (hi - lo + 1);
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  jacobi_generic<<<(unsigned)blocks, 256, 0, s>>>(g);
  return after_launch("jacobi_generic");
}

}  // namespace

// Used by the distributed layer: one sweep over planes [lo, hi] of the last dim.
ftn_status_t jacobi_sweep(const ftn_desc_t* src, const ftn_desc_t* dst, double coeff, int64_t lo, int64_t hi,
                          cudaStream_t stream) {
  CUtensorMap m;
  const CUtensorMap* mp = nullptr;
  if (stencil_tma_able(src)) {
    FTN_CHECK(make_stencil_map(&m, src));
    mp = &m;
  }
  return sweep(src, dst, mp, coeff, lo, hi, stream);
}

ftn_status_t jacobi_check(const ftn_desc_t* u, const ftn_desc_t* unew) {
  FTN_CHECK(check_desc(u, "ftn_jacobi(u)", 2, 3));
  FTN_CHECK(check_desc(unew, "ftn_jacobi(unew)", 2, 3));
  if (u->type != FTN_F64 || unew->type != FTN_F64) return fail(FTN_ERR_TYPE, "ftn_jacobi: real(8) only");
  if (!same_shape(u, unew)) return fail(FTN_ERR_SHAPE, "ftn_jacobi: u and unew are not conformable");
  if (desc_overlap(u, unew)) return fail(FTN_ERR_SHAPE, "ftn_jacobi: u and unew overlap");
  return FTN_OK;
}

static std::atomic<bool> g_attr_done[64] = {};  // per device (idempotent)

// Sweeps fused per launch for 2-D arrays (1 = off, 2..12): ftn_jacobi_set_fusion, else the
// FTN_JACOBI_FUSE environment variable, else a size-dependent default (jacobi_fuse_for).
static std::atomic<int> g_fuse{0};
static std::atomic<bool> g_fuse_explicit{false};  // set by ftn_jacobi_set_fusion or FTN_JACOBI_FUSE
int jacobi_fuse_T() {
  int t = g_fuse.load();
  if (t == 0) {
    const char* e = getenv("FTN_JACOBI_FUSE");
    if (e) g_fuse_explicit.store(true);
    t = e ? atoi(e) : 8;
    t = t < 1 ? 1 : (t > 12 ? 12 : t);
    g_fuse.store(t);
  }
  return t;
}

// Sweeps per launch for this array: T for TMA-able rank-2 arrays, 2 for TMA-able rank-3 arrays
// (jacobi3d_tb2, when T >= 2), 1 otherwise.  Unless T was set explicitly, the rank-2 default
// depends on the grid (measured on B200, DESIGN.md §4.3 / §4.6): > 2^23 points 8 (jacobi2d_wq:
// 8192^2 x 100 1981 GLUPS vs 1600 at T = 5), <= 2^23 points 5 (2048^2: 929 vs 792 at 8),
// <= 2^21 points 6 (1024^2: 548 vs 422 at 5; launches there are latency bound).
// Sweeps fused per launch for rank-3 arrays (FTN_J3_T overrides, 1..4): 3 by default --
// jacobi3d_wr<3> (stencil3d_wr.cu), measured at 2048^3 x 100: T = 2 jacobi3d_tb2 539-570,
// T = 3 631, T = 4 620 GLUPS.  Launches of 2 sweeps use jacobi3d_tb2 (faster
// than jacobi3d_wr<2>: 539 vs 486), launches of 3 or 4 jacobi3d_wr.
int jacobi2d_max_T();  // stencil_wq.cu

int jacobi3d_T() {
  static const int t = [] {
    const char* e = getenv("FTN_J3_T");
    int v = e ? atoi(e) : 3;
    return v < 1 ? 1 : (v > 4 ? 4 : v);
  }();
  return t;
}
int jacobi_fuse_for(const ftn_desc_t* u, const ftn_desc_t* unew) {
  int T = jacobi_fuse_T();
  if (T < 2 || !stencil_tma_able(u) || !stencil_tma_able(unew)) return 1;
  for (int d = 0; d < u->rank; ++d)
    if (u->dim[d].extent < 3) return 1;
  if (u->rank == 2 && !g_fuse_explicit.load()) {
    const int64_t pts = u->dim[0].extent * u->dim[1].extent;
    // measured best: 1024^2 6 (wf), 1536^2 / 2048^2 6 (wq), 3072^2 7, 4096^2+ 8
    T = pts <= (int64_t(1) << 22) ? 6 : pts < (int64_t(1) << 24) ? 7 : 8;
  }
  return u->rank == 2 ? (T < jacobi2d_max_T() ? T : jacobi2d_max_T()) : (T < jacobi3d_T() ? T : jacobi3d_T());
}

// k >= 2 fused sweeps src -> dst
ftn_status_t jacobi_fused(const ftn_desc_t* src, const ftn_desc_t* dst, int k, double coeff, cudaStream_t s) {
  if (src->rank == 2) return jacobi2d_fused(src, dst, k, coeff, s);
  if (k == 2) return jacobi3d_fused2(src, dst, coeff, s);
  const int64_t n3 = src->dim[2].extent;
  return jacobi3d_wr_planes(src, dst, k, coeff, 1, n3 - 2, 0, n3 - 1, s);
}

ftn_status_t jacobi_prepare() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (!g_attr_done[dev & 63]) {
    FTN_CUDA(cudaFuncSetAttribute(jacobi2d_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, S2_SMEM));
    FTN_CUDA(cudaFuncSetAttribute(jacobi3d_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, S3_SMEM));
    g_attr_done[dev & 63] = true;
  }
  return FTN_OK;
}

}  // namespace ftn

using namespace ftn;

// Padded packed copies of u / unew (even leading dimension: TMA-able) for arrays the TMA
// kernels cannot address; copies both in.  false (nothing enqueued) when an extent is
// unsuitable or the temporaries cannot be allocated.
static int64_t jacobi_pad_min() {
  static const int64_t v = getenv("FTN_JACOBI_PAD_MIN") ? atoll(getenv("FTN_JACOBI_PAD_MIN")) : 8;
  return v > 0 ? v : INT64_MAX;
}

// Bytes of the two padded packed copies (each 256-byte aligned); 0 when an extent is unsuitable.
static size_t padded_bytes(const ftn_desc_t* u) {
  for (int d = 0; d < u->rank; ++d)
    if (u->dim[d].extent < 3 || u->dim[d].extent >= (1ll << 31)) return 0;
  const int64_t n1 = u->dim[0].extent, ld = n1 + (n1 & 1);  // even leading dimension: 16-byte rows
  size_t elems = (size_t)ld;
  for (int d = 1; d < u->rank; ++d) elems *= (size_t)u->dim[d].extent;
  return 2 * ((elems * 8 + 255) / 256 * 256);
}

// The padded path applies: arrays the TMA kernels cannot address, enough sweeps.
static bool padded_wanted(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t sweeps) {
  return !(stencil_tma_able(u) && stencil_tma_able(unew)) && sweeps >= jacobi_pad_min() && padded_bytes(u) > 0;
}

// Padded packed copies du / dw of u / unew in the caller's workspace ws (padded_bytes(u)
// bytes, 256-byte aligned); copies both in.
static ftn_status_t padded_pair(const ftn_desc_t* u, const ftn_desc_t* unew, cudaStream_t s, char* ws,
                                ftn_desc_t* du, ftn_desc_t* dw) {
  const int64_t n1 = u->dim[0].extent, ld = n1 + (n1 & 1);
  const size_t half = padded_bytes(u) / 2;
  for (ftn_desc_t* d : {du, dw}) {
    memset(d, 0, sizeof(*d));
    d->base_addr = d == du ? ws : ws + half;
    d->elem_len = 8;
    d->rank = u->rank;
    d->type = FTN_F64;
    int64_t sm = 8;
    for (int k = 0; k < u->rank; ++k) {
      d->dim[k].lower_bound = 1;
      d->dim[k].extent = u->dim[k].extent;
      d->dim[k].sm = sm;
      sm *= k == 0 ? ld : u->dim[k].extent;
    }
  }
  FTN_CHECK(launch_copy(du, u, s));
  return launch_copy(dw, unew, s);
}

// Interior section (lb+1 : ub-1 in every dimension) of a Jacobi array: the points a sweep
// updates; false when it is empty.
static bool interior_section(const ftn_desc_t* u, ftn_desc_t* out) {
  int64_t lo[3], hi[3], st[3] = {1, 1, 1};
  for (int d = 0; d < u->rank; ++d) {
    if (u->dim[d].extent < 3) return false;
    lo[d] = u->dim[d].lower_bound + 1;
    hi[d] = u->dim[d].lower_bound + u->dim[d].extent - 2;
  }
  return ftn_desc_section(out, u, lo, hi, st) == FTN_OK;
}

extern "C" ftn_status_t ftn_jacobi_set_fusion(int32_t sweeps_per_launch) {
  if (sweeps_per_launch == 0) {  // back to the default (FTN_JACOBI_FUSE, else size-dependent)
    const char* e = getenv("FTN_JACOBI_FUSE");
    int t = e ? atoi(e) : 8;
    g_fuse.store(t < 1 ? 1 : (t > 12 ? 12 : t));
    g_fuse_explicit.store(e != nullptr);
    return FTN_OK;
  }
  if (sweeps_per_launch < 1 || sweeps_per_launch > 12)
    return fail(FTN_ERR_UNSUPPORTED, "ftn_jacobi_set_fusion: 1..12 sweeps per launch");
  g_fuse.store(sweeps_per_launch);
  g_fuse_explicit.store(true);
  return FTN_OK;
}

extern "C" int32_t ftn_jacobi_get_fusion(void) { return jacobi_fuse_T(); }

extern "C" int32_t ftn_jacobi_fusion_for(const ftn_desc_t* u) {
  if (check_desc(u, "ftn_jacobi_fusion_for(u)", 2, 3) != FTN_OK) return 0;
  return jacobi_fuse_for(u, u);
}

// Launch plan for S sweeps with at most T per launch: the fewest launches n
// >= ceil(S/T) whose count has the parity of S (every launch swaps u/unew, so the result then
// lands in unew iff S is odd), with the sweeps spread as evenly as possible over them (sizes
// ceil(S/n) first, then floor(S/n)): no short launch that pays a whole HBM pass for one or two
// sweeps.  Each entry is the number of sweeps of one launch.
extern "C" int64_t ftn_jacobi_plan(int64_t sweeps, int32_t T, int32_t* sizes, int64_t cap) {
  if (T < 1) T = 1;
  if (sweeps <= 0) return 0;
  int64_t n = (sweeps + T - 1) / T;
  if ((n & 1) != (sweeps & 1)) ++n;  // n <= sweeps: when n = ceil(S/T) <= S has the wrong parity, n + 1 <= S
  const int64_t q = sweeps / n, r = sweeps % n;  // r launches of q + 1, n - r of q
  for (int64_t i = 0; i < n && i < cap; ++i) sizes[i] = (int32_t)(i < r ? q + 1 : q);
  return n;
}

extern "C" ftn_status_t ftn_jacobi_workspace_size(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t sweeps,
                                                  size_t* bytes) {
  FTN_CHECK(jacobi_check(u, unew));
  if (!bytes) return fail(FTN_ERR_NULL, "ftn_jacobi_workspace_size: bytes NULL");
  *bytes = padded_wanted(u, unew, sweeps) ? padded_bytes(u) : 0;
  return FTN_OK;
}

extern "C" ftn_status_t ftn_jacobi(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t sweeps, double coeff,
                                   int32_t* result_in_unew, ftn_stream_t stream) {
  return ftn_jacobi_ws(u, unew, sweeps, coeff, nullptr, 0, result_in_unew, stream);
}

extern "C" ftn_status_t ftn_jacobi_ws(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t sweeps, double coeff,
                                      void* ws, size_t ws_bytes, int32_t* result_in_unew, ftn_stream_t stream) {
  NvtxRange nvtx_("ftn_jacobi");
  FTN_CHECK(jacobi_check(u, unew));
  if (sweeps < 0) return fail(FTN_ERR_SHAPE, "ftn_jacobi: negative sweep count");
  if (ws && ((uintptr_t)ws % 256)) return fail(FTN_ERR_WORKSPACE, "ftn_jacobi_ws: workspace must be 256-byte aligned");
  FTN_CHECK(require_sm100());
  FTN_CHECK(jacobi_prepare());
  cudaStream_t s = (cudaStream_t)stream;
  const bool tma = stencil_tma_able(u) && stencil_tma_able(unew);
  CUtensorMap mu, mw;
  if (tma) {
    FTN_CHECK(make_stencil_map(&mu, u));
    FTN_CHECK(make_stencil_map(&mw, unew));
  }
  const int64_t nlast = u->dim[u->rank - 1].extent;
  // Arrays the TMA kernels cannot address (odd leading dimension, sections with a non-unit
  // first stride or unaligned strides): for enough sweeps and a caller workspace of
  // ftn_jacobi_workspace_size bytes, run the temporally blocked kernels on padded packed
  // copies in the workspace (copy both arrays in, the sweeps, copy both back: 4 extra passes
  // instead of `sweeps` passes of the generic one-point-per-thread kernel).  Same results,
  // same result array; without the workspace the generic kernel runs.  Nothing is allocated.
  if (padded_wanted(u, unew, sweeps) && ws && ws_bytes >= padded_bytes(u)) {
    ftn_desc_t du, dw;
    FTN_CHECK(padded_pair(u, unew, s, (char*)ws, &du, &dw));
    int32_t in_new = 0;
    FTN_CHECK(ftn_jacobi_ws(&du, &dw, sweeps, coeff, nullptr, 0, &in_new, stream));
    FTN_CHECK(launch_copy(u, &du, s));
    FTN_CHECK(launch_copy(unew, &dw, s));
    if (result_in_unew) *result_in_unew = in_new;
    return FTN_OK;
  }
  // Temporal blocking: launches of up to T fused sweeps (ftn_jacobi_plan).
  // Every launch swaps u/unew; the plan's launch count has the parity of `sweeps`, so the
  // result lands in unew iff sweeps is odd.
  const int T = jacobi_fuse_for(u, unew);
  const bool can_fuse = T >= 2 && u->rank == 2;
  static const bool wf1 = getenv("FTN_JACOBI_WF1") && atoi(getenv("FTN_JACOBI_WF1")) != 0;
  const int64_t nplan = ftn_jacobi_plan(sweeps, T, nullptr, 0);
  std::vector<int32_t> plan((size_t)nplan);
  ftn_jacobi_plan(sweeps, T, plan.data(), nplan);
  int64_t launches = 0;
  for (; launches < nplan; ++launches) {
    const bool even = (launches % 2) == 0;
    const ftn_desc_t* src = even ? u : unew;
    const ftn_desc_t* dst = even ? unew : u;
    const int k = plan[(size_t)launches];
    if (k >= 2 || (wf1 && can_fuse))
      FTN_CHECK(jacobi_fused(src, dst, k, coeff, s));
    else
      FTN_CHECK(sweep(src, dst, tma ? (even ? &mu : &mw) : nullptr, coeff, 1, nlast - 2, s));
  }
  if (result_in_unew) *result_in_unew = (int32_t)(launches % 2);
  return FTN_OK;
}

extern "C" ftn_status_t ftn_jacobi_host(const double* host_u, double* host_result, const ftn_desc_t* u,
                                        const ftn_desc_t* unew, int64_t sweeps, double coeff, int32_t* result_in_unew,
                                        ftn_stream_t stream) {
  FTN_CHECK(jacobi_check(u, unew));
  if (!desc_contiguous(u) || !desc_contiguous(unew))
    return fail(FTN_ERR_SHAPE, "ftn_jacobi_host: u and unew must be packed device arrays");
  if ((!host_u || !host_result) && desc_size(u) > 0) return fail(FTN_ERR_SHAPE, "ftn_jacobi_host: null host buffer");
  if (sweeps < 0) return fail(FTN_ERR_SHAPE, "ftn_jacobi_host: negative sweep count");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = (size_t)desc_size(u) * 8;
  int32_t in_new = 0;
  if (bytes) {
    FTN_CUDA(cudaMemcpyAsync(u->base_addr, host_u, bytes, cudaMemcpyHostToDevice, s));
    FTN_CUDA(cudaMemcpyAsync(unew->base_addr, u->base_addr, bytes, cudaMemcpyDeviceToDevice, s));
  }
  FTN_CHECK(ftn_jacobi(u, unew, sweeps, coeff, &in_new, stream));
  if (bytes)
    FTN_CUDA(cudaMemcpyAsync(host_result, (in_new ? unew : u)->base_addr, bytes, cudaMemcpyDeviceToHost, s));
  if (result_in_unew) *result_in_unew = in_new;
  return FTN_OK;
}

// Output planes [out_lo, out_hi] (within the owned planes [halo, n_last - halo)) of one
// local step of the distributed DO nest: `sweeps` fused sweeps with the global boundary
// planes of a first / last slab held fixed.  No validation (callers validate).
namespace ftn {
ftn_status_t jacobi_slab_part(const ftn_desc_t* src, const ftn_desc_t* dst, int32_t sweeps, double coeff,
                              int32_t halo, int32_t first, int32_t last, int64_t out_lo, int64_t out_hi,
                              cudaStream_t s, double* res) {
  const int r = src->rank;
  const int64_t nl = src->dim[r - 1].extent;
  const bool tma = stencil_tma_able(src) && stencil_tma_able(dst);
  const int64_t lo = halo, hi = nl - halo - 1;
  if (out_lo > out_hi) return FTN_OK;
  if (res && !(tma && r == 2)) return fail(FTN_ERR_UNSUPPORTED, "fused residual: rank-2 TMA-able slabs only");
  if (sweeps == 1 && !res) {
    CUtensorMap m;
    const CUtensorMap* mp = nullptr;
    if (tma) {
      FTN_CHECK(make_stencil_map(&m, src));
      mp = &m;
    }
    return sweep(src, dst, mp, coeff, out_lo, out_hi, s);
  }
  const int64_t fix_lo = first ? lo - 1 : INT64_MIN / 4;
  const int64_t fix_hi = last ? hi + 1 : INT64_MAX / 4;
  if (r == 3) {
    if (sweeps == 2) {
      // 32-bit plane arithmetic in the kernel: clamp the "no boundary" sentinels to the slab
      const int64_t flo = first ? fix_lo : lo - 3, fhi = last ? fix_hi : hi + 3;
      return jacobi3d_fused2_planes(src, dst, coeff, out_lo, out_hi, flo, fhi, s);
    }
    return jacobi3d_wr_planes(src, dst, sweeps, coeff, out_lo, out_hi, fix_lo, fix_hi, s);  // clamps the sentinels
  }
  return jacobi2d_fused_rows(src, dst, sweeps, coeff, out_lo, out_hi, fix_lo, fix_hi, s, res);
}
}  // namespace ftn

// One local step of the distributed DO nest, no communication: `sweeps`
// (1 <= sweeps <= halo) sweeps of the owned planes [halo, n_last - halo) of a slab whose
// halo planes are current; reads src planes [halo - sweeps, n_last - halo + sweeps).
extern "C" ftn_status_t ftn_jacobi_slab(const ftn_desc_t* src, const ftn_desc_t* dst, int32_t sweeps, double coeff,
                                        int32_t halo, int32_t first, int32_t last, ftn_stream_t stream) {
  FTN_CHECK(jacobi_check(src, dst));
  const int r = src->rank;
  const int64_t nl = src->dim[r - 1].extent;
  if (halo < 1 || nl - 2 * (int64_t)halo < 1)
    return fail(FTN_ERR_SHAPE, "ftn_jacobi_slab: need halo >= 1 and at least one owned plane");
  if (sweeps < 1 || sweeps > halo) return fail(FTN_ERR_SHAPE, "ftn_jacobi_slab: need 1 <= sweeps <= halo");
  const bool tma = stencil_tma_able(src) && stencil_tma_able(dst);
  if (sweeps > 1 && !(tma && (r == 2 ? sweeps <= 8 : sweeps <= 4)))
    return fail(FTN_ERR_UNSUPPORTED,
                "ftn_jacobi_slab: several sweeps per step need a TMA-able slab (rank 2: up to 8, rank 3: up to 4)");
  FTN_CHECK(require_sm100());
  FTN_CHECK(jacobi_prepare());
  return jacobi_slab_part(src, dst, sweeps, coeff, halo, first, last, halo, nl - halo - 1, (cudaStream_t)stream,
                          nullptr);
}

// Jacobi iteration to convergence (R#25): blocks of check_every
// sweeps, then res = MAXVAL(ABS(u_s - u_{s-1})) over the interior points (exact: a max of
// exactly rounded differences); stop when res <= tol or after max_sweeps.  Rank-2 TMA-able
// arrays: the block runs the plan of ftn_jacobi and its LAST launch (jacobi2d_wq) folds the
// residual of its last two levels into an fmax slot as it stores them -- no extra pass over
// the arrays.  Otherwise the block's last sweep is a single sweep (the two arrays then hold
// consecutive iterates) followed by a MAXVAL(ABS(x - y)) pass over the interior sections.
// Synchronises the stream once per block to read res.
namespace ftn {
// Workspace layout of the solve: [0, 16) the residual slot, [16, 16 + rws) the reduction
// workspace, then (optionally, 256-byte aligned) the padded copies of ftn_jacobi_ws.
static size_t solve_head(const ftn_desc_t* u) {
  size_t rws = 0;
  ftn_reduce_workspace_size(u, &rws);
  return (16 + rws + 255) / 256 * 256;
}

// One block of k sweeps of the solve on the caller's stream; *cur flips per launch; the
// block's residual is left in the device slot res_dev (NaN when the interior is empty).
static ftn_status_t solve_block(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t k, int T, double coeff,
                                double* res_dev, void* rw, size_t rw_bytes, int* cur, cudaStream_t s) {
  const bool tma = stencil_tma_able(u) && stencil_tma_able(unew);
  const int64_t nlast = u->dim[u->rank - 1].extent;
  const bool fused_res = tma && u->rank == 2;
  FTN_CUDA(cudaMemsetAsync(res_dev, 0xff, sizeof(double), s));  // NaN: the empty fmax slot
  const int64_t np = ftn_jacobi_plan(fused_res ? k : k - 1, T, nullptr, 0);
  std::vector<int32_t> plan((size_t)np);
  ftn_jacobi_plan(fused_res ? k : k - 1, T, plan.data(), np);
  if (!fused_res) plan.push_back(1);  // the last sweep alone: consecutive iterates in u / unew
  for (size_t q = 0; q < plan.size(); ++q) {
    const ftn_desc_t* src = *cur ? unew : u;
    const ftn_desc_t* dst = *cur ? u : unew;
    const int32_t kk = plan[q];
    if (fused_res && q + 1 == plan.size()) {
      FTN_CHECK(jacobi2d_fused_rows(src, dst, kk, coeff, 1, nlast - 2, 0, nlast - 1, s, res_dev));
    } else if (kk >= 2) {
      FTN_CHECK(jacobi_fused(src, dst, kk, coeff, s));
    } else {
      CUtensorMap m;
      const CUtensorMap* mp = nullptr;
      if (tma) {
        FTN_CHECK(make_stencil_map(&m, src));
        mp = &m;
      }
      FTN_CHECK(sweep(src, dst, mp, coeff, 1, nlast - 2, s));
    }
    *cur ^= 1;
  }
  if (!fused_res) {
    ftn_desc_t iu, iw;
    if (interior_section(u, &iu) && interior_section(unew, &iw))
      FTN_CHECK(ftn_maxval_absdiff(&iu, &iw, res_dev, rw, rw_bytes, (ftn_stream_t)s));
  }
  return FTN_OK;
}
}  // namespace ftn

extern "C" ftn_status_t ftn_jacobi_solve_workspace_size(const ftn_desc_t* u, const ftn_desc_t* unew,
                                                        int64_t max_sweeps, int64_t check_every, size_t* bytes) {
  FTN_CHECK(jacobi_check(u, unew));
  if (!bytes) return fail(FTN_ERR_NULL, "ftn_jacobi_solve_workspace_size: bytes NULL");
  *bytes = solve_head(u) + (padded_wanted(u, unew, max_sweeps) && check_every >= 3 ? padded_bytes(u) : 0);
  return FTN_OK;
}

extern "C" ftn_status_t ftn_jacobi_solve(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t max_sweeps,
                                         int64_t check_every, double tol, double coeff, void* ws, size_t ws_bytes,
                                         int64_t* sweeps_done, double* residual, int32_t* result_in_unew,
                                         ftn_stream_t stream) {
  NvtxRange nvtx_("ftn_jacobi_solve");
  FTN_CHECK(jacobi_check(u, unew));
  if (max_sweeps < 0 || check_every < 1) return fail(FTN_ERR_SHAPE, "ftn_jacobi_solve: need max_sweeps >= 0, check_every >= 1");
  size_t rws = 0;
  FTN_CHECK(ftn_reduce_workspace_size(u, &rws));
  if (!ws || ws_bytes < rws + 16 || ((uintptr_t)ws % 256))
    return fail(FTN_ERR_WORKSPACE,
                "ftn_jacobi_solve: workspace must hold ftn_reduce_workspace_size(u) + 16 bytes, 256-byte aligned");
  FTN_CHECK(require_sm100());
  FTN_CHECK(jacobi_prepare());
  cudaStream_t s = (cudaStream_t)stream;
  // arrays the TMA kernels cannot address: padded copies in the workspace when it has room
  const size_t head = solve_head(u);
  if (padded_wanted(u, unew, max_sweeps) && check_every >= 3 && ws_bytes >= head + padded_bytes(u)) {
    ftn_desc_t du, dw;
    FTN_CHECK(padded_pair(u, unew, s, (char*)ws + head, &du, &dw));
    FTN_CHECK(ftn_jacobi_solve(&du, &dw, max_sweeps, check_every, tol, coeff, ws, head, sweeps_done, residual,
                               result_in_unew, stream));
    FTN_CHECK(launch_copy(u, &du, s));
    FTN_CHECK(launch_copy(unew, &dw, s));
    return FTN_OK;
  }
  const int T = jacobi_fuse_for(u, unew);
  double* res_dev = reinterpret_cast<double*>(ws);
  char* rw = reinterpret_cast<char*>(ws) + 16;
  int cur = 0;  // 0: u holds the newest iterate
  int64_t done = 0;
  double res = INFINITY;
  while (done < max_sweeps) {
    const int64_t k = check_every < max_sweeps - done ? check_every : max_sweeps - done;
    FTN_CHECK(solve_block(u, unew, k, T, coeff, res_dev, rw, ws_bytes - 16, &cur, s));
    done += k;
    FTN_CUDA(cudaMemcpyAsync(&res, res_dev, sizeof(double), cudaMemcpyDeviceToHost, s));
    FTN_CUDA(cudaStreamSynchronize(s));
    if (res != res) res = -INFINITY;  // empty interior (R#10); NaN data are outside the parity inputs (R#11)
    if (res <= tol) break;
  }
  if (sweeps_done) *sweeps_done = done;
  if (residual) *residual = done ? res : 0.0;
  if (result_in_unew) *result_in_unew = cur;
  return FTN_OK;
}
