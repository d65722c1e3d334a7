// Temporally blocked 3-D Jacobi: two sweeps of the 7-point DO nest (R#16,
// R#23) per launch, bit-identical to two single sweeps, with one HBM pass (16 B per 2 LUP).
//
// A CTA owns a (64-4) x (32-4) column of output points and streams it along k:
//   * level 0 (the input u) arrives plane by plane as TMA boxes {64 x 32 x 1} (start 2
//     columns/rows before the tile: halo 2 for two sweeps; dim-0 start 16-byte aligned, the
//     output rows 32-byte aligned) into an 8-slot mbarrier ring; thread 0 refills the slot of
//     plane q-1 right after the block barrier of step q (every warp has finished reading it
//     by then), so there is no producer warp and no empty barrier: 16 warps = 4 per SM
//     sub-partition share the register file evenly;
//   * thread (x, y0) owns box column x, rows y0 .. y0+R-1 of every plane and keeps its own
//     values of three consecutive planes of level 0 and of level 1 in register rings
//     (slot = plane mod 3, compile-time after unrolling the plane loop by 3);
//   * at step q (input plane q landed) it computes level 1 (sweep 1) of plane q-1: the k and
//     own-row j neighbours come from registers, the i neighbours and the two halo rows from
//     shared memory; level 1 is also written to a 3-slot shared ring for the neighbours'
//     benefit; then, after one block barrier, level 2 (sweep 2) of plane q-2 the same way,
//     stored to HBM.
// The 3-slot level-1 ring is safe with one barrier per step: the slot written at step q was
// last read at step q-2, before the barrier of step q-1.  Global boundary points keep their
// value at every level.
#include "ftn_internal.cuh"

#include <algorithm>
#include <cstdlib>

#ifndef FTN_J3_ROWS
#define FTN_J3_ROWS 4
#endif

namespace ftn {

void plan_units_halo(int64_t tiles, int64_t len, int64_t grid, int64_t halo_rows, int64_t* seg, int64_t* units);

namespace {

#ifndef FTN_J3_BOX_X
#define FTN_J3_BOX_X 64
#endif
#ifndef FTN_J3_BOX_Y
#define FTN_J3_BOX_Y 32
#endif
#ifndef FTN_J3_JFAST
#define FTN_J3_JFAST 0
#endif
#ifndef FTN_J3_CTAS
#define FTN_J3_CTAS 1
#endif
constexpr int B3_X = FTN_J3_BOX_X, B3_Y = FTN_J3_BOX_Y;  // box (level 0) extent in i, j
constexpr int B3_OX = B3_X - 4, B3_OY = B3_Y - 4;    // output tile 60 x 28
constexpr int B3_PE = B3_X * B3_Y;                   // elements per plane
constexpr int B3_PLANE = B3_PE * 8;                  // 16 KB
#ifndef FTN_J3_LAG2
#define FTN_J3_LAG2 0  // measured: lag 2 512 vs lag 1 566 GLUPS at 2048^3 x 100
#endif
// level 2 lags level 1 by two planes (LAG2: the two levels of a step are independent) or one
constexpr int B3_NS0 = 8, B3_NS1 = FTN_J3_LAG2 ? 4 : 3;  // level-0 TMA ring, level-1 ring
constexpr int B3_ROWS = FTN_J3_ROWS;                 // j rows per thread
constexpr int B3_THREADS = B3_X * (B3_Y / B3_ROWS);  // 512 at 4 rows
constexpr int B3_SMEM = (B3_NS0 + B3_NS1) * B3_PLANE + 128 + 8 * B3_NS0;

struct J3TParams {
  char* dst;
  int64_t d_sm1, d_sm2, d_sm3;
  int64_t n1, n2, n3;
  int64_t tiles_i, tiles_j;
  int64_t seg, units;   // output planes per unit, units = tiles * segments
  int64_t plane_lo, plane_hi;  // output planes [plane_lo, plane_hi] (0-based positions in dim 3)
  int64_t fix_lo, fix_hi;      // planes <= fix_lo and >= fix_hi keep their value at every level
  double coeff;
};

// Unit u -> (tile origin, output planes [ka, kb)); 32-bit (units, tiles < 2^31).
struct J3Geom {
  int32_t ntile, tiles_i, seg, plane_lo, plane_end;  // output planes [plane_lo, plane_end)
  __device__ __forceinline__ void unit(uint32_t u, int32_t& i0, int32_t& j0, int32_t& ka, int32_t& kb) const {
    const uint32_t t = u % (uint32_t)ntile, sgi = u / (uint32_t)ntile;
#if FTN_J3_JFAST
    // j fastest: CTAs launched together hold j-neighbour tiles, whose 4 shared halo rows
    // (of 32 per box) can then come from L2
    const uint32_t tiles_j = (uint32_t)ntile / (uint32_t)tiles_i;
    i0 = (int32_t)(t / tiles_j) * B3_OX - 2;
    j0 = (int32_t)(t % tiles_j) * B3_OY - 2;
#else
    i0 = (int32_t)(t % (uint32_t)tiles_i) * B3_OX - 2;
    j0 = (int32_t)(t / (uint32_t)tiles_i) * B3_OY - 2;
#endif
    ka = plane_lo + (int32_t)sgi * seg;
    kb = min(ka + seg, plane_end);
  }
};

// Plane cursor of the TMA issuer (thread 0): walks (unit, k) in consumption order.
struct J3Cursor {
  uint32_t u;
  int32_t kk, kend, ci, cj;
};

__device__ __forceinline__ void cursor_unit(J3Cursor& c, const J3Geom& G) {
  int32_t ka, kb;
  G.unit(c.u, c.ci, c.cj, ka, kb);
  c.kk = ka - 2;
  c.kend = kb + 2;
}

// Issues the next plane (if any) into slot g % NS0.
__device__ __forceinline__ void cursor_issue(J3Cursor& c, const J3Geom& G, uint32_t units, const CUtensorMap* map,
                                             uint8_t* smem, uint64_t* full, uint32_t g) {
  if (c.u >= units) return;
  const int s = (int)(g % B3_NS0);
  dev::mbar_arrive_expect_tx(&full[s], B3_PLANE);
  dev::tma_load_3d(smem + s * B3_PLANE, map, &full[s], c.ci, c.cj, c.kk);
  if (++c.kk == c.kend) {
    c.u += gridDim.x;
    if (c.u < units) cursor_unit(c, G);
  }
}

// Per-thread state of the compute warps (smem offsets in elements).
struct J3Unit {
  const double* L0;   // level-0 ring base
  double* L1;         // level-1 ring base
  uint64_t* full;
  char* out;          // &dst(gi, gj0 + y0, 0)
  int64_t d_sm2, d_sm3;
  double c;
  int own, xm, xp, ylo, yhi;  // element offsets in a plane: own (y0, x), x-1, x+1, rows y0-1, y0+R (clamped)
  int qlo, qhi;       // level 1 keeps plane q-1 when q <= qlo or q >= qhi (global boundary planes)
  int ka;
  uint32_t fix_rows;  // bit r: level 1 keeps row r (boundary row or boundary column)
  uint32_t st_rows;   // bit r: level 2 stores row r (0 for a column that is not stored)
};

template <int PH>
__device__ __forceinline__ void tb3_step(const J3Unit& U, int q, uint32_t gq, double (&a)[3][B3_ROWS],
                                         double (&b)[3][B3_ROWS]) {
  constexpr int P0 = PH, P1 = (PH + 2) % 3, P2 = (PH + 1) % 3;  // ring slots of planes q, q-1, q-2
  dev::mbar_wait(&U.full[gq % B3_NS0], (uint32_t)((gq / B3_NS0) & 1));
  {
    const double* Lq = U.L0 + (gq % B3_NS0) * B3_PE + U.own;
#pragma unroll
    for (int r = 0; r < B3_ROWS; ++r) a[P0][r] = Lq[r * B3_X];
  }
  if (q >= 2) {  // level 1 of plane q-1 (ring slot P1 of the 3-slot shared level-1 ring too)
    const double* Lp = U.L0 + ((gq - 1) % B3_NS0) * B3_PE;
    double xl[B3_ROWS], xr[B3_ROWS];
#pragma unroll
    for (int r = 0; r < B3_ROWS; ++r) {
      xl[r] = Lp[U.xm + r * B3_X];
      xr[r] = Lp[U.xp + r * B3_X];
    }
    const double ylo = Lp[U.ylo], yhi = Lp[U.yhi];
    const uint32_t keep = (q <= U.qlo || q >= U.qhi) ? 0xffffffffu : U.fix_rows;
    double* W = U.L1 + P1 * B3_PE + U.own;
#pragma unroll
    for (int r = 0; r < B3_ROWS; ++r) {
      const double up = r == 0 ? ylo : a[P1][r - 1];
      const double dn = r == B3_ROWS - 1 ? yhi : a[P1][r + 1];
      double v = xl[r] + xr[r];
      v = v + up;
      v = v + dn;
      v = v + a[P2][r];
      v = v + a[P0][r];
      v = U.c * v;
      v = ((keep >> r) & 1) ? a[P1][r] : v;
      b[P1][r] = v;
      W[r * B3_X] = v;
    }
  }
  __syncthreads();
  if (q >= 4) {  // level 2 of plane q-2 (an output plane of this unit): level-1 slots P1, P2, P0 = planes q-1, q-2, q-3
    const double* Lr = U.L1 + P2 * B3_PE;
    double xl[B3_ROWS], xr[B3_ROWS];
#pragma unroll
    for (int r = 0; r < B3_ROWS; ++r) {
      xl[r] = Lr[U.xm + r * B3_X];
      xr[r] = Lr[U.xp + r * B3_X];
    }
    const double ylo = Lr[U.ylo], yhi = Lr[U.yhi];
    char* out = U.out + (int64_t)(U.ka - 4 + q) * U.d_sm3;
#pragma unroll
    for (int r = 0; r < B3_ROWS; ++r) {
      const double up = r == 0 ? ylo : b[P2][r - 1];
      const double dn = r == B3_ROWS - 1 ? yhi : b[P2][r + 1];
      double v = xl[r] + xr[r];
      v = v + up;
      v = v + dn;
      v = v + b[P0][r];
      v = v + b[P1][r];
      v = U.c * v;
      if ((U.st_rows >> r) & 1) *reinterpret_cast<double*>(out + r * U.d_sm2) = v;
    }
  }
}

// Lag-2 step (PH = q mod 4): level 1 of plane q-1 and level 2 of plane q-3 are independent
// (level 2 reads level-1 planes q-4 .. q-2, finished in earlier steps), so their instruction
// streams interleave; 4-slot register rings (a: level 0, b: level 1) and a 4-slot shared
// level-1 ring (the slot written at step q, plane q-1, was last read at step q-2).  Step nq
// (no new plane) only drains level 2.
template <int PH>
__device__ __forceinline__ void tb3_step_l2(const J3Unit& U, int q, int nq, uint32_t gq, double (&a)[4][B3_ROWS],
                                            double (&b)[4][B3_ROWS]) {
  constexpr int A0 = PH, A1 = (PH + 3) % 4, A2 = (PH + 2) % 4;  // a slots of planes q, q-1, q-2
  constexpr int B1 = (PH + 3) % 4;                              // b slot of level-1 plane q-1
  constexpr int C2 = (PH + 2) % 4, C3 = (PH + 1) % 4, C4 = PH;  // b slots of planes q-2, q-3, q-4
  const bool load = q < nq;
  if (load) {
    dev::mbar_wait(&U.full[gq % B3_NS0], (uint32_t)((gq / B3_NS0) & 1));
    const double* Lq = U.L0 + (gq % B3_NS0) * B3_PE + U.own;
#pragma unroll
    for (int r = 0; r < B3_ROWS; ++r) a[A0][r] = Lq[r * B3_X];
  }
  if (load && q >= 2) {  // level 1 of plane q-1 -> b[B1] and shared slot B1
    const double* Lp = U.L0 + ((gq - 1) % B3_NS0) * B3_PE;
    double xl[B3_ROWS], xr[B3_ROWS];
#pragma unroll
    for (int r = 0; r < B3_ROWS; ++r) {
      xl[r] = Lp[U.xm + r * B3_X];
      xr[r] = Lp[U.xp + r * B3_X];
    }
    const double ylo = Lp[U.ylo], yhi = Lp[U.yhi];
    const uint32_t keep = (q <= U.qlo || q >= U.qhi) ? 0xffffffffu : U.fix_rows;
    double* W = U.L1 + B1 * B3_PE + U.own;
#pragma unroll
    for (int r = 0; r < B3_ROWS; ++r) {
      const double up = r == 0 ? ylo : a[A1][r - 1];
      const double dn = r == B3_ROWS - 1 ? yhi : a[A1][r + 1];
      double v = xl[r] + xr[r];
      v = v + up;
      v = v + dn;
      v = v + a[A2][r];
      v = v + a[A0][r];
      v = U.c * v;
      v = ((keep >> r) & 1) ? a[A1][r] : v;
      b[B1][r] = v;
      W[r * B3_X] = v;
    }
  }
  if (q >= 5) {  // level 2 of plane q-3 (an output plane) from level-1 planes q-4, q-3, q-2
    const double* Lr = U.L1 + C3 * B3_PE;
    double xl[B3_ROWS], xr[B3_ROWS];
#pragma unroll
    for (int r = 0; r < B3_ROWS; ++r) {
      xl[r] = Lr[U.xm + r * B3_X];
      xr[r] = Lr[U.xp + r * B3_X];
    }
    const double ylo = Lr[U.ylo], yhi = Lr[U.yhi];
    char* out = U.out + (int64_t)(U.ka - 5 + q) * U.d_sm3;
#pragma unroll
    for (int r = 0; r < B3_ROWS; ++r) {
      const double up = r == 0 ? ylo : b[C3][r - 1];
      const double dn = r == B3_ROWS - 1 ? yhi : b[C3][r + 1];
      double v = xl[r] + xr[r];
      v = v + up;
      v = v + dn;
      v = v + b[C4][r];
      v = v + b[C2][r];
      v = U.c * v;
      if ((U.st_rows >> r) & 1) *reinterpret_cast<double*>(out + r * U.d_sm2) = v;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(B3_THREADS, FTN_J3_CTAS) jacobi3d_tb2(const __grid_constant__ CUtensorMap map,
                                                              const __grid_constant__ J3TParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const uint32_t soff = (uint32_t)(smem - smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (B3_NS0 + B3_NS1) * B3_PLANE);
  J3Geom G;
  G.ntile = (int32_t)(p.tiles_i * p.tiles_j);
  G.tiles_i = (int32_t)p.tiles_i;
  G.seg = (int32_t)p.seg;
  G.plane_lo = (int32_t)p.plane_lo;
  G.plane_end = (int32_t)(p.plane_hi + 1);
  const uint32_t units = (uint32_t)p.units;
  J3Cursor cur;
  cur.u = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < B3_NS0; ++s) dev::mbar_init(&full[s], 1);
    dev::fence_barrier_init();
    dev::prefetch_tma(&map);
    if (cur.u < units) cursor_unit(cur, G);
    for (uint32_t g = 0; g < B3_NS0; ++g) cursor_issue(cur, G, units, &map, smem, full, g);
  }
  __syncthreads();

  J3Unit U;
  U.L0 = reinterpret_cast<const double*>(smem_raw + soff);
  U.L1 = reinterpret_cast<double*>(smem_raw + soff + B3_NS0 * B3_PLANE);
  U.full = full;
  U.d_sm2 = p.d_sm2;
  U.d_sm3 = p.d_sm3;
  U.c = p.coeff;
  const int x = threadIdx.x % B3_X, y0 = (threadIdx.x / B3_X) * B3_ROWS;
  U.own = y0 * B3_X + x;
  U.xm = y0 * B3_X + (x > 0 ? x - 1 : 0);
  U.xp = y0 * B3_X + (x < B3_X - 1 ? x + 1 : B3_X - 1);
  U.ylo = (y0 > 0 ? y0 - 1 : 0) * B3_X + x;                            // unused when y0 == 0
  U.yhi = (y0 + B3_ROWS < B3_Y ? y0 + B3_ROWS : B3_Y - 1) * B3_X + x;  // unused when y0 + R == 32
#if !FTN_J3_LAG2
  double a[3][B3_ROWS], b[3][B3_ROWS];
#endif
  uint32_t g = 0;  // level-0 planes consumed so far (ring slot / phase)
  for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
    int32_t i0, j0, ka, kb;
    G.unit(u, i0, j0, ka, kb);
    const int64_t gi = i0 + x;
    U.ka = ka;
    // level 1 at step q is plane ka - 3 + q: a boundary plane when <= 0 or >= n3 - 1
    // level 1 at step q is plane ka - 3 + q: held fixed when <= fix_lo or >= fix_hi
    U.qlo = (int)(p.fix_lo + 3 - ka);
    U.qhi = (int)(p.fix_hi + 3 - ka);
    const bool col_fixed = gi <= 0 || gi >= p.n1 - 1;
    const bool st_col = x >= 2 && x < B3_X - 2 && gi >= 1 && gi <= p.n1 - 2;
    U.out = p.dst + gi * p.d_sm1 + (int64_t)(j0 + y0) * p.d_sm2;
    U.fix_rows = 0;
    U.st_rows = 0;
#pragma unroll
    for (int r = 0; r < B3_ROWS; ++r) {
      const int y = y0 + r;
      const int64_t gj = j0 + y;
      if (col_fixed || gj <= 0 || gj >= p.n2 - 1) U.fix_rows |= 1u << r;
      if (st_col && y >= 2 && y < B3_Y - 2 && gj >= 1 && gj <= p.n2 - 2) U.st_rows |= 1u << r;
    }
    const int nq = kb - ka + 4;  // level-0 planes ka-2 .. kb+1
#if FTN_J3_LAG2
    double a4[4][B3_ROWS], b4[4][B3_ROWS];
    // steps 0 .. nq-1 consume a plane; step nq drains level 2; thread 0 refills the slot of
    // level-0 plane gq-1 after the barrier of step gq (consuming steps only)
    for (int q = 0; q <= nq; q += 4) {
      tb3_step_l2<0>(U, q, nq, g + q, a4, b4);
      if (threadIdx.x == 0 && q < nq && g + q >= 1) {
        dev::fence_proxy_async();
        cursor_issue(cur, G, units, &map, smem, full, g + q - 1 + B3_NS0);
      }
#pragma unroll
      for (int d = 1; d < 4; ++d) {
        if (q + d > nq) break;
        if (d == 1) tb3_step_l2<1>(U, q + 1, nq, g + q + 1, a4, b4);
        if (d == 2) tb3_step_l2<2>(U, q + 2, nq, g + q + 2, a4, b4);
        if (d == 3) tb3_step_l2<3>(U, q + 3, nq, g + q + 3, a4, b4);
        if (threadIdx.x == 0 && q + d < nq) {
          dev::fence_proxy_async();
          cursor_issue(cur, G, units, &map, smem, full, g + q + d - 1 + B3_NS0);
        }
      }
    }
#else
    for (int q = 0; q < nq; q += 3) {
      tb3_step<0>(U, q, g + q, a, b);
      if (threadIdx.x == 0 && g + q >= 1) {  // level-0 plane g+q-1 is free: refill its slot
        dev::fence_proxy_async();
        cursor_issue(cur, G, units, &map, smem, full, g + q - 1 + B3_NS0);
      }
      if (q + 1 < nq) {
        tb3_step<1>(U, q + 1, g + q + 1, a, b);
        if (threadIdx.x == 0) {
          dev::fence_proxy_async();
          cursor_issue(cur, G, units, &map, smem, full, g + q + B3_NS0);
        }
      }
      if (q + 2 < nq) {
        tb3_step<2>(U, q + 2, g + q + 2, a, b);
        if (threadIdx.x == 0) {
          dev::fence_proxy_async();
          cursor_issue(cur, G, units, &map, smem, full, g + q + 1 + B3_NS0);
        }
      }
    }
#endif
    g += nq;
  }
}

}  // namespace

// Two fused 3-D sweeps src -> dst on output planes [plane_lo, plane_hi] (0-based positions in
// dim 3) of a TMA-able rank-3 src; planes <= fix_lo and >= fix_hi are held fixed (the global
// boundary; for a slab of the distributed path the planes outside the global array are never
// consumed).  Reads src planes [plane_lo - 2, plane_hi + 2].
ftn_status_t jacobi3d_fused2_planes(const ftn_desc_t* src, const ftn_desc_t* dst, double coeff, int64_t plane_lo,
                                    int64_t plane_hi, int64_t fix_lo, int64_t fix_hi, cudaStream_t s) {
  static std::atomic<bool> attr[64] = {};  // per device: dynamic smem attribute set (idempotent)
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    FTN_CUDA(cudaFuncSetAttribute(jacobi3d_tb2, cudaFuncAttributeMaxDynamicSharedMemorySize, B3_SMEM));
    attr[dev & 63] = true;
  }
  J3TParams p;
  p.dst = (char*)dst->base_addr;
  p.d_sm1 = dst->dim[0].sm;
  p.d_sm2 = dst->dim[1].sm;
  p.d_sm3 = dst->dim[2].sm;
  p.n1 = src->dim[0].extent;
  p.n2 = src->dim[1].extent;
  p.n3 = src->dim[2].extent;
  p.plane_lo = plane_lo;
  p.plane_hi = plane_hi;
  p.fix_lo = fix_lo;
  p.fix_hi = fix_hi;
  const int64_t nk = plane_hi - plane_lo + 1;
  if (p.n1 < 3 || p.n2 < 3 || nk <= 0) return FTN_OK;
  p.tiles_i = (p.n1 - 1 + B3_OX - 1) / B3_OX;
  p.tiles_j = (p.n2 - 1 + B3_OY - 1) / B3_OY;
  p.coeff = coeff;
  CUtensorMap m;
  uint64_t dims[3] = {(uint64_t)p.n1, (uint64_t)p.n2, (uint64_t)p.n3};
  uint64_t strides[2] = {(uint64_t)src->dim[1].sm, (uint64_t)src->dim[2].sm};
  uint32_t box[3] = {B3_X, B3_Y, 1};
  FTN_CHECK(encode_tma(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, src->base_addr, dims, strides, box,
                       CU_TENSOR_MAP_SWIZZLE_NONE));
  int occ = 0;
  FTN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jacobi3d_tb2, B3_THREADS, B3_SMEM));
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)num_sms() * occ;
  plan_units_halo(p.tiles_i * p.tiles_j, nk, grid, 4, &p.seg, &p.units);
  // Cap the unit length so that a wave's units span at most ~4 GiB of k-planes (measured at
  // 2048^3, 32 MiB planes: 128-plane units 503 GLUPS vs 432 with the cost-model choice of
  // 1023; at 1024^3 the cap is 512 planes and changes nothing).  FTN_J3_MAXSEG overrides.
  static const int64_t env_maxseg = getenv("FTN_J3_MAXSEG") ? atoll(getenv("FTN_J3_MAXSEG")) : -1;
  const int64_t plane_bytes = src->dim[2].sm > 0 ? src->dim[2].sm : 1;
  const int64_t maxseg = env_maxseg >= 0 ? env_maxseg : std::max<int64_t>(32, (int64_t(4) << 30) / plane_bytes);
  if (maxseg > 0 && p.seg > maxseg) {
    p.seg = maxseg;
    p.units = p.tiles_i * p.tiles_j * ((nk + p.seg - 1) / p.seg);
  }
  if (grid > p.units) grid = p.units;
  jacobi3d_tb2<<<(unsigned)grid, B3_THREADS, B3_SMEM, s>>>(m, p);
  return after_launch("jacobi3d_tb2");
}

// Two fused 3-D sweeps src -> dst over the whole interior.
ftn_status_t jacobi3d_fused2(const ftn_desc_t* src, const ftn_desc_t* dst, double coeff, cudaStream_t s) {
  const int64_t n3 = src->dim[2].extent;
  return jacobi3d_fused2_planes(src, dst, coeff, 1, n3 - 2, 0, n3 - 1, s);
}

}  // namespace ftn
