// Temporally blocked 3-D Jacobi: two sweeps of the 7-point DO nest (R#16,
// R#23) per launch, bit-identical to two single sweeps, with one HBM pass (16 B per 2 LUP).
//
// A CTA owns a (64-4) x (32-4) column of output points and streams it along k:
//   * level 0 (the input u) arrives plane by plane as TMA boxes {64 x 32 x 1} (start 2
//     columns/rows before the tile: halo 2 for two sweeps; dim-0 start 16-byte aligned) into
//     a 6-slot mbarrier ring filled by one producer lane;
//   * when input plane q has landed, every thread computes level 1 (sweep 1) of plane q-1 on
//     the box interior [1,63) x [1,31) into a 4-slot shared-memory ring, then (one block
//     barrier) level 2 (sweep 2) of plane q-2 on [2,62) x [2,30), which is stored;
//   * thread (x, jb) owns box column x and rows 8 jb .. 8 jb + 7 of every plane.
// The 4-slot level-1 ring makes one barrier per plane sufficient: the slot written by
// level 1 of plane q+1 was last read by level 2 of plane q-2, which every thread finished
// before the barrier of step q+1.  Global boundary points keep their value at every level.
#include "ftn_internal.cuh"

namespace ftn {

void plan_units_halo(int64_t tiles, int64_t len, int64_t grid, int64_t halo_rows, int64_t* seg, int64_t* units);

namespace {

constexpr int B3_X = 64, B3_Y = 32;                  // box (level 0) extent in i, j
constexpr int B3_OX = B3_X - 4, B3_OY = B3_Y - 4;    // output tile 60 x 28
constexpr int B3_PLANE = B3_X * B3_Y * 8;            // 16 KB
constexpr int B3_NS0 = 6, B3_NS1 = 4;        // level-0 TMA ring, level-1 ring
constexpr int B3_ROWS = 8;                           // j rows per thread
constexpr int B3_CT = B3_X * (B3_Y / B3_ROWS);       // 256 compute threads
constexpr int B3_THREADS = B3_CT + 32;
constexpr int B3_SMEM = (B3_NS0 + B3_NS1) * B3_PLANE + 128 + 64;

struct J3TParams {
  char* dst;
  int64_t d_sm1, d_sm2, d_sm3;
  int64_t n1, n2, n3;
  int64_t tiles_i, tiles_j;
  int64_t seg, units;   // output planes per unit, units = tiles * segments
  double coeff;
};

__device__ __forceinline__ void bar_compute3() { asm volatile("bar.sync 1, %0;" ::"n"(B3_CT) : "memory"); }

__global__ void __launch_bounds__(B3_THREADS, 1) jacobi3d_tb2(const __grid_constant__ CUtensorMap map,
                                                              const __grid_constant__ J3TParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const uint32_t soff = (uint32_t)(smem - smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (B3_NS0 + B3_NS1) * B3_PLANE);
  uint64_t* empty = full + B3_NS0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < B3_NS0; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], B3_CT / 32);
    }
    dev::fence_barrier_init();
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  const int64_t ntile = p.tiles_i * p.tiles_j;
  const int64_t nk = p.n3 - 2;

  if (warp == B3_CT / 32) {
    if (lane == 0) {
      dev::prefetch_tma(&map);
      int64_t g = 0;
      for (int64_t u = blockIdx.x; u < p.units; u += G) {
        const int64_t t = u % ntile;
        const int32_t ci = (int32_t)((t % p.tiles_i) * B3_OX - 2), cj = (int32_t)((t / p.tiles_i) * B3_OY - 2);
        const int64_t ka = 1 + (u / ntile) * p.seg, kb = min(ka + p.seg, 1 + nk);
        for (int64_t kk = ka - 2; kk < kb + 2; ++kk, ++g) {
          const int s = (int)(g % B3_NS0);
          if (g >= B3_NS0) dev::mbar_wait(&empty[s], (uint32_t)(((g / B3_NS0) - 1) & 1));
          dev::mbar_arrive_expect_tx(&full[s], B3_PLANE);
          dev::tma_load_3d(smem + s * B3_PLANE, &map, &full[s], ci, cj, (int32_t)kk);
        }
      }
      for (int64_t q = g - B3_NS0 > 0 ? g - B3_NS0 : 0; q < g; ++q)  // producer tail
        dev::mbar_wait(&empty[q % B3_NS0], (uint32_t)((q / B3_NS0) & 1));
    }
    return;
  }

  const int x = threadIdx.x % B3_X;            // box column
  const int y0 = (threadIdx.x / B3_X) * B3_ROWS;  // first box row of this thread
  const double c = p.coeff;
  const double* L0 = reinterpret_cast<const double*>(smem_raw + soff);
  double* L1 = reinterpret_cast<double*>(smem_raw + soff + B3_NS0 * B3_PLANE);
  int64_t g = 0;  // global level-0 plane counter (ring slots / phases)
  for (int64_t u = blockIdx.x; u < p.units; u += G) {
    const int64_t t = u % ntile;
    const int64_t gi0 = (t % p.tiles_i) * B3_OX - 2, gj0 = (t / p.tiles_i) * B3_OY - 2;  // global (i, j) of box (0, 0)
    const int64_t ka = 1 + (u / ntile) * p.seg, kb = min(ka + p.seg, 1 + nk);
    const int nq = (int)(kb - ka + 4);                 // level-0 planes ka-2 .. kb+1
    const int64_t gi = gi0 + x;
    const bool col_fixed = gi <= 0 || gi >= p.n1 - 1;
    const int64_t g0 = g;
    for (int q = 0; q < nq; ++q) {
      const int64_t gq = g0 + q;
      dev::mbar_wait(&full[gq % B3_NS0], (uint32_t)((gq / B3_NS0) & 1));
      // ---- level 1 of plane q-1 (global k = ka - 2 + q - 1) from level-0 planes q-2, q-1, q
      if (q >= 2) {
        const double* P0 = L0 + ((gq - 1) % B3_NS0) * (B3_X * B3_Y);
        const double* Pm = L0 + ((gq - 2) % B3_NS0) * (B3_X * B3_Y);
        const double* Pp = L0 + (gq % B3_NS0) * (B3_X * B3_Y);
        double* O = L1 + ((q - 1) & 3) * (B3_X * B3_Y);
        const int64_t gk = ka - 2 + q - 1;
        const bool plane_fixed = gk <= 0 || gk >= p.n3 - 1;
        if (x >= 1 && x < B3_X - 1) {
#pragma unroll
          for (int r = 0; r < B3_ROWS; ++r) {
            const int y = y0 + r;
            if (y < 1 || y >= B3_Y - 1) continue;
            const int o = y * B3_X + x;
            const int64_t gj = gj0 + y;
            double v = P0[o - 1] + P0[o + 1];
            v = v + P0[o - B3_X];
            v = v + P0[o + B3_X];
            v = v + Pm[o];
            v = v + Pp[o];
            v = c * v;
            if (col_fixed || plane_fixed || gj <= 0 || gj >= p.n2 - 1) v = P0[o];
            O[o] = v;
          }
        }
        // level-0 plane q-2 is no longer needed by anyone after this step's level 1
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&empty[(gq - 2) % B3_NS0]);
      }
      bar_compute3();
      // ---- level 2 of plane q-2 (global k = ka - 2 + q - 2) from level-1 planes q-3, q-2, q-1
      if (q >= 4) {
        const double* Q0 = L1 + ((q - 2) & 3) * (B3_X * B3_Y);
        const double* Qm = L1 + ((q - 3) & 3) * (B3_X * B3_Y);
        const double* Qp = L1 + ((q - 1) & 3) * (B3_X * B3_Y);
        const int64_t gk = ka - 2 + q - 2;  // in [ka, kb): an interior plane
        if (x >= 2 && x < B3_X - 2 && gi >= 1 && gi <= p.n1 - 2) {
          char* out = p.dst + gi * p.d_sm1 + gk * p.d_sm3;
#pragma unroll
          for (int r = 0; r < B3_ROWS; ++r) {
            const int y = y0 + r;
            if (y < 2 || y >= B3_Y - 2) continue;
            const int64_t gj = gj0 + y;
            if (gj < 1 || gj > p.n2 - 2) continue;
            const int o = y * B3_X + x;
            double v = Q0[o - 1] + Q0[o + 1];
            v = v + Q0[o - B3_X];
            v = v + Q0[o + B3_X];
            v = v + Qm[o];
            v = v + Qp[o];
            *reinterpret_cast<double*>(out + gj * p.d_sm2) = c * v;
          }
        }
      }
    }
    // the unit's last two level-0 planes (nq-2, nq-1) were never released by a level 1
    __syncwarp();
    if (lane == 0) {
      dev::mbar_arrive(&empty[(g0 + nq - 2) % B3_NS0]);
      dev::mbar_arrive(&empty[(g0 + nq - 1) % B3_NS0]);
    }
    g = g0 + nq;
    bar_compute3();  // level-1 ring reuse across units
  }
}

}  // namespace

// Two fused 3-D sweeps src -> dst over the whole interior (TMA-able rank-3 src).
ftn_status_t jacobi3d_fused2(const ftn_desc_t* src, const ftn_desc_t* dst, double coeff, cudaStream_t s) {
  static bool attr[64] = {false};
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
  if (p.n1 < 3 || p.n2 < 3 || p.n3 < 3) return FTN_OK;
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
  plan_units_halo(p.tiles_i * p.tiles_j, p.n3 - 2, grid, 4, &p.seg, &p.units);
  if (grid > p.units) grid = p.units;
  jacobi3d_tb2<<<(unsigned)grid, B3_THREADS, B3_SMEM, s>>>(m, p);
  return after_launch("jacobi3d_tb2");
}

}  // namespace ftn
