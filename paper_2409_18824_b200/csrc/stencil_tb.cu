// Temporally blocked 2-D Jacobi ("k sweeps per HBM pass"):
// one launch performs T consecutive sweeps of the DO-nest of R#16, bit-identical to
// T single sweeps (same neighbour order, same single rounding per operation), while
// reading u from HBM once and writing the result once: 16 B per T lattice updates
// instead of 16 B per update.
//
// Register wavefront (no shared-memory levels, no block barriers):
//   * A CTA owns a strip of NW*(32-2T) output columns; one TMA box row per input row
//     covers the strip plus an H-column halo on each side (H = T rounded up to even: a
//     box must start on a 16-byte boundary, tools/microbench/tma_probe.cu).  Rows arrive
//     through an NS-stage mbarrier ring of {BW x R} boxes issued by one producer lane.
//   * Warp w reads its own 32-column window of each row (overlapping its neighbours by
//     2T columns) and runs the T sweeps as a pipeline along j: when input row s arrives,
//     level 1 (sweep 1) produces row s-1, level 2 row s-2, ..., level T row s-T, which
//     is stored.  Each level keeps its last three rows in registers; the i-1 / i+1
//     neighbours come from the adjacent lanes (shfl), so lane l is valid at level t for
//     t <= l < 32-t (a trapezoid) and lanes T..31-T are the warp's outputs.
//   * Global boundary points keep their value at every level (the caller presets the
//     boundary of both arrays, R#16); values outside the array are never consumed.
// Work units (strip, row segment) are taken round-robin with the strip fastest, as in
// the single-sweep kernels.
#include "ftn_internal.cuh"

#include <cstring>

namespace ftn {

void plan_units_halo(int64_t tiles, int64_t len, int64_t grid, int64_t halo_rows, int64_t* seg, int64_t* units);

namespace {

constexpr int WF_NW = 8;   // compute warps per CTA
constexpr int WF_R = 8;    // rows per TMA box
constexpr int WF_NS = 4;   // ring stages

template <int T> struct WFCfg {
  static constexpr int H = T + (T & 1);
  static constexpr int WO = 32 - 2 * T;           // output columns per warp
  static constexpr int OUT = WF_NW * WO;          // output columns per CTA strip
  static constexpr int BW = OUT + 2 * H;          // box width (<= 256, even)
  static constexpr int STAGE = (BW * WF_R * 8 + 127) / 128 * 128;
  static constexpr int SMEM = WF_NS * STAGE + 128 + 64;
  static constexpr int THREADS = (WF_NW + 1) * 32;
  static_assert(BW <= 256, "TMA box width");
};

struct WFParams {
  char* dst;
  int64_t d_sm1, d_sm2;
  int64_t n1, n2;
  int64_t strips;
  int64_t nrows;   // rows to update (interior rows 1 .. n2-2)
  int64_t seg;     // output rows per unit
  int64_t units;
  double coeff;
};

template <int T>
__global__ void __launch_bounds__(WFCfg<T>::THREADS) jacobi2d_wf(const __grid_constant__ CUtensorMap src_map,
                                                                 const __grid_constant__ WFParams p) {
  using C = WFCfg<T>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + WF_NS * C::STAGE);
  uint64_t* empty = full + WF_NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < WF_NS; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], WF_NW);
    }
    dev::fence_barrier_init();
  }
  __syncthreads();
  const int64_t G = gridDim.x;

  if (warp == WF_NW) {
    // ---------------- producer lane: every box of every unit of this CTA, in order
    if (lane == 0) {
      dev::prefetch_tma(&src_map);
      int64_t k = 0;
      for (int64_t u = blockIdx.x; u < p.units; u += G) {
        const int64_t c = u % p.strips;
        const int64_t ja = 1 + (u / p.strips) * p.seg;
        const int64_t jb = min(ja + p.seg, 1 + p.nrows);
        const int64_t nch = (jb - ja + 2 * T + WF_R - 1) / WF_R;
        for (int64_t q = 0; q < nch; ++q, ++k) {
          const int s = (int)(k % WF_NS);
          if (k >= WF_NS) dev::mbar_wait(&empty[s], (uint32_t)(((k / WF_NS) - 1) & 1));
          dev::mbar_arrive_expect_tx(&full[s], C::BW * WF_R * 8);
          dev::tma_load_2d(smem + s * C::STAGE, &src_map, &full[s], (int32_t)(c * C::OUT - C::H),
                           (int32_t)(ja - T + q * WF_R));
        }
      }
      for (int64_t q = k - WF_NS > 0 ? k - WF_NS : 0; q < k; ++q)  // producer tail
        dev::mbar_wait(&empty[q % WF_NS], (uint32_t)((q / WF_NS) & 1));
    }
    return;
  }

  // ---------------- compute warps
  const int col = C::H - T + warp * C::WO + lane;  // box column of this lane
  const bool out_lane = lane >= T && lane < 32 - T;
  const double coeff = p.coeff;
  int64_t k = 0;
  for (int64_t u = blockIdx.x; u < p.units; u += G) {
    const int64_t c = u % p.strips;
    const int64_t ja = 1 + (u / p.strips) * p.seg;
    const int64_t jb = min(ja + p.seg, 1 + p.nrows);
    const int64_t nr = jb - ja + 2 * T;  // input rows, relative 0 .. nr-1 (global ja - T + r)
    const int64_t gcol = c * C::OUT - C::H + col;
    const bool col_fixed = gcol <= 0 || gcol >= p.n1 - 1;
    const bool store_col = out_lane && gcol >= 1 && gcol <= p.n1 - 2;
    char* outp = p.dst + gcol * p.d_sm1 + ja * p.d_sm2;  // row ja = relative row T of level T
    // relative rows r whose global row ja - T + r is interior: r_lo <= r <= r_hi
    const int r_lo = (int)(1 - (ja - T)), r_hi = (int)(p.n2 - 2 - (ja - T));
    // level t keeps rows (s-t-1, s-t, s-t+1) = (up, mid, dn) after step s
    double up[T + 1], mid[T + 1], dn[T + 1];
#pragma unroll
    for (int t = 0; t <= T; ++t) up[t] = mid[t] = dn[t] = 0.0;
    const int64_t nch = (nr + WF_R - 1) / WF_R;
    int s = 0;
    // one pipeline step: input row s -> level t rows s - t
    auto step = [&](const double* row) {
      up[0] = mid[0];
      mid[0] = dn[0];
      dn[0] = *row;
#pragma unroll
      for (int t = 1; t <= T; ++t) {
        const double lf = __shfl_up_sync(0xffffffffu, mid[t - 1], 1);
        const double rt = __shfl_down_sync(0xffffffffu, mid[t - 1], 1);
        const int r = s - t;
        double v = lf + rt;
        v = v + up[t - 1];
        v = v + dn[t - 1];
        v = coeff * v;
        const bool upd = !col_fixed && r >= r_lo && r <= r_hi;
        up[t] = mid[t];
        mid[t] = dn[t];
        dn[t] = upd ? v : mid[t - 1];
      }
      if (s >= 2 * T) {
        if (store_col) *reinterpret_cast<double*>(outp) = dn[T];
        outp += p.d_sm2;
      }
      ++s;
    };
    for (int64_t q = 0; q < nch; ++q, ++k) {
      dev::mbar_wait(&full[k % WF_NS], (uint32_t)((k / WF_NS) & 1));
      const double* st = reinterpret_cast<const double*>(smem + (k % WF_NS) * C::STAGE) + col;
      const int rows = (int)min((int64_t)WF_R, nr - q * WF_R);
      if (rows == WF_R) {
#pragma unroll
        for (int rr = 0; rr < WF_R; ++rr) step(st + rr * C::BW);
      } else {
        for (int rr = 0; rr < rows; ++rr) step(st + rr * C::BW);
      }
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&empty[k % WF_NS]);
    }
  }
}

template <int T>
ftn_status_t launch_wf(const ftn_desc_t* src, const ftn_desc_t* dst, double coeff, cudaStream_t s) {
  using C = WFCfg<T>;
  static bool attr[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    FTN_CUDA(cudaFuncSetAttribute(jacobi2d_wf<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr[dev & 63] = true;
  }
  CUtensorMap m;
  uint64_t dims[2] = {(uint64_t)src->dim[0].extent, (uint64_t)src->dim[1].extent};
  uint64_t strides[1] = {(uint64_t)src->dim[1].sm};
  uint32_t box[2] = {(uint32_t)C::BW, (uint32_t)WF_R};
  FTN_CHECK(encode_tma(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, src->base_addr, dims, strides, box,
                       CU_TENSOR_MAP_SWIZZLE_NONE));
  WFParams p;
  p.dst = (char*)dst->base_addr;
  p.d_sm1 = dst->dim[0].sm;
  p.d_sm2 = dst->dim[1].sm;
  p.n1 = src->dim[0].extent;
  p.n2 = src->dim[1].extent;
  p.strips = (p.n1 - 1 + C::OUT - 1) / C::OUT;  // output columns 1 .. n1-2 lie in [0, strips*OUT)
  p.nrows = p.n2 - 2;
  p.coeff = coeff;
  int occ = 0;
  FTN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jacobi2d_wf<T>, C::THREADS, C::SMEM));
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)num_sms() * occ;
  plan_units_halo(p.strips, p.nrows, grid, 2 * T, &p.seg, &p.units);
  if (grid > p.units) grid = p.units;
  jacobi2d_wf<T><<<(unsigned)grid, C::THREADS, C::SMEM, s>>>(m, p);
  return after_launch("jacobi2d_wf");
}

}  // namespace

// T fused sweeps src -> dst (rank 2, TMA-able src): see the header comment.
ftn_status_t jacobi2d_fused(const ftn_desc_t* src, const ftn_desc_t* dst, int T, double coeff, cudaStream_t s) {
  switch (T) {
    case 1: return launch_wf<1>(src, dst, coeff, s);
    case 2: return launch_wf<2>(src, dst, coeff, s);
    case 3: return launch_wf<3>(src, dst, coeff, s);
    case 4: return launch_wf<4>(src, dst, coeff, s);
  }
  return fail(FTN_ERR_UNSUPPORTED, "jacobi2d_fused: T must be 1..4");
}

}  // namespace ftn
