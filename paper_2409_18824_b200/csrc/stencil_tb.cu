// Temporally blocked 2-D Jacobi ("k sweeps per HBM pass"):
// one launch performs T consecutive sweeps of the DO-nest of R#16, bit-identical to
// T single sweeps (same neighbour order, same single rounding per operation), while
// reading u from HBM once and writing the result once: 16 B per T lattice updates
// instead of 16 B per update.
//
// Register wavefront (no shared-memory levels, no block barriers):
//   * A CTA owns a strip of NW*(64-2T) output columns; one TMA box row per input row
//     covers the strip plus an H-column halo on each side (H = T rounded up to even: a
//     box must start on a 16-byte boundary, tools/microbench/tma_probe.cu).  Rows arrive
//     through an NS-stage mbarrier ring of {BW x R} boxes issued by one producer lane.
//   * Warp w reads its own 64-column window of each row (two adjacent columns per
//     lane; windows of neighbouring warps overlap by 2T columns) and runs the T sweeps
//     as a pipeline along j: when input row s arrives, level 1 (sweep 1) produces row
//     s-1, level 2 row s-2, ..., level T row s-T, which is stored.  Each level keeps its
//     last three rows in registers; the i-1 / i+1 neighbours are the lane's other column
//     or come from the adjacent lane (one shfl each way per level), so column k of the
//     window is valid at level t for t <= k < 64-t (a trapezoid) and columns T..63-T are
//     the warp's outputs.
//   * Global boundary points keep their value at every level (the caller presets the
//     boundary of both arrays, R#16); values outside the array are never consumed.  Warps
//     whose window and row chunk touch no global boundary take a select-free fast path.
// Work units (strip, row segment) are taken round-robin with the strip fastest, as in
// the single-sweep kernels.
#include "ftn_internal.cuh"

#include <cstring>
#include <cstdlib>

namespace ftn {

void plan_units_halo(int64_t tiles, int64_t len, int64_t grid, int64_t halo_rows, int64_t* seg, int64_t* units);

namespace {

template <int T, int WF_NW = 4 /*compute warps per CTA*/, int WF_R = 8 /*rows per TMA box*/,
          int WF_NS = 4 /*ring stages*/, int WF_LAG = 1 /*rows of lag per level*/,
          int WF_MINB = 1 /*__launch_bounds__ min blocks per SM*/,
          int WF_NOPROD = 0 /*1: no producer warp; the last warp to release a slot refills it*/>
struct WFCfg {
  static constexpr int NW = WF_NW, R = WF_R, NS = WF_NS, LAG = WF_LAG, MINB = WF_MINB, NOPROD = WF_NOPROD;
  // level t produces row s - LAG*t at step s; extra input rows beyond the dependency cone
  static constexpr int EXTRA = (WF_LAG - 1) * T;
  static constexpr int H = T + (T & 1);
  static constexpr int WO = 64 - 2 * T;           // output columns per warp
  static constexpr int OUT = WF_NW * WO;          // output columns per CTA strip
  static constexpr int BW = OUT + 2 * H;          // box width (<= 256, even)
  static constexpr int STAGE = (BW * WF_R * 8 + 127) / 128 * 128;
  static constexpr int SMEM = WF_NS * STAGE + 128 + 128;
  static constexpr int THREADS = (WF_NW + (WF_NOPROD ? 0 : 1)) * 32;
  static constexpr bool ALIGNED = ((H - T) % 2) == 0;  // lane column pairs 16-byte aligned in smem
  static_assert(BW <= 256, "TMA box width");
  static_assert(WF_R % 3 == 0, "rows per box: a multiple of 3 (register ring slots are compile-time)");
  static_assert(WF_LAG == 1 || WF_LAG == 2, "lag 1 (levels in sequence) or 2 (levels independent)");
};

struct WFParams {
  char* dst;
  int64_t d_sm1, d_sm2;
  int64_t n1, n2;
  int64_t strips;
  int64_t row_lo;  // first output row (0-based position in dim 2)
  int64_t nrows;   // output rows row_lo .. row_lo + nrows - 1
  int64_t fix_lo;  // rows <= fix_lo and >= fix_hi keep their value at every level
  int64_t fix_hi;  //   (the global boundary; outside it nothing is consumed)
  int64_t seg;     // output rows per unit
  int64_t units;
  double coeff;
};

// Box cursor for the producer-less variant: the position of a box in this CTA's sequence
// (unit, chunk); every compute warp keeps one NS boxes ahead of the box it consumes, so the
// warp that releases a slot last can refill it at once (no producer warp, no polling).
template <int T, class C>
struct WFCursor {
  int64_t u, q, nch, c, ja;
  __device__ __forceinline__ void unit(const WFParams& p) {
    c = u % p.strips;
    ja = p.row_lo + (u / p.strips) * p.seg;
    const int64_t jb = min(ja + p.seg, p.row_lo + p.nrows);
    nch = (jb - ja + 2 * T + C::EXTRA + C::R - 1) / C::R;
    q = 0;
  }
  __device__ __forceinline__ void start(const WFParams& p) {
    u = blockIdx.x;
    if (u < p.units) unit(p);
  }
  __device__ __forceinline__ void advance(const WFParams& p) {
    if (u < p.units && ++q == nch) {
      u += gridDim.x;
      if (u < p.units) unit(p);
    }
  }
  __device__ __forceinline__ void issue(const WFParams& p, const CUtensorMap* map, uint8_t* smem, uint64_t* full,
                                        int s) const {
    dev::mbar_arrive_expect_tx(&full[s], C::BW * C::R * 8);
    dev::tma_load_2d(smem + s * C::STAGE, map, &full[s], (int32_t)(c * C::OUT - C::H), (int32_t)(ja - T + q * C::R));
  }
};

template <int T, class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB) jacobi2d_wf(const __grid_constant__ CUtensorMap src_map,
                                                          const __grid_constant__ WFParams p) {
  constexpr int WF_NW = C::NW, WF_R = C::R, WF_NS = C::NS;
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
  uint32_t* relcnt = reinterpret_cast<uint32_t*>(empty + WF_NS);  // NOPROD: warps done with a slot
  if (C::NOPROD && threadIdx.x == 0) {
    for (int s = 0; s < WF_NS; ++s) relcnt[s] = 0;
  }
  __syncthreads();
  // programmatic dependent launch: the next launch of the plan may start its prologue now;
  // nothing of this grid touches global memory before the previous grid has completed
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t G = gridDim.x;
  WFCursor<T, C> icur;  // NOPROD: NS boxes ahead of the consumed one
  if (C::NOPROD) {
    icur.start(p);
    if (threadIdx.x == 0) dev::prefetch_tma(&src_map);
    for (int s = 0; s < WF_NS; ++s) {
      if (threadIdx.x == 0 && icur.u < p.units) icur.issue(p, &src_map, smem, full, s);
      icur.advance(p);
    }
  }

  if (!C::NOPROD && warp == WF_NW) {
    // ---------------- producer lane: every box of every unit of this CTA, in order
    if (lane == 0) {
      dev::prefetch_tma(&src_map);
      int64_t k = 0;
      for (int64_t u = blockIdx.x; u < p.units; u += G) {
        const int64_t c = u % p.strips;
        const int64_t ja = p.row_lo + (u / p.strips) * p.seg;
        const int64_t jb = min(ja + p.seg, p.row_lo + p.nrows);
        const int64_t nch = (jb - ja + 2 * T + C::EXTRA + WF_R - 1) / WF_R;
        for (int64_t q = 0; q < nch; ++q, ++k) {
          const int s = (int)(k % WF_NS);
          if (k >= WF_NS) dev::mbar_wait_idle(&empty[s], (uint32_t)(((k / WF_NS) - 1) & 1));
          dev::mbar_arrive_expect_tx(&full[s], C::BW * WF_R * 8);
          dev::tma_load_2d(smem + s * C::STAGE, &src_map, &full[s], (int32_t)(c * C::OUT - C::H),
                           (int32_t)(ja - T + q * WF_R));
        }
      }
      for (int64_t q = k - WF_NS > 0 ? k - WF_NS : 0; q < k; ++q)  // producer tail
        dev::mbar_wait_idle(&empty[q % WF_NS], (uint32_t)((q / WF_NS) & 1));
    }
    return;
  }

  // ---------------- compute warps: lane owns window columns 2*lane, 2*lane+1
  const uint32_t smem_off = (uint32_t)(smem - smem_raw);
  const int wbase = C::H - T + warp * C::WO;  // box column of window column 0
  const int col0 = wbase + 2 * lane;          // box column of this lane's first column
  const double coeff = p.coeff;
  int64_t k = 0;
  for (int64_t u = blockIdx.x; u < p.units; u += G) {
    const int64_t c = u % p.strips;
    const int64_t ja = p.row_lo + (u / p.strips) * p.seg;
    const int64_t jb = min(ja + p.seg, p.row_lo + p.nrows);
    const int64_t nr = jb - ja + 2 * T;  // input rows, relative 0 .. nr-1 (global ja - T + r)
    const int64_t gbase = c * C::OUT - C::H;     // global column of box column 0
    const int64_t g0 = gbase + col0;              // global column of this lane's first column
    bool fixed[2], store[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int kk = 2 * lane + e;  // window column
      const int64_t g = g0 + e;
      fixed[e] = g <= 0 || g >= p.n1 - 1;
      store[e] = kk >= T && kk < 64 - T && g >= 1 && g <= p.n1 - 2;
    }
    // warp-uniform fast path, decided per chunk: no point of this window that a level
    // computes in the chunk is a boundary point
    const int64_t wg_lo = gbase + wbase + 1, wg_hi = gbase + wbase + 62;
    const bool colfast = wg_lo >= 1 && wg_hi <= p.n1 - 2;
    // relative rows r whose row ja - T + r is updated: r_lo <= r <= r_hi
    const int64_t rl = p.fix_lo + 1 - (ja - T), rh = p.fix_hi - 1 - (ja - T);
    const int r_lo = (int)max(rl, (int64_t)-1), r_hi = (int)min(rh, (int64_t)(1 << 30));
    char* outp = p.dst + g0 * p.d_sm1 + ja * p.d_sm2;  // row ja = relative row T of level T
    // Level t keeps its last three rows in a register ring: row r in slot r mod 3.  Every
    // chunk starts at a row s0 = 0 mod 3 (R is a multiple of 3) and is processed fully
    // unrolled, so every slot index is a compile-time constant (no register moves); rows of
    // the last chunk beyond nr compute garbage that is never stored or consumed.
    double L[T + 1][3][2];
#pragma unroll
    for (int t = 0; t <= T; ++t)
#pragma unroll
      for (int q3 = 0; q3 < 3; ++q3) L[t][q3][0] = L[t][q3][1] = 0.0;
    const int64_t nch = (nr + C::EXTRA + WF_R - 1) / WF_R;
    const int nri = (int)nr;
    // one level: level t row s - LAG*t from level t-1 rows (s - LAG*t) - 1, s - LAG*t, (s - LAG*t) + 1
    auto level = [&](int t, int rr, int s, bool fastpath) {
      const int su = ((rr - C::LAG * t - 1) % 3 + 3) % 3, sm = ((rr - C::LAG * t) % 3 + 3) % 3,
                sd = ((rr - C::LAG * t + 1) % 3 + 3) % 3;
      const double left0 = __shfl_up_sync(0xffffffffu, L[t - 1][sm][1], 1);
      const double right1 = __shfl_down_sync(0xffffffffu, L[t - 1][sm][0], 1);
      double v0 = left0 + L[t - 1][sm][1];
      v0 = v0 + L[t - 1][su][0];
      v0 = v0 + L[t - 1][sd][0];
      v0 = coeff * v0;
      double v1 = L[t - 1][sm][0] + right1;
      v1 = v1 + L[t - 1][su][1];
      v1 = v1 + L[t - 1][sd][1];
      v1 = coeff * v1;
      if (!fastpath) {
        const int r = s - C::LAG * t;
        const bool rowok = r >= r_lo && r <= r_hi;
        if (!(rowok && !fixed[0])) v0 = L[t - 1][sm][0];
        if (!(rowok && !fixed[1])) v1 = L[t - 1][sm][1];
      }
      L[t][sm][0] = v0;  // level t row s - LAG*t -> slot (s - LAG*t) mod 3
      L[t][sm][1] = v1;
    };
    auto chunk = [&](const double* st, int s0, bool fastpath) {
      char* orow = outp + (int64_t)(s0 - (C::LAG + 1) * T) * p.d_sm2;  // formed, stored only when ok
#pragma unroll
      for (int rr = 0; rr < WF_R; ++rr) {
        const int s = s0 + rr;
        const double* row = st + rr * C::BW;
        double in0, in1;
        if constexpr (C::ALIGNED) {
          const double2 v = *reinterpret_cast<const double2*>(row);
          in0 = v.x;
          in1 = v.y;
        } else {
          in0 = row[0];
          in1 = row[1];
        }
        const int sl0 = rr % 3;
        if constexpr (C::LAG == 1) {
          // level t needs level t-1's row produced in this same step: ascending order
          L[0][sl0][0] = in0;
          L[0][sl0][1] = in1;
#pragma unroll
          for (int t = 1; t <= T; ++t) level(t, rr, s, fastpath);
        } else {
          // level t reads level t-1 rows produced in earlier steps only, so the T levels of a
          // step are independent; descending order lets level t read the ring slot that
          // level t-1 overwrites later in the same step
#pragma unroll
          for (int t = T; t >= 1; --t) level(t, rr, s, fastpath);
          L[0][sl0][0] = in0;
          L[0][sl0][1] = in1;
        }
        // level T row s - LAG*T is output row ja + (s - (LAG+1)T) when (LAG+1)T <= s < nr + (LAG-1)T;
        // the destination has unit stride in dim 1 (TMA-able, checked on the host): the
        // lane's second column is at +8 bytes.  The fast path only runs on chunks whose rows
        // are all stored, so its stores need no row test and walk a row pointer.
        const int so = ((rr - C::LAG * T) % 3 + 3) % 3;
        const bool ok = s >= (C::LAG + 1) * T && s < nri + C::EXTRA;
        if (ok && store[0]) *reinterpret_cast<double*>(orow) = L[T][so][0];
        if (ok && store[1]) *reinterpret_cast<double*>(orow + 8) = L[T][so][1];
        orow += p.d_sm2;
      }
    };
    for (int64_t q = 0; q < nch; ++q, ++k) {
      dev::mbar_wait(&full[k % WF_NS], (uint32_t)((k / WF_NS) & 1));
      // index the __shared__ array itself so the loads are LDS (not generic LD)
      const double* st = reinterpret_cast<const double*>(smem_raw + smem_off + (k % WF_NS) * C::STAGE) + col0;
      // rows computed by levels 1..T in this chunk: s - LAG*t for s in [s0, s0+R), t in [1, T]
      const int s0 = (int)(q * WF_R);
      const bool fast = colfast && s0 - C::LAG * T >= r_lo && s0 + WF_R - 1 - C::LAG <= r_hi;
      if (fast) chunk(st, s0, true);
      else chunk(st, (int)(q * WF_R), false);
      __syncwarp();
      if constexpr (C::NOPROD) {
        if (lane == 0) {
          const int sl = (int)(k % WF_NS);
          __threadfence_block();  // this warp's reads of the slot happen before its release
          if (atomicAdd(&relcnt[sl], 1u) == WF_NW - 1) {  // last warp out: refill with box k + NS
            relcnt[sl] = 0;
            __threadfence_block();
            if (icur.u < p.units) {
              dev::fence_proxy_async();
              icur.issue(p, &src_map, smem, full, sl);
            }
          }
        }
        icur.advance(p);
      } else {
        if (lane == 0) dev::mbar_arrive(&empty[k % WF_NS]);
      }
    }
  }
}

template <int T, class C>
ftn_status_t launch_wf(const ftn_desc_t* src, const ftn_desc_t* dst, double coeff, int64_t row_lo, int64_t row_hi,
                       int64_t fix_lo, int64_t fix_hi, cudaStream_t s) {
  constexpr int WF_R = C::R;
  static std::atomic<bool> attr[64] = {};  // per device: dynamic smem attribute set (idempotent)
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    FTN_CUDA(cudaFuncSetAttribute(jacobi2d_wf<T, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr[dev & 63] = true;
  }
  if (dst->dim[0].sm != 8) return fail(FTN_ERR_UNSUPPORTED, "jacobi2d_wf: destination must have unit stride in dim 1");
  // host cost per launch matters for small grids (a launch of 5 sweeps of 1024^2 is ~10 us of
  // device time): the tensor map, the occupancy and the unit plan are cached per thread
  struct MapEntry {
    const void* base;
    int64_t n1, n2, sm2;
    CUtensorMap map;
  };
  thread_local MapEntry maps[4] = {};
  thread_local int next_map = 0;
  const CUtensorMap* mp = nullptr;
  for (auto& e : maps)
    if (e.base == src->base_addr && e.n1 == src->dim[0].extent && e.n2 == src->dim[1].extent &&
        e.sm2 == src->dim[1].sm)
      mp = &e.map;
  if (!mp) {
    MapEntry& e = maps[next_map];
    next_map = (next_map + 1) % 4;
    uint64_t dims[2] = {(uint64_t)src->dim[0].extent, (uint64_t)src->dim[1].extent};
    uint64_t strides[1] = {(uint64_t)src->dim[1].sm};
    uint32_t box[2] = {(uint32_t)C::BW, (uint32_t)WF_R};
    e.base = nullptr;
    FTN_CHECK(encode_tma(&e.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, src->base_addr, dims, strides, box,
                         CU_TENSOR_MAP_SWIZZLE_NONE));
    e.base = src->base_addr;
    e.n1 = src->dim[0].extent;
    e.n2 = src->dim[1].extent;
    e.sm2 = src->dim[1].sm;
    mp = &e.map;
  }
  WFParams p;
  p.dst = (char*)dst->base_addr;
  p.d_sm1 = dst->dim[0].sm;
  p.d_sm2 = dst->dim[1].sm;
  p.n1 = src->dim[0].extent;
  p.n2 = src->dim[1].extent;
  p.strips = (p.n1 - 1 + C::OUT - 1) / C::OUT;  // output columns 1 .. n1-2 lie in [0, strips*OUT)
  p.row_lo = row_lo;
  p.nrows = row_hi - row_lo + 1;
  p.fix_lo = fix_lo;
  p.fix_hi = fix_hi;
  p.coeff = coeff;
  if (p.nrows <= 0 || p.n1 < 3) return FTN_OK;
  static std::atomic<int> occ_cache[64] = {};
  int occ = occ_cache[dev & 63].load();
  if (occ == 0) {
    FTN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jacobi2d_wf<T, C>, C::THREADS, C::SMEM));
    if (occ < 1) occ = 1;
    occ_cache[dev & 63].store(occ);
  }
  int64_t grid = (int64_t)num_sms() * occ;
  struct PlanEntry {
    int64_t strips = -1, nrows, grid, seg, units;
  };
  thread_local PlanEntry pc;
  if (pc.strips == p.strips && pc.nrows == p.nrows && pc.grid == grid) {
    p.seg = pc.seg;
    p.units = pc.units;
  } else {
    plan_units_halo(p.strips, p.nrows, grid, 2 * T, &p.seg, &p.units);
    pc = {p.strips, p.nrows, grid, p.seg, p.units};
  }
  static const int64_t nseg_env = getenv("FTN_WF_NSEG") ? atoll(getenv("FTN_WF_NSEG")) : 0;  // tuning probe
  if (nseg_env > 0) {
    p.seg = (p.nrows + nseg_env - 1) / nseg_env;
    p.units = p.strips * ((p.nrows + p.seg - 1) / p.seg);
  }
  if (grid > p.units) grid = p.units;
  static const bool pdl = !getenv("FTN_WF_PDL") || atoi(getenv("FTN_WF_PDL")) != 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = pdl ? 1 : 0;
  FTN_CUDA(cudaLaunchKernelEx(&cfg, jacobi2d_wf<T, C>, *mp, p));
  return after_launch("jacobi2d_wf");
}

}  // namespace

// T fused sweeps src -> dst (rank 2, TMA-able src) on output rows [row_lo, row_hi], with
// rows <= fix_lo and >= fix_hi held fixed (the global boundary): see the header comment.
// Input rows [row_lo - T, row_hi + T] are read.
ftn_status_t jacobi2d_wq_rows(const ftn_desc_t* src, const ftn_desc_t* dst, int T, double coeff, int64_t row_lo,
                              int64_t row_hi, int64_t fix_lo, int64_t fix_hi, double* res, cudaStream_t s);
// res != nullptr: also fold MAXVAL(ABS(iterate T - iterate T-1)) over the stored points into
// the fmax slot *res (jacobi2d_wq's fused residual).
ftn_status_t jacobi2d_fused_rows(const ftn_desc_t* src, const ftn_desc_t* dst, int T, double coeff, int64_t row_lo,
                                 int64_t row_hi, int64_t fix_lo, int64_t fix_hi, cudaStream_t s, double* res) {
  if (res) return jacobi2d_wq_rows(src, dst, T, coeff, row_lo, row_hi, fix_lo, fix_hi, res, s);
  // jacobi2d_wq (stencil_wq.cu) for T = 7, 8, for T = 4..6 on launches of more than 2^21
  // points, or for every T with FTN_WF_WQ=1 (=0: wf whenever T <= 6).  GLUPS over 100 sweeps
  // (wf / wq, both 2 CTAs per SM for wq at T = 4..6): 8192^2 T=4 1218 / 1395, T=5 1600 / 1771,
  // T=6 1469 / 1916; 2048^2 T=5 905 / 990, T=6 892 / 1027; 1536^2 T=6 670 / 723; but 1024^2
  // T=6 463 / 360 and T <= 3 at every size favour wf
  static const int wq_env = getenv("FTN_WF_WQ") ? atoi(getenv("FTN_WF_WQ")) : -1;
  const int64_t pts = src->dim[0].extent * (row_hi - row_lo + 1);
  const bool wq = wq_env > 0 || (wq_env < 0 && T >= 4 && pts > (int64_t(1) << 21));
  if (wq || T > 6) return jacobi2d_wq_rows(src, dst, T, coeff, row_lo, row_hi, fix_lo, fix_hi, nullptr, s);
  // FTN_WF_CFG selects a tuning variant for every T that has one; other T use the default
  static const int cfg = getenv("FTN_WF_CFG") ? atoi(getenv("FTN_WF_CFG")) : -1;
  int key = cfg < 0 ? T * 10 + 9 : T * 10 + cfg;
  for (int attempt = 0; attempt < 2; ++attempt, key = T * 10 + 9) {
#define WF_ARGS src, dst, coeff, row_lo, row_hi, fix_lo, fix_hi, s
  switch (key) {
    // defaults (cfg 9): measured on B200 (R=6 NS=4 1253 vs R=12 NS=3 1230 GLUPS at T=4),
    // DESIGN.md §4.3; R must be a multiple of 3
    case 19: return launch_wf<1, WFCfg<1, 4, 6, 4, 1>>(WF_ARGS);
    case 29: return launch_wf<2, WFCfg<2, 4, 6, 4, 1>>(WF_ARGS);
    case 39: return launch_wf<3, WFCfg<3, 4, 6, 4, 1>>(WF_ARGS);
    case 49: return launch_wf<4, WFCfg<4, 4, 6, 4, 1>>(WF_ARGS);
    // T = 5: no producer warp (the last warp to release a slot refills it), 128 registers,
    // 4 CTAs x 4 warps per SM: 1570 GLUPS vs 1500 with a producer warp (3 CTAs x 5 warps)
    case 59: return launch_wf<5, WFCfg<5, 4, 6, 4, 1, 4, 1>>(WF_ARGS);
    case 69: return launch_wf<6, WFCfg<6, 4, 6, 4, 1>>(WF_ARGS);
#ifdef FTN_WF_TUNING
    // tuning variants (FTN_WF_CFG), compiled only into tuning builds (-DFTN_WF_TUNING)
    case 58: return launch_wf<5, WFCfg<5, 4, 6, 4, 1, 3>>(WF_ARGS);   // producer warp, 3 CTAs/SM
    case 52: return launch_wf<5, WFCfg<5, 4, 6, 4, 1, 3, 1>>(WF_ARGS);  // no producer, 3 CTAs/SM (168 regs)
    case 53: return launch_wf<5, WFCfg<5, 4, 12, 3, 1, 3, 1>>(WF_ARGS); // 12-row boxes, 3 CTAs/SM
    case 51: return launch_wf<5, WFCfg<5, 4, 6, 4, 1>>(WF_ARGS);
    case 50: return launch_wf<5, WFCfg<5, 4, 6, 5, 1, 4, 1>>(WF_ARGS);
    case 40: return launch_wf<4, WFCfg<4, 4, 6, 4, 1, 4, 1>>(WF_ARGS);
    case 30: return launch_wf<3, WFCfg<3, 4, 6, 4, 1, 4, 1>>(WF_ARGS);
    case 20: return launch_wf<2, WFCfg<2, 4, 6, 4, 1, 4, 1>>(WF_ARGS);
    case 60: return launch_wf<6, WFCfg<6, 4, 6, 4, 1, 4, 1>>(WF_ARGS);
    case 61: return launch_wf<6, WFCfg<6, 4, 3, 8, 1, 4, 1>>(WF_ARGS);
    case 68: return launch_wf<6, WFCfg<6, 4, 6, 4, 1, 3>>(WF_ARGS);
    case 57: return launch_wf<5, WFCfg<5, 4, 12, 3, 1, 3>>(WF_ARGS);
    case 56: return launch_wf<5, WFCfg<5, 4, 6, 6, 1, 3>>(WF_ARGS);
    case 55: return launch_wf<5, WFCfg<5, 4, 3, 8, 1, 3>>(WF_ARGS);
    case 67: return launch_wf<6, WFCfg<6, 4, 3, 8, 1, 3>>(WF_ARGS);
    case 66: return launch_wf<6, WFCfg<6, 3, 6, 4, 1, 4>>(WF_ARGS);
    case 38: return launch_wf<3, WFCfg<3, 4, 12, 3, 2>>(WF_ARGS);   // lag 2: levels independent
    case 48: return launch_wf<4, WFCfg<4, 4, 12, 3, 2>>(WF_ARGS);
    case 37: return launch_wf<3, WFCfg<3, 4, 6, 6, 1>>(WF_ARGS);
    case 47: return launch_wf<4, WFCfg<4, 4, 6, 6, 1>>(WF_ARGS);
    case 36: return launch_wf<3, WFCfg<3, 3, 12, 3, 1>>(WF_ARGS);
    case 46: return launch_wf<4, WFCfg<4, 3, 12, 3, 1>>(WF_ARGS);
    case 35: return launch_wf<3, WFCfg<3, 4, 3, 8, 1>>(WF_ARGS);
    case 45: return launch_wf<4, WFCfg<4, 4, 3, 8, 1>>(WF_ARGS);
    case 31: return launch_wf<3, WFCfg<3, 4, 12, 3, 1>>(WF_ARGS);
    case 41: return launch_wf<4, WFCfg<4, 4, 12, 3, 1>>(WF_ARGS);
    case 32: return launch_wf<3, WFCfg<3, 4, 12, 4, 1>>(WF_ARGS);
    case 42: return launch_wf<4, WFCfg<4, 4, 12, 4, 1>>(WF_ARGS);
    case 33: return launch_wf<3, WFCfg<3, 4, 18, 3, 1>>(WF_ARGS);
    case 43: return launch_wf<4, WFCfg<4, 4, 18, 3, 1>>(WF_ARGS);
    case 34: return launch_wf<3, WFCfg<3, 2, 12, 3, 1>>(WF_ARGS);
    case 44: return launch_wf<4, WFCfg<4, 2, 12, 3, 1>>(WF_ARGS);
#endif
  }
#undef WF_ARGS
  }
  return fail(FTN_ERR_UNSUPPORTED, "jacobi2d_fused: T must be 1..6 (and FTN_WF_CFG a known variant)");
}

// The whole interior of a single array: rows 1 .. n2-2, boundary rows 0 and n2-1.
ftn_status_t jacobi2d_fused(const ftn_desc_t* src, const ftn_desc_t* dst, int T, double coeff, cudaStream_t s) {
  const int64_t n2 = src->dim[1].extent;
  return jacobi2d_fused_rows(src, dst, T, coeff, 1, n2 - 2, 0, n2 - 1, s, nullptr);
}

}  // namespace ftn
