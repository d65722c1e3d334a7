// Temporally blocked 2-D Jacobi, second design ("k sweeps per HBM
// pass"): one launch performs T consecutive sweeps of the DO-nest of R#16, bit-identical to
// T single sweeps (same neighbour order, one rounding per operation), reading u from HBM
// once and writing the T-th iterate once: 16 B per T lattice updates.
//
//   unew(i,j) = c * (((u(i-1,j) + u(i+1,j)) + u(i,j-1)) + u(i,j+1))
//
// Streaming partial sums.  A warp walks the rows j of a 128-column window (four adjacent
// columns i per lane) and runs the T sweeps as a pipeline along j: when row s of level t-1
// (sweep t-1) arrives, level t
//   - finishes row s-1:   L_t(s-1) = c * (P_t(s-1) + L_{t-1}(s))        (the "+ u(i,j+1)")
//   - starts row s:       P_t(s)   = (L_{t-1}(s,i-1) + L_{t-1}(s,i+1)) + L_{t-1}(s-1)
// which is exactly the DO-nest's evaluation order ((left + right) + up) + down.  A level
// therefore keeps two values per column (the previous row of its input and the pending
// partial), 16 doubles per lane, and the lane's four columns need only two 64-bit shuffles
// per level and row (the left neighbour of its first column, the right one of its last).
// Column k of the window is valid at level t for t <= k < 128-t; the window's outputs are
// columns H .. 127-H (H = T rounded up to even, so that box starts and lane column pairs are
// 16-byte aligned), windows of neighbouring warps overlap by 2H columns.
//
// Input rows arrive by TMA: every warp owns an NS-stage ring of {128 x R} boxes with one
// mbarrier per stage; lane 0 refills a stage as soon as the warp has consumed it (no
// producer warp, no cross-warp synchronisation).  Work units (strip, row segment) are taken
// round-robin by the warps of a persistent grid with the strip fastest, so warps running
// together read neighbouring strips of the same rows (the overlap columns and the segment
// halo rows come from L2).
//
// Global boundary points (column 0 / n1-1, rows <= fix_lo or >= fix_hi) keep their value
// at every level (the caller presets the boundary of both arrays, R#16); values outside the
// array (TMA zero fill) are never consumed by a point that is stored.  Chunks whose window
// and rows touch no boundary take a select-free path.
#include "ftn_internal.cuh"

#include <cstdlib>

// Tuning (tools/variants.py): rows per box, ring stages, row-loop unrolling, CTAs per SM.
#ifndef FTN_WQ_R
#define FTN_WQ_R 4
#endif
#ifndef FTN_WQ_NS
#define FTN_WQ_NS 2  // ring stages per warp: 8192^2, T = 8: 2 -> 2022, 3 -> 1971, 4 -> 1919 GLUPS
#endif
#ifndef FTN_WQ_UNROLL
#define FTN_WQ_UNROLL 2
#endif
#ifndef FTN_WQ_MINB_LO   // T <= 3 (the fused-residual launches): 2 CTAs per SM (8192^2 T=3 963 vs 860 GLUPS with 4)
#define FTN_WQ_MINB_LO 2
#endif
#ifndef FTN_WQ_MINB_MID  // T = 4..6: 2 CTAs per SM (8192^2 T=6: 3.50 vs 4.77 ms per 100 sweeps with 3)
#define FTN_WQ_MINB_MID 2
#endif
#ifndef FTN_WQ_MINB_HI   // T = 7, 8
#define FTN_WQ_MINB_HI 2
#endif

namespace ftn {

constexpr int kWqUnroll = FTN_WQ_UNROLL;

void plan_units_halo(int64_t tiles, int64_t len, int64_t grid, int64_t halo_rows, int64_t* seg, int64_t* units);

namespace {

template <int T_, int NW_, int R_, int NS_, int MINB_>
struct WQCfg {
  static constexpr int T = T_, NW = NW_, R = R_, NS = NS_, MINB = MINB_;
  static constexpr int H = T + (T & 1);        // window halo columns per side (even)
  static constexpr int WO = 128 - 2 * H;       // output columns per window
  static constexpr int BOX = 128 * R * 8;      // bytes per box
  static constexpr int SMEM = NW * NS * BOX + NW * NS * 8 + 128;
  static constexpr int THREADS = NW * 32;
  static_assert(T >= 1 && T <= 12, "1..12 sweeps per launch");
};

struct WQParams {
  char* dst;
  int64_t d_sm2;    // dst row stride in bytes (dim 1 has unit stride)
  int64_t n1, n2;
  int64_t strips;   // windows across dim 1
  int64_t row_lo;   // first output row (0-based position in dim 2)
  int64_t nrows;    // output rows row_lo .. row_lo + nrows - 1
  int64_t fix_lo;   // rows <= fix_lo and >= fix_hi keep their value at every level
  int64_t fix_hi;
  // Flattened, weighted work split (no units of fixed size): the strips' rows are laid end to
  // end, strip by strip, each row weighing w_edge (first / last strip: their windows touch the
  // global boundary columns and run the select path) or w_in (every other strip); warp gw of
  // the grid takes the rows whose weighted start lies in [gw*W/GW, (gw+1)*W/GW).  Every warp
  // then carries the same weighted work -- one or two pieces (a row range of one strip) instead
  // of a whole number of equal units, so neither wave quantisation nor the slower edge strips
  // leave a straggler.
  int64_t w_edge, w_in;   // row weights
  int64_t W;              // total weight
  int64_t GW;             // warps of the grid
  double coeff;
  double* res;      // RES: fmax slot of MAXVAL(ABS(L_T - L_{T-1})) over the stored points
};

__device__ __forceinline__ int64_t wq_ceil_div(int64_t a, int64_t b) { return a <= 0 ? 0 : (a + b - 1) / b; }

// First weighted position of strip s (s in [0, strips]).
__device__ __forceinline__ int64_t wq_strip_start(const WQParams& p, int64_t s) {
  if (s <= 0) return 0;
  if (s >= p.strips) return p.W;
  return p.w_edge * p.nrows + (s - 1) * p.w_in * p.nrows;
}

// Strip holding weighted position x in [0, W).
__device__ __forceinline__ int64_t wq_strip_of(const WQParams& p, int64_t x) {
  const int64_t e = p.w_edge * p.nrows;
  if (x < e) return 0;
  const int64_t s = 1 + (x - e) / (p.w_in * p.nrows);
  return s < p.strips - 1 ? s : p.strips - 1;
}

// Piece k of warp gw: strip c, output rows [ja, jb) (absolute positions in dim 2).  false:
// no piece k; an empty piece (ja == jb) is possible and carries no rows.
__device__ __forceinline__ bool wq_piece(const WQParams& p, int64_t gw, int64_t k, int64_t& c, int64_t& ja,
                                         int64_t& jb) {
  const int64_t A = gw * p.W / p.GW, B = (gw + 1) * p.W / p.GW;
  if (A >= B) return false;
  const int64_t s = wq_strip_of(p, A) + k;
  if (s > wq_strip_of(p, B - 1)) return false;
  const int64_t P0 = wq_strip_start(p, s), P1 = wq_strip_start(p, s + 1);
  const int64_t w = (s == 0 || s == p.strips - 1) ? p.w_edge : p.w_in;
  int64_t lo = wq_ceil_div(A - P0, w), hi = wq_ceil_div((B < P1 ? B : P1) - P0, w);
  if (hi > p.nrows) hi = p.nrows;
  if (lo > hi) lo = hi;
  c = s;
  ja = p.row_lo + lo;
  jb = p.row_lo + hi;
  return true;
}

// The box sequence of one warp: piece k of the warp, chunk q of the piece (pieces without
// rows are skipped).
template <class C>
struct WQCursor {
  int64_t gw, k, q, nch, c, ja;
  bool live;
  __device__ __forceinline__ void find(const WQParams& p) {
    int64_t jb;
    for (;;) {
      live = wq_piece(p, gw, k, c, ja, jb);
      if (!live || jb > ja) break;
      ++k;
    }
    if (live) nch = (jb - ja + 2 * C::T + C::R - 1) / C::R;
    q = 0;
  }
  __device__ __forceinline__ void start(const WQParams& p, int64_t gw_) {
    gw = gw_;
    k = 0;
    find(p);
  }
  __device__ __forceinline__ void advance(const WQParams& p) {
    if (live && ++q == nch) {
      ++k;
      find(p);
    }
  }
  __device__ __forceinline__ void issue(const CUtensorMap* map, uint8_t* ring, uint64_t* full, int s) const {
    dev::mbar_arrive_expect_tx(&full[s], C::BOX);
    dev::tma_load_2d(ring + s * C::BOX, map, &full[s], (int32_t)(c * C::WO - C::H),
                     (int32_t)(ja - C::T + q * C::R));
  }
};

__device__ __forceinline__ void st_v2(char* p, double a, double b) {
  asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}

template <class C, bool RES>
__global__ void __launch_bounds__(C::THREADS, C::MINB) jacobi2d_wq(const __grid_constant__ CUtensorMap src_map,
                                                                  const __grid_constant__ WQParams p) {
  constexpr int T = C::T, R = C::R, NS = C::NS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * NS * C::BOX;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::NW * NS * C::BOX) + warp * NS;
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) dev::mbar_init(&full[s], 1);
    dev::fence_barrier_init();
  }
  __syncwarp();
  // programmatic dependent launch: the next launch of the plan may start its prologue now;
  // nothing of this grid touches global memory before the previous grid has completed
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t gw = (int64_t)blockIdx.x * C::NW + warp;
  WQCursor<C> icur;  // NS boxes ahead of the consumed one
  icur.start(p, gw);
  if (lane == 0) dev::prefetch_tma(&src_map);
  for (int s = 0; s < NS; ++s) {
    if (lane == 0 && icur.live) icur.issue(&src_map, ring, full, s);
    icur.advance(p);
  }
  const uint32_t ring_off = (uint32_t)(ring - smem_raw);
  const double coeff = p.coeff;
  double rmax = __longlong_as_double(0x7ff8000000000000ll);  // RES: fmax over this lane's stored points
  int64_t k = 0;  // boxes consumed by this warp
  int64_t c, ja, jb;
  for (int64_t pk = 0; wq_piece(p, gw, pk, c, ja, jb); ++pk) {
    if (jb <= ja) continue;
    const int nr = (int)(jb - ja) + 2 * T;       // input rows, relative 0 .. nr-1 (global ja - T + r)
    const int64_t gcol0 = c * C::WO - C::H;       // global column of window column 0
    const int64_t g0 = gcol0 + 4 * lane;          // global column of this lane's first column
    bool fixed[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) fixed[e] = g0 + e <= 0 || g0 + e >= p.n1 - 1;
    // stored columns: window columns H .. 127-H inside the interior 1 .. n1-2 (pairs of
    // columns are stored or not together in the fast path: H and g0 are even)
    bool store[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int kk = 4 * lane + e;
      store[e] = kk >= C::H && kk < 128 - C::H && g0 + e >= 1 && g0 + e <= p.n1 - 2;
    }
    // no point a level computes in this window is a boundary column
    const bool colfast = gcol0 >= 0 && gcol0 + 127 <= p.n1 - 1;
    // relative rows r whose global row ja - T + r is updated: r_lo <= r <= r_hi
    const int64_t rl = p.fix_lo + 1 - (ja - T), rh = p.fix_hi - 1 - (ja - T);
    const int r_lo = (int)max(rl, (int64_t)-(1 << 20)), r_hi = (int)min(rh, (int64_t)(1 << 30));
    // level T row s - T is output row ja + s - 2T; rows s < 2T are not stored
    char* orow = p.dst + g0 * 8 + (ja - 2 * T) * p.d_sm2;
    double prev[T][4], part[T][4];
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) prev[t][e] = part[t][e] = 0.0;
    const int nch = (nr + R - 1) / R;
    auto chunk = [&](const double* st, int s0, bool fastpath) {
#pragma unroll kWqUnroll
      for (int rr = 0; rr < R; ++rr) {
        const int s = s0 + rr;
        double x[4], pb[4];  // pb: level T-1 at the row level T finishes (RES)
        {
          const double2 a = *reinterpret_cast<const double2*>(st + rr * 128);
          const double2 b = *reinterpret_cast<const double2*>(st + rr * 128 + 2);
          x[0] = a.x;
          x[1] = a.y;
          x[2] = b.x;
          x[3] = b.y;
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
          // x: level t row s - t (input of level t+1, which finishes row s - t - 1)
          const double left = __shfl_up_sync(0xffffffffu, x[3], 1);
          const double right = __shfl_down_sync(0xffffffffu, x[0], 1);
          double o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) o[e] = coeff * (part[t][e] + x[e]);
          if (!fastpath) {
            const int r = s - t - 1;
            const bool rowok = r >= r_lo && r <= r_hi;
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (!rowok || fixed[e]) o[e] = prev[t][e];
          }
          part[t][0] = (left + x[1]) + prev[t][0];
          part[t][1] = (x[0] + x[2]) + prev[t][1];
          part[t][2] = (x[1] + x[3]) + prev[t][2];
          part[t][3] = (x[2] + right) + prev[t][3];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (RES && t == T - 1) pb[e] = prev[t][e];
            prev[t][e] = x[e];
            x[e] = o[e];
          }
        }
        // x: level T row s - T = global row ja - 2T + s
        if (s >= 2 * T && s < nr) {
          char* q = orow + (int64_t)s * p.d_sm2;
          if (fastpath) {
            if (store[0]) st_v2(q, x[0], x[1]);
            if (store[2]) st_v2(q + 16, x[2], x[3]);
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (store[e]) *reinterpret_cast<double*>(q + 8 * e) = x[e];
          }
          if (RES) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (store[e]) rmax = fmax(rmax, fabs(x[e] - pb[e]));
          }
        }
      }
    };
    for (int q = 0; q < nch; ++q, ++k) {
      const int sl = (int)(k % NS);
      dev::mbar_wait(&full[sl], (uint32_t)((k / NS) & 1));
      // index the __shared__ array itself so the loads are LDS (not generic loads)
      const double* st = reinterpret_cast<const double*>(smem_raw + ring_off + sl * C::BOX) + 4 * lane;
      const int s0 = q * R;
      // rows finished by levels 1..T in this chunk: s - t for s in [s0, s0+R), t in [1, T]
      const bool fast = colfast && s0 - T >= r_lo && s0 + R - 2 <= r_hi;
      if (fast)
        chunk(st, s0, true);
      else
        chunk(st, s0, false);
      __syncwarp();
      if (lane == 0 && icur.live) {
        dev::fence_proxy_async();  // this warp's reads of the slot precede the TMA overwrite
        icur.issue(&src_map, ring, full, sl);
      }
      icur.advance(p);
    }
  }
  if (RES) {
    rmax = dev::warp_fmax(rmax);
    if (lane == 0) dev::atomic_fmax_slot(p.res, rmax);
  }
}

template <class C, bool RES>
ftn_status_t launch_wq(const ftn_desc_t* src, const ftn_desc_t* dst, double coeff, int64_t row_lo, int64_t row_hi,
                       int64_t fix_lo, int64_t fix_hi, double* res, cudaStream_t s) {
  static std::atomic<bool> attr[64] = {};  // per device: dynamic smem attribute set (idempotent)
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    FTN_CUDA(cudaFuncSetAttribute(jacobi2d_wq<C, RES>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr[dev & 63] = true;
  }
  if (dst->dim[0].sm != 8 || ((uintptr_t)dst->base_addr % 16) || (dst->dim[1].sm % 16))
    return fail(FTN_ERR_UNSUPPORTED, "jacobi2d_wq: destination must be TMA-able");
  // host cost per launch matters for small grids: the tensor map, the occupancy and the unit
  // plan are cached per thread
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
    uint32_t box[2] = {128u, (uint32_t)C::R};
    e.base = nullptr;
    FTN_CHECK(encode_tma(&e.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, src->base_addr, dims, strides, box,
                         CU_TENSOR_MAP_SWIZZLE_NONE));
    e.base = src->base_addr;
    e.n1 = src->dim[0].extent;
    e.n2 = src->dim[1].extent;
    e.sm2 = src->dim[1].sm;
    mp = &e.map;
  }
  WQParams p;
  p.dst = (char*)dst->base_addr;
  p.d_sm2 = dst->dim[1].sm;
  p.n1 = src->dim[0].extent;
  p.n2 = src->dim[1].extent;
  p.strips = (p.n1 - 1 + C::WO - 1) / C::WO;  // output columns 1 .. n1-2 lie in [0, strips*WO)
  p.row_lo = row_lo;
  p.nrows = row_hi - row_lo + 1;
  p.fix_lo = fix_lo;
  p.fix_hi = fix_hi;
  p.coeff = coeff;
  p.res = res;
  if (p.nrows <= 0 || p.n1 < 3) return FTN_OK;
  static std::atomic<int> occ_cache[64] = {};
  int occ = occ_cache[dev & 63].load();
  if (occ == 0) {
    FTN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jacobi2d_wq<C, RES>, C::THREADS, C::SMEM));
    if (occ < 1) occ = 1;
    occ_cache[dev & 63].store(occ);
  }
  // one persistent wave: every resident warp takes an equal share of the weighted rows
  int64_t grid = (int64_t)num_sms() * occ;
  const int64_t need = (p.strips * p.nrows + 63) / 64;  // at least ~64 rows per CTA's warps
  if (grid > need) grid = need < 1 ? 1 : need;
  p.GW = grid * C::NW;
  // row weights: edge strips run the select path (FTN_WQ_EDGE_W = its cost in 1/8 of an
  // interior row; measured at 8192^2, T = 8: 8 -> 1521, 12 -> 1852, 16 -> 1924-1930,
  // 20 -> 1908, 24 -> 1878 GLUPS)
  static const int64_t w_edge = getenv("FTN_WQ_EDGE_W") ? atoll(getenv("FTN_WQ_EDGE_W")) : 16;
  p.w_in = 8;
  p.w_edge = w_edge > 0 ? w_edge : 8;
  p.W = (p.strips == 1 ? p.w_edge : 2 * p.w_edge + (p.strips - 2) * p.w_in) * p.nrows;
  // Strip-aligned shares (FTN_WQ_ALIGN, default on): with u = (row weight of all strips) /
  // w_in warps' worth per row, GW = a multiple of u gives every interior strip the same whole
  // number of warps and the same row cuts, so the warps of neighbouring strips sweep the same
  // rows at the same time and their shared overlap columns meet in L2.  The left-over warps
  // (< u) get no work: for gw >= GW the range [gw W / GW, ...) starts at or past W, so every
  // piece wq_piece returns for them is empty.
  static const bool align = !getenv("FTN_WQ_ALIGN") || atoi(getenv("FTN_WQ_ALIGN")) != 0;
  if (align && p.strips > 2 && p.w_edge % p.w_in == 0) {
    const int64_t u = 2 * (p.w_edge / p.w_in) + (p.strips - 2);
    if (p.GW >= u) {
      p.GW = p.GW / u * u;
      grid = (p.GW + C::NW - 1) / C::NW;
    }
  }
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
  FTN_CUDA(cudaLaunchKernelEx(&cfg, jacobi2d_wq<C, RES>, *mp, p));
  return after_launch("jacobi2d_wq");
}

}  // namespace

// T fused sweeps src -> dst (rank 2, TMA-able src and dst) on output rows [row_lo, row_hi],
// with rows <= fix_lo and >= fix_hi held fixed (the global boundary).  Input rows
// [row_lo - T, row_hi + T] are read.
ftn_status_t jacobi2d_wq_rows(const ftn_desc_t* src, const ftn_desc_t* dst, int T, double coeff, int64_t row_lo,
                              int64_t row_hi, int64_t fix_lo, int64_t fix_hi, double* res, cudaStream_t s) {
#define WQ_ARGS src, dst, coeff, row_lo, row_hi, fix_lo, fix_hi, res, s
#define WQ_CASE(T_, MINB)                                              \
  case T_:                                                             \
    return res ? launch_wq<WQCfg<T_, 4, FTN_WQ_R, FTN_WQ_NS, MINB>, true>(WQ_ARGS)    \
               : launch_wq<WQCfg<T_, 4, FTN_WQ_R, FTN_WQ_NS, MINB>, false>(WQ_ARGS);
  switch (T) {
    WQ_CASE(1, FTN_WQ_MINB_LO)
    WQ_CASE(2, FTN_WQ_MINB_LO)
    WQ_CASE(3, FTN_WQ_MINB_LO)
    WQ_CASE(4, FTN_WQ_MINB_MID)
    WQ_CASE(5, FTN_WQ_MINB_MID)
    WQ_CASE(6, FTN_WQ_MINB_MID)
    WQ_CASE(7, FTN_WQ_MINB_HI)
    WQ_CASE(8, FTN_WQ_MINB_HI)
#ifdef FTN_WQ_BIG_T
    WQ_CASE(9, FTN_WQ_MINB_HI)
    WQ_CASE(10, FTN_WQ_MINB_HI)
    WQ_CASE(11, FTN_WQ_MINB_HI)
    WQ_CASE(12, FTN_WQ_MINB_HI)
#endif
  }
#undef WQ_CASE
#undef WQ_ARGS
  return fail(FTN_ERR_UNSUPPORTED, "jacobi2d_wq: T must be 1..8 (1..12 in -DFTN_WQ_BIG_T builds)");
}

// The most sweeps one rank-2 launch of this build fuses (ftn_jacobi caps the fusion at it).
int jacobi2d_max_T() {
#ifdef FTN_WQ_BIG_T
  return 12;
#else
  return 8;
#endif
}

}  // namespace ftn
