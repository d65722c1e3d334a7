// Temporally blocked 3-D Jacobi, register design ("k sweeps per HBM pass";
// DESIGN.md §4.4): one launch performs T = 3 or 4 consecutive sweeps of the 7-point DO nest of
// R#16 / R#23, bit-identical to T single sweeps, reading u from HBM once and writing the T-th
// iterate once (16 B per T lattice updates).
//
//   unew(i,j,k) = c * (((((u(i-1) + u(i+1)) + u(j-1)) + u(j+1)) + u(k-1)) + u(k+1))
//
// A CTA of 8 warps owns a box of 64 (i) x 32 (j) points and streams it along k.  Lane l of
// warp w holds columns 2l, 2l+1 of rows 4w .. 4w+3 of every level in registers:
//   * i neighbours are the lane's other column or one 64-bit shuffle from the adjacent lane;
//   * j neighbours are the lane's own rows, except the band's first / last row, whose
//     neighbours are the adjacent warps' edge rows, exchanged through shared memory;
//   * k is streamed with partial sums, in the DO nest's evaluation order: when plane m of
//     level t-1 arrives, level t finishes plane m-1,  L_t(m-1) = c * (P_t(m-1) + L_{t-1}(m)),
//     and starts plane m,  P_t(m) = ((((xl + xr) + yl) + yh) + L_{t-1}(m-1)).
//     A level keeps two values per point (the previous plane of its input and the pending
//     partial sum), 16 doubles per lane.
// Level 0 arrives by TMA, boxes {64 x 32 x 1} into an NS-slot mbarrier ring; all T levels
// advance one plane per step (level t finishes plane q - t at step q), with one block barrier
// after each level but the last (its band-edge rows must be visible to the neighbouring
// warps) -- T-1 barriers per plane; after the first one thread 0 refills the TMA slot that
// level 1 has consumed.  Level t is valid on box columns [t, 63-t] and rows [t, 31-t]; the
// outputs are columns [H, 63-H] (H = T rounded up to even: 16-byte TMA starts) and rows
// [T, 31-T].  Global boundary points and planes keep their value at every level (the caller
// presets the boundary of both arrays, R#16); values outside the array are never consumed by
// a stored point.  Boxes touching no global boundary take a select-free path.
//
// Work: tiles (i fastest) x planes laid end to end, the tiles touching the global i / j
// boundary weighted by their select path's cost; CTA b of one persistent wave takes the
// planes whose weighted start lies in [b W / G, (b+1) W / G) -- one or a few pieces (a tile's
// plane range) per CTA, equal weighted work, no wave quantisation.  Large grids instead deal
// (tile, 512-plane band) cells in order -- taken from a ticket counter, or round-robin under
// stream capture (launch_wr): neighbouring tiles are then swept at the same planes at the same
// time and share their box halos through L2.
#include "ftn_internal.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <numeric>
#include <type_traits>
#include <vector>

namespace ftn {
namespace {

#ifndef FTN_W3_NW
#define FTN_W3_NW 8
#endif
#ifndef FTN_W3_R
#define FTN_W3_R 4
#endif
constexpr int W3_NW = FTN_W3_NW;          // warps per CTA (bands of W3_R rows)
constexpr int W3_R = FTN_W3_R;            // rows per lane
constexpr int W3_BX = 64, W3_BY = W3_NW * W3_R;  // box 64 x 32
constexpr int W3_PLANE = W3_BX * W3_BY * 8;      // 16 KB
constexpr int W3_THREADS = W3_NW * 32;
#ifndef FTN_W3_NS
#define FTN_W3_NS 4
#endif
constexpr int W3_NS = FTN_W3_NS;          // TMA ring slots
constexpr int W3_HALO = W3_NW * 2 * W3_BX * 8;  // edge rows of every warp, one level: 8 KB

template <int T>
struct W3Cfg {
  static constexpr int H = T + (T & 1);
  static constexpr int OX = W3_BX - 2 * H, OY = W3_BY - 2 * T;
  static constexpr int NHALO = T > 1 ? 2 * (T - 1) : 1;  // edge-row slots: level x step parity
  static constexpr int SMEM = W3_NS * W3_PLANE + NHALO * W3_HALO + 128 + 8 * W3_NS + 32;  // + the cell queue
};

struct W3Params {
  char* dst;
  int64_t d_sm2, d_sm3;  // dst strides in bytes (dim 1 has unit stride)
  int32_t n1, n2;
  int32_t tiles_i, tiles_j;
  int32_t plane_lo, nplanes;   // output planes [plane_lo, plane_lo + nplanes)
  int32_t fix_lo, fix_hi;      // planes <= fix_lo and >= fix_hi keep their value at every level
  int64_t w_iedge, w_jedge, w_in, W;  // weighted flattened split (see the header comment)
  int64_t G;                   // CTAs
  int64_t rr_band;             // > 0: (tile, k-band) cells instead of the weighted split
  unsigned long long* ticket;  // dynamic cells: [0] next cell, [1] CTAs done (zero at launch; reset by the last CTA)
  double coeff;
};

#ifndef FTN_W3_TRACE
#define FTN_W3_TRACE 0
#endif
#if FTN_W3_TRACE
__device__ long long* w3_trace;  // per CTA: start, end (globaltimer ns), edge / interior tile-planes
#endif

__device__ __forceinline__ int64_t w3_cdiv(int64_t a, int64_t b) { return a <= 0 ? 0 : (a + b - 1) / b; }

// Tile weights: the tiles of the first / last tile column (their boxes start or end outside
// the array in the contiguous dimension and run the select path) weigh w_iedge, the other
// tiles of the first / last tile row w_jedge, every other tile w_in (per plane).
__device__ __forceinline__ int64_t w3_weight(const W3Params& p, int64_t t) {
  const int64_t ti = t % p.tiles_i, tj = t / p.tiles_i;
  if (ti == 0 || ti == p.tiles_i - 1) return p.w_iedge;
  return (tj == 0 || tj == p.tiles_j - 1) ? p.w_jedge : p.w_in;
}
__device__ __forceinline__ bool w3_edge_tile(const W3Params& p, int64_t t) { return w3_weight(p, t) != p.w_in; }

// Per-plane weight of tiles [0, ti) of a row whose middle tiles weigh wm.
__device__ __forceinline__ int64_t w3_row_prefix(const W3Params& p, int64_t ti, int64_t wm) {
  if (ti <= 0) return 0;
  if (ti >= p.tiles_i) return p.tiles_i == 1 ? p.w_iedge : 2 * p.w_iedge + (p.tiles_i - 2) * wm;
  return p.w_iedge + (ti - 1) * wm;
}

// Weighted start of tile t (tiles i fastest; rows tj = 0 and tj = tiles_j - 1 are j-edge rows).
__device__ __forceinline__ int64_t w3_tile_start(const W3Params& p, int64_t t) {
  const int64_t ti = t % p.tiles_i, tj = t / p.tiles_i, N = p.nplanes;
  const int64_t row_j = w3_row_prefix(p, p.tiles_i, p.w_jedge), row_m = w3_row_prefix(p, p.tiles_i, p.w_in);
  int64_t s = 0;
  if (tj > 0) s += (row_j + (tj - 1) * row_m) * N;   // row 0 (a j-edge row) and the middle rows before tj
  const bool jrow = tj == 0 || tj == p.tiles_j - 1;
  return s + w3_row_prefix(p, ti, jrow ? p.w_jedge : p.w_in) * N;
}

// Tile holding weighted position x (binary search over the monotone tile starts).
__device__ __forceinline__ int64_t w3_tile_of(const W3Params& p, int64_t x) {
  int64_t lo = 0, hi = (int64_t)p.tiles_i * p.tiles_j - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (w3_tile_start(p, mid) <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Cell c of the banded order (tile fastest, then 512-plane band): tile t, planes [ka, kb).
__device__ __forceinline__ bool w3_cell(const W3Params& p, int64_t c, int64_t& t, int32_t& ka, int32_t& kb) {
  const int64_t nt = (int64_t)p.tiles_i * p.tiles_j, nb = (p.nplanes + p.rr_band - 1) / p.rr_band;
  if (c >= nt * nb) return false;
  t = c % nt;
  const int64_t band = c / nt, e = (band + 1) * p.rr_band;
  ka = p.plane_lo + (int32_t)(band * p.rr_band);
  kb = p.plane_lo + (int32_t)(e < p.nplanes ? e : p.nplanes);
  return true;
}

// Piece k of CTA b: tile t, output planes [ka, kb) (absolute); false: no piece k.  Banded
// cells: cell b + k G (static), or the k-th cell this CTA's TMA issuer took from the ticket
// counter (dynamic; cellq holds the last four).
__device__ __forceinline__ bool w3_piece(const W3Params& p, int64_t b, int64_t k, int64_t t0, int64_t t1,
                                         int64_t& t, int32_t& ka, int32_t& kb, const int64_t* cellq) {
  if (p.rr_band > 0) return w3_cell(p, p.ticket ? cellq[k & 3] : b + k * p.G, t, ka, kb);
  const int64_t A = b * p.W / p.G, B = (b + 1) * p.W / p.G;
  t = t0 + k;
  if (A >= B || t > t1) return false;
  const int64_t P0 = w3_tile_start(p, t);
  const int64_t P1 = t + 1 < (int64_t)p.tiles_i * p.tiles_j ? w3_tile_start(p, t + 1) : p.W;
  const int64_t w = w3_weight(p, t);
  int64_t lo = w3_cdiv(A - P0, w), hi = w3_cdiv((B < P1 ? B : P1) - P0, w);
  if (hi > p.nplanes) hi = p.nplanes;
  if (lo > hi) lo = hi;
  ka = p.plane_lo + (int32_t)lo;
  kb = p.plane_lo + (int32_t)hi;
  return true;
}

// TMA issuer's cursor over (piece, level-0 plane) in consumption order (thread 0 only).
template <int T>
struct W3Cursor {
  int64_t k, t;
  int32_t plane, pend, i0, j0;
  bool live;
  __device__ __forceinline__ void find(const W3Params& p, int64_t b, int64_t t0, int64_t t1, int64_t* cellq) {
    int32_t ka, kb;
    for (;;) {
      if (p.ticket) cellq[k & 3] = (int64_t)atomicAdd(p.ticket, 1ull);  // take the next cell
      live = w3_piece(p, b, k, t0, t1, t, ka, kb, cellq);
      if (!live || kb > ka) break;
      ++k;
    }
    if (live) {
      plane = ka - T;
      pend = kb + T;  // level-0 planes ka-T .. kb+T-1
      i0 = (int32_t)(t % p.tiles_i) * W3Cfg<T>::OX - W3Cfg<T>::H;
      j0 = (int32_t)(t / p.tiles_i) * W3Cfg<T>::OY - T;
    }
  }
  __device__ __forceinline__ void issue(const CUtensorMap* map, uint8_t* ring, uint64_t* full, uint32_t g) const {
    const int s = (int)(g % W3_NS);
    dev::mbar_arrive_expect_tx(&full[s], W3_PLANE);
    dev::tma_load_3d(ring + s * W3_PLANE, map, &full[s], i0, j0, plane);
  }
  __device__ __forceinline__ void advance(const W3Params& p, int64_t b, int64_t t0, int64_t t1, int64_t* cellq) {
    if (live && ++plane == pend) {
      ++k;
      find(p, b, t0, t1, cellq);
    }
  }
};

__device__ __forceinline__ void lds2(uint32_t a, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a) : "memory");
}
__device__ __forceinline__ void sts2(uint32_t a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void stg2(char* p, double x, double y) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ double shfl_up1(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shfl_dn1(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }

template <int T>
__global__ void __launch_bounds__(W3_THREADS, 1) jacobi3d_wr(const __grid_constant__ CUtensorMap map,
                                                             const __grid_constant__ W3Params p) {
  using C = W3Cfg<T>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const uint32_t soff = (uint32_t)(smem - smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + W3_NS * W3_PLANE + C::NHALO * W3_HALO);
  int64_t* cellq = reinterpret_cast<int64_t*>(full + W3_NS);  // dynamic cells taken by thread 0
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = blockIdx.x;
  // this CTA's tile range
  const int64_t A = b * p.W / p.G, Bw = (b + 1) * p.W / p.G;
  const int64_t t0 = A < Bw ? w3_tile_of(p, A) : 0, t1 = A < Bw ? w3_tile_of(p, Bw - 1) : -1;
  W3Cursor<T> cur;
  if (threadIdx.x == 0) {
    for (int s = 0; s < W3_NS; ++s) dev::mbar_init(&full[s], 1);
    dev::fence_barrier_init();
    dev::prefetch_tma(&map);
    cur.k = 0;
    cur.find(p, b, t0, t1, cellq);
    for (uint32_t g = 0; g < W3_NS && cur.live; ++g) {
      cur.issue(&map, smem, full, g);
      cur.advance(p, b, t0, t1, cellq);
    }
  }
  __syncthreads();

  const double c = p.coeff;
  const int y0 = warp * W3_R;       // first row of this warp's band
  const int x0 = 2 * lane;          // first column of this lane
  // shared-memory byte addresses (32-bit, shared window) of this lane's pairs
  const uint32_t sbase = dev::smem_u32(smem);
  const uint32_t ring_own = sbase + (uint32_t)((y0 * W3_BX + x0) * 8);           // + slot * PLANE + r * BX * 8
  const int ru = y0 > 0 ? y0 - 1 : 0, rd = y0 + W3_R < W3_BY ? y0 + W3_R : W3_BY - 1;
  const uint32_t ring_up = sbase + (uint32_t)((ru * W3_BX + x0) * 8);
  const uint32_t ring_dn = sbase + (uint32_t)((rd * W3_BX + x0) * 8);
  const int wu = warp > 0 ? warp - 1 : 0, wd = warp < W3_NW - 1 ? warp + 1 : W3_NW - 1;
  const uint32_t hbase = sbase + W3_NS * W3_PLANE;                               // + slot * HALO
  const uint32_t h_up = hbase + (uint32_t)(((wu * 2 + 1) * W3_BX + x0) * 8);     // warp above: its last row
  const uint32_t h_dn = hbase + (uint32_t)(((wd * 2 + 0) * W3_BX + x0) * 8);     // warp below: its first row
  const uint32_t h_w0 = hbase + (uint32_t)(((warp * 2 + 0) * W3_BX + x0) * 8);   // my first row
  const uint32_t h_w1 = hbase + (uint32_t)(((warp * 2 + 1) * W3_BX + x0) * 8);   // my last row
  // warp-uniform output rows, lane-uniform output columns (the pair is stored or not together)
  bool st_row[W3_R];
#pragma unroll
  for (int r = 0; r < W3_R; ++r) st_row[r] = y0 + r >= T && y0 + r < W3_BY - T;
  const bool st_col = x0 >= C::H && x0 + 1 < W3_BX - C::H;
  uint32_t g = 0;  // level-0 planes consumed by this CTA
  int64_t t;
  int32_t ka, kb;
#if FTN_W3_TRACE
  uint64_t tr0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
  int64_t tr_edge = 0, tr_in = 0;
#endif
  for (int64_t pk = 0; w3_piece(p, b, pk, t0, t1, t, ka, kb, cellq); ++pk) {
    if (kb <= ka) continue;
#if FTN_W3_TRACE
    if (w3_edge_tile(p, t)) tr_edge += kb - ka;
    else tr_in += kb - ka;
#endif
    const int32_t i0 = (int32_t)(t % p.tiles_i) * C::OX - C::H, j0 = (int32_t)(t / p.tiles_i) * C::OY - T;
    const int nq = (kb - ka) + 2 * T;  // level-0 planes ka-T .. kb+T-1 (steps q)
    const int32_t gi0 = i0 + x0;
    // slow path: per point fixed in i / j (global boundary) and stored
    uint32_t fixed = 0, store = 0;  // bit 2r + e
#pragma unroll
    for (int r = 0; r < W3_R; ++r)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int32_t gi = gi0 + e, gj = j0 + y0 + r;
        const bool fx = gi <= 0 || gi >= p.n1 - 1 || gj <= 0 || gj >= p.n2 - 1;
        const bool st = !fx && st_col && st_row[r];
        fixed |= (uint32_t)fx << (2 * r + e);
        store |= (uint32_t)st << (2 * r + e);
      }
    const bool tilefast = i0 >= 1 && i0 + W3_BX - 1 <= p.n1 - 2 && j0 >= 1 && j0 + W3_BY - 1 <= p.n2 - 2;
    // output pointer of row y0, column gi0, walking one plane per step from output plane ka
    char* ob = p.dst + (int64_t)gi0 * 8 + (int64_t)(j0 + y0) * p.d_sm2 + (int64_t)ka * p.d_sm3;
    const int64_t sm2 = p.d_sm2, sm3 = p.d_sm3;
    double part[T][W3_R][2], prev[T][W3_R][2];
#pragma unroll
    for (int tt = 0; tt < T; ++tt)
#pragma unroll
      for (int r = 0; r < W3_R; ++r) part[tt][r][0] = part[tt][r][1] = prev[tt][r][0] = prev[tt][r][1] = 0.0;

    auto step = [&](int q, bool fast) {
      const uint32_t slot = g % W3_NS;
      dev::mbar_wait(&full[slot], (g / W3_NS) & 1);
      // level 0: own rows and the band's outer rows (box rows y0-1, y0+4, clamped) from the TMA slot
      double x[W3_R][2], yl[2], yh[2];
      {
        const uint32_t so = slot * W3_PLANE;
#pragma unroll
        for (int r = 0; r < W3_R; ++r) lds2(ring_own + so + r * (W3_BX * 8), x[r][0], x[r][1]);
        lds2(ring_up + so, yl[0], yl[1]);
        lds2(ring_dn + so, yh[0], yh[1]);
      }
      const uint32_t hpar = (g & 1) * (T - 1) * W3_HALO;  // this step's edge-row slots
#pragma unroll
      for (int tt = 0; tt < T; ++tt) {  // level tt+1 from level tt (x: its plane q - tt)
        if (tt > 0) {  // neighbouring warps' edge rows of level tt (written before the last barrier)
          const uint32_t ho = hpar + (tt - 1) * W3_HALO;
          lds2(h_up + ho, yl[0], yl[1]);
          lds2(h_dn + ho, yh[0], yh[1]);
        }
        // level tt+1 finishes plane q - tt - 1 (global ka - T + q - tt - 1)
        bool pfixed = false;
        if (!fast) {
          const int32_t fplane = ka - T + q - tt - 1;
          pfixed = fplane <= p.fix_lo || fplane >= p.fix_hi;
        }
        double o[W3_R][2];
#pragma unroll
        for (int r = 0; r < W3_R; ++r) {
          const double xl = shfl_up1(x[r][1]);
          const double xr = shfl_dn1(x[r][0]);
          const double up0 = r == 0 ? yl[0] : x[r - 1][0], up1 = r == 0 ? yl[1] : x[r - 1][1];
          const double dn0 = r == W3_R - 1 ? yh[0] : x[r + 1][0], dn1 = r == W3_R - 1 ? yh[1] : x[r + 1][1];
          o[r][0] = c * (part[tt][r][0] + x[r][0]);
          o[r][1] = c * (part[tt][r][1] + x[r][1]);
          if (!fast) {
            if (pfixed || ((fixed >> (2 * r)) & 1)) o[r][0] = prev[tt][r][0];
            if (pfixed || ((fixed >> (2 * r + 1)) & 1)) o[r][1] = prev[tt][r][1];
          }
          double v0 = xl + x[r][1];
          v0 = v0 + up0;
          v0 = v0 + dn0;
          part[tt][r][0] = v0 + prev[tt][r][0];
          double v1 = x[r][0] + xr;
          v1 = v1 + up1;
          v1 = v1 + dn1;
          part[tt][r][1] = v1 + prev[tt][r][1];
          prev[tt][r][0] = x[r][0];
          prev[tt][r][1] = x[r][1];
        }
        if (tt + 1 < T) {
          // this level's band-edge rows for the neighbouring warps' next level; the slots
          // alternate with the step parity, so a warp writing step q+1's rows never meets a warp
          // still reading step q's (the last level has no barrier after it)
          const uint32_t ho = hpar + tt * W3_HALO;
          sts2(h_w0 + ho, o[0][0], o[0][1]);
          sts2(h_w1 + ho, o[W3_R - 1][0], o[W3_R - 1][1]);
          __syncthreads();
          if (tt == 0 && threadIdx.x == 0 && cur.live) {  // level-0 plane of this step consumed
            dev::fence_proxy_async();
            cur.issue(&map, smem, full, g + W3_NS);
            cur.advance(p, b, t0, t1, cellq);
          }
#pragma unroll
          for (int r = 0; r < W3_R; ++r) {
            x[r][0] = o[r][0];
            x[r][1] = o[r][1];
          }
        } else if (q >= 2 * T) {
          // level T, plane q - T = output plane ka + q - 2T (ob)
          if (fast) {
            if (st_col) {
#pragma unroll
              for (int r = 0; r < W3_R; ++r)
                if (st_row[r]) stg2(ob + r * sm2, o[r][0], o[r][1]);
            }
          } else if (!pfixed) {
#pragma unroll
            for (int r = 0; r < W3_R; ++r) {
              if ((store >> (2 * r)) & 1u) *reinterpret_cast<double*>(ob + r * sm2) = o[r][0];
              if ((store >> (2 * r + 1)) & 1u) *reinterpret_cast<double*>(ob + r * sm2 + 8) = o[r][1];
            }
          }
          ob += sm3;
        }
      }
      if (T == 1) {
        __syncthreads();
        if (threadIdx.x == 0 && cur.live) {
          dev::fence_proxy_async();
          cur.issue(&map, smem, full, g + W3_NS);
          cur.advance(p, b, t0, t1, cellq);
        }
      }
      ++g;
    };
    for (int q = 0; q < nq; ++q) {
      // planes finished in this step: ka - T + q - 1 - tt, tt = 0 .. T-1
      const int32_t lo_pl = ka - T + q - T, hi_pl = ka - T + q - 1;
      const bool fast = tilefast && lo_pl > p.fix_lo && hi_pl < p.fix_hi;
      if (fast) step(q, true);
      else step(q, false);
    }
  }
  if (p.ticket && threadIdx.x == 0) {  // the last CTA to finish leaves the ticket slot zeroed
    __threadfence();
    if (atomicAdd(p.ticket + 1, 1ull) == (unsigned long long)(p.G - 1)) {
      p.ticket[0] = 0;
      p.ticket[1] = 0;
    }
  }
#if FTN_W3_TRACE
  if (threadIdx.x == 0 && w3_trace) {
    uint64_t tr1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr1));
    w3_trace[4 * b + 0] = (long long)tr0;
    w3_trace[4 * b + 1] = (long long)tr1;
    w3_trace[4 * b + 2] = tr_edge;
    w3_trace[4 * b + 3] = tr_in;
  }
#endif
}

// Ticket slots for the dynamic cell order: per device, 256 slots of {next cell, CTAs done},
// zeroed once; a launch takes the next slot and its last CTA leaves it zeroed again (a slot
// is reused only 256 launches later).
unsigned long long* ticket_slot() {
  static std::mutex mu;
  static unsigned long long* slots[64] = {};
  static unsigned next[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!slots[dev & 63]) {
    if (cudaMalloc(&slots[dev & 63], 256 * 2 * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    if (cudaMemset(slots[dev & 63], 0, 256 * 2 * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
  }
  return slots[dev & 63] + 2 * (next[dev & 63]++ % 256);
}

template <int T>
ftn_status_t launch_wr(const ftn_desc_t* src, const ftn_desc_t* dst, double coeff, int64_t plane_lo,
                       int64_t plane_hi, int64_t fix_lo, int64_t fix_hi, cudaStream_t s) {
  using C = W3Cfg<T>;
  static std::atomic<bool> attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    FTN_CUDA(cudaFuncSetAttribute(jacobi3d_wr<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr[dev & 63] = true;
  }
  if (dst->dim[0].sm != 8 || ((uintptr_t)dst->base_addr % 16) || (dst->dim[1].sm % 16) || (dst->dim[2].sm % 16))
    return fail(FTN_ERR_UNSUPPORTED, "jacobi3d_wr: destination must be TMA-able");
  W3Params p;
  p.dst = (char*)dst->base_addr;
  p.d_sm2 = dst->dim[1].sm;
  p.d_sm3 = dst->dim[2].sm;
  p.n1 = (int32_t)src->dim[0].extent;
  p.n2 = (int32_t)src->dim[1].extent;
  const int64_t n3 = src->dim[2].extent;
  const int64_t nk = plane_hi - plane_lo + 1;
  if (p.n1 < 3 || p.n2 < 3 || nk <= 0) return FTN_OK;
  p.plane_lo = (int32_t)plane_lo;
  p.nplanes = (int32_t)nk;
  p.fix_lo = (int32_t)std::max<int64_t>(fix_lo, plane_lo - 3 * T - 2);  // 32-bit: clamp the sentinels
  p.fix_hi = (int32_t)std::min<int64_t>(fix_hi, plane_hi + 3 * T + 2);
  p.tiles_i = (p.n1 - 1 + C::OX - 1) / C::OX;  // output columns 1 .. n1-2 lie in [0, tiles_i*OX)
  p.tiles_j = (p.n2 - 1 + C::OY - 1) / C::OY;
  p.coeff = coeff;
  (void)n3;
  // tensor map (cached per thread for repeated launches on the same array)
  struct MapEntry {
    const void* base;
    int64_t n1, n2, n3, sm2, sm3;
    CUtensorMap map;
  };
  thread_local MapEntry maps[4] = {};
  thread_local int next_map = 0;
  const CUtensorMap* mp = nullptr;
  for (auto& e : maps)
    if (e.base == src->base_addr && e.n1 == src->dim[0].extent && e.n2 == src->dim[1].extent &&
        e.n3 == src->dim[2].extent && e.sm2 == src->dim[1].sm && e.sm3 == src->dim[2].sm)
      mp = &e.map;
  if (!mp) {
    MapEntry& e = maps[next_map];
    next_map = (next_map + 1) % 4;
    uint64_t dims[3] = {(uint64_t)src->dim[0].extent, (uint64_t)src->dim[1].extent, (uint64_t)src->dim[2].extent};
    uint64_t strides[2] = {(uint64_t)src->dim[1].sm, (uint64_t)src->dim[2].sm};
    uint32_t box[3] = {W3_BX, W3_BY, 1};
    e.base = nullptr;
    FTN_CHECK(encode_tma(&e.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, src->base_addr, dims, strides, box,
                         CU_TENSOR_MAP_SWIZZLE_NONE));
    e.base = src->base_addr;
    e.n1 = src->dim[0].extent;
    e.n2 = src->dim[1].extent;
    e.n3 = src->dim[2].extent;
    e.sm2 = src->dim[1].sm;
    e.sm3 = src->dim[2].sm;
    mp = &e.map;
  }
  // one persistent wave, equal weighted work per CTA.  Weights in eighths of an interior tile
  // (FTN_W3_EDGE_W = "i,j"); per-CTA durations at 2048^3 (FTN_W3_TRACE builds): a tile of the first /
  // last tile column costs ~1.75x an interior one, another tile of the first / last tile row
  // ~1.4x (their boxes overhang the array in the contiguous dimension resp. by whole rows).
  static int64_t wi_e = 16, wj_e = 11;  // 2048^3 / 512^3 GLUPS: (12,12) 611 / 405, (14,11) 616 / 455, (16,11) 618 / 497
  static const bool parsed = [] {
    if (const char* e = getenv("FTN_W3_EDGE_W")) {
      long long a = 0, b = 0;
      const int n = sscanf(e, "%lld,%lld", &a, &b);
      if (n >= 1 && a > 0) wi_e = a;
      wj_e = n == 2 && b > 0 ? b : wi_e;
    }
    return true;
  }();
  (void)parsed;
  p.w_in = 8;
  p.w_iedge = wi_e;
  p.w_jedge = wj_e;
  const int64_t TI = p.tiles_i, TJ = p.tiles_j;
  auto row_total = [&](int64_t wm) { return TI == 1 ? p.w_iedge : 2 * p.w_iedge + (TI - 2) * wm; };
  p.W = (TJ == 1 ? row_total(p.w_jedge) : 2 * row_total(p.w_jedge) + (TJ - 2) * row_total(p.w_in)) * nk;
  int64_t grid = num_sms();
  const int64_t need = (TI * TJ * nk + 15) / 16;  // at least ~16 planes of a tile per CTA
  if (grid > need) grid = need < 1 ? 1 : need;
  // Large grids: deal (tile, 512-plane band) cells round-robin instead (cell c to CTA c mod G).
  // CTAs launched together then sweep neighbouring tiles at the same planes and share the box
  // halos through L2: at 2048^3 the DRAM reads fall from 1.92x to 1.34x the algorithmic bytes,
  // and under the board's power cap that is +5.5 % (602-605 -> 635-637 GLUPS; bands of 384-768
  // planes are equal, 1024 623).  The grid is made coprime to the tile-row length so a CTA's
  // cells rotate through the tile columns (the edge tiles spread over all CTAs).  It needs >= 40
  // cells per CTA for the statistical balance (512^3: 390 vs 495, 1024^3: 514 vs 595 GLUPS with
  // 10 cells per CTA), so smaller grids keep the weighted split.  FTN_W3_RR = band (0: off).
  // By default the cells are not dealt but taken, in order, from a per-launch ticket counter
  // (FTN_W3_DYN=1): a CTA that finishes early takes the next cell, so no grid adjustment is
  // needed and the load balances exactly (+2.7 % over the static deal at 2048^3).
  static const int64_t rr_env = getenv("FTN_W3_RR") ? atoll(getenv("FTN_W3_RR")) : -1;
  static const int dyn_env = getenv("FTN_W3_DYN") ? atoi(getenv("FTN_W3_DYN")) : 1;
  p.ticket = nullptr;
  {
    const int64_t band = rr_env >= 0 ? rr_env : 512;
    int64_t g2 = grid;
    while (g2 > 1 && std::gcd(g2, (int64_t)p.tiles_i) != 1) --g2;
    const int64_t cells = band > 0 ? TI * TJ * ((nk + band - 1) / band) : 0;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) {  // e.g. the legacy stream during a global capture
      cudaGetLastError();
      cap = cudaStreamCaptureStatusActive;
    }
    const bool large = band > 0 && (rr_env > 0 || cells >= 40 * g2);
    if (large && dyn_env && cap == cudaStreamCaptureStatusNone) {
      // dynamic cells: CTAs take (tile, band) cells from a ticket counter in launch order
      // (2048^3: 649 vs 630-632 GLUPS for the static round-robin; no capture: a replayed graph
      // would share the slot between replays)
      p.rr_band = band;
      p.ticket = ticket_slot();
      if (!p.ticket) return fail(FTN_ERR_CUDA, "jacobi3d_wr: ticket slots");
    } else {
      p.rr_band = large ? band : 0;
      if (p.rr_band > 0) grid = g2;
    }
  }
  p.G = grid;
#if FTN_W3_TRACE
  {
    static long long* buf = nullptr;
    if (!buf) cudaMalloc(&buf, 4 * 8 * 1024);
    cudaMemcpyToSymbolAsync(w3_trace, &buf, sizeof(buf), 0, cudaMemcpyHostToDevice, s);
    static int calls = 0;
    if (getenv("FTN_W3_TRACE_DUMP") && ++calls == atoi(getenv("FTN_W3_TRACE_DUMP"))) {
      jacobi3d_wr<T><<<(unsigned)grid, W3_THREADS, C::SMEM, s>>>(*mp, p);
      std::vector<long long> h(4 * grid);
      cudaMemcpyAsync(h.data(), buf, h.size() * 8, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      long long t0 = h[0];
      for (int64_t i = 0; i < grid; ++i) t0 = std::min(t0, h[4 * i]);
      for (int64_t i = 0; i < grid; ++i)
        fprintf(stderr, "W3TRACE %lld %lld %lld %lld %lld\n", (long long)i, h[4 * i] - t0, h[4 * i + 1] - t0,
                h[4 * i + 2], h[4 * i + 3]);
      return after_launch("jacobi3d_wr");
    }
  }
#endif
  jacobi3d_wr<T><<<(unsigned)grid, W3_THREADS, C::SMEM, s>>>(*mp, p);
  return after_launch("jacobi3d_wr");
}

}  // namespace

// T fused 3-D sweeps src -> dst (TMA-able rank-3 arrays) on output planes [plane_lo, plane_hi]
// (0-based positions in dim 3); planes <= fix_lo and >= fix_hi are held fixed (the global
// boundary).  Reads src planes [plane_lo - T, plane_hi + T].
ftn_status_t jacobi3d_wr_planes(const ftn_desc_t* src, const ftn_desc_t* dst, int T, double coeff, int64_t plane_lo,
                                int64_t plane_hi, int64_t fix_lo, int64_t fix_hi, cudaStream_t s) {
  switch (T) {
    case 3: return launch_wr<3>(src, dst, coeff, plane_lo, plane_hi, fix_lo, fix_hi, s);
    case 4: return launch_wr<4>(src, dst, coeff, plane_lo, plane_hi, fix_lo, fix_hi, s);
  }
  return fail(FTN_ERR_UNSUPPORTED, "jacobi3d_wr: T must be 3 or 4 (2 sweeps: jacobi3d_tb2)");
}

}  // namespace ftn
