// tra-adv (R#28): the NEMO tracer-advection benchmark the paper
// runs ("six fields on a three dimensional grid of size 1024 by 512 by 512, running over
// 20 iterations"), its loop nests as recalled in R#28 -- the same statements, with the same
// Fortran evaluation order as oracle/ftn_oracle.c's orc_tra_adv_f64, so results are
// bit-identical (-fmad=false; SIGN = copysign, MIN / MAX / ABS exact).  Fields are indexed
// (ji, jj, jk), ji contiguous.
//
// Default: two fused passes per iteration (ta_h, ta_v below), ~115 B per cell moved against
// the algorithmic 72 B.  FTN_TA_PASSES=8: the eight-pass version (K1..K8, one kernel per group
// of loop nests, every temporary through HBM: 288 B per cell), kept as the plain reference
// of the fusion:
//   K1  steps 1-2   zind (all points); zwx, zwy (ji < jpi-1, jj < jpj-1, jk < jpk-1; 0 at jk = jpk-1)
//   K2  steps 3-4   slopes zslpx, zslpy (ji >= 1, jj >= 1, jk < jpk-1; 0 at jk = jpk-1): step 4
//                   at a point reads only step 3's value at that point, so the two fuse per point
//   K3  step 5      horizontal fluxes zwx, zwy (interior) -- reads no zwx / zwy
//   K4  step 6      md += -(flux divergence) (interior)
//   K5  step 7      vertical gradients zwx (all ji, jj; 0 at jk = 0 and jpk-1)
//   K6  steps 8-9   vertical slopes zslpx (all ji, jj, 1 <= jk < jpk-1; 0 at jk = 0)
//   K7  steps 10-11 vertical fluxes: zwx(:,:,0) = pwn md, zwx(jk+1) (interior) -- reads no zwx
//   K8  step 12     md = -(zwx - zwx(jk+1)) (interior)
// The temporaries live in the caller's workspace (5 packed arrays), zeroed at the start of the
// call (R#28).
#include "ftn_internal.cuh"

#include <cstdlib>
#include <cstring>

namespace ftn {
namespace {

struct F3 {
  char* b;
  int64_t s1, s2, s3;
  __device__ __forceinline__ double& operator()(int64_t i, int64_t j, int64_t k) const {
    return *reinterpret_cast<double*>(b + i * s1 + j * s2 + k * s3);
  }
};
struct F2 {
  const char* b;
  int64_t s1, s2;
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const {
    return *reinterpret_cast<const double*>(b + i * s1 + j * s2);
  }
};

struct TAParams {
  F3 md, tsn, pun, pvn, pwn, umask, vmask, tmask;
  F3 zind, zwx, zwy, zslpx, zslpy;
  F2 ztfreez, rnfmsk, upsmsk;
  const char* rz;
  int64_t rz_s;
  int64_t ni, nj, nk;
};

__device__ __forceinline__ double fsign(double a, double b) { return copysign(fabs(a), b); }

// Block (x, y = jj - j_lo, z = jk - k_lo): ji = i_lo + x * 256 + threadIdx.x.
struct Range {
  int64_t i_lo, i_hi, j_lo, k_lo;
};
__device__ __forceinline__ bool at(const Range& r, int64_t& i, int64_t& j, int64_t& k) {
  i = r.i_lo + (int64_t)blockIdx.x * 256 + threadIdx.x;
  j = r.j_lo + blockIdx.y;
  k = r.k_lo + blockIdx.z;
  return i < r.i_hi;
}

// K1: steps 1 and 2
__global__ void __launch_bounds__(256) ta_k1(const __grid_constant__ TAParams p, const Range r) {
  int64_t i, j, k;
  if (!at(r, i, j, k)) return;
  const double zice = p.tsn(i, j, k) <= p.ztfreez(i, j) + 0.1 ? 1.0 : 0.0;
  double m = p.rnfmsk(i, j) * *reinterpret_cast<const double*>(p.rz + k * p.rz_s);
  m = fmax(fmax(m, p.upsmsk(i, j)), zice);
  p.zind(i, j, k) = 1.0 - m * p.tmask(i, j, k);
  if (k == p.nk - 1) {
    p.zwx(i, j, k) = 0.0;
    p.zwy(i, j, k) = 0.0;
  } else if (i < p.ni - 1 && j < p.nj - 1) {
    const double c = p.md(i, j, k);
    p.zwx(i, j, k) = p.umask(i, j, k) * (p.md(i + 1, j, k) - c);
    p.zwy(i, j, k) = p.vmask(i, j, k) * (p.md(i, j + 1, k) - c);
  }
}

// K2: steps 3 and 4 (range jk < jpk-1 with jj >= 1, ji >= 1; and the zero plane jk = jpk-1)
__global__ void __launch_bounds__(256) ta_k2(const __grid_constant__ TAParams p, const Range r) {
  int64_t i, j, k;
  if (!at(r, i, j, k)) return;
  if (k == p.nk - 1) {
    p.zslpx(i, j, k) = 0.0;
    p.zslpy(i, j, k) = 0.0;
    return;
  }
  if (i < 1 || j < 1) return;
  const double ax = p.zwx(i, j, k), bx = p.zwx(i - 1, j, k);
  const double sx = (ax + bx) * (0.25 + fsign(0.25, ax * bx));
  p.zslpx(i, j, k) = fsign(1.0, sx) * fmin(fmin(fabs(sx), 2.0 * fabs(bx)), 2.0 * fabs(ax));
  const double ay = p.zwy(i, j, k), by = p.zwy(i, j - 1, k);
  const double sy = (ay + by) * (0.25 + fsign(0.25, ay * by));
  p.zslpy(i, j, k) = fsign(1.0, sy) * fmin(fmin(fabs(sy), 2.0 * fabs(by)), 2.0 * fabs(ay));
}

// K3: step 5 (interior ji, jj; jk < jpk-1)
__global__ void __launch_bounds__(256) ta_k3(const __grid_constant__ TAParams p, const Range r) {
  int64_t i, j, k;
  if (!at(r, i, j, k)) return;
  const double zi = p.zind(i, j, k), u = p.pun(i, j, k), v = p.pvn(i, j, k), c = p.md(i, j, k);
  const double z0u = fsign(0.5, u);
  double zalpha = 0.5 - z0u;
  const double zu = z0u - (0.5 * u) * 1.0;
  double zzwx = p.md(i + 1, j, k) + zi * (zu * p.zslpx(i + 1, j, k));
  double zzwy = c + zi * (zu * p.zslpx(i, j, k));
  p.zwx(i, j, k) = u * (zalpha * zzwx + (1.0 - zalpha) * zzwy);
  const double z0v = fsign(0.5, v);
  zalpha = 0.5 - z0v;
  const double zv = z0v - (0.5 * v) * 1.0;
  zzwx = p.md(i, j + 1, k) + zi * (zv * p.zslpy(i, j + 1, k));
  zzwy = c + zi * (zv * p.zslpy(i, j, k));
  p.zwy(i, j, k) = v * (zalpha * zzwx + (1.0 - zalpha) * zzwy);
}

// K4: step 6 (interior)
__global__ void __launch_bounds__(256) ta_k4(const __grid_constant__ TAParams p, const Range r) {
  int64_t i, j, k;
  if (!at(r, i, j, k)) return;
  const double ztra =
      -(1.0 * (((p.zwx(i, j, k) - p.zwx(i - 1, j, k)) + p.zwy(i, j, k)) - p.zwy(i, j - 1, k)));
  p.md(i, j, k) = p.md(i, j, k) + ztra;
}

// K5: step 7 (all ji, jj, jk)
__global__ void __launch_bounds__(256) ta_k5(const __grid_constant__ TAParams p, const Range r) {
  int64_t i, j, k;
  if (!at(r, i, j, k)) return;
  if (k == 0 || k == p.nk - 1) {
    p.zwx(i, j, k) = 0.0;
    return;
  }
  p.zwx(i, j, k) = p.tmask(i, j, k) * (p.md(i, j, k - 1) - p.md(i, j, k));
}

// K6: steps 8 and 9 (all ji, jj; jk <= jpk-2; zero at jk = 0)
__global__ void __launch_bounds__(256) ta_k6(const __grid_constant__ TAParams p, const Range r) {
  int64_t i, j, k;
  if (!at(r, i, j, k)) return;
  if (k == 0) {
    p.zslpx(i, j, k) = 0.0;
    return;
  }
  const double a = p.zwx(i, j, k), b = p.zwx(i, j, k + 1);
  const double s = (a + b) * (0.25 + fsign(0.25, a * b));
  p.zslpx(i, j, k) = fsign(1.0, s) * fmin(fmin(fabs(s), 2.0 * fabs(b)), 2.0 * fabs(a));
}

// K7: steps 10 and 11: block z = 0 writes zwx(:,:,0) = pwn md (all ji, jj); block z = kk >= 1
// writes zwx(:,:,kk) from level k = kk-1 (interior ji, jj only)
__global__ void __launch_bounds__(256) ta_k7(const __grid_constant__ TAParams p, const Range r) {
  int64_t i, j, kk;
  if (!at(r, i, j, kk)) return;
  if (kk == 0) {
    p.zwx(i, j, 0) = p.pwn(i, j, 0) * p.md(i, j, 0);
    return;
  }
  if (i < 1 || i > p.ni - 2 || j < 1 || j > p.nj - 2) return;
  const int64_t k = kk - 1;
  const double w1 = p.pwn(i, j, kk), zi = p.zind(i, j, k);
  const double z0w = fsign(0.5, w1);
  const double zalpha = 0.5 + z0w;
  const double zw = z0w - ((0.5 * w1) * 1.0) * 1.0;
  const double zzwx = p.md(i, j, kk) + zi * (zw * p.zslpx(i, j, kk));
  const double zzwy = p.md(i, j, k) + zi * (zw * p.zslpx(i, j, k));
  p.zwx(i, j, kk) = w1 * (zalpha * zzwx + (1.0 - zalpha) * zzwy);
}

// K8: step 12 (interior)
__global__ void __launch_bounds__(256) ta_k8(const __grid_constant__ TAParams p, const Range r) {
  int64_t i, j, k;
  if (!at(r, i, j, k)) return;
  p.md(i, j, k) = -(1.0 * (p.zwx(i, j, k) - p.zwx(i, j, k + 1)));
}

// ---------------------------------------------------------------- fused: two passes per iteration
// H: steps 1-6 for one (jk, 32 x 8 tile), every intermediate in shared memory (halo 2 in ji
//    and jj); writes zind and md6 (the tracer after step 6) -- 72 B per cell instead of 192.
// V: steps 7-12 for one (ji, jj) column, streaming jk with the vertical gradients, slopes and
//    fluxes in registers; writes md and, for the column ji = jpi-1, the side buffer S(jj, jk)
//    = its final zwx, which the next iteration's step 3 reads (R#28: the temporaries carry
//    over) -- 40 B per cell instead of 96.
#ifndef FTN_TA_TX
#define FTN_TA_TX 32
#endif
#ifndef FTN_TA_TY
#define FTN_TA_TY 32
#endif
constexpr int TH_X = FTN_TA_TX, TH_Y = FTN_TA_TY;  // output tile per CTA of 32 x 8 threads

struct TAFused {
  F3 md6;       // workspace: the tracer after step 6
  double* side; // workspace: zwx(jpi-1, jj, jk), jj + jpj * jk
};

__device__ __forceinline__ double ta_limit(double a, double b) {  // steps 3-4 / 8-9: slope of (a, b)
  const double s = (a + b) * (0.25 + fsign(0.25, a * b));
  return fsign(1.0, s) * fmin(fmin(fabs(s), 2.0 * fabs(b)), 2.0 * fabs(a));
}

__device__ __forceinline__ double ta_zind(const TAParams& p, int64_t i, int64_t j, int64_t k) {
  const double zice = p.tsn(i, j, k) <= p.ztfreez(i, j) + 0.1 ? 1.0 : 0.0;
  double m = p.rnfmsk(i, j) * *reinterpret_cast<const double*>(p.rz + k * p.rz_s);
  m = fmax(fmax(m, p.upsmsk(i, j)), zice);
  return 1.0 - m * p.tmask(i, j, k);
}

// Shared-memory regions of one tile (origin i0, j0), each [rows][cols] with its own offsets:
//   md  i0-2 .. i0+33, j0-2 .. j0+33    zi  i0-1 .. i0+31, j0-1 .. j0+31 (zind)
//   wx  s = i0-2 .. i0+32, tile rows    wy  tile columns, t = j0-2 .. j0+32   (step 2)
//   sx  s = i0-1 .. i0+32, tile rows    sy  tile columns, t = j0-1 .. j0+32   (steps 3-4)
//   fx  f = i0-1 .. i0+31, tile rows    fy  tile columns, g = j0-1 .. j0+31   (step 5)
// Loops walk rows with the 8 thread rows and columns with the 32 lanes (no divisions).
struct TASmem {
  double md[TH_Y + 4][TH_X + 4];
  double zi[TH_Y + 1][TH_X + 1];
  double wx[TH_Y][TH_X + 3];
  double wy[TH_Y + 3][TH_X];
  double sx[TH_Y][TH_X + 2];
  double sy[TH_Y + 2][TH_X];
};

__global__ void __launch_bounds__(256) ta_h(const __grid_constant__ TAParams p, const __grid_constant__ TAFused q) {
  extern __shared__ double ta_smem_raw[];
  TASmem& S = *reinterpret_cast<TASmem*>(ta_smem_raw);
  constexpr int MX = TH_X / 32, RY = TH_Y / 8;  // columns per lane, rows per thread row
  const int64_t ni = p.ni, nj = p.nj, nk = p.nk;
  const int64_t i0 = (int64_t)blockIdx.x * TH_X, j0 = (int64_t)blockIdx.y * TH_Y, k = blockIdx.z;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (k == nk - 1) {  // top plane: zind only, md6 = md
    for (int ly = ty; ly < TH_Y; ly += 8)
#pragma unroll
      for (int m = 0; m < MX; ++m) {
        const int64_t i = i0 + tx + 32 * m, j = j0 + ly;
        if (i < ni && j < nj) {
          p.zind(i, j, k) = ta_zind(p, i, j, k);
          q.md6(i, j, k) = p.md(i, j, k);
        }
      }
    return;
  }
  // md over the halo-2 region
  for (int ly = ty; ly < TH_Y + 4; ly += 8) {
    const int64_t j = j0 - 2 + ly;
    for (int lx = tx; lx < TH_X + 4; lx += 32) {
      const int64_t i = i0 - 2 + lx;
      S.md[ly][lx] = (i >= 0 && i < ni && j >= 0 && j < nj) ? p.md(i, j, k) : 0.0;
    }
  }
  // zind over i0-1 .. i0+TH_X-1, j0-1 .. j0+TH_Y-1; the tile's own points go to global for pass V
  for (int ly = ty; ly < TH_Y + 1; ly += 8) {
    const int64_t j = j0 - 1 + ly;
    for (int lx = tx; lx < TH_X + 1; lx += 32) {
      const int64_t i = i0 - 1 + lx;
      double z = 0.0;
      if (i >= 0 && i < ni && j >= 0 && j < nj) {
        z = ta_zind(p, i, j, k);
        if (lx >= 1 && ly >= 1) p.zind(i, j, k) = z;
      }
      S.zi[ly][lx] = z;
    }
  }
  __syncthreads();
  // step 2 (and the carried-over zwx of the last column, R#28)
  for (int ly = ty; ly < TH_Y; ly += 8) {
    const int64_t j = j0 + ly;
    for (int lx = tx; lx < TH_X + 3; lx += 32) {
      const int64_t s = i0 - 2 + lx;
      double v = 0.0;
      if (j < nj - 1 && s >= 0 && s < ni - 1) v = p.umask(s, j, k) * (S.md[ly + 2][lx + 1] - S.md[ly + 2][lx]);
      else if (j < nj && s == ni - 1) v = q.side[j + nj * k];
      S.wx[ly][lx] = v;
    }
  }
  for (int ly = ty; ly < TH_Y + 3; ly += 8) {
    const int64_t t = j0 - 2 + ly;
#pragma unroll
    for (int m = 0; m < MX; ++m) {
      const int c = tx + 32 * m;
      const int64_t i = i0 + c;
      double v = 0.0;
      if (i < ni - 1 && t >= 0 && t < nj - 1) v = p.vmask(i, t, k) * (S.md[ly + 1][c + 2] - S.md[ly][c + 2]);
      S.wy[ly][c] = v;
    }
  }
  __syncthreads();
  // steps 3-4
  for (int ly = ty; ly < TH_Y; ly += 8)
    for (int lx = tx; lx < TH_X + 2; lx += 32) S.sx[ly][lx] = ta_limit(S.wx[ly][lx + 1], S.wx[ly][lx]);
  for (int ly = ty; ly < TH_Y + 2; ly += 8)
#pragma unroll
    for (int m = 0; m < MX; ++m) {
      const int c = tx + 32 * m;
      S.sy[ly][c] = ta_limit(S.wy[ly + 1][c], S.wy[ly][c]);
    }
  __syncthreads();
  // step 5: x fluxes at f = i0-1 .. i0+TH_X-1 (zwx2(0) where step 5 leaves the boundary
  // column), y fluxes at g = j0-1 .. j0+TH_Y-1, kept in registers; the y fluxes then replace wy
  auto xflux = [&](int ly, int lx) {  // f = i0-1+lx, row j0+ly
    const int64_t f = i0 - 1 + lx, j = j0 + ly;
    if (f >= 1 && f <= ni - 2 && j >= 1 && j <= nj - 2) {
      const double zi = S.zi[ly + 1][lx], u = p.pun(f, j, k);
      const double z0u = fsign(0.5, u);
      const double zalpha = 0.5 - z0u;
      const double zu = z0u - (0.5 * u) * 1.0;
      const double zzwx = S.md[ly + 2][lx + 2] + zi * (zu * S.sx[ly][lx + 1]);
      const double zzwy = S.md[ly + 2][lx + 1] + zi * (zu * S.sx[ly][lx]);
      return u * (zalpha * zzwx + (1.0 - zalpha) * zzwy);
    }
    return f == 0 ? S.wx[ly][lx + 1] : 0.0;
  };
  double fx[RY][MX][2], fy[RY + 1][MX];
#pragma unroll
  for (int r = 0; r < RY; ++r)
#pragma unroll
    for (int m = 0; m < MX; ++m) {
      const int ly = ty + 8 * r, c = tx + 32 * m;
      fx[r][m][0] = xflux(ly, c);       // f = i0 + c - 1
      fx[r][m][1] = xflux(ly, c + 1);   // f = i0 + c
    }
#pragma unroll
  for (int r = 0; r < RY + 1; ++r)
#pragma unroll
    for (int m = 0; m < MX; ++m) {
      const int ly = ty + 8 * r, c = tx + 32 * m;  // g = j0-1+ly (ly < TH_Y + 1)
      fy[r][m] = 0.0;
      if (ly >= TH_Y + 1) continue;
      const int64_t i = i0 + c, g = j0 - 1 + ly;
      if (g >= 1 && g <= nj - 2 && i >= 1 && i <= ni - 2) {
        const double zi = S.zi[ly][c + 1], w = p.pvn(i, g, k);
        const double z0v = fsign(0.5, w);
        const double zalpha = 0.5 - z0v;
        const double zv = z0v - (0.5 * w) * 1.0;
        const double zzwx = S.md[ly + 2][c + 2] + zi * (zv * S.sy[ly + 1][c]);
        const double zzwy = S.md[ly + 1][c + 2] + zi * (zv * S.sy[ly][c]);
        fy[r][m] = w * (zalpha * zzwx + (1.0 - zalpha) * zzwy);
      } else if (g == 0) {
        fy[r][m] = S.wy[ly + 1][c];
      }
    }
  __syncthreads();  // every read of wy / sy is done: wy[ly][c] now holds the y flux at g = j0-1+ly
#pragma unroll
  for (int r = 0; r < RY + 1; ++r)
#pragma unroll
    for (int m = 0; m < MX; ++m) {
      const int ly = ty + 8 * r, c = tx + 32 * m;
      if (ly < TH_Y + 1) S.wy[ly][c] = fy[r][m];
    }
  __syncthreads();
  // step 6
#pragma unroll
  for (int r = 0; r < RY; ++r)
#pragma unroll
    for (int m = 0; m < MX; ++m) {
      const int ly = ty + 8 * r, c = tx + 32 * m;
      const int64_t i = i0 + c, j = j0 + ly;
      if (i >= ni || j >= nj) continue;
      double v = S.md[ly + 2][c + 2];
      if (i >= 1 && i <= ni - 2 && j >= 1 && j <= nj - 2) {
        const double ztra = -(1.0 * (((fx[r][m][1] - fx[r][m][0]) + S.wy[ly + 1][c]) - S.wy[ly][c]));
        v = v + ztra;
      }
      q.md6(i, j, k) = v;
    }
}

// ---------------------------------------------------------------- ta_h with TMA (the default
// when all seven 3-D inputs are TMA-able): a CTA walks KC consecutive k-planes of one 32 x 32
// tile; the seven inputs of plane k+1 (36 x 36 boxes at (i0-2, j0-2), zero outside the array)
// arrive by TMA into the other half of a double buffer while plane k is computed, so the
// loads are in flight during the whole step instead of between barriers.
constexpr int TB = TH_X + 4;                 // box edge (36)
constexpr int TBOX = TB * TB * 8;            // bytes per field box
constexpr int TNF = 7;                       // md, tsn, tmask, umask, vmask, pun, pvn
constexpr int TKC = 16;                      // planes per CTA
struct TAMaps {
  CUtensorMap m[TNF];
};
struct TAHsmem {
  double box[2][TNF][TB][TB];                // double-buffered input boxes
  double zi[TH_Y + 1][TH_X + 1];
  double wx[TH_Y][TH_X + 3];
  double wy[TH_Y + 3][TH_X];
  double sx[TH_Y][TH_X + 2];
  double sy[TH_Y + 2][TH_X];
  double f2[3][TH_Y + 1][TH_X + 1];          // ztfreez, rnfmsk, upsmsk at the zind region
  uint64_t full[2];
};

__global__ void __launch_bounds__(256, 1) ta_h_tma(const __grid_constant__ TAMaps maps,
                                                   const __grid_constant__ TAParams p,
                                                   const __grid_constant__ TAFused q) {
  extern __shared__ __align__(128) uint8_t ta_tma_raw[];
  TAHsmem& S = *reinterpret_cast<TAHsmem*>((reinterpret_cast<uintptr_t>(ta_tma_raw) + 127) & ~uintptr_t(127));
  constexpr int MX = TH_X / 32, RY = TH_Y / 8;
  enum { MD = 0, TSN = 1, TM = 2, UM = 3, VM = 4, PU = 5, PV = 6 };
  const int64_t ni = p.ni, nj = p.nj, nk = p.nk;
  const int64_t i0 = (int64_t)blockIdx.x * TH_X, j0 = (int64_t)blockIdx.y * TH_Y;
  const int64_t ka = (int64_t)blockIdx.z * TKC, kb = min(ka + TKC, nk);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  auto issue = [&](int64_t k, int st) {
    dev::mbar_arrive_expect_tx(&S.full[st], TNF * TBOX);
    for (int f = 0; f < TNF; ++f)
      dev::tma_load_3d(&S.box[st][f][0][0], &maps.m[f], &S.full[st], (int32_t)(i0 - 2), (int32_t)(j0 - 2), (int32_t)k);
  };
  if (threadIdx.x == 0) {
    dev::mbar_init(&S.full[0], 1);
    dev::mbar_init(&S.full[1], 1);
    dev::fence_barrier_init();
    for (int f = 0; f < TNF; ++f) dev::prefetch_tma(&maps.m[f]);
    issue(ka, 0);
  }
  // the 2-D fields of the zind region (constant over k)
  for (int ly = ty; ly < TH_Y + 1; ly += 8) {
    const int64_t j = j0 - 1 + ly;
    for (int lx = tx; lx < TH_X + 1; lx += 32) {
      const int64_t i = i0 - 1 + lx;
      const bool in = i >= 0 && i < ni && j >= 0 && j < nj;
      S.f2[0][ly][lx] = in ? p.ztfreez(i, j) : 0.0;
      S.f2[1][ly][lx] = in ? p.rnfmsk(i, j) : 0.0;
      S.f2[2][ly][lx] = in ? p.upsmsk(i, j) : 0.0;
    }
  }
  __syncthreads();
  for (int64_t k = ka; k < kb; ++k) {
    const int st = (int)((k - ka) & 1);
    if (threadIdx.x == 0 && k + 1 < kb) issue(k + 1, st ^ 1);  // its buffer was released at the end of k-1
    dev::mbar_wait(&S.full[st], (uint32_t)(((k - ka) >> 1) & 1));
    double (*B)[TB][TB] = S.box[st];
    const double rzk = *reinterpret_cast<const double*>(p.rz + k * p.rz_s);
    // zind over i0-1 .. i0+31, j0-1 .. j0+31 (box offset +1); the tile's own points to global
    for (int ly = ty; ly < TH_Y + 1; ly += 8) {
      const int64_t j = j0 - 1 + ly;
      for (int lx = tx; lx < TH_X + 1; lx += 32) {
        const int64_t i = i0 - 1 + lx;
        const double zice = B[TSN][ly + 1][lx + 1] <= S.f2[0][ly][lx] + 0.1 ? 1.0 : 0.0;
        double m = S.f2[1][ly][lx] * rzk;
        m = fmax(fmax(m, S.f2[2][ly][lx]), zice);
        const double z = 1.0 - m * B[TM][ly + 1][lx + 1];
        S.zi[ly][lx] = z;
        if (lx >= 1 && ly >= 1 && i < ni && j < nj) p.zind(i, j, k) = z;
      }
    }
    if (k == nk - 1) {  // top plane: zind only, md6 = md
#pragma unroll
      for (int r = 0; r < RY; ++r)
#pragma unroll
        for (int m = 0; m < MX; ++m) {
          const int ly = ty + 8 * r, c = tx + 32 * m;
          const int64_t i = i0 + c, j = j0 + ly;
          if (i < ni && j < nj) q.md6(i, j, k) = B[MD][ly + 2][c + 2];
        }
      __syncthreads();
      continue;
    }
    // step 2 (and the carried-over zwx of the last column, R#28)
    for (int ly = ty; ly < TH_Y; ly += 8) {
      const int64_t j = j0 + ly;
      for (int lx = tx; lx < TH_X + 3; lx += 32) {
        const int64_t s2 = i0 - 2 + lx;
        double v = 0.0;
        if (j < nj - 1 && s2 >= 0 && s2 < ni - 1) v = B[UM][ly + 2][lx] * (B[MD][ly + 2][lx + 1] - B[MD][ly + 2][lx]);
        else if (j < nj && s2 == ni - 1) v = q.side[j + nj * k];
        S.wx[ly][lx] = v;
      }
    }
    for (int ly = ty; ly < TH_Y + 3; ly += 8) {
      const int64_t t = j0 - 2 + ly;
#pragma unroll
      for (int m = 0; m < MX; ++m) {
        const int c = tx + 32 * m;
        const int64_t i = i0 + c;
        double v = 0.0;
        if (i < ni - 1 && t >= 0 && t < nj - 1) v = B[VM][ly][c + 2] * (B[MD][ly + 1][c + 2] - B[MD][ly][c + 2]);
        S.wy[ly][c] = v;
      }
    }
    __syncthreads();
    // steps 3-4
    for (int ly = ty; ly < TH_Y; ly += 8)
      for (int lx = tx; lx < TH_X + 2; lx += 32) S.sx[ly][lx] = ta_limit(S.wx[ly][lx + 1], S.wx[ly][lx]);
    for (int ly = ty; ly < TH_Y + 2; ly += 8)
#pragma unroll
      for (int m = 0; m < MX; ++m) {
        const int c = tx + 32 * m;
        S.sy[ly][c] = ta_limit(S.wy[ly + 1][c], S.wy[ly][c]);
      }
    __syncthreads();
    // step 5
    auto xflux = [&](int ly, int lx) {  // f = i0-1+lx, row j0+ly
      const int64_t f = i0 - 1 + lx, j = j0 + ly;
      if (f >= 1 && f <= ni - 2 && j >= 1 && j <= nj - 2) {
        const double zi = S.zi[ly + 1][lx], u = B[PU][ly + 2][lx + 1];
        const double z0u = fsign(0.5, u);
        const double zalpha = 0.5 - z0u;
        const double zu = z0u - (0.5 * u) * 1.0;
        const double zzwx = B[MD][ly + 2][lx + 2] + zi * (zu * S.sx[ly][lx + 1]);
        const double zzwy = B[MD][ly + 2][lx + 1] + zi * (zu * S.sx[ly][lx]);
        return u * (zalpha * zzwx + (1.0 - zalpha) * zzwy);
      }
      return f == 0 ? S.wx[ly][lx + 1] : 0.0;
    };
    double fx[RY][MX][2], fy[RY + 1][MX];
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int m = 0; m < MX; ++m) {
        const int ly = ty + 8 * r, c = tx + 32 * m;
        fx[r][m][0] = xflux(ly, c);
        fx[r][m][1] = xflux(ly, c + 1);
      }
#pragma unroll
    for (int r = 0; r < RY + 1; ++r)
#pragma unroll
      for (int m = 0; m < MX; ++m) {
        const int ly = ty + 8 * r, c = tx + 32 * m;
        fy[r][m] = 0.0;
        if (ly >= TH_Y + 1) continue;
        const int64_t i = i0 + c, g = j0 - 1 + ly;
        if (g >= 1 && g <= nj - 2 && i >= 1 && i <= ni - 2) {
          const double zi = S.zi[ly][c + 1], w = B[PV][ly + 1][c + 2];
          const double z0v = fsign(0.5, w);
          const double zalpha = 0.5 - z0v;
          const double zv = z0v - (0.5 * w) * 1.0;
          const double zzwx = B[MD][ly + 2][c + 2] + zi * (zv * S.sy[ly + 1][c]);
          const double zzwy = B[MD][ly + 1][c + 2] + zi * (zv * S.sy[ly][c]);
          fy[r][m] = w * (zalpha * zzwx + (1.0 - zalpha) * zzwy);
        } else if (g == 0) {
          fy[r][m] = S.wy[ly + 1][c];
        }
      }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RY + 1; ++r)
#pragma unroll
      for (int m = 0; m < MX; ++m) {
        const int ly = ty + 8 * r, c = tx + 32 * m;
        if (ly < TH_Y + 1) S.wy[ly][c] = fy[r][m];
      }
    __syncthreads();
    // step 6
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int m = 0; m < MX; ++m) {
        const int ly = ty + 8 * r, c = tx + 32 * m;
        const int64_t i = i0 + c, j = j0 + ly;
        if (i >= ni || j >= nj) continue;
        double v = B[MD][ly + 2][c + 2];
        if (i >= 1 && i <= ni - 2 && j >= 1 && j <= nj - 2) {
          const double ztra = -(1.0 * (((fx[r][m][1] - fx[r][m][0]) + S.wy[ly + 1][c]) - S.wy[ly][c]));
          v = v + ztra;
        }
        q.md6(i, j, k) = v;
      }
    __syncthreads();  // the boxes of plane k are free for plane k+2 (and S.zi / wx / ... for k+1)
    if (threadIdx.x == 0) dev::fence_proxy_async();
  }
}

__global__ void __launch_bounds__(256) ta_v(const __grid_constant__ TAParams p, const __grid_constant__ TAFused q) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x, j = blockIdx.y;
  const int64_t ni = p.ni, nj = p.nj, nk = p.nk;
  if (i >= ni) return;
  const bool inner = i >= 1 && i <= ni - 2 && j >= 1 && j <= nj - 2;
  const bool last_col = i == ni - 1;
  // step 7: zwx7(kk) = tmask (md6(kk-1) - md6(kk)) for 1 <= kk <= nk-2, 0 at kk = 0, nk-1
  auto zwx7 = [&](int64_t kk, double m_lo, double m_hi) {
    return (kk >= 1 && kk <= nk - 2) ? p.tmask(i, j, kk) * (m_lo - m_hi) : 0.0;
  };
  double m0 = q.md6(i, j, 0);
  double m1 = nk > 1 ? q.md6(i, j, 1) : 0.0;
  double z7_0 = 0.0;                                // zwx7(0)
  double z7_1 = nk > 1 ? zwx7(1, m0, m1) : 0.0;     // zwx7(1)
  // steps 8-9: zslpx(kk) = limit(zwx7(kk), zwx7(kk+1)) for 1 <= kk <= nk-2, 0 at kk = 0, nk-1
  double s_prev = 0.0;                              // zslpx(0)
  // step 10
  double flux_prev = p.pwn(i, j, 0) * m0;           // zwx(0)
  if (last_col) q.side[j + nj * 0] = flux_prev;
  double zi_prev = p.zind(i, j, 0);
  double m_prev = m0, m_cur = m1, z7_cur = z7_1;
  (void)z7_0;
  for (int64_t kk = 1; kk < nk; ++kk) {
    // plane kk: md6(kk) = m_cur, zwx7(kk) = z7_cur; look ahead to kk+1
    const double m_next = kk + 1 < nk ? q.md6(i, j, kk + 1) : 0.0;
    const double z7_next = kk + 1 < nk ? zwx7(kk + 1, m_cur, m_next) : 0.0;
    const double s_cur = (kk <= nk - 2) ? ta_limit(z7_cur, z7_next) : 0.0;
    double flux;  // zwx(kk) after steps 7, 10, 11
    if (inner) {
      const double w1 = p.pwn(i, j, kk);
      const double z0w = fsign(0.5, w1);
      const double zalpha = 0.5 + z0w;
      const double zw = z0w - ((0.5 * w1) * 1.0) * 1.0;
      const double zzwx = m_cur + zi_prev * (zw * s_cur);
      const double zzwy = m_prev + zi_prev * (zw * s_prev);
      flux = w1 * (zalpha * zzwx + (1.0 - zalpha) * zzwy);
      p.md(i, j, kk - 1) = -(1.0 * (flux_prev - flux));   // step 12 for plane kk-1
    } else {
      flux = z7_cur;
      p.md(i, j, kk - 1) = m_prev;                        // boundary columns: md6 = md
    }
    if (last_col) q.side[j + nj * kk] = flux;
    zi_prev = p.zind(i, j, kk);
    flux_prev = flux;
    s_prev = s_cur;
    m_prev = m_cur;
    m_cur = m_next;
    z7_cur = z7_next;
  }
  p.md(i, j, nk - 1) = m_prev;  // the top plane: never updated (md6 = md there)
}

F3 f3_of(const ftn_desc_t* d) {
  F3 f;
  f.b = (char*)d->base_addr;
  f.s1 = d->dim[0].sm;
  f.s2 = d->dim[1].sm;
  f.s3 = d->dim[2].sm;
  return f;
}
F2 f2_of(const ftn_desc_t* d) {
  F2 f;
  f.b = (const char*)d->base_addr;
  f.s1 = d->dim[0].sm;
  f.s2 = d->dim[1].sm;
  return f;
}

template <class K>
ftn_status_t ta_launch(K kern, const TAParams& p, int64_t i_lo, int64_t i_hi, int64_t j_lo, int64_t j_hi, int64_t k_lo,
                       int64_t k_hi, cudaStream_t s) {
  if (i_hi <= i_lo || j_hi <= j_lo || k_hi <= k_lo) return FTN_OK;
  if (j_hi - j_lo > 65535 || k_hi - k_lo > 65535)
    return fail(FTN_ERR_UNSUPPORTED, "ftn_tra_adv: jpj and jpk must be <= 65535");
  Range r{i_lo, i_hi, j_lo, k_lo};
  dim3 grid((unsigned)((i_hi - i_lo + 255) / 256), (unsigned)(j_hi - j_lo), (unsigned)(k_hi - k_lo));
  kern<<<grid, 256, 0, s>>>(p, r);
  return after_launch("tra_adv");
}

size_t ta_ws_bytes(const ftn_desc_t* md) {
  const size_t n = (size_t)desc_size(md);
  return 5 * ((n * 8 + 255) / 256 * 256);
}

}  // namespace
}  // namespace ftn

using namespace ftn;

extern "C" {

ftn_status_t ftn_tra_adv_workspace_size(const ftn_desc_t* md, size_t* bytes) {
  FTN_CHECK(check_desc(md, "ftn_tra_adv_workspace_size(md)", 3, 3));
  if (!bytes) return fail(FTN_ERR_NULL, "ftn_tra_adv_workspace_size: bytes NULL");
  *bytes = ta_ws_bytes(md);
  return FTN_OK;
}

ftn_status_t ftn_tra_adv(const ftn_desc_t* md, const ftn_desc_t* tsn, const ftn_desc_t* pun, const ftn_desc_t* pvn,
                         const ftn_desc_t* pwn, const ftn_desc_t* umask, const ftn_desc_t* vmask,
                         const ftn_desc_t* tmask, const ftn_desc_t* ztfreez, const ftn_desc_t* rnfmsk,
                         const ftn_desc_t* upsmsk, const ftn_desc_t* rnfmsk_z, int64_t iters, void* ws,
                         size_t ws_bytes, ftn_stream_t stream) {
  NvtxRange nvtx_("ftn_tra_adv");
  const ftn_desc_t* f3[8] = {md, tsn, pun, pvn, pwn, umask, vmask, tmask};
  static const char* n3[8] = {"md", "tsn", "pun", "pvn", "pwn", "umask", "vmask", "tmask"};
  for (int q = 0; q < 8; ++q) {
    FTN_CHECK(check_desc(f3[q], (std::string("ftn_tra_adv(") + n3[q] + ")").c_str(), 3, 3));
    if (f3[q]->type != FTN_F64) return fail(FTN_ERR_TYPE, "ftn_tra_adv: real(8) fields only");
    for (int d = 0; d < 3; ++d)
      if (f3[q]->dim[d].extent != md->dim[d].extent) return fail(FTN_ERR_SHAPE, "ftn_tra_adv: fields not conformable");
    if (q > 0 && desc_overlap(md, f3[q])) return fail(FTN_ERR_SHAPE, "ftn_tra_adv: md overlaps an input field");
  }
  const ftn_desc_t* f2[3] = {ztfreez, rnfmsk, upsmsk};
  for (int q = 0; q < 3; ++q) {
    FTN_CHECK(check_desc(f2[q], "ftn_tra_adv(2-D field)", 2, 2));
    if (f2[q]->type != FTN_F64) return fail(FTN_ERR_TYPE, "ftn_tra_adv: real(8) fields only");
    if (f2[q]->dim[0].extent != md->dim[0].extent || f2[q]->dim[1].extent != md->dim[1].extent)
      return fail(FTN_ERR_SHAPE, "ftn_tra_adv: 2-D fields must be (jpi, jpj)");
    if (desc_overlap(md, f2[q])) return fail(FTN_ERR_SHAPE, "ftn_tra_adv: md overlaps an input field");
  }
  FTN_CHECK(check_desc(rnfmsk_z, "ftn_tra_adv(rnfmsk_z)", 1, 1));
  if (rnfmsk_z->type != FTN_F64 || rnfmsk_z->dim[0].extent != md->dim[2].extent)
    return fail(FTN_ERR_SHAPE, "ftn_tra_adv: rnfmsk_z must be real(8) of extent jpk");
  if (iters < 0) return fail(FTN_ERR_SHAPE, "ftn_tra_adv: negative iteration count");
  const size_t need = ta_ws_bytes(md);
  if (!ws || ws_bytes < need || ((uintptr_t)ws % 256))
    return fail(FTN_ERR_WORKSPACE, "ftn_tra_adv: workspace must hold ftn_tra_adv_workspace_size bytes, 256-byte aligned");
  FTN_CHECK(require_sm100());
  const int64_t ni = md->dim[0].extent, nj = md->dim[1].extent, nk = md->dim[2].extent;
  if (ni * nj * nk == 0 || iters == 0) return FTN_OK;
  cudaStream_t s = (cudaStream_t)stream;
  TAParams p;
  p.md = f3_of(md);
  p.tsn = f3_of(tsn);
  p.pun = f3_of(pun);
  p.pvn = f3_of(pvn);
  p.pwn = f3_of(pwn);
  p.umask = f3_of(umask);
  p.vmask = f3_of(vmask);
  p.tmask = f3_of(tmask);
  F3* tmp[5] = {&p.zind, &p.zwx, &p.zwy, &p.zslpx, &p.zslpy};
  const size_t one = need / 5;
  for (int q = 0; q < 5; ++q) {
    tmp[q]->b = (char*)ws + q * one;
    tmp[q]->s1 = 8;
    tmp[q]->s2 = 8 * ni;
    tmp[q]->s3 = 8 * ni * nj;
  }
  p.ztfreez = f2_of(ztfreez);
  p.rnfmsk = f2_of(rnfmsk);
  p.upsmsk = f2_of(upsmsk);
  p.rz = (const char*)rnfmsk_z->base_addr;
  p.rz_s = rnfmsk_z->dim[0].sm;
  p.ni = ni;
  p.nj = nj;
  p.nk = nk;
  FTN_CUDA(cudaMemsetAsync(ws, 0, need, s));  // R#28: the temporaries start at zero
  static const bool passes8 = getenv("FTN_TA_PASSES") && atoi(getenv("FTN_TA_PASSES")) == 8;
  if (!passes8) {
    if (nj > 65535 || nk > 65535) return fail(FTN_ERR_UNSUPPORTED, "ftn_tra_adv: jpj and jpk must be <= 65535");
    static std::atomic<bool> attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[dev & 63]) {
      FTN_CUDA(cudaFuncSetAttribute(ta_h, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TASmem)));
      attr[dev & 63] = true;
    }
    TAFused q;
    q.md6 = p.zwx;                                        // workspace array 1
    q.side = reinterpret_cast<double*>(p.zwy.b);          // workspace array 2 (jpj x jpk used)
    const dim3 gh((unsigned)((ni + TH_X - 1) / TH_X), (unsigned)((nj + TH_Y - 1) / TH_Y), (unsigned)nk);
    const dim3 gv((unsigned)((ni + 255) / 256), (unsigned)nj);
    // TMA path: every 3-D input TMA-able (unit stride in ji, 16-byte aligned base and strides)
    const ftn_desc_t* tf[TNF] = {md, tsn, tmask, umask, vmask, pun, pvn};
    bool tma = getenv("FTN_TA_TMA") == nullptr || atoi(getenv("FTN_TA_TMA")) != 0;
    for (int f = 0; f < TNF && tma; ++f)
      tma = tf[f]->dim[0].sm == 8 && ((uintptr_t)tf[f]->base_addr % 16) == 0 && tf[f]->dim[1].sm > 0 &&
            tf[f]->dim[2].sm > 0 && (tf[f]->dim[1].sm % 16) == 0 && (tf[f]->dim[2].sm % 16) == 0;
    TAMaps maps;
    if (tma) {
      for (int f = 0; f < TNF; ++f) {
        uint64_t dims[3] = {(uint64_t)ni, (uint64_t)nj, (uint64_t)nk};
        uint64_t strides[2] = {(uint64_t)tf[f]->dim[1].sm, (uint64_t)tf[f]->dim[2].sm};
        uint32_t box[3] = {TB, TB, 1};
        FTN_CHECK(encode_tma(&maps.m[f], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, tf[f]->base_addr, dims, strides, box,
                             CU_TENSOR_MAP_SWIZZLE_NONE));
      }
      static std::atomic<bool> attr2[64] = {};
      if (!attr2[dev & 63]) {
        FTN_CUDA(cudaFuncSetAttribute(ta_h_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TAHsmem) + 128));
        attr2[dev & 63] = true;
      }
    }
    const dim3 ght((unsigned)((ni + TH_X - 1) / TH_X), (unsigned)((nj + TH_Y - 1) / TH_Y), (unsigned)((nk + TKC - 1) / TKC));
    for (int64_t it = 0; it < iters; ++it) {
      if (tma)
        ta_h_tma<<<ght, 256, sizeof(TAHsmem) + 128, s>>>(maps, p, q);
      else
        ta_h<<<gh, 256, sizeof(TASmem), s>>>(p, q);
      FTN_CHECK(after_launch("tra_adv_h"));
      ta_v<<<gv, 256, 0, s>>>(p, q);
      FTN_CHECK(after_launch("tra_adv_v"));
    }
    return FTN_OK;
  }
  for (int64_t it = 0; it < iters; ++it) {
    FTN_CHECK(ta_launch(ta_k1, p, 0, ni, 0, nj, 0, nk, s));
    FTN_CHECK(ta_launch(ta_k2, p, 0, ni, 0, nj, 0, nk, s));
    FTN_CHECK(ta_launch(ta_k3, p, 1, ni - 1, 1, nj - 1, 0, nk - 1, s));
    FTN_CHECK(ta_launch(ta_k4, p, 1, ni - 1, 1, nj - 1, 0, nk - 1, s));
    FTN_CHECK(ta_launch(ta_k5, p, 0, ni, 0, nj, 0, nk, s));
    FTN_CHECK(ta_launch(ta_k6, p, 0, ni, 0, nj, 0, nk - 1, s));
    FTN_CHECK(ta_launch(ta_k7, p, 0, ni, 0, nj, 0, nk, s));
    FTN_CHECK(ta_launch(ta_k8, p, 1, ni - 1, 1, nj - 1, 0, nk - 1, s));
  }
  return FTN_OK;
}

}  // extern "C"
