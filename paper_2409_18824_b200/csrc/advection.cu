// pw-advection (R#26, R#27): the 3-field advection stencil of the
// paper's pw-advection benchmark (body reproduced in DESIGN.md R#26):
// su, sv, sw at every interior point from u, v, w and their neighbours at k±1, j±1, i±1 (plus
// three diagonal points), the per-level coefficients tzc1, tzc2, tzd1, tzd2 (k) and the scalars
// tcx, tcy.  Fields are indexed (k, j, i) = dims (1, 2, 3), k contiguous.
//
// HBM-bound: 24 B read + 24 B written per interior point (48 B/cell).
//
// TMA path (u, v, w TMA-able): a CTA owns a 128 (k) x 8 (j) tile of output columns and marches
// along i.  Each i-plane of the three fields arrives as TMA boxes {132 x 10 x 1} (k-2 .. k+129,
// j-1 .. j+8; the k start 128t-2 is 16-byte aligned; 1 KB box rows keep DRAM efficient) into a
// 5-slot mbarrier ring; when plane i+1 has landed the 512 threads compute output plane i from
// the slots of planes i-1, i, i+1 (thread = a pair k, k+1 of one j row: its neighbours come as
// 16-byte pairs, LDS.128, and its results leave as 16-byte stores), then one block barrier,
// after which thread 0 refills the slot
// of plane i-1 (no producer warp, no empty barriers).  Work units = (tile, i-segment), tile
// fastest, round-robin (plan_units_halo).
// Generic path (any strides): one thread per output point, direct loads.
//
// Arithmetic: exactly the DO-nest expression of R#26 in Fortran order ((a*b)*c, x+(a-b)), one
// rounding per operation (-fmad=false), so results are bit-identical to the oracle.
#include "ftn_internal.cuh"

#include <algorithm>
#include <type_traits>
#include <cstdlib>

namespace ftn {

void plan_units_halo(int64_t tiles, int64_t len, int64_t grid, int64_t halo_rows, int64_t* seg, int64_t* units);
bool stencil_tma_able(const ftn_desc_t* d);

namespace {

#ifndef FTN_AD_OK
#define FTN_AD_OK 128
#endif
#ifndef FTN_AD_OJ
#define FTN_AD_OJ 8
#endif
constexpr int AD_OK = FTN_AD_OK, AD_OJ = FTN_AD_OJ;  // output tile (k, j)
#ifndef FTN_AD_PP
#define FTN_AD_PP 2
#endif
constexpr int AD_PP = FTN_AD_PP;                    // consecutive k points per thread (2 or 4)
constexpr int AD_PAIRS = AD_OK / AD_PP;             // threads per j row
constexpr int AD_BK = AD_OK + 4, AD_BJ = AD_OJ + 2;  // box 132 x 10: k-2 .. k+129, j-1 .. j+8
constexpr int AD_FIELD = (AD_BK * AD_BJ * 8 + 127) / 128 * 128;  // 9856 B per field box
constexpr int AD_SLOT = 3 * AD_FIELD;
constexpr int AD_THREADS = AD_PAIRS * AD_OJ;
template <int NS>
constexpr int ad_smem() { return NS * AD_SLOT + 128 + 8 * NS; }

struct AdvOut {
  char* base;
  int64_t sm1, sm2, sm3;
};

struct AdvParams {
  AdvOut su, sv, sw;
  const double* tz[4];  // tzc1, tzc2, tzd1, tzd2 (contiguous device vectors of length nz)
  int64_t tz_sm[4];     // byte strides of the coefficient vectors
  int32_t nz, ny, nx;
  int32_t tiles_k, tiles_j;
  int32_t seg;          // output i-planes per unit
  uint32_t units;
  int32_t vec_out;      // outputs: unit stride in k, 16-byte aligned base and strides
  double tcx, tcy;
};

// One output point from the three fields' (k, j) neighbourhoods.  P(f, dk, dj, di) reads field
// f at (k + dk, j + dj, i + di); the expression is the DO nest of R#26.
template <class P>
__device__ __forceinline__ void adv_point(const P& F, double tzc1, double tzc2, double tzd1, double tzd2, double tcx,
                                          double tcy, double& su, double& sv, double& sw) {
  double a, b, s;
  // su = tcx*(x flux) ; su = su + tcy*(y flux) ; su = su + (tzc1*(z flux in) - tzc2*(z flux out))
  a = F(0, 0, 0, -1) * (F(0, 0, 0, 0) + F(0, 0, 0, -1));
  b = F(0, 0, 0, 1) * (F(0, 0, 0, 0) + F(0, 0, 0, 1));
  s = tcx * (a - b);
  a = F(0, 0, -1, 0) * (F(1, 0, -1, 0) + F(1, 0, -1, 1));
  b = F(0, 0, 1, 0) * (F(1, 0, 0, 0) + F(1, 0, 0, 1));
  s = s + tcy * (a - b);
  a = (tzc1 * F(0, -1, 0, 0)) * (F(2, -1, 0, 0) + F(2, -1, 0, 1));
  b = (tzc2 * F(0, 1, 0, 0)) * (F(2, 0, 0, 0) + F(2, 0, 0, 1));
  su = s + (a - b);
  // sv: the same three terms in the same order (x, y, z)
  a = F(1, 0, 0, -1) * (F(0, 0, 0, -1) + F(0, 0, 1, -1));
  b = F(1, 0, 0, 1) * (F(0, 0, 0, 0) + F(0, 0, 1, 0));
  s = tcx * (a - b);
  a = F(1, 0, -1, 0) * (F(1, 0, 0, 0) + F(1, 0, -1, 0));
  b = F(1, 0, 1, 0) * (F(1, 0, 0, 0) + F(1, 0, 1, 0));
  s = s + tcy * (a - b);
  a = (tzc1 * F(1, -1, 0, 0)) * (F(2, -1, 0, 0) + F(2, -1, 1, 0));
  b = (tzc2 * F(1, 1, 0, 0)) * (F(2, 0, 0, 0) + F(2, 0, 1, 0));
  sv = s + (a - b);
  // sw: x, y, then the z term with tzd1 / tzd2
  a = F(2, 0, 0, -1) * (F(0, 0, 0, -1) + F(0, 1, 0, -1));
  b = F(2, 0, 0, 1) * (F(0, 0, 0, 0) + F(0, 1, 0, 0));
  s = tcx * (a - b);
  a = F(2, 0, -1, 0) * (F(1, 0, -1, 0) + F(1, 1, -1, 0));
  b = F(2, 0, 1, 0) * (F(1, 0, 0, 0) + F(1, 1, 0, 0));
  s = s + tcy * (a - b);
  a = (tzd1 * F(2, -1, 0, 0)) * (F(2, 0, 0, 0) + F(2, -1, 0, 0));
  b = (tzd2 * F(2, 1, 0, 0)) * (F(2, 0, 0, 0) + F(2, 1, 0, 0));
  sw = s + (a - b);
}

__device__ __forceinline__ double tz_at(const AdvParams& p, int q, int k) {
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(p.tz[q]) + (int64_t)k * p.tz_sm[q]);
}

// Unit u -> tile origin (first output k, j) and output planes [ia, ib).
__device__ __forceinline__ void adv_unit(const AdvParams& p, uint32_t u, int& k0, int& j0, int& ia, int& ib) {
  const uint32_t ntile = (uint32_t)(p.tiles_k * p.tiles_j);
  const uint32_t t = u % ntile, sgi = u / ntile;
  k0 = (int)(t % (uint32_t)p.tiles_k) * AD_OK;  // outputs k0 .. k0+AD_OK-1 (k = 0 is boundary)
  j0 = 1 + (int)(t / (uint32_t)p.tiles_k) * AD_OJ;
  ia = 1 + (int)sgi * p.seg;
  ib = min(ia + p.seg, p.nx - 1);
}

struct AdvCursor {
  uint32_t u;
  int ck, cj, ci, cend;
};

__device__ __forceinline__ void adv_cursor_unit(AdvCursor& c, const AdvParams& p) {
  int k0, j0, ia, ib;
  adv_unit(p, c.u, k0, j0, ia, ib);
  c.ck = k0 - 2;  // = 64 t - 2: 16-byte aligned box start
  c.cj = j0 - 1;
  c.ci = ia - 1;
  c.cend = ib + 1;
}

template <int AD_NS>
__device__ __forceinline__ void adv_issue(AdvCursor& c, const AdvParams& p, const CUtensorMap* mu, const CUtensorMap* mv,
                                          const CUtensorMap* mw, uint8_t* smem, uint64_t* full, uint32_t g) {
  if (c.u >= p.units) return;
  const int s = (int)(g % AD_NS);
  uint8_t* dst = smem + s * AD_SLOT;
  dev::mbar_arrive_expect_tx(&full[s], 3 * AD_BK * AD_BJ * 8);
  dev::tma_load_3d(dst, mu, &full[s], c.ck, c.cj, c.ci);
  dev::tma_load_3d(dst + AD_FIELD, mv, &full[s], c.ck, c.cj, c.ci);
  dev::tma_load_3d(dst + 2 * AD_FIELD, mw, &full[s], c.ck, c.cj, c.ci);
  if (++c.ci == c.cend) {
    c.u += gridDim.x;
    if (c.u < p.units) adv_cursor_unit(c, p);
  }
}

// Reads field f at (k + E + dk, j + dj, i + di) for the thread's pair (k, k+1), E = 0 or 1: the
// row segment is read as 16-byte pairs L = (k-2, k-1), C = (k, k+1), R = (k+2, k+3) (LDS.128;
// identical loads are shared between the calls).
template <int E>
struct SmemPair {
  const double* pl[3];  // plane i-1, i, i+1 (field 0 base)
  int row0;             // element offset of the thread's row (j) and pair L in a field box
  __device__ __forceinline__ double operator()(int f, int dk, int dj, int di) const {
    const double2* seg = reinterpret_cast<const double2*>(pl[di + 1] + f * (AD_FIELD / 8) + row0 + dj * AD_BK);
    const int m = E + dk + 2;  // element index from the L pair; pair m / 2, component m % 2
    return (m & 1) ? seg[m >> 1].y : seg[m >> 1].x;
  }
};

// AD_NS ring slots: NS-2 planes in flight ahead of the step
template <int AD_NS>
__global__ void __launch_bounds__(AD_THREADS, 1) adv_tma_kernel(const __grid_constant__ CUtensorMap mu,
                                                                const __grid_constant__ CUtensorMap mv,
                                                                const __grid_constant__ CUtensorMap mw,
                                                                const __grid_constant__ AdvParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const uint32_t soff = (uint32_t)(smem - smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + AD_NS * AD_SLOT);
  AdvCursor cur;
  cur.u = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < AD_NS; ++s) dev::mbar_init(&full[s], 1);
    dev::fence_barrier_init();
    dev::prefetch_tma(&mu);
    dev::prefetch_tma(&mv);
    dev::prefetch_tma(&mw);
    if (cur.u < p.units) adv_cursor_unit(cur, p);
    for (uint32_t g = 0; g < AD_NS; ++g) adv_issue<AD_NS>(cur, p, &mu, &mv, &mw, smem, full, g);
  }
  __syncthreads();
  const double* base = reinterpret_cast<const double*>(smem_raw + soff);
  const int lane = threadIdx.x % AD_PAIRS, jr = threadIdx.x / AD_PAIRS;  // pair (2 lane, 2 lane + 1), row jr
  uint32_t g = 0;  // planes consumed so far
  for (uint32_t u = blockIdx.x; u < p.units; u += gridDim.x) {
    int k0, j0, ia, ib;
    adv_unit(p, u, k0, j0, ia, ib);
    const int k = k0 + AD_PP * lane;
    const int j = j0 + jr;
    const bool jin = j <= p.ny - 2;
    double cz[AD_PP][4];
    bool st[AD_PP];
    bool all_st = jin;
#pragma unroll
    for (int e = 0; e < AD_PP; ++e) {
      const bool in = k + e >= 1 && k + e <= p.nz - 2;
      const int kc = in ? k + e : 1;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) cz[e][q4] = tz_at(p, q4, kc);
      st[e] = jin && in;
      all_st = all_st && in;
    }
    const int np = ib - ia + 2;  // planes ia-1 .. ib
    for (int q = 0; q < np; ++q) {
      const uint32_t gq = g + q;
      dev::mbar_wait(&full[gq % AD_NS], (gq / AD_NS) & 1);
      if (q >= 2) {  // output plane i from planes i-1, i, i+1 (steps q-2, q-1, q)
        const int i = ia + q - 2;
        const double* pl0 = base + ((gq - 2) % AD_NS) * (AD_SLOT / 8);
        const double* pl1 = base + ((gq - 1) % AD_NS) * (AD_SLOT / 8);
        const double* pl2 = base + (gq % AD_NS) * (AD_SLOT / 8);
        const int row0 = (jr + 1) * AD_BK + AD_PP * lane;
        double su[AD_PP], sv[AD_PP], sw[AD_PP];
        auto point = [&](auto E_) {
          constexpr int E = decltype(E_)::value;
          SmemPair<E> F;
          F.pl[0] = pl0;
          F.pl[1] = pl1;
          F.pl[2] = pl2;
          F.row0 = row0;
          adv_point(F, cz[E][0], cz[E][1], cz[E][2], cz[E][3], p.tcx, p.tcy, su[E], sv[E], sw[E]);
        };
        point(std::integral_constant<int, 0>{});
        point(std::integral_constant<int, 1>{});
        if constexpr (AD_PP == 4) {
          point(std::integral_constant<int, 2>{});
          point(std::integral_constant<int, 3>{});
        }
        const int64_t ok = (int64_t)k, oj = (int64_t)j, oi = (int64_t)i;
        char* a0 = p.su.base + ok * p.su.sm1 + oj * p.su.sm2 + oi * p.su.sm3;
        char* a1 = p.sv.base + ok * p.sv.sm1 + oj * p.sv.sm2 + oi * p.sv.sm3;
        char* a2 = p.sw.base + ok * p.sw.sm1 + oj * p.sw.sm2 + oi * p.sw.sm3;
        if (p.vec_out && all_st) {
#pragma unroll
          for (int e = 0; e < AD_PP; e += 2) {
            *reinterpret_cast<double2*>(a0 + e * 8) = make_double2(su[e], su[e + 1]);
            *reinterpret_cast<double2*>(a1 + e * 8) = make_double2(sv[e], sv[e + 1]);
            *reinterpret_cast<double2*>(a2 + e * 8) = make_double2(sw[e], sw[e + 1]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < AD_PP; ++e)
            if (st[e]) {
              *reinterpret_cast<double*>(a0 + e * p.su.sm1) = su[e];
              *reinterpret_cast<double*>(a1 + e * p.sv.sm1) = sv[e];
              *reinterpret_cast<double*>(a2 + e * p.sw.sm1) = sw[e];
            }
        }
      }
      __syncthreads();
      // plane gq-2 is not read after this step (the next step reads gq-1 .. gq+1 or, at a new
      // unit, nothing before its third plane): refill its slot with plane gq-2+NS
      if (threadIdx.x == 0 && gq >= 2) {
        dev::fence_proxy_async();
        adv_issue<AD_NS>(cur, p, &mu, &mv, &mw, smem, full, gq - 2 + AD_NS);
      }
    }
    g += np;
  }
}

struct GlobalNbr {
  const char* f[3];
  int64_t sm[3][3];
  int64_t k, j, i;
  __device__ __forceinline__ double operator()(int q, int dk, int dj, int di) const {
    return *reinterpret_cast<const double*>(f[q] + (k + dk) * sm[q][0] + (j + dj) * sm[q][1] + (i + di) * sm[q][2]);
  }
};

struct AdvGenParams {
  AdvParams p;
  const char* in[3];
  int64_t in_sm[3][3];
};

__global__ void __launch_bounds__(256) adv_generic_kernel(const __grid_constant__ AdvGenParams G) {
  const AdvParams& p = G.p;
  const int64_t mk = p.nz - 2, mj = p.ny - 2, mi = p.nx - 2;
  const int64_t total = mk * mj * mi;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    GlobalNbr F;
    for (int q = 0; q < 3; ++q) {
      F.f[q] = G.in[q];
      for (int d = 0; d < 3; ++d) F.sm[q][d] = G.in_sm[q][d];
    }
    F.k = 1 + t % mk;
    F.j = 1 + (t / mk) % mj;
    F.i = 1 + t / (mk * mj);
    double su, sv, sw;
    const int k = (int)F.k;
    adv_point(F, tz_at(p, 0, k), tz_at(p, 1, k), tz_at(p, 2, k), tz_at(p, 3, k), p.tcx, p.tcy, su, sv, sw);
    *reinterpret_cast<double*>(p.su.base + F.k * p.su.sm1 + F.j * p.su.sm2 + F.i * p.su.sm3) = su;
    *reinterpret_cast<double*>(p.sv.base + F.k * p.sv.sm1 + F.j * p.sv.sm2 + F.i * p.sv.sm3) = sv;
    *reinterpret_cast<double*>(p.sw.base + F.k * p.sw.sm1 + F.j * p.sw.sm2 + F.i * p.sw.sm3) = sw;
  }
}

template <int NS>
ftn_status_t launch_adv(unsigned grid, const CUtensorMap& mu, const CUtensorMap& mv, const CUtensorMap& mw,
                        const AdvParams& p, cudaStream_t s) {
  static std::atomic<bool> attr[64] = {};  // per device: dynamic smem attribute set (idempotent)
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    FTN_CUDA(cudaFuncSetAttribute(adv_tma_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, ad_smem<NS>()));
    attr[dev & 63] = true;
  }
  adv_tma_kernel<NS><<<grid, AD_THREADS, ad_smem<NS>(), s>>>(mu, mv, mw, p);
  return FTN_OK;
}

AdvOut out_of(const ftn_desc_t* d) {
  AdvOut o;
  o.base = (char*)d->base_addr;
  o.sm1 = d->dim[0].sm;
  o.sm2 = d->dim[1].sm;
  o.sm3 = d->dim[2].sm;
  return o;
}

ftn_status_t make_map(CUtensorMap* m, const ftn_desc_t* d) {
  uint64_t dims[3] = {(uint64_t)d->dim[0].extent, (uint64_t)d->dim[1].extent, (uint64_t)d->dim[2].extent};
  uint64_t strides[2] = {(uint64_t)d->dim[1].sm, (uint64_t)d->dim[2].sm};
  uint32_t box[3] = {AD_BK, AD_BJ, 1};
  return encode_tma(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d->base_addr, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
}

}  // namespace
}  // namespace ftn

using namespace ftn;

extern "C" ftn_status_t ftn_pw_advection(const ftn_desc_t* su, const ftn_desc_t* sv, const ftn_desc_t* sw,
                                         const ftn_desc_t* u, const ftn_desc_t* v, const ftn_desc_t* w,
                                         const ftn_desc_t* tzc1, const ftn_desc_t* tzc2, const ftn_desc_t* tzd1,
                                         const ftn_desc_t* tzd2, double tcx, double tcy, ftn_stream_t stream) {
  NvtxRange nvtx_("ftn_pw_advection");
  const ftn_desc_t* f6[6] = {su, sv, sw, u, v, w};
  const char* names[6] = {"ftn_pw_advection(su)", "ftn_pw_advection(sv)", "ftn_pw_advection(sw)",
                          "ftn_pw_advection(u)", "ftn_pw_advection(v)", "ftn_pw_advection(w)"};
  for (int q = 0; q < 6; ++q) {
    FTN_CHECK(check_desc(f6[q], names[q], 3, 3));
    if (f6[q]->type != FTN_F64) return fail(FTN_ERR_TYPE, "ftn_pw_advection: fields must be real(8)");
    if (!same_shape(f6[q], u)) return fail(FTN_ERR_SHAPE, "ftn_pw_advection: fields are not conformable");
  }
  const ftn_desc_t* z4[4] = {tzc1, tzc2, tzd1, tzd2};
  for (int q = 0; q < 4; ++q) {
    FTN_CHECK(check_desc(z4[q], "ftn_pw_advection(tz)", 1, 1));
    if (z4[q]->type != FTN_F64) return fail(FTN_ERR_TYPE, "ftn_pw_advection: coefficients must be real(8)");
    if (z4[q]->dim[0].extent != u->dim[0].extent)
      return fail(FTN_ERR_SHAPE, "ftn_pw_advection: coefficient vectors must have extent size(u, 1)");
  }
  for (int a = 0; a < 3; ++a)
    for (int b = 3; b < 6; ++b)
      if (desc_overlap(f6[a], f6[b])) return fail(FTN_ERR_SHAPE, "ftn_pw_advection: an output overlaps an input");
  for (int a = 0; a < 3; ++a)
    for (int b = a + 1; b < 3; ++b)
      if (desc_overlap(f6[a], f6[b])) return fail(FTN_ERR_SHAPE, "ftn_pw_advection: outputs overlap");
  FTN_CHECK(require_sm100());
  cudaStream_t s = (cudaStream_t)stream;
  AdvParams p;
  p.su = out_of(su);
  p.sv = out_of(sv);
  p.sw = out_of(sw);
  for (int q = 0; q < 4; ++q) {
    p.tz[q] = (const double*)z4[q]->base_addr;
    p.tz_sm[q] = z4[q]->dim[0].sm;
  }
  const int64_t nz = u->dim[0].extent, ny = u->dim[1].extent, nx = u->dim[2].extent;
  if (nz < 3 || ny < 3 || nx < 3) return FTN_OK;  // no interior
  if (nz >= (1ll << 31) || ny >= (1ll << 31) || nx >= (1ll << 31))
    return fail(FTN_ERR_UNSUPPORTED, "ftn_pw_advection: extents must be < 2^31");
  p.nz = (int32_t)nz;
  p.ny = (int32_t)ny;
  p.nx = (int32_t)nx;
  p.tcx = tcx;
  p.tcy = tcy;
  const bool tma = stencil_tma_able(u) && stencil_tma_able(v) && stencil_tma_able(w);
  if (tma) {
    CUtensorMap mu, mv, mw;
    FTN_CHECK(make_map(&mu, u));
    FTN_CHECK(make_map(&mv, v));
    FTN_CHECK(make_map(&mw, w));
    p.tiles_k = (int32_t)((nz - 1 + AD_OK - 1) / AD_OK);  // outputs k in [1, nz-2] within [0, AD_OK tiles_k)
    p.vec_out = 1;
    for (const ftn_desc_t* o : {su, sv, sw})
      if (o->dim[0].sm != 8 || ((uintptr_t)o->base_addr % 16) || (o->dim[1].sm % 16) || (o->dim[2].sm % 16))
        p.vec_out = 0;
    p.tiles_j = (int32_t)((ny - 2 + AD_OJ - 1) / AD_OJ);
    const int64_t grid0 = num_sms();
    int64_t seg = 0, units = 0;
    plan_units_halo((int64_t)p.tiles_k * p.tiles_j, nx - 2, grid0, 2, &seg, &units);
    // units spanning at most ~4 GiB of i-planes (three fields), as for jacobi3d_tb2
    const int64_t plane_bytes = 3 * std::max<int64_t>(u->dim[2].sm, 1);
    static const int64_t env_maxseg = getenv("FTN_AD_MAXSEG") ? atoll(getenv("FTN_AD_MAXSEG")) : -1;
    const int64_t maxseg = env_maxseg > 0 ? env_maxseg : std::max<int64_t>(16, (int64_t(4) << 30) / plane_bytes);
    if (seg > maxseg) {
      seg = maxseg;
      units = (int64_t)p.tiles_k * p.tiles_j * ((nx - 2 + seg - 1) / seg);
    }
    if (units >= (1ll << 32)) return fail(FTN_ERR_UNSUPPORTED, "ftn_pw_advection: too many work units");
    p.seg = (int32_t)seg;
    p.units = (uint32_t)units;
    const int64_t grid = std::min<int64_t>(grid0, units);
    // measured at 2048x1024x1024 (Gcells/s): tile 64x16: NS 3: 56, 4: 94, 5: 94-97, 6: 86;
    // tile 128x8: NS 4: 100, 5: 110, 6: 96, 7: 95; tile 192x5: NS 5: 107, 6: 109
    static const int ns = getenv("FTN_AD_NS") ? atoi(getenv("FTN_AD_NS")) : 5;
    switch (ns) {
      case 3: FTN_CHECK(launch_adv<3>((unsigned)grid, mu, mv, mw, p, s)); break;
      case 5: FTN_CHECK(launch_adv<5>((unsigned)grid, mu, mv, mw, p, s)); break;
      case 6: FTN_CHECK(launch_adv<6>((unsigned)grid, mu, mv, mw, p, s)); break;
      case 7: FTN_CHECK(launch_adv<7>((unsigned)grid, mu, mv, mw, p, s)); break;
      default: FTN_CHECK(launch_adv<4>((unsigned)grid, mu, mv, mw, p, s)); break;
    }
    return after_launch("adv_tma_kernel");
  }
  AdvGenParams G;
  G.p = p;
  const ftn_desc_t* in3[3] = {u, v, w};
  for (int q = 0; q < 3; ++q) {
    G.in[q] = (const char*)in3[q]->base_addr;
    for (int d = 0; d < 3; ++d) G.in_sm[q][d] = in3[q]->dim[d].sm;
  }
  const int64_t total = (nz - 2) * (ny - 2) * (nx - 2);
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
  adv_generic_kernel<<<(unsigned)blocks, 256, 0, s>>>(G);
  return after_launch("adv_generic_kernel");
}
