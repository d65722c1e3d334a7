// tra-adv (R#28): the NEMO tracer-advection benchmark the paper
// runs ("six fields on a three dimensional grid of size 1024 by 512 by 512, running over
// 20 iterations"), its loop nests as recalled in R#28 -- the same statements, in the same
// order, with the same Fortran evaluation order as oracle/ftn_oracle.c's orc_tra_adv_f64, so
// results are bit-identical (-fmad=false; SIGN = copysign, MIN / MAX / ABS exact).
//
// Fields are indexed (ji, jj, jk), ji contiguous.  One iteration is eight passes, each a
// kernel over its index range with one thread per ji (coalesced) and a block per (jj, jk) row:
//   K1  steps 1-2   zind (all points); zwx, zwy (ji < jpi-1, jj < jpj-1, jk < jpk-1; 0 at jk = jpk-1)
//   K2  steps 3-4   slopes zslpx, zslpy (ji >= 1, jj >= 1, jk < jpk-1; 0 at jk = jpk-1): step 4
//                   at a point reads only step 3's value at that point, so the two fuse per point
//   K3  step 5      horizontal fluxes zwx, zwy (interior) -- reads no zwx / zwy
//   K4  step 6      md += -(flux divergence) (interior)
//   K5  step 7      vertical gradients zwx (all ji, jj; 0 at jk = 0 and jpk-1)
//   K6  steps 8-9   vertical slopes zslpx (all ji, jj, 1 <= jk < jpk-1; 0 at jk = 0)
//   K7  steps 10-11 vertical fluxes: zwx(:,:,0) = pwn md, zwx(jk+1) (interior) -- reads no zwx
//   K8  step 12     md = -(zwx - zwx(jk+1)) (interior)
// Each pass is HBM-bound; the temporaries live in the caller's workspace (5 packed arrays),
// zeroed at the start of the call (R#28).
#include "ftn_internal.cuh"

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
