// Descriptor / C-ABI layer (b): construction, sections,
// inquiry, validation, dimension collapsing, overlap tests, errors, TMA encoding.
//
// "a subtraction of the index from its starting index is undertaken";
//          here folded once into base_addr (base = element (lb_1, ..., lb_r)).
// slices are memref subviews: "the same underlying memory ... different
//          offsets, sizes and strides"; ftn_desc_section builds exactly that.
// negative DO steps; S:329 trip count max(0, (u-l+s) div s).
#include "ftn_internal.cuh"

#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>
#include <algorithm>

namespace ftn {

static thread_local std::string t_last_error;
std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { t_last_error = msg; }

ftn_status_t fail(ftn_status_t s, const std::string& msg) {
  t_last_error = msg;
  return s;
}

ftn_status_t cuda_fail(cudaError_t e, const char* what) {
  t_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return FTN_ERR_CUDA;
}

ftn_status_t after_launch(const char* what, uint64_t n) {
  g_launches.fetch_add(n, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, what);
  return FTN_OK;
}

namespace {
struct DevInfo {
  int checked = 0;
  int ok = 0;
  int sms = 0;
};
std::mutex g_dev_mu;
DevInfo g_dev[64];
}  // namespace

ftn_status_t require_sm100() {
  int d = 0;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (d < 0 || d >= 64) return fail(FTN_ERR_DEVICE, "device index out of range");
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DevInfo& info = g_dev[d];
  if (!info.checked) {
    int major = 0, minor = 0, sms = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, d);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    info.ok = (major == 10 && minor == 0);
    info.sms = sms;
    info.checked = 1;
  }
  if (!info.ok) return fail(FTN_ERR_DEVICE, "libftn is built for sm_100a (B200); current device is not sm_100");
  return FTN_OK;
}

thread_local int t_sm_reserve = 0;  // ScopedSmReserve (dist.cu): SMs left free for concurrent kernels

int num_sms() {
  int d = 0;
  cudaGetDevice(&d);
  std::lock_guard<std::mutex> lk(g_dev_mu);
  const int n = g_dev[d].sms > 0 ? g_dev[d].sms : 148;
  return n - t_sm_reserve > 1 ? n - t_sm_reserve : 1;
}

ScopedSmReserve::ScopedSmReserve(int n) : saved(t_sm_reserve) { t_sm_reserve = n; }
ScopedSmReserve::~ScopedSmReserve() { t_sm_reserve = saved; }

int64_t type_len(int32_t type) {
  switch (type) {
    case FTN_I32:
    case FTN_F32:
      return 4;
    case FTN_I64:
    case FTN_F64:
      return 8;
    default:
      return 0;
  }
}
bool type_ok(int32_t type) { return type_len(type) != 0; }

ftn_status_t check_desc(const ftn_desc_t* d, const char* name, int min_rank, int max_rank) {
  if (!d) return fail(FTN_ERR_NULL, std::string(name) + ": descriptor is NULL");
  if (d->rank < min_rank || d->rank > max_rank || d->rank > FTN_MAX_RANK)
    return fail(FTN_ERR_RANK, std::string(name) + ": rank " + std::to_string(d->rank) + " not accepted");
  if (!type_ok(d->type) || d->elem_len != type_len(d->type))
    return fail(FTN_ERR_TYPE, std::string(name) + ": bad type / elem_len");
  for (int k = 0; k < d->rank; ++k)
    if (d->dim[k].extent < 0) return fail(FTN_ERR_SHAPE, std::string(name) + ": negative extent");
  if (!d->base_addr && desc_size(d) > 0) return fail(FTN_ERR_NULL, std::string(name) + ": base_addr is NULL");
  return FTN_OK;
}

int64_t desc_size(const ftn_desc_t* d) {
  int64_t n = 1;
  for (int k = 0; k < d->rank; ++k) n *= d->dim[k].extent;
  return n;
}

bool same_shape(const ftn_desc_t* a, const ftn_desc_t* b) {
  if (a->rank != b->rank) return false;
  for (int k = 0; k < a->rank; ++k)
    if (a->dim[k].extent != b->dim[k].extent) return false;
  return true;
}

void desc_byte_range(const ftn_desc_t* d, uintptr_t* lo, uintptr_t* hi) {
  intptr_t l = 0, h = 0;
  for (int k = 0; k < d->rank; ++k) {
    intptr_t span = (intptr_t)(d->dim[k].extent - 1) * d->dim[k].sm;
    if (d->dim[k].extent == 0) span = 0;
    if (span < 0) l += span; else h += span;
  }
  *lo = (uintptr_t)d->base_addr + l;
  *hi = (uintptr_t)d->base_addr + h + d->elem_len;
}

static uint64_t gcd_u64(uint64_t x, uint64_t y) {
  while (y) {
    const uint64_t t = x % y;
    x = y;
    y = t;
  }
  return x;
}

// Conservative alias test (R#5): false only if a and b provably share no byte.  Beyond the
// bounding intervals: every element of a starts at base_a + (a multiple of g), every element
// of b at base_b + (a multiple of g), g = gcd of all strides of both with extent > 1; with
// elem_len <= g the elements occupy the residue intervals [ra, ra + len_a) and
// [rb, rb + len_b) modulo g, and disjoint residue intervals mean disjoint memory.
bool desc_overlap(const ftn_desc_t* a, const ftn_desc_t* b) {
  if (desc_size(a) == 0 || desc_size(b) == 0) return false;
  uintptr_t al, ah, bl, bh;
  desc_byte_range(a, &al, &ah);
  desc_byte_range(b, &bl, &bh);
  if (!(al < bh && bl < ah)) return false;
  uint64_t g = 0;
  for (const ftn_desc_t* d : {a, b})
    for (int k = 0; k < d->rank; ++k)
      if (d->dim[k].extent > 1) g = gcd_u64(g, (uint64_t)(d->dim[k].sm < 0 ? -d->dim[k].sm : d->dim[k].sm));
  const uint64_t la = (uint64_t)a->elem_len, lb = (uint64_t)b->elem_len;
  if (g == 0 || la > g || lb > g) return true;  // a single element each, or elements wider than g
  const uint64_t ra = (uint64_t)(uintptr_t)a->base_addr % g, rb = (uint64_t)(uintptr_t)b->base_addr % g;
  const uint64_t d = (rb + g - ra) % g;  // b's residue interval starts d bytes after a's
  return d < la || d + lb > g;           // [0, la) and [d, d + lb) intersect modulo g
}


bool desc_identical(const ftn_desc_t* a, const ftn_desc_t* b) {
  if (a->base_addr != b->base_addr || a->rank != b->rank || a->elem_len != b->elem_len) return false;
  for (int k = 0; k < a->rank; ++k)
    if (a->dim[k].extent != b->dim[k].extent || (a->dim[k].extent > 1 && a->dim[k].sm != b->dim[k].sm))
      return false;
  return true;
}

bool desc_contiguous(const ftn_desc_t* d) {
  int64_t expect = d->elem_len;
  for (int k = 0; k < d->rank; ++k) {
    if (d->dim[k].extent > 1 && d->dim[k].sm != expect) return false;
    expect *= d->dim[k].extent;
  }
  return true;
}

KDesc to_kdesc(const ftn_desc_t* d) {
  KDesc k;
  k.base = (char*)d->base_addr;
  for (int i = 0; i < 3; ++i) {
    k.ext[i] = i < d->rank ? d->dim[i].extent : 1;
    k.sm[i] = i < d->rank ? d->dim[i].sm : 0;
  }
  return k;
}

int collapse(const ftn_desc_t* const* arrays, int n, KDesc* out) {
  // arrays[0] gives the shape; rank-0 members are scalars (left as is)
  const ftn_desc_t* s = arrays[0];
  int64_t ext[3];
  int64_t sm[4][3];
  int r = 0;
  for (int k = 0; k < s->rank; ++k) {
    if (s->dim[k].extent == 1) continue;  // a unit dimension never contributes an offset
    ext[r] = s->dim[k].extent;
    for (int a = 0; a < n; ++a) sm[a][r] = arrays[a]->rank ? arrays[a]->dim[k].sm : 0;
    ++r;
  }
  if (r == 0) {
    ext[0] = 1;
    for (int a = 0; a < n; ++a) sm[a][0] = 0;
    r = 1;
  }
  // merge d and d+1 when contiguous in every non-scalar array
  int w = 0;
  for (int k = 1; k < r; ++k) {
    bool merge = true;
    for (int a = 0; a < n && merge; ++a)
      if (arrays[a]->rank && sm[a][k] != sm[a][w] * ext[w]) merge = false;
    if (merge) {
      ext[w] *= ext[k];
    } else {
      ++w;
      ext[w] = ext[k];
      for (int a = 0; a < n; ++a) sm[a][w] = sm[a][k];
    }
  }
  r = w + 1;
  for (int a = 0; a < n; ++a) {
    out[a].base = (char*)arrays[a]->base_addr;
    for (int k = 0; k < 3; ++k) {
      out[a].ext[k] = k < r ? ext[k] : 1;
      out[a].sm[k] = (k < r && arrays[a]->rank) ? sm[a][k] : 0;
    }
  }
  return r;
}

StreamTemp::~StreamTemp() {
  if (ptr) cudaFreeAsync(ptr, stream);
}

ftn_status_t StreamTemp::alloc(size_t bytes, cudaStream_t s) {
  stream = s;
  // Fortran-semantics temporaries (R#5: an overlapping assignment, TRANSPOSE or MATMUL result)
  // come from a memory pool owned by this library, one per device: the device's default pool
  // and the caller's allocator are left alone.  The pool keeps up to 256 MiB of freed blocks
  // for reuse (small temporaries of repeated calls cost no new mapping) and returns anything
  // above that to the driver at the next synchronisation.
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev & 63]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      FTN_CUDA(cudaMemPoolCreate(&pools[dev & 63], &props));
      uint64_t keep = uint64_t(256) << 20;
      FTN_CUDA(cudaMemPoolSetAttribute(pools[dev & 63], cudaMemPoolAttrReleaseThreshold, &keep));
    }
    pool = pools[dev & 63];
  }
  FTN_CUDA(cudaMallocFromPoolAsync(&ptr, bytes > 0 ? bytes : 16, pool, s));
  return FTN_OK;
}

ftn_status_t make_packed(ftn_desc_t* out, void* base, const ftn_desc_t* like) {
  int64_t lb[3] = {1, 1, 1}, ext[3] = {1, 1, 1};
  for (int k = 0; k < like->rank; ++k) ext[k] = like->dim[k].extent;
  return ftn_desc_contiguous(out, base, like->type, like->rank, lb, ext);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

ftn_status_t encode_tma(CUtensorMap* map, CUtensorMapDataType dt, int rank, void* base, const uint64_t* dims,
                        const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swizzle) {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) return fail(FTN_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, dt, (cuuint32_t)rank, base, (const cuuint64_t*)dims, (const cuuint64_t*)strides_bytes,
                  (const cuuint32_t*)box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FTN_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return FTN_OK;
}

}  // namespace ftn

using namespace ftn;

extern "C" {

ftn_status_t ftn_desc_may_overlap(const ftn_desc_t* a, const ftn_desc_t* b, int32_t* out) {
  FTN_CHECK(ftn::check_desc(a, "ftn_desc_may_overlap", 0, FTN_MAX_RANK));
  FTN_CHECK(ftn::check_desc(b, "ftn_desc_may_overlap", 0, FTN_MAX_RANK));
  if (!out) return ftn::fail(FTN_ERR_NULL, "ftn_desc_may_overlap: out NULL");
  *out = ftn::desc_overlap(a, b) ? 1 : 0;
  return FTN_OK;
}

ftn_status_t ftn_desc_contiguous(ftn_desc_t* out, void* base, int32_t type, int32_t rank,
                                 const int64_t* lower_bounds, const int64_t* extents) {
  if (!out) return fail(FTN_ERR_NULL, "ftn_desc_contiguous: out is NULL");
  if (rank < 0 || rank > FTN_MAX_RANK) return fail(FTN_ERR_RANK, "ftn_desc_contiguous: rank must be 0..3");
  if (!type_ok(type)) return fail(FTN_ERR_TYPE, "ftn_desc_contiguous: unknown type");
  if (rank > 0 && (!lower_bounds || !extents)) return fail(FTN_ERR_NULL, "ftn_desc_contiguous: bounds NULL");
  ftn_desc_t d;
  memset(&d, 0, sizeof(d));
  d.base_addr = base;
  d.elem_len = type_len(type);
  d.rank = rank;
  d.type = type;
  int64_t sm = d.elem_len;
  for (int k = 0; k < rank; ++k) {
    if (extents[k] < 0) return fail(FTN_ERR_SHAPE, "ftn_desc_contiguous: negative extent");
    d.dim[k].lower_bound = lower_bounds[k];
    d.dim[k].extent = extents[k];
    d.dim[k].sm = sm;
    sm *= extents[k];
  }
  *out = d;
  return FTN_OK;
}

ftn_status_t ftn_desc_section(ftn_desc_t* out, const ftn_desc_t* parent, const int64_t* lo, const int64_t* hi,
                              const int64_t* step) {
  if (!out || !lo || !hi || !step) return fail(FTN_ERR_NULL, "ftn_desc_section: NULL argument");
  FTN_CHECK(check_desc(parent, "ftn_desc_section(parent)", 1, FTN_MAX_RANK));
  ftn_desc_t r = *parent;
  char* base = (char*)parent->base_addr;
  for (int k = 0; k < parent->rank; ++k) {
    if (step[k] == 0) return fail(FTN_ERR_BOUNDS, "ftn_desc_section: zero step in dim " + std::to_string(k + 1));
    int64_t n = (hi[k] - lo[k] + step[k]) / step[k];
    if (n < 0) n = 0;
    const int64_t lb = parent->dim[k].lower_bound, ub = lb + parent->dim[k].extent - 1;
    if (n > 0) {
      const int64_t first = lo[k], last = lo[k] + (n - 1) * step[k];
      if (first < lb || first > ub || last < lb || last > ub)
        return fail(FTN_ERR_BOUNDS, "ftn_desc_section: dim " + std::to_string(k + 1) + " selects outside " +
                                        std::to_string(lb) + ":" + std::to_string(ub));
      base += (first - lb) * parent->dim[k].sm;
    }
    r.dim[k].lower_bound = 1;
    r.dim[k].extent = n;
    r.dim[k].sm = step[k] * parent->dim[k].sm;
  }
  r.base_addr = base;
  *out = r;
  return FTN_OK;
}

ftn_status_t ftn_lbound(const ftn_desc_t* x, int32_t dim, int64_t* out) {
  FTN_CHECK(check_desc(x, "ftn_lbound", 0, FTN_MAX_RANK));
  if (!out) return fail(FTN_ERR_NULL, "ftn_lbound: out NULL");
  if (dim < 1 || dim > x->rank) return fail(FTN_ERR_DIM, "ftn_lbound: DIM out of range");
  // F2018 16.9.109: LBOUND of a zero-extent dimension is 1
  *out = x->dim[dim - 1].extent == 0 ? 1 : x->dim[dim - 1].lower_bound;
  return FTN_OK;
}

ftn_status_t ftn_ubound(const ftn_desc_t* x, int32_t dim, int64_t* out) {
  FTN_CHECK(check_desc(x, "ftn_ubound", 0, FTN_MAX_RANK));
  if (!out) return fail(FTN_ERR_NULL, "ftn_ubound: out NULL");
  if (dim < 1 || dim > x->rank) return fail(FTN_ERR_DIM, "ftn_ubound: DIM out of range");
  *out = x->dim[dim - 1].extent == 0 ? 0 : x->dim[dim - 1].lower_bound + x->dim[dim - 1].extent - 1;
  return FTN_OK;
}

ftn_status_t ftn_size(const ftn_desc_t* x, int32_t dim, int64_t* out) {
  FTN_CHECK(check_desc(x, "ftn_size", 0, FTN_MAX_RANK));
  if (!out) return fail(FTN_ERR_NULL, "ftn_size: out NULL");
  if (dim == 0) {
    *out = desc_size(x);
    return FTN_OK;
  }
  if (dim < 1 || dim > x->rank) return fail(FTN_ERR_DIM, "ftn_size: DIM out of range");
  *out = x->dim[dim - 1].extent;
  return FTN_OK;
}

ftn_status_t ftn_shape(const ftn_desc_t* x, int64_t* out) {
  FTN_CHECK(check_desc(x, "ftn_shape", 0, FTN_MAX_RANK));
  if (!out && x->rank > 0) return fail(FTN_ERR_NULL, "ftn_shape: out NULL");
  for (int k = 0; k < x->rank; ++k) out[k] = x->dim[k].extent;
  return FTN_OK;
}

uint64_t ftn_launch_count(void) { return g_launches.load(); }

const char* ftn_status_string(ftn_status_t s) {
  switch (s) {
    case FTN_OK: return "FTN_OK";
    case FTN_ERR_NULL: return "FTN_ERR_NULL";
    case FTN_ERR_RANK: return "FTN_ERR_RANK";
    case FTN_ERR_TYPE: return "FTN_ERR_TYPE";
    case FTN_ERR_SHAPE: return "FTN_ERR_SHAPE";
    case FTN_ERR_BOUNDS: return "FTN_ERR_BOUNDS";
    case FTN_ERR_DIM: return "FTN_ERR_DIM";
    case FTN_ERR_ALIGN: return "FTN_ERR_ALIGN";
    case FTN_ERR_UNSUPPORTED: return "FTN_ERR_UNSUPPORTED";
    case FTN_ERR_WORKSPACE: return "FTN_ERR_WORKSPACE";
    case FTN_ERR_DEVICE: return "FTN_ERR_DEVICE";
    case FTN_ERR_CUDA: return "FTN_ERR_CUDA";
    case FTN_ERR_NCCL: return "FTN_ERR_NCCL";
  }
  return "FTN_ERR_?";
}

const char* ftn_last_error(void) { return t_last_error.c_str(); }

}  // extern "C"
