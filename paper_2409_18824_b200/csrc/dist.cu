// Multi-GPU layer: one process per GPU, NCCL over
// NVLink 5 / NVSwitch.  The paper itself only threads with OpenMP;
// BASELINE's north star partitions the work where it shards naturally:
//   * reductions: each rank reduces its slab in order R, the p rank partials are
//     all-gathered and combined by the same balanced tree on every rank
//     (deterministic; equal to the 1-GPU result when slabs are equal power-of-two
//     multiples of the R chunk);
//   * Jacobi: last-dimension slabs with `halo` planes per side; per launch of the plan the
//     k owned planes next to each neighbour go out with grouped ncclSend/ncclRecv and the
//     slab advances k fused sweeps (k <= halo: deep halos, one exchange per k sweeps);
//   * MATMUL: column blocks of b and c, a replicated (ftn_bcast once).
#include "ftn_internal.cuh"

#include <algorithm>

#include <nccl.h>
#include <cstring>
#include <vector>

struct ftn_comm_s {
  ncclComm_t nccl;
  int nranks, rank, device;
  int overlap = 1;                 // 0 off, 1 when nranks > 1, 2 always (ftn_comm_set_overlap)
  cudaStream_t side = nullptr;     // interior sweeps while the halo exchange runs
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
};

namespace ftn {
size_t matmul_ws(const ftn_desc_t* a, const ftn_desc_t* b);
ftn_status_t matmul_local(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, void* ws, size_t ws_bytes,
                          cudaStream_t s);
ftn_status_t jacobi_check(const ftn_desc_t* u, const ftn_desc_t* unew);
ftn_status_t jacobi_prepare();
int jacobi_fuse_T();
bool stencil_tma_able(const ftn_desc_t* d);
ftn_status_t jacobi_slab_part(const ftn_desc_t* src, const ftn_desc_t* dst, int32_t sweeps, double coeff,
                              int32_t halo, int32_t first, int32_t last, int64_t out_lo, int64_t out_hi,
                              cudaStream_t s);

namespace {

ftn_status_t nccl_fail(ncclResult_t r, const char* what) {
  return fail(FTN_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
#define FTN_NCCL(expr)                                         \
  do {                                                         \
    ncclResult_t r__ = (expr);                                 \
    if (r__ != ncclSuccess) return nccl_fail(r__, #expr);      \
  } while (0)

ncclDataType_t nccl_type(int32_t t) {
  switch (t) {
    case FTN_I32: return ncclInt32;
    case FTN_I64: return ncclInt64;
    case FTN_F32: return ncclFloat32;
    default: return ncclFloat64;
  }
}

ftn_status_t global_reduce(int kind, ftn_comm_t comm, const ftn_desc_t* x, const ftn_desc_t* y, void* result,
                           void* ws, size_t ws_bytes, cudaStream_t s) {
  if (!comm) return fail(FTN_ERR_NULL, "global reduction: comm NULL");
  if (!result) return fail(FTN_ERR_NULL, "global reduction: result NULL");
  const size_t head = 8 * ((size_t)comm->nranks + 1);
  if (!ws || ws_bytes < head + reduce_ws_bytes(desc_size(x)) || ((uintptr_t)ws % 8))
    return fail(FTN_ERR_WORKSPACE, "global reduction: workspace must hold reduce_workspace_size + 8*(nranks+1) bytes");
  if (x->type == FTN_I32)
    return fail(FTN_ERR_UNSUPPORTED, "global reductions of integer(4) are not offered; use integer(8)");
  char* w = (char*)ws;
  void* local = w;
  void* gathered = w + 8;
  FTN_CHECK(reduce_local(kind, x, y, local, w + head, ws_bytes - head, s));
  FTN_NCCL(ncclAllGather(local, gathered, 1, nccl_type(x->type), comm->nccl, s));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return tree_combine_launch(kind, x->type, gathered, comm->nranks, result, s);
}

bool plane_contiguous(const ftn_desc_t* d) {
  int64_t expect = d->elem_len;
  for (int k = 0; k < d->rank - 1; ++k) {
    if (d->dim[k].sm != expect) return false;
    expect *= d->dim[k].extent;
  }
  return true;
}

}  // namespace
}  // namespace ftn

using namespace ftn;

extern "C" {

ftn_status_t ftn_comm_unique_id(uint8_t id[FTN_COMM_ID_BYTES]) {
  static_assert(sizeof(ncclUniqueId) == FTN_COMM_ID_BYTES, "ncclUniqueId size");
  if (!id) return fail(FTN_ERR_NULL, "ftn_comm_unique_id: id NULL");
  ncclUniqueId u;
  FTN_NCCL(ncclGetUniqueId(&u));
  memcpy(id, &u, sizeof(u));
  return FTN_OK;
}

ftn_status_t ftn_comm_init(ftn_comm_t* comm, int32_t nranks, int32_t rank, const uint8_t id[FTN_COMM_ID_BYTES],
                           int32_t device) {
  if (!comm || !id) return fail(FTN_ERR_NULL, "ftn_comm_init: NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FTN_ERR_SHAPE, "ftn_comm_init: bad rank / nranks");
  FTN_CUDA(cudaSetDevice(device));
  FTN_CHECK(require_sm100());
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ftn_comm_s* c = new ftn_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming) != cudaSuccess) {
    ncclCommDestroy(c->nccl);
    delete c;
    return fail(FTN_ERR_CUDA, "ftn_comm_init: stream / event creation failed");
  }
  *comm = c;
  return FTN_OK;
}

ftn_status_t ftn_comm_set_overlap(ftn_comm_t comm, int32_t mode) {
  if (!comm) return fail(FTN_ERR_NULL, "ftn_comm_set_overlap: comm NULL");
  if (mode < 0 || mode > 2) return fail(FTN_ERR_SHAPE, "ftn_comm_set_overlap: mode must be 0, 1 or 2");
  comm->overlap = mode;
  return FTN_OK;
}

ftn_status_t ftn_comm_destroy(ftn_comm_t comm) {
  if (!comm) return FTN_OK;
  if (comm->ev_in) cudaEventDestroy(comm->ev_in);
  if (comm->ev_out) cudaEventDestroy(comm->ev_out);
  if (comm->side) cudaStreamDestroy(comm->side);
  ncclResult_t r = ncclCommDestroy(comm->nccl);
  delete comm;
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return FTN_OK;
}

ftn_status_t ftn_sum_global(ftn_comm_t comm, const ftn_desc_t* x_local, void* result_dev, void* ws, size_t ws_bytes,
                            ftn_stream_t stream) {
  FTN_CHECK(check_desc(x_local, "ftn_sum_global(x)", 1, FTN_MAX_RANK));
  FTN_CHECK(require_sm100());
  return global_reduce(RK_SUM, comm, x_local, nullptr, result_dev, ws, ws_bytes, (cudaStream_t)stream);
}
ftn_status_t ftn_maxval_global(ftn_comm_t comm, const ftn_desc_t* x_local, void* result_dev, void* ws,
                               size_t ws_bytes, ftn_stream_t stream) {
  FTN_CHECK(check_desc(x_local, "ftn_maxval_global(x)", 1, FTN_MAX_RANK));
  FTN_CHECK(require_sm100());
  return global_reduce(RK_MAX, comm, x_local, nullptr, result_dev, ws, ws_bytes, (cudaStream_t)stream);
}
ftn_status_t ftn_minval_global(ftn_comm_t comm, const ftn_desc_t* x_local, void* result_dev, void* ws,
                               size_t ws_bytes, ftn_stream_t stream) {
  FTN_CHECK(check_desc(x_local, "ftn_minval_global(x)", 1, FTN_MAX_RANK));
  FTN_CHECK(require_sm100());
  return global_reduce(RK_MIN, comm, x_local, nullptr, result_dev, ws, ws_bytes, (cudaStream_t)stream);
}
ftn_status_t ftn_dot_product_global(ftn_comm_t comm, const ftn_desc_t* x_local, const ftn_desc_t* y_local,
                                    void* result_dev, void* ws, size_t ws_bytes, ftn_stream_t stream) {
  FTN_CHECK(check_desc(x_local, "ftn_dot_product_global(x)", 1, 1));
  FTN_CHECK(check_desc(y_local, "ftn_dot_product_global(y)", 1, 1));
  if (x_local->type != FTN_F64 || y_local->type != FTN_F64) return fail(FTN_ERR_TYPE, "dot: real(8) only");
  if (x_local->dim[0].extent != y_local->dim[0].extent) return fail(FTN_ERR_SHAPE, "dot: sizes differ");
  FTN_CHECK(require_sm100());
  return global_reduce(RK_DOT, comm, x_local, y_local, result_dev, ws, ws_bytes, (cudaStream_t)stream);
}

ftn_status_t ftn_jacobi_dist(ftn_comm_t comm, const ftn_desc_t* u, const ftn_desc_t* unew, int64_t sweeps,
                             double coeff, int32_t halo, int32_t* result_in_unew, ftn_stream_t stream) {
  NvtxRange nvtx_("ftn_jacobi_dist");
  if (!comm) return fail(FTN_ERR_NULL, "ftn_jacobi_dist: comm NULL");
  FTN_CHECK(jacobi_check(u, unew));
  if (!plane_contiguous(u) || !plane_contiguous(unew))
    return fail(FTN_ERR_UNSUPPORTED, "ftn_jacobi_dist: last-dimension planes must be contiguous");
  if (sweeps < 0) return fail(FTN_ERR_SHAPE, "ftn_jacobi_dist: negative sweep count");
  const int r = u->rank;
  const int64_t nl = u->dim[r - 1].extent;
  if (halo < 1 || nl - 2 * (int64_t)halo < 1)
    return fail(FTN_ERR_SHAPE, "ftn_jacobi_dist: a slab needs >= 1 owned plane + halo planes on each side");
  FTN_CHECK(require_sm100());
  FTN_CHECK(jacobi_prepare());
  cudaStream_t s = (cudaStream_t)stream;
  // temporal blocking: up to T sweeps per exchange (rank 2: the fusion setting, rank 3: 2),
  // at most the halo depth
  int T = 1;
  if (stencil_tma_able(u) && stencil_tma_able(unew)) {
    T = r == 2 ? jacobi_fuse_T() : std::min(2, jacobi_fuse_T());
    if (T > halo) T = halo;
  }
  const int64_t nplan = ftn_jacobi_plan(sweeps, T, nullptr, 0);
  std::vector<int32_t> plan((size_t)nplan);
  ftn_jacobi_plan(sweeps, T, plan.data(), nplan);
  const size_t plane = (size_t)(desc_size(u) / nl);
  const int lower = comm->rank - 1, upper = comm->rank + 1;
  const int first = comm->rank == 0, last = comm->rank == comm->nranks - 1;
  const bool overlap = comm->overlap == 2 || (comm->overlap == 1 && comm->nranks > 1);
  const int64_t lo = halo, hi = nl - halo - 1;
  int64_t launches = 0;
  for (; launches < nplan; ++launches) {
    const int k = plan[(size_t)launches];
    const ftn_desc_t* src = (launches % 2 == 0) ? u : unew;
    const ftn_desc_t* dst = (launches % 2 == 0) ? unew : u;
    char* b = (char*)src->base_addr;
    const int64_t sm = src->dim[r - 1].sm;
    // Overlap: the owned planes whose k-sweep dependence cone stays inside the owned planes,
    // [lo + k, hi - k], are advanced on the side stream while the halos travel; the k planes
    // next to each halo follow on the caller's stream after the exchange.
    const bool split = overlap && hi - lo + 1 >= 4 * (int64_t)k;
    if (split) {
      NvtxRange r_("jacobi_dist interior (side stream)");
      FTN_CUDA(cudaEventRecord(comm->ev_in, s));
      FTN_CUDA(cudaStreamWaitEvent(comm->side, comm->ev_in, 0));
      FTN_CHECK(jacobi_slab_part(src, dst, k, coeff, halo, first, last, lo + k, hi - k, comm->side));
      FTN_CUDA(cudaEventRecord(comm->ev_out, comm->side));
    }
    if (comm->nranks > 1) {
      NvtxRange r_("jacobi_dist halo exchange");
      // the k owned planes next to each neighbour -> its k halo planes next to its owned planes
      FTN_NCCL(ncclGroupStart());
      if (lower >= 0) {
        FTN_NCCL(ncclSend(b + halo * sm, plane * k, ncclFloat64, lower, comm->nccl, s));
        FTN_NCCL(ncclRecv(b + (halo - k) * sm, plane * k, ncclFloat64, lower, comm->nccl, s));
      }
      if (upper < comm->nranks) {
        FTN_NCCL(ncclSend(b + (nl - halo - k) * sm, plane * k, ncclFloat64, upper, comm->nccl, s));
        FTN_NCCL(ncclRecv(b + (nl - halo) * sm, plane * k, ncclFloat64, upper, comm->nccl, s));
      }
      FTN_NCCL(ncclGroupEnd());
      g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    if (split) {
      NvtxRange r_("jacobi_dist halo-adjacent planes");
      FTN_CHECK(jacobi_slab_part(src, dst, k, coeff, halo, first, last, lo, lo + k - 1, s));
      FTN_CHECK(jacobi_slab_part(src, dst, k, coeff, halo, first, last, hi - k + 1, hi, s));
      FTN_CUDA(cudaStreamWaitEvent(s, comm->ev_out, 0));
    } else {
      FTN_CHECK(ftn_jacobi_slab(src, dst, k, coeff, halo, first, last, stream));
    }
  }
  if (result_in_unew) *result_in_unew = (int32_t)(launches % 2);
  return FTN_OK;
}

ftn_status_t ftn_matmul_colsharded(ftn_comm_t comm, const ftn_desc_t* c_local, const ftn_desc_t* a_full,
                                   const ftn_desc_t* b_local, void* ws, size_t ws_bytes, ftn_stream_t stream) {
  if (!comm) return fail(FTN_ERR_NULL, "ftn_matmul_colsharded: comm NULL");
  size_t need = 0;
  FTN_CHECK(ftn_matmul_workspace_size(c_local, a_full, b_local, &need));
  FTN_CHECK(require_sm100());
  return matmul_local(c_local, a_full, b_local, ws, ws_bytes, (cudaStream_t)stream);
}

ftn_status_t ftn_bcast(ftn_comm_t comm, const ftn_desc_t* x, int32_t root, ftn_stream_t stream) {
  if (!comm) return fail(FTN_ERR_NULL, "ftn_bcast: comm NULL");
  FTN_CHECK(check_desc(x, "ftn_bcast(x)", 1, FTN_MAX_RANK));
  if (!desc_contiguous(x)) return fail(FTN_ERR_UNSUPPORTED, "ftn_bcast: array must be contiguous");
  if (root < 0 || root >= comm->nranks) return fail(FTN_ERR_SHAPE, "ftn_bcast: bad root");
  FTN_NCCL(ncclBroadcast(x->base_addr, x->base_addr, (size_t)desc_size(x), nccl_type(x->type), root, comm->nccl,
                         (cudaStream_t)stream));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return FTN_OK;
}

}  // extern "C"
