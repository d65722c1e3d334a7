// Multi-GPU layer: one process per GPU, NCCL over
// NVLink 5 / NVSwitch.  The paper itself only threads with OpenMP;
// BASELINE's north star partitions the work where it shards naturally:
//   * reductions: each rank reduces its slab in order R, the p rank partials are
//     all-gathered and combined by the same balanced tree on every rank
//     (deterministic; equal to the 1-GPU result when slabs are equal power-of-two
//     multiples of the R chunk);
//   * Jacobi: last-dimension slabs with `halo` planes per side; per launch of the plan the
//     k owned planes next to each neighbour go out (grouped send/recv) and the slab
//     advances k fused sweeps (k <= halo: deep halos, one exchange per k sweeps);
//   * MATMUL: column blocks of b and c, a replicated (ftn_bcast once).
//
// The exchange sits behind a small transport interface with two implementations:
//   * NcclTransport: ncclSend/ncclRecv in a group, ncclAllGather, ncclBroadcast;
//   * VirtualTransport: p ranks of ONE process (one host thread per rank, any devices,
//     typically all on one GPU) -- every message is one cudaMemcpyAsync on the receiver's
//     stream, ordered by CUDA events against the sender's stream, with the same blocking
//     semantics as NCCL's grouped send/recv (a send completes, in stream order, once the
//     receiver's copy has).  It runs the library's own distributed loops -- plans, deep
//     halos, buffer offsets, the interior/halo overlap on the side stream -- at p > 1 on a
//     single GPU (ftn_comm_init_virtual).
#include "ftn_internal.cuh"

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <vector>

#include <nccl.h>

namespace ftn {

// One message of a grouped exchange (bytes of contiguous device memory to / from `peer`).
struct P2POp {
  bool send;
  void* buf;
  size_t bytes;
  int peer;
};

struct Transport {
  virtual ~Transport() {}
  // All sends and receives of one exchange step; every rank posts the matching ops.
  virtual ftn_status_t group(const P2POp* ops, int n, cudaStream_t s) = 0;
  // recv[r * bytes .. (r+1) * bytes) = rank r's send (every rank).
  virtual ftn_status_t allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  // buf on every rank = buf on root.
  virtual ftn_status_t bcast(void* buf, size_t bytes, int root, cudaStream_t s) = 0;
};

namespace {

ftn_status_t nccl_fail(ncclResult_t r, const char* what) {
  return fail(FTN_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
#define FTN_NCCL(expr)                                         \
  do {                                                         \
    ncclResult_t r__ = (expr);                                 \
    if (r__ != ncclSuccess) return nccl_fail(r__, #expr);      \
  } while (0)

struct NcclTransport : Transport {
  ncclComm_t nccl = nullptr;
  ~NcclTransport() override {
    if (nccl) ncclCommDestroy(nccl);
  }
  ftn_status_t group(const P2POp* ops, int n, cudaStream_t s) override {
    FTN_NCCL(ncclGroupStart());
    for (int i = 0; i < n; ++i) {
      if (ops[i].send)
        FTN_NCCL(ncclSend(ops[i].buf, ops[i].bytes, ncclUint8, ops[i].peer, nccl, s));
      else
        FTN_NCCL(ncclRecv(ops[i].buf, ops[i].bytes, ncclUint8, ops[i].peer, nccl, s));
    }
    FTN_NCCL(ncclGroupEnd());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return FTN_OK;
  }
  ftn_status_t allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    FTN_NCCL(ncclAllGather(send, recv, bytes, ncclUint8, nccl, s));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return FTN_OK;
  }
  ftn_status_t bcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
    FTN_NCCL(ncclBroadcast(buf, buf, bytes, ncclUint8, root, nccl, s));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return FTN_OK;
  }
};

// ---------------------------------------------------------------- virtual ranks
// Channel a -> b of a virtual group: a queue of posted messages.  Per group the sender
// records `ready` on its stream once and posts its messages (buf, bytes, sequence number);
// the receiver waits for each post, makes its stream wait on `ready`, copies, records `done`
// on its stream and acknowledges; once every message of the group is acknowledged the
// sender's stream waits on `done` (recorded after the last copy).  Event reuse is safe:
// `ready` is re-recorded only in the sender's next group, after every receiver's wait on it
// was enqueued; `done` only for a message of the next group, after the sender's wait on it
// was enqueued.
struct VMsg {
  const void* buf;
  size_t bytes;
  uint64_t seq;
};

struct VChannel {
  cudaEvent_t ready = nullptr, done = nullptr;
  std::vector<VMsg> q;   // posted, not yet taken
  uint64_t acked = 0;    // highest acknowledged sequence number
};

struct VGroup {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<VChannel> ch;  // ch[a * n + b]: a -> b
  explicit VGroup(int n_) : n(n_), ch((size_t)n_ * n_) {}
  ~VGroup() {
    for (auto& c : ch) {
      if (c.ready) cudaEventDestroy(c.ready);
      if (c.done) cudaEventDestroy(c.done);
    }
  }
};

constexpr auto kVirtualTimeout = std::chrono::seconds(300);

struct VirtualTransport : Transport {
  std::shared_ptr<VGroup> g;
  int rank, device;
  std::vector<uint64_t> sent, recvd;  // per peer: messages sent to / received from it

  VirtualTransport(std::shared_ptr<VGroup> g_, int rank_, int device_)
      : g(std::move(g_)), rank(rank_), device(device_), sent((size_t)g->n, 0), recvd((size_t)g->n, 0) {}

  ftn_status_t wait_for(std::unique_lock<std::mutex>& lk, const char* what, int peer,
                        const std::function<bool()>& pred) {
    if (!g->cv.wait_for(lk, kVirtualTimeout, pred))
      return fail(FTN_ERR_NCCL, std::string("virtual transport: rank ") + std::to_string(rank) + " timed out waiting for " +
                                    what + " of rank " + std::to_string(peer));
    return FTN_OK;
  }

  ftn_status_t group(const P2POp* ops, int n, cudaStream_t s) override {
    for (int i = 0; i < n; ++i)
      if (ops[i].peer < 0 || ops[i].peer >= g->n || ops[i].peer == rank)
        return fail(FTN_ERR_NCCL, "virtual transport: bad peer");
    // 1. post every send (never blocks)
    std::vector<char> to(g->n, 0);
    for (int i = 0; i < n; ++i)
      if (ops[i].send && !to[(size_t)ops[i].peer]) {
        to[(size_t)ops[i].peer] = 1;
        FTN_CUDA(cudaEventRecord(g->ch[(size_t)rank * g->n + ops[i].peer].ready, s));
      }
    {
      std::lock_guard<std::mutex> lk(g->mu);
      for (int i = 0; i < n; ++i) {
        if (!ops[i].send) continue;
        const int b = ops[i].peer;
        g->ch[(size_t)rank * g->n + b].q.push_back({ops[i].buf, ops[i].bytes, ++sent[(size_t)b]});
      }
    }
    g->cv.notify_all();
    // 2. every receive, in posting order per peer: wait for the post, copy on this rank's
    //    stream, acknowledge
    for (int i = 0; i < n; ++i) {
      if (ops[i].send) continue;
      const int a = ops[i].peer;
      VChannel& c = g->ch[(size_t)a * g->n + rank];
      const uint64_t seq = ++recvd[(size_t)a];
      VMsg m{};
      {
        std::unique_lock<std::mutex> lk(g->mu);
        FTN_CHECK(wait_for(lk, "a send", a, [&] {
          for (const VMsg& x : c.q)
            if (x.seq == seq) return true;
          return false;
        }));
        for (size_t j = 0; j < c.q.size(); ++j)
          if (c.q[j].seq == seq) {
            m = c.q[j];
            c.q.erase(c.q.begin() + (long)j);
            break;
          }
      }
      if (m.bytes != ops[i].bytes)
        return fail(FTN_ERR_NCCL, "virtual transport: message size differs between sender and receiver");
      FTN_CUDA(cudaStreamWaitEvent(s, c.ready, 0));
      if (m.bytes) FTN_CUDA(cudaMemcpyAsync(ops[i].buf, m.buf, m.bytes, cudaMemcpyDefault, s));
      FTN_CUDA(cudaEventRecord(c.done, s));
      {
        std::lock_guard<std::mutex> lk(g->mu);
        c.acked = seq;
      }
      g->cv.notify_all();
    }
    // 3. the sends complete (in stream order) when their receivers' copies have
    for (int b = 0; b < g->n; ++b) {
      if (!to[(size_t)b]) continue;
      VChannel& c = g->ch[(size_t)rank * g->n + b];
      const uint64_t seq = sent[(size_t)b];
      {
        std::unique_lock<std::mutex> lk(g->mu);
        FTN_CHECK(wait_for(lk, "the acknowledgement", b, [&] { return c.acked >= seq; }));
      }
      FTN_CUDA(cudaStreamWaitEvent(s, c.done, 0));
    }
    return FTN_OK;
  }

  ftn_status_t allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    std::vector<P2POp> ops;
    for (int r = 0; r < g->n; ++r) {
      if (r == rank) continue;
      ops.push_back({true, const_cast<void*>(send), bytes, r});
      ops.push_back({false, (char*)recv + (size_t)r * bytes, bytes, r});
    }
    if (bytes) FTN_CUDA(cudaMemcpyAsync((char*)recv + (size_t)rank * bytes, send, bytes, cudaMemcpyDefault, s));
    return group(ops.data(), (int)ops.size(), s);
  }

  ftn_status_t bcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
    std::vector<P2POp> ops;
    if (rank == root) {
      for (int r = 0; r < g->n; ++r)
        if (r != root) ops.push_back({true, buf, bytes, r});
    } else {
      ops.push_back({false, buf, bytes, root});
    }
    return group(ops.data(), (int)ops.size(), s);
  }
};

}  // namespace
}  // namespace ftn

struct ftn_comm_s {
  std::unique_ptr<ftn::Transport> tr;
  int nranks, rank, device;
  bool is_virtual = false;
  int overlap = 1;                 // 0 off, 1 when nranks > 1, 2 always (ftn_comm_set_overlap)
  int sm_reserve = 8;              // SMs left free by the interior sweeps while the exchange runs
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
int jacobi_fuse_for(const ftn_desc_t* u, const ftn_desc_t* unew);
bool stencil_tma_able(const ftn_desc_t* d);
ftn_status_t jacobi_slab_part(const ftn_desc_t* src, const ftn_desc_t* dst, int32_t sweeps, double coeff,
                              int32_t halo, int32_t first, int32_t last, int64_t out_lo, int64_t out_hi,
                              cudaStream_t s, double* res);

namespace {

ftn_status_t comm_streams(ftn_comm_s* c) {
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming) != cudaSuccess)
    return fail(FTN_ERR_CUDA, "ftn_comm_init: stream / event creation failed");
  return FTN_OK;
}

void comm_free(ftn_comm_s* c) {
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_out) cudaEventDestroy(c->ev_out);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
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
  FTN_CHECK(comm->tr->allgather(local, gathered, 8, s));
  return tree_combine_launch(kind, x->type, gathered, comm->nranks, result, s);
}

// Each last-dimension plane is one packed block (dims 1..r-1 packed column-major).
bool plane_contiguous(const ftn_desc_t* d) {
  int64_t expect = d->elem_len;
  for (int k = 0; k < d->rank - 1; ++k) {
    if (d->dim[k].sm != expect) return false;
    expect *= d->dim[k].extent;
  }
  return d->dim[d->rank - 1].sm > 0;
}

// The sends / receives that move the k planes [from, from + k) of `a` to / from `peer`: one
// message for k adjacent planes, else one per plane (a padded leading dimension leaves gaps
// between the planes of a 2-D slab).
void plane_ops(std::vector<P2POp>& ops, bool send, const ftn_desc_t* a, int64_t from, int k, int peer) {
  const int r = a->rank;
  const int64_t sm = a->dim[r - 1].sm;
  const size_t plane = (size_t)(desc_size(a) / a->dim[r - 1].extent) * (size_t)a->elem_len;
  char* b = (char*)a->base_addr;
  if ((size_t)sm == plane) {
    ops.push_back({send, b + from * sm, plane * (size_t)k, peer});
  } else {
    for (int q = 0; q < k; ++q) ops.push_back({send, b + (from + q) * sm, plane, peer});
  }
}

// Exchange of the k owned planes next to each neighbour into its k halo planes next to its
// owned planes (array `a`, local planes [halo, nl - halo) owned).
ftn_status_t halo_exchange(ftn_comm_t comm, const ftn_desc_t* a, int halo, int k, cudaStream_t s) {
  if (comm->nranks == 1) return FTN_OK;
  const int r = a->rank;
  const int64_t nl = a->dim[r - 1].extent;
  std::vector<P2POp> ops;
  if (comm->rank > 0) {
    plane_ops(ops, true, a, halo, k, comm->rank - 1);
    plane_ops(ops, false, a, halo - k, k, comm->rank - 1);
  }
  if (comm->rank < comm->nranks - 1) {
    plane_ops(ops, true, a, nl - halo - k, k, comm->rank + 1);
    plane_ops(ops, false, a, nl - halo, k, comm->rank + 1);
  }
  NvtxRange r_("jacobi_dist halo exchange");
  return comm->tr->group(ops.data(), (int)ops.size(), s);
}

ftn_status_t dist_check(ftn_comm_t comm, const ftn_desc_t* u, const ftn_desc_t* unew, int32_t halo, const char* who) {
  if (!comm) return fail(FTN_ERR_NULL, std::string(who) + ": comm NULL");
  FTN_CHECK(jacobi_check(u, unew));
  if (!plane_contiguous(u) || !plane_contiguous(unew))
    return fail(FTN_ERR_UNSUPPORTED, std::string(who) + ": each last-dimension plane must be packed");
  const int r = u->rank;
  const int64_t nl = u->dim[r - 1].extent;
  if (halo < 1 || nl - 2 * (int64_t)halo < 1)
    return fail(FTN_ERR_SHAPE, std::string(who) + ": a slab needs >= 1 owned plane + halo planes on each side");
  return FTN_OK;
}

// Sweeps per exchange: the local fusion factor for the slab (as ftn_jacobi), at most the
// halo depth.
int dist_T(const ftn_desc_t* u, const ftn_desc_t* unew, int32_t halo) {
  int T = stencil_tma_able(u) && stencil_tma_able(unew) ? jacobi_fuse_for(u, unew) : 1;
  return T > halo ? halo : T;
}

// The launches `plan` of the distributed DO nest starting from the array `*cur` (0: u holds
// the newest iterate), each preceded by the exchange of its k planes; flips *cur per launch.
// res_last != nullptr: the last launch also folds MAXVAL(ABS(last two iterates)) over the
// owned interior into that fmax slot (rank-2 TMA-able slabs).
ftn_status_t dist_run(ftn_comm_t comm, const ftn_desc_t* u, const ftn_desc_t* unew, const std::vector<int32_t>& plan,
                      double coeff, int32_t halo, int* cur, cudaStream_t s, double* res_last = nullptr) {
  const int r = u->rank;
  const int64_t nl = u->dim[r - 1].extent;
  const int first = comm->rank == 0, last = comm->rank == comm->nranks - 1;
  const bool overlap = comm->overlap == 2 || (comm->overlap == 1 && comm->nranks > 1);
  const int64_t lo = halo, hi = nl - halo - 1;
  for (size_t q = 0; q < plan.size(); ++q) {
    const int32_t k = plan[q];
    double* res = q + 1 == plan.size() ? res_last : nullptr;
    const ftn_desc_t* src = *cur ? unew : u;
    const ftn_desc_t* dst = *cur ? u : unew;
    // Overlap: the owned planes whose k-sweep dependence cone stays inside the owned planes,
    // [lo + k, hi - k], are advanced on the side stream (leaving sm_reserve SMs for the
    // exchange kernels) while the halos travel; the k planes next to each halo follow on the
    // caller's stream after the exchange.
    const bool split = overlap && hi - lo + 1 >= 4 * (int64_t)k;
    if (split) {
      NvtxRange r_("jacobi_dist interior (side stream)");
      FTN_CUDA(cudaEventRecord(comm->ev_in, s));
      FTN_CUDA(cudaStreamWaitEvent(comm->side, comm->ev_in, 0));
      ScopedSmReserve reserve(comm->nranks > 1 ? comm->sm_reserve : 0);
      FTN_CHECK(jacobi_slab_part(src, dst, k, coeff, halo, first, last, lo + k, hi - k, comm->side, res));
      FTN_CUDA(cudaEventRecord(comm->ev_out, comm->side));
    }
    FTN_CHECK(halo_exchange(comm, src, halo, k, s));
    if (split) {
      NvtxRange r_("jacobi_dist halo-adjacent planes");
      FTN_CHECK(jacobi_slab_part(src, dst, k, coeff, halo, first, last, lo, lo + k - 1, s, res));
      FTN_CHECK(jacobi_slab_part(src, dst, k, coeff, halo, first, last, hi - k + 1, hi, s, res));
      FTN_CUDA(cudaStreamWaitEvent(s, comm->ev_out, 0));
    } else {
      FTN_CHECK(jacobi_slab_part(src, dst, k, coeff, halo, first, last, lo, hi, s, res));
    }
    *cur ^= 1;
  }
  return FTN_OK;
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
  auto t = std::make_unique<NcclTransport>();
  FTN_NCCL(ncclCommInitRank(&t->nccl, nranks, u, rank));
  ftn_comm_s* c = new ftn_comm_s();
  c->tr = std::move(t);
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ftn_status_t st = comm_streams(c);
  if (st != FTN_OK) {
    comm_free(c);
    return st;
  }
  *comm = c;
  return FTN_OK;
}

ftn_status_t ftn_comm_init_virtual(ftn_comm_t* comms, int32_t nranks, const int32_t* devices) {
  if (!comms || !devices) return fail(FTN_ERR_NULL, "ftn_comm_init_virtual: NULL argument");
  if (nranks < 1 || nranks > 1024) return fail(FTN_ERR_SHAPE, "ftn_comm_init_virtual: nranks must be 1..1024");
  int saved = 0;
  FTN_CUDA(cudaGetDevice(&saved));
  auto g = std::make_shared<VGroup>(nranks);
  std::vector<ftn_comm_s*> made;
  ftn_status_t st = FTN_OK;
  for (int a = 0; a < nranks && st == FTN_OK; ++a) {
    if (cudaSetDevice(devices[a]) != cudaSuccess) {
      st = fail(FTN_ERR_DEVICE, "ftn_comm_init_virtual: bad device");
      break;
    }
    st = require_sm100();
    if (st != FTN_OK) break;
    for (int b = 0; b < nranks && st == FTN_OK; ++b) {
      VChannel& c = g->ch[(size_t)a * nranks + b];  // a's events live on a's device (ready); done on b's
      if (cudaEventCreateWithFlags(&c.ready, cudaEventDisableTiming) != cudaSuccess)
        st = fail(FTN_ERR_CUDA, "ftn_comm_init_virtual: event creation failed");
    }
    for (int b = 0; b < nranks && st == FTN_OK; ++b) {
      VChannel& c = g->ch[(size_t)b * nranks + a];
      if (cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming) != cudaSuccess)
        st = fail(FTN_ERR_CUDA, "ftn_comm_init_virtual: event creation failed");
    }
    if (st != FTN_OK) break;
    ftn_comm_s* c = new ftn_comm_s();
    c->tr = std::make_unique<VirtualTransport>(g, a, devices[a]);
    c->nranks = nranks;
    c->rank = a;
    c->device = devices[a];
    c->is_virtual = true;
    st = comm_streams(c);
    made.push_back(c);
  }
  cudaSetDevice(saved);
  if (st != FTN_OK) {
    for (auto* c : made) comm_free(c);
    return st;
  }
  for (int a = 0; a < nranks; ++a) comms[a] = made[(size_t)a];
  return FTN_OK;
}

ftn_status_t ftn_comm_set_overlap(ftn_comm_t comm, int32_t mode) {
  if (!comm) return fail(FTN_ERR_NULL, "ftn_comm_set_overlap: comm NULL");
  if (mode < 0 || mode > 2) return fail(FTN_ERR_SHAPE, "ftn_comm_set_overlap: mode must be 0, 1 or 2");
  comm->overlap = mode;
  return FTN_OK;
}

ftn_status_t ftn_comm_set_sm_reserve(ftn_comm_t comm, int32_t sms) {
  if (!comm) return fail(FTN_ERR_NULL, "ftn_comm_set_sm_reserve: comm NULL");
  if (sms < 0 || sms > 64) return fail(FTN_ERR_SHAPE, "ftn_comm_set_sm_reserve: 0..64 SMs");
  comm->sm_reserve = sms;
  return FTN_OK;
}

ftn_status_t ftn_comm_destroy(ftn_comm_t comm) {
  if (!comm) return FTN_OK;
  comm_free(comm);  // the transport's destructor releases the NCCL communicator / virtual group
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
  FTN_CHECK(dist_check(comm, u, unew, halo, "ftn_jacobi_dist"));
  if (sweeps < 0) return fail(FTN_ERR_SHAPE, "ftn_jacobi_dist: negative sweep count");
  FTN_CHECK(require_sm100());
  FTN_CHECK(jacobi_prepare());
  // temporal blocking: up to T sweeps per exchange, at most the halo depth
  const int T = dist_T(u, unew, halo);
  const int64_t nplan = ftn_jacobi_plan(sweeps, T, nullptr, 0);
  std::vector<int32_t> plan((size_t)nplan);
  ftn_jacobi_plan(sweeps, T, plan.data(), nplan);
  int cur = 0;
  FTN_CHECK(dist_run(comm, u, unew, plan, coeff, halo, &cur, (cudaStream_t)stream));
  if (result_in_unew) *result_in_unew = cur;
  return FTN_OK;
}

// Distributed Jacobi to convergence: blocks of check_every sweeps by
// the plan of ftn_jacobi_dist; each rank's residual over its owned interior points (fused
// into the block's last launch for rank-2 TMA-able slabs, else a single last sweep and a
// MAXVAL(ABS(x - y)) pass over the owned interior section), all-gathered, and the maximum of
// the p values (exact, identical on every rank) decides the stop.  One stream synchronisation
// per block.
ftn_status_t ftn_jacobi_solve_dist(ftn_comm_t comm, const ftn_desc_t* u, const ftn_desc_t* unew, int32_t halo,
                                   int64_t max_sweeps, int64_t check_every, double tol, double coeff, void* ws,
                                   size_t ws_bytes, int64_t* sweeps_done, double* residual, int32_t* result_in_unew,
                                   ftn_stream_t stream) {
  NvtxRange nvtx_("ftn_jacobi_solve_dist");
  FTN_CHECK(dist_check(comm, u, unew, halo, "ftn_jacobi_solve_dist"));
  if (max_sweeps < 0 || check_every < 1)
    return fail(FTN_ERR_SHAPE, "ftn_jacobi_solve_dist: need max_sweeps >= 0, check_every >= 1");
  size_t rws = 0;
  FTN_CHECK(ftn_reduce_workspace_size(u, &rws));
  const size_t head = 8 * ((size_t)comm->nranks + 2);
  if (!ws || ws_bytes < head + rws || ((uintptr_t)ws % 16))
    return fail(FTN_ERR_WORKSPACE,
                "ftn_jacobi_solve_dist: workspace must hold 8*(nranks+2) + ftn_reduce_workspace_size(u) bytes, 16-byte aligned");
  FTN_CHECK(require_sm100());
  FTN_CHECK(jacobi_prepare());
  cudaStream_t s = (cudaStream_t)stream;
  const int r = u->rank;
  const int T = dist_T(u, unew, halo);
  const bool fused_res = r == 2 && stencil_tma_able(u) && stencil_tma_able(unew);
  double* slot = reinterpret_cast<double*>(ws);
  double* gathered = slot + 2;
  char* rw = reinterpret_cast<char*>(ws) + head;
  // owned interior sections (local planes [halo, nl - halo), interior in the other dims)
  ftn_desc_t iu, iw;
  bool have_interior = true;
  {
    int64_t lo[3], hi[3], st[3] = {1, 1, 1};
    for (int d = 0; d < r; ++d) {
      const int64_t lb = u->dim[d].lower_bound, ext = u->dim[d].extent;
      lo[d] = d == r - 1 ? lb + halo : lb + 1;
      hi[d] = d == r - 1 ? lb + ext - halo - 1 : lb + ext - 2;
      if (hi[d] < lo[d]) have_interior = false;
    }
    if (have_interior) {
      FTN_CHECK(ftn_desc_section(&iu, u, lo, hi, st));
      FTN_CHECK(ftn_desc_section(&iw, unew, lo, hi, st));
    }
  }
  std::vector<double> host((size_t)comm->nranks);
  int cur = 0;
  int64_t done = 0;
  double res = INFINITY;
  while (done < max_sweeps) {
    const int64_t k = check_every < max_sweeps - done ? check_every : max_sweeps - done;
    FTN_CUDA(cudaMemsetAsync(slot, 0xff, sizeof(double), s));  // NaN: the empty fmax slot
    const int64_t np = ftn_jacobi_plan(fused_res ? k : k - 1, T, nullptr, 0);
    std::vector<int32_t> plan((size_t)np);
    ftn_jacobi_plan(fused_res ? k : k - 1, T, plan.data(), np);
    if (!fused_res) plan.push_back(1);  // consecutive iterates in u / unew for the residual pass
    FTN_CHECK(dist_run(comm, u, unew, plan, coeff, halo, &cur, s, fused_res ? slot : nullptr));
    if (!fused_res && have_interior) FTN_CHECK(ftn_maxval_absdiff(&iu, &iw, slot, rw, ws_bytes - head, stream));
    FTN_CHECK(comm->tr->allgather(slot, gathered, 8, s));
    FTN_CUDA(cudaMemcpyAsync(host.data(), gathered, 8 * (size_t)comm->nranks, cudaMemcpyDeviceToHost, s));
    FTN_CUDA(cudaStreamSynchronize(s));
    done += k;
    res = -INFINITY;  // max over the ranks' values, empty (NaN) ones skipped: exact, the same on every rank
    for (double v : host)
      if (v == v && v > res) res = v;
    if (res <= tol) break;
  }
  if (sweeps_done) *sweeps_done = done;
  if (residual) *residual = done ? res : 0.0;
  if (result_in_unew) *result_in_unew = cur;
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
  return comm->tr->bcast(x->base_addr, (size_t)desc_size(x) * (size_t)x->elem_len, root, (cudaStream_t)stream);
}

}  // extern "C"
