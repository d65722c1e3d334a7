// SMEM-resident 2-D Jacobi for grids that fit the aggregate shared memory of the GPU (the
// paper's own jacobi shape, 1024^2 x 10^5 sweeps: a 16 MiB working set that other
// kernels re-read from L2 at one launch per few sweeps).  The DO nest of R#16, bit-identical
// to T single sweeps; one cooperative launch runs all `sweeps`:
//   * CTA b (one per SM) owns the interior rows [lo_b, hi_b] (Fortran dim 2) and keeps them,
//     plus K halo rows per side, in two shared-memory buffers: buffer p holds the iterates of
//     parity p (buffer 0 starts from u, buffer 1 from unew, so each array keeps its own
//     boundary values exactly as the DO nest with swapped arrays does).
//   * A phase runs k <= K sweeps without communication on a shrinking row range (sweep q of
//     a phase computes rows lo-(K-q) .. hi+(K-q)), then the CTA writes its first and last K
//     owned rows to global memory, publishes an epoch flag, waits for the flags of its two
//     neighbours only (no grid barrier) and reads their rows into its halo.
//   * Epoch e's rows go to unew (e even) or u (e odd): a CTA writes epoch e+2 into the same
//     array only after both neighbours published e+1, i.e. after they read epoch e; epoch 0
//     goes to unew, so no CTA overwrites u rows that a slower neighbour still has to load.
//   * After a final flag round (neighbours done reading) every CTA writes iterate S of its rows
//     to the result array (unew iff S is odd) and iterate S-1 to the other one, exactly the
//     state the swapped DO nest leaves behind.
// Spin waits are bounded (a trap instead of a hang if a neighbour never arrives).
#include "ftn_internal.cuh"

#include <cstdlib>

namespace ftn {

namespace {

constexpr int RES_THREADS = 512;
constexpr int RES_SMEM_MAX = 227 * 1024;

struct ResParams {
  char* u;
  char* w;
  int64_t u_sm1, u_sm2, w_sm1, w_sm2;
  int32_t n1, n2;
  int32_t pitch;    // doubles per shared-memory row (even)
  int32_t K;        // halo depth = sweeps per exchange
  int32_t rows_max; // shared-memory rows per buffer
  int64_t sweeps;
  double coeff;
  uint32_t* flags;  // one per CTA, zeroed before the launch
  uint64_t* trace;  // FTN_RES_TRACE only: publish times [CTA][64 epochs]
  double* xbuf;     // exchange rows: [epoch parity][CTA][side: first / last K owned rows][K][pitch]
};

// Publish: a release reduction (the flag counts the epochs).  A plain st.release measured
// ~4.5 us per neighbour handshake with 148 polling CTAs, the reduction ~1.4 us
// (tools/microbench/flag_probe.cu).
__device__ __forceinline__ void publish(uint32_t* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// thread 0: wait until the flags of CTAs b-1 and b+1 (those that exist) reach `epoch`
__device__ void wait_neighbours(const ResParams& p, int b, uint32_t epoch) {
  for (int nb = b - 1; nb <= b + 1; nb += 2) {
    if (nb < 0 || nb >= (int)gridDim.x) continue;
    uint64_t spins = 0;
    while (ld_acquire(&p.flags[nb]) < epoch) {
      if (++spins > (1ull << 24)) __trap();  // a neighbour that never arrives: fail, do not hang
    }
  }
}

// n double2 from global (L2, never a stale L1 line) to shared memory: batches of 8 loads in
// flight per thread before their stores
__device__ __forceinline__ void copy_g2s(double2* dst, const double2* src, int n) {
  for (int base = 0; base < n; base += 4 * RES_THREADS) {
    double2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = base + q * RES_THREADS + threadIdx.x;
      if (i < n) v[q] = __ldcg(src + i);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = base + q * RES_THREADS + threadIdx.x;
      if (i < n) dst[i] = v[q];
    }
  }
}

__device__ __forceinline__ void copy_s2g(double2* dst, const double2* src, int n) {
  for (int i = threadIdx.x; i < n; i += RES_THREADS) dst[i] = src[i];
}

#ifndef FTN_RES_TRACE
#define FTN_RES_TRACE 0
#endif
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(RES_THREADS, 1) jacobi2d_resident(const __grid_constant__ ResParams p) {
  uint64_t tr_c0 = 0, tr_c1 = 0, tr_w = 0, tr_h = 0;  // FTN_RES_TRACE: compute / wait / halo ns
  extern __shared__ __align__(16) double sm[];
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int interior = p.n2 - 2;
  const int lo = 1 + (int)((int64_t)interior * b / G);
  const int hi = (int)((int64_t)interior * (b + 1) / G);  // owned rows lo .. hi
  const int K = p.K;
  const int rb = max(0, lo - K), re = min(p.n2 - 1, hi + K);  // rows held: rb .. re
  const int nr = re - rb + 1;
  const int pitch = p.pitch;
  double* const buf0 = sm;
  double* const buf1 = sm + (size_t)p.rows_max * pitch;
  auto bufp = [&](int q) { return q ? buf1 : buf0; };
  auto srow = [&](int q, int r) { return bufp(q) + (size_t)(r - rb) * pitch; };
  auto gptr = [&](int arr, int r, int c) -> double* {
    return arr == 0 ? reinterpret_cast<double*>(p.u + (int64_t)c * p.u_sm1 + (int64_t)r * p.u_sm2)
                    : reinterpret_cast<double*>(p.w + (int64_t)c * p.w_sm1 + (int64_t)r * p.w_sm2);
  };
  // exchange slot of CTA c, side s (0: its first K owned rows, 1: its last K), epoch parity e
  auto xrow = [&](int e, int c, int side) {
    return p.xbuf + ((((size_t)e * G + c) * 2 + side) * K) * pitch;
  };
  // initial slab: buffer 0 from u, buffer 1 from unew (all columns: the boundary stays per array)
  for (int q = 0; q < 2; ++q)
    for (int idx = tid; idx < nr * p.n1; idx += RES_THREADS) {
      const int r = rb + idx / p.n1, c = idx % p.n1;
      srow(q, r)[c] = __ldcg(gptr(q, r, c));
    }
  __syncthreads();

  const double coeff = p.coeff;
  int64_t done = 0;
  uint32_t epoch = 0;
  while (done < p.sweeps) {
    const int k = (int)min((int64_t)K, p.sweeps - done);
    if (FTN_RES_TRACE && tid == 0) tr_c0 = gtimer();
    for (int q = 1; q <= k; ++q) {
      const int sp = (int)((done + q - 1) & 1);  // source parity: iterate done+q-1
      const int ra = max(1, lo - (K - q)), rz = min(p.n2 - 2, hi + (K - q));
      const double* S = bufp(sp);
      double* D = bufp(sp ^ 1);
      // a warp task = 64 consecutive columns (lane = column pair (c, c+1)) x one part of the
      // rows; the i-1 / i+1 neighbours come from the adjacent lanes, the warp's edge lanes
      // read them from smem
      const int nch = (p.n1 + 63) / 64;
      const int parts = max(1, (RES_THREADS / 32) / nch);
      const int nrow = rz - ra + 1;
      for (int task = warp; task < nch * parts; task += RES_THREADS / 32) {
        const int c = (task % nch) * 64 + 2 * lane;
        const int part = task / nch;
        const int pa = ra + (int)((int64_t)nrow * part / parts), pz = ra + (int)((int64_t)nrow * (part + 1) / parts) - 1;
        if (pa > pz) continue;  // warp-uniform
        const bool valid = c < p.n1;
        const int cc = valid ? c : 0;  // idle lanes of the last chunk read column 0
        const double* col = S + cc;
        double2 up = *reinterpret_cast<const double2*>(col + (size_t)(pa - 1 - rb) * pitch);
        double2 mid = *reinterpret_cast<const double2*>(col + (size_t)(pa - rb) * pitch);
        const bool in0 = valid && c >= 1 && c <= p.n1 - 2, in1 = valid && c + 1 <= p.n1 - 2;
#pragma unroll 2
        for (int r = pa; r <= pz; ++r) {
          const double* row = col + (size_t)(r - rb) * pitch;
          const double2 dn = *reinterpret_cast<const double2*>(row + pitch);
          double left = __shfl_up_sync(0xffffffffu, mid.y, 1);
          double right = __shfl_down_sync(0xffffffffu, mid.x, 1);
          if (lane == 0) left = c >= 1 ? row[-1] : 0.0;
          if (lane == 31) right = c + 2 < p.n1 ? row[2] : 0.0;
          // R#16: coeff * (((u(i-1,j) + u(i+1,j)) + u(i,j-1)) + u(i,j+1))
          double v0 = left + mid.y;
          v0 = v0 + up.x;
          v0 = v0 + dn.x;
          v0 = coeff * v0;
          double v1 = mid.x + right;
          v1 = v1 + up.y;
          v1 = v1 + dn.y;
          v1 = coeff * v1;
          double* drow = D + (size_t)(r - rb) * pitch + cc;
          if (in0 && in1) {
            *reinterpret_cast<double2*>(drow) = make_double2(v0, v1);
          } else {
            if (in0) drow[0] = v0;
            if (in1) drow[1] = v1;
          }
          up = mid;
          mid = dn;
        }
      }
      __syncthreads();
    }
    done += k;
    const int cp = (int)(done & 1);  // buffer of iterate `done`
    if (done < p.sweeps) {
      // exchange: the first and last K owned rows (whole rows: the boundary columns of buffer
      // cp come from the same array in every CTA) -> exchange slots of epoch parity
      const int e = (int)(epoch & 1);
      const int n2v = K * pitch / 2;
      if (b > 0) copy_s2g(reinterpret_cast<double2*>(xrow(e, b, 0)), reinterpret_cast<const double2*>(srow(cp, lo)), n2v);
      if (b < G - 1)
        copy_s2g(reinterpret_cast<double2*>(xrow(e, b, 1)), reinterpret_cast<const double2*>(srow(cp, hi - K + 1)), n2v);
      ++epoch;
      __syncthreads();
      if (tid == 0) {
        if (FTN_RES_TRACE) tr_c1 += gtimer() - tr_c0, tr_c0 = gtimer();
        if (FTN_RES_TRACE && epoch <= 64) p.trace[(size_t)b * 64 + epoch - 1] = tr_c0;
        publish(&p.flags[b]);
        wait_neighbours(p, b, epoch);
        if (FTN_RES_TRACE) tr_w += gtimer() - tr_c0, tr_c0 = gtimer();
      }
      __syncthreads();
      // halo rows: lo-K .. lo-1 are CTA b-1's last K rows, hi+1 .. hi+K CTA b+1's first K
      if (b > 0) copy_g2s(reinterpret_cast<double2*>(srow(cp, lo - K)), reinterpret_cast<const double2*>(xrow(e, b - 1, 1)), n2v);
      if (b < G - 1) copy_g2s(reinterpret_cast<double2*>(srow(cp, hi + 1)), reinterpret_cast<const double2*>(xrow(e, b + 1, 0)), n2v);
      __syncthreads();
      if (FTN_RES_TRACE && tid == 0) tr_h += gtimer() - tr_c0;
    }
  }
  if (FTN_RES_TRACE && tid == 0 && b == 0) {
    for (int c = 0; c < G; ++c)
      while (ld_relaxed(&p.flags[c]) < epoch) {
      }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    for (int e = 40; e < 44; ++e) {
      uint64_t t0 = ~0ull;
      for (int c = 0; c < G; ++c) t0 = min(t0, p.trace[(size_t)c * 64 + e]);
      printf("epoch %d:", e);
      for (int c = 0; c < G; c += 4) printf(" %.1f", (p.trace[(size_t)c * 64 + e] - t0) / 1e3);
      printf("\n");
    }
  }
  if (FTN_RES_TRACE && tid == 0 && (b % 37 == 1 || b == G - 1))
    printf("res CTA %d: phases %u compute+write %.2f us wait %.2f us halo %.2f us per phase\n", b, epoch,
           tr_c1 / 1e3 / epoch, tr_w / 1e3 / epoch, tr_h / 1e3 / epoch);
  // final round: neighbours have loaded their initial rows of u / unew before they are overwritten
  ++epoch;
  __syncthreads();
  if (tid == 0) {
    publish(&p.flags[b]);
    wait_neighbours(p, b, epoch);
  }
  __syncthreads();
  const int last = (int)(p.sweeps & 1);  // iterate S in buffer `last`, array unew iff S odd
  const int cols = p.n1 - 2;
  for (int q = 0; q < 2; ++q) {
    const int parity = q == 0 ? last : last ^ 1;  // iterate S, then iterate S-1
    const int arr = parity;                       // parity 1 -> unew, 0 -> u
    for (int idx = tid; idx < (hi - lo + 1) * cols; idx += RES_THREADS) {
      const int r = lo + idx / cols, c = 1 + idx % cols;
      *gptr(arr, r, c) = srow(parity, r)[c];
    }
  }
}

// Register-resident variant (n1 <= 2 * RES_THREADS, slab rows <= RR_MAX): thread = column pair
// (c, c+1) holding its two columns of every slab row in registers, so a sweep reads no shared
// memory except the two warp-edge columns; the i-1 / i+1 neighbours come from the adjacent
// lanes.  The boundary columns / rows take the values of the array of the new iterate's parity
// from small shared tables (u's and unew's rings may differ, as in the swapped DO nest).
constexpr int RR_MAX = 16;
constexpr int RES_WARPS = RES_THREADS / 32;

__global__ void __launch_bounds__(RES_THREADS, 1) jacobi2d_resident_reg(const __grid_constant__ ResParams p) {
  extern __shared__ __align__(16) double sm[];
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int interior = p.n2 - 2;
  const int lo = 1 + (int)((int64_t)interior * b / G);
  const int hi = (int)((int64_t)interior * (b + 1) / G);
  const int K = p.K;
  const int rb = max(0, lo - K), re = min(p.n2 - 1, hi + K);
  const int nr = re - rb + 1;  // <= RR_MAX
  const int pitch = p.pitch;
  const int n1 = p.n1;
  const int c = 2 * tid;
  const bool valid = c < n1, has1 = c + 1 < n1;
  // shared tables: bcol[array][side: column 0 / n1-1][RR_MAX], brow[array][side: row 0 / n2-1][pitch],
  // edge[sweep parity][warp][lane 0 .x / lane 31 .y][RR_MAX]
  double* bcol = sm;
  double* brow = bcol + 2 * 2 * RR_MAX;
  double* edge = brow + 2 * 2 * (size_t)pitch;
  auto gptr = [&](int arr, int r, int col) -> double* {
    return arr == 0 ? reinterpret_cast<double*>(p.u + (int64_t)col * p.u_sm1 + (int64_t)r * p.u_sm2)
                    : reinterpret_cast<double*>(p.w + (int64_t)col * p.w_sm1 + (int64_t)r * p.w_sm2);
  };
  auto xrow = [&](int e, int cta, int side) {
    return p.xbuf + ((((size_t)e * G + cta) * 2 + side) * K) * pitch;
  };
  double x[RR_MAX][2];
#pragma unroll
  for (int i = 0; i < RR_MAX; ++i) {
    x[i][0] = x[i][1] = 0.0;
    if (i < nr && valid) {
      x[i][0] = __ldcg(gptr(0, rb + i, c));
      if (has1) x[i][1] = __ldcg(gptr(0, rb + i, c + 1));
    }
  }
  for (int idx = tid; idx < 2 * 2 * nr; idx += RES_THREADS) {
    const int arr = idx / (2 * nr), side = (idx / nr) % 2, i = idx % nr;
    bcol[(arr * 2 + side) * RR_MAX + i] = __ldcg(gptr(arr, rb + i, side ? n1 - 1 : 0));
  }
  for (int idx = tid; idx < 2 * n1; idx += RES_THREADS) {
    const int arr = idx / n1, col = idx % n1;
    if (rb == 0) brow[(arr * 2 + 0) * pitch + col] = __ldcg(gptr(arr, 0, col));
    if (re == p.n2 - 1) brow[(arr * 2 + 1) * pitch + col] = __ldcg(gptr(arr, p.n2 - 1, col));
  }
  __syncthreads();
  uint32_t epoch = 0;
  if (p.sweeps <= K) {  // no exchange will order the neighbours' initial loads before our writes
    ++epoch;
    if (tid == 0) {
      publish(&p.flags[b]);
      wait_neighbours(p, b, epoch);
    }
    __syncthreads();
  }
  const double coeff = p.coeff;
  int64_t done = 0;
  uint64_t tr0 = 0, trc = 0, trw = 0, trh = 0;
  while (done < p.sweeps) {
    const int k = (int)min((int64_t)K, p.sweeps - done);
    if (FTN_RES_TRACE && tid == 0) tr0 = gtimer();
    for (int q = 1; q <= k; ++q) {
      const int64_t t = done + q - 1;  // iterate t -> t + 1
      const int np = (int)((t + 1) & 1);  // parity (array) of the new iterate
      const int ia = max(1, lo - (K - q)) - rb, iz = min(p.n2 - 2, hi + (K - q)) - rb;
      uint64_t ts0 = 0;
      if (FTN_RES_TRACE && tid == 0) ts0 = gtimer();
      double* ed = edge + (size_t)(t & 1) * RES_WARPS * 2 * RR_MAX;
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < RR_MAX; ++i) ed[(warp * 2 + 0) * RR_MAX + i] = x[i][0];
      }
      if (lane == 31) {
#pragma unroll
        for (int i = 0; i < RR_MAX; ++i) ed[(warp * 2 + 1) * RR_MAX + i] = x[i][1];
      }
      __syncthreads();
      if (FTN_RES_TRACE && tid == 0) trh += gtimer() - ts0;
      if (t + 1 == p.sweeps) {  // last sweep: iterate S-1 of the owned rows -> its array
#pragma unroll
        for (int i = 0; i < RR_MAX; ++i) {
          const int r = rb + i;
          if (r >= lo && r <= hi) {
            if (valid && c >= 1 && c <= n1 - 2) *gptr(np ^ 1, r, c) = x[i][0];
            if (has1 && c + 1 <= n1 - 2) *gptr(np ^ 1, r, c + 1) = x[i][1];
          }
        }
      }
      // every row 1 .. RR_MAX-2 is computed (no divergent branches around the shuffles); rows
      // outside [ia, iz] keep their value through a select
      const double* edL = ed + (max(warp - 1, 0) * 2 + 1) * RR_MAX;
      const double* edR = ed + (min(warp + 1, RES_WARPS - 1) * 2 + 0) * RR_MAX;
      const bool in0 = valid && c >= 1 && c <= n1 - 2, in1 = has1 && c + 1 <= n1 - 2;
      double pv0 = x[0][0], pv1 = x[0][1];  // old values of the row above
#pragma unroll
      for (int i = 1; i < RR_MAX - 1; ++i) {
        const double o0 = x[i][0], o1 = x[i][1];
        double left = __shfl_up_sync(0xffffffffu, o1, 1);
        double right = __shfl_down_sync(0xffffffffu, o0, 1);
        const double eL = edL[i], eR = edR[i];
        left = lane == 0 ? eL : left;    // warp 0 lane 0 holds column 0: its left is never used
        right = lane == 31 ? eR : right;
        // R#16: coeff * (((u(i-1,j) + u(i+1,j)) + u(i,j-1)) + u(i,j+1))
        double v0 = left + o1;
        v0 = v0 + pv0;
        v0 = v0 + x[i + 1][0];
        v0 = coeff * v0;
        double v1 = o0 + right;
        v1 = v1 + pv1;
        v1 = v1 + x[i + 1][1];
        v1 = coeff * v1;
        const bool act = i >= ia && i <= iz;
        x[i][0] = act && in0 ? v0 : o0;
        x[i][1] = act && in1 ? v1 : o1;
        pv0 = o0;
        pv1 = o1;
      }
      // boundary columns (the lanes holding column 0 or n1-1) switch to the new iterate's array
      if (valid && (c == 0 || c == n1 - 1 || c + 1 == n1 - 1)) {
        const double* b0 = bcol + (np * 2 + (c == 0 ? 0 : 1)) * RR_MAX;
        const double* b1 = bcol + (np * 2 + 1) * RR_MAX;
#pragma unroll
        for (int i = 1; i < RR_MAX - 1; ++i)
          if (i >= ia && i <= iz) {
            if (!in0) x[i][0] = b0[i];
            if (has1 && !in1) x[i][1] = b1[i];
          }
      }
      // boundary rows switch to the new iterate's array
      if (rb == 0 && valid) {
        x[0][0] = brow[(np * 2 + 0) * pitch + c];
        if (has1) x[0][1] = brow[(np * 2 + 0) * pitch + c + 1];
      }
      if (re == p.n2 - 1 && valid) {
#pragma unroll
        for (int i = 0; i < RR_MAX; ++i)
          if (i == nr - 1) {
            x[i][0] = brow[(np * 2 + 1) * pitch + c];
            if (has1) x[i][1] = brow[(np * 2 + 1) * pitch + c + 1];
          }
      }
    }
    done += k;
    if (done < p.sweeps) {
      const int e = (int)(epoch & 1);
      // first / last K owned rows -> exchange slots (whole pairs, incl. the boundary columns)
#pragma unroll
      for (int i = 0; i < RR_MAX; ++i) {
        const int r = rb + i;
        if (valid && b > 0 && r >= lo && r < lo + K)
          *reinterpret_cast<double2*>(xrow(e, b, 0) + (size_t)(r - lo) * pitch + c) = make_double2(x[i][0], x[i][1]);
        if (valid && b < G - 1 && r > hi - K && r <= hi)
          *reinterpret_cast<double2*>(xrow(e, b, 1) + (size_t)(r - (hi - K + 1)) * pitch + c) =
              make_double2(x[i][0], x[i][1]);
      }
      ++epoch;
      __syncthreads();
      if (tid == 0) {
        if (FTN_RES_TRACE) trc += gtimer() - tr0, tr0 = gtimer();
        publish(&p.flags[b]);
        wait_neighbours(p, b, epoch);
        if (FTN_RES_TRACE) trw += gtimer() - tr0, tr0 = gtimer();
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < RR_MAX; ++i) {
        const int r = rb + i;
        if (valid && b > 0 && r < lo) {
          const double2 v = __ldcg(reinterpret_cast<const double2*>(xrow(e, b - 1, 1) + (size_t)(r - (lo - K)) * pitch + c));
          x[i][0] = v.x;
          x[i][1] = v.y;
        }
        if (valid && b < G - 1 && r > hi && i < nr) {
          const double2 v = __ldcg(reinterpret_cast<const double2*>(xrow(e, b + 1, 0) + (size_t)(r - (hi + 1)) * pitch + c));
          x[i][0] = v.x;
          x[i][1] = v.y;
        }
      }
    }
  }
  if (FTN_RES_TRACE && tid == 0 && (b % 37 == 1 || b == G - 1))
    printf("reg CTA %d: phases %u compute+write %.2f us wait %.2f us; per sweep edge+barrier %.2f us\n", b, epoch,
           trc / 1e3 / epoch, trw / 1e3 / epoch, trh / 1e3 / p.sweeps);
  // iterate S of the owned rows -> its array (unew iff S odd)
  const int fa = (int)(p.sweeps & 1);
#pragma unroll
  for (int i = 0; i < RR_MAX; ++i) {
    const int r = rb + i;
    if (r >= lo && r <= hi) {
      if (valid && c >= 1 && c <= n1 - 2) *gptr(fa, r, c) = x[i][0];
      if (has1 && c + 1 <= n1 - 2) *gptr(fa, r, c + 1) = x[i][1];
    }
  }
}

}  // namespace

// ftn_jacobi_set_resident: minimum sweep count for the resident path (0: never) and the halo
// depth K (0: the largest K <= 4 that fits)
static std::atomic<int64_t> g_res_min{-1};
static std::atomic<int> g_res_k{0};

int64_t jacobi_resident_min() {
  int64_t v = g_res_min.load();
  if (v < 0) {
    v = getenv("FTN_JACOBI_RES_MIN") ? atoll(getenv("FTN_JACOBI_RES_MIN")) : 0;
    if (v < 0) v = 0;
    g_res_min.store(v);
  }
  return v;
}

// Plan for the resident kernels: grid, halo depth, shared memory and the variant (register
// slab when n1 <= 2 * RES_THREADS and owned + 2K rows <= RR_MAX, else the shared-memory slab);
// false when the grid does not fit (then the caller uses the streaming kernels).
struct ResPlan {
  int grid, K, rows_max, pitch;
  size_t smem;
  bool reg;
};

static bool resident_plan(int64_t n1, int64_t n2, ResPlan* pl) {
  if (n1 < 3 || n2 < 3 || n1 > (1 << 20) || n2 > (1 << 20)) return false;
  const int64_t interior = n2 - 2;
  const int pt = (int)((n1 + 1) & ~int64_t(1));
  const int kenv = g_res_k.load();
  for (int pass = 0; pass < 2; ++pass) {  // 0: register slab, 1: shared-memory slab
    if (pass == 0 && n1 > 2 * RES_THREADS) continue;
    for (int k = (kenv > 0 ? kenv : 4); k >= 1; --k) {
      const int64_t G = std::min<int64_t>(num_sms(), interior / k);  // every CTA owns >= k rows
      if (G >= 1) {
        const int64_t own_max = (interior + G - 1) / G;
        const int64_t rows = own_max + 2 * k;
        const size_t bytes = pass == 0 ? (size_t)(4 * RR_MAX + 4 * (size_t)pt + 2 * RES_WARPS * 2 * RR_MAX) * 8
                                       : 2 * (size_t)rows * pt * 8;
        if ((pass == 0 ? rows <= RR_MAX : true) && bytes <= (size_t)RES_SMEM_MAX) {
          *pl = {(int)G, k, (int)rows, pt, bytes, pass == 0};
          return true;
        }
      }
      if (kenv > 0) break;
    }
  }
  return false;
}

bool jacobi2d_resident_fits(const ftn_desc_t* u) {
  ResPlan pl;
  return u->rank == 2 && resident_plan(u->dim[0].extent, u->dim[1].extent, &pl);
}

// All `sweeps` of the DO nest in one cooperative launch (sweeps >= 1); the result lands in
// unew iff sweeps is odd, the other array holds iterate sweeps-1.
ftn_status_t jacobi2d_resident_run(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t sweeps, double coeff,
                                   cudaStream_t s) {
  ResPlan pl;
  if (!resident_plan(u->dim[0].extent, u->dim[1].extent, &pl))
    return fail(FTN_ERR_UNSUPPORTED, "jacobi2d_resident: grid does not fit the aggregate shared memory");
  const int grid = pl.grid, K = pl.K, rows_max = pl.rows_max, pitch = pl.pitch;
  const size_t smem = pl.smem;
  const void* fn = pl.reg ? (const void*)jacobi2d_resident_reg : (const void*)jacobi2d_resident;
  static std::atomic<bool> attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    FTN_CUDA(cudaFuncSetAttribute(jacobi2d_resident, cudaFuncAttributeMaxDynamicSharedMemorySize, RES_SMEM_MAX));
    FTN_CUDA(cudaFuncSetAttribute(jacobi2d_resident_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, RES_SMEM_MAX));
    attr[dev & 63] = true;
  }
  // one stream-ordered temporary: flags (zeroed) + exchange slots (2 parities x grid x 2 x K rows)
  const size_t flag_bytes = ((size_t)grid * sizeof(uint32_t) + 255) / 256 * 256;
  const size_t xbytes = (size_t)2 * grid * 2 * K * pitch * sizeof(double) + (FTN_RES_TRACE ? (size_t)grid * 64 * 8 : 0);
  StreamTemp tmp;
  FTN_CHECK(tmp.alloc(flag_bytes + xbytes, s));
  FTN_CUDA(cudaMemsetAsync(tmp.ptr, 0, (size_t)grid * sizeof(uint32_t), s));
  ResParams p;
  p.u = (char*)u->base_addr;
  p.w = (char*)unew->base_addr;
  p.u_sm1 = u->dim[0].sm;
  p.u_sm2 = u->dim[1].sm;
  p.w_sm1 = unew->dim[0].sm;
  p.w_sm2 = unew->dim[1].sm;
  p.n1 = (int32_t)u->dim[0].extent;
  p.n2 = (int32_t)u->dim[1].extent;
  p.pitch = pitch;
  p.K = K;
  p.rows_max = rows_max;
  p.sweeps = sweeps;
  p.coeff = coeff;
  p.flags = (uint32_t*)tmp.ptr;
  p.xbuf = (double*)((char*)tmp.ptr + flag_bytes);
  p.trace = FTN_RES_TRACE ? (uint64_t*)((char*)tmp.ptr + flag_bytes + (size_t)2 * grid * 2 * K * pitch * sizeof(double)) : nullptr;
  void* args[] = {&p};
  FTN_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(RES_THREADS), args, smem, s));
  return after_launch("jacobi2d_resident");
}

}  // namespace ftn

extern "C" ftn_status_t ftn_jacobi_set_resident(int64_t min_sweeps, int32_t halo_depth) {
  if (min_sweeps < 0 || halo_depth < 0 || halo_depth > 8)
    return ftn::fail(FTN_ERR_SHAPE, "ftn_jacobi_set_resident: need min_sweeps >= 0 and 0 <= halo_depth <= 8");
  ftn::g_res_min.store(min_sweeps);
  ftn::g_res_k.store(halo_depth);
  return FTN_OK;
}
