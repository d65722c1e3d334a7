// MATMUL: c = MATMUL(a, b) in real(8) on the fp64 tensor
// cores (DMMA, mma.sync.m16n8k4.f64), P:298 / P:310 / P:317.
//
// The paper's linalg.matmul gained ~5x from affine-loop-tile; this is the
// B200 version of that tiling.  sm_100a has no tcgen05 kind for f64, so the fp64
// tensor path is the warp-level DMMA, which the probe (tools/microbench) measured
// at 37.1 TFLOP/s chip-wide, the same as cuBLAS' ceiling (35.5) and DFMA (36.6).
//
// CTA tile 128 x 128, k-step 32, 3-stage TMA -> shared memory pipeline with
// mbarriers (lane 0 of warp 0 issues the TMA loads STAGES-1 steps ahead; eight MMA
// warps each own a 64 x 32 sub-tile as 4 x 4 m16n8 accumulators = 64 fp64
// registers).  A ninth, producer-only warp would put 3 warps on one SMSP and cap
// every thread at 168 registers (spills); folding the producer in keeps 2 warps
// per SMSP.
//
// Shared-memory layout (fragment loads spread over the banks, DESIGN.md §4 kernel table; ncu still
// counts ~200 M bank conflicts per 4096^3 product -- harmless, the DMMA pipe is at 97 %):
//   A stage = 8 TMA boxes {16 (i), 32 (l)}, B stage = 2 boxes {16 (l), 128 (j)},
//   all with the 128-byte swizzle.  Fortran A is i-fastest, but the m16n8k4 A
//   fragment puts k across lanes; the MMA's k index t is therefore mapped to the
//   physical l offset {0,4,1,5} (first k4 of each 8) and {2,6,3,7} (second),
//   which with the swizzle spreads the four t-rows over all 32 banks.  The same
//   permutation is applied to B, so each product a(i,l) b(l,j) is still formed
//   for every l exactly once.
#include "ftn_internal.cuh"

#include <algorithm>
#include <cstdlib>

#include <cstring>

namespace ftn {
namespace {

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3;
constexpr int MMA_WARPS = 8;
constexpr int THREADS = MMA_WARPS * 32;  // 2 warps per SMSP -> up to 255 registers each
constexpr int A_BOX_BYTES = 16 * BK * 8;         // 4 KB
constexpr int B_BOX_BYTES = 16 * BN * 8;         // 16 KB
constexpr int A_STAGE = (BM / 16) * A_BOX_BYTES; // 32 KB
constexpr int B_STAGE = (BK / 16) * B_BOX_BYTES; // 32 KB
constexpr int STAGE_BYTES = A_STAGE + B_STAGE;   // 64 KB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int GROUP_M = 8;

struct MParams {
  char* c;
  int64_t c_sm0, c_sm1;
  int64_t M, N, K;
  int64_t tiles_m, tiles_n;
  int kt;  // number of BK steps
  // Work: tiles [0, dp_tiles) whole, one per CTA in turn (data parallel); tiles
  // [dp_tiles, dp_tiles + sk_tiles) by stream-K: their sk_tiles * kt k-steps split evenly over
  // the CTAs of one persistent wave, a tile's partial sums combined in k order by the CTA that
  // finishes it last (sk_part: 2 slots of BM x BN per CTA, sk_cnt: one counter per tile, zero
  // at launch and left zero).
  int64_t dp_tiles, sk_tiles;
  double* sk_part;
  int* sk_cnt;
};

// byte offset of element (row, x) inside a 128B-swizzled box (rows of 16 doubles)
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t x) {
  return row * 128u + ((((x >> 1) ^ (row & 7u)) << 4) | ((x & 1u) << 3));
}


__device__ __forceinline__ void dmma(double* d, double a0, double a1, double b0) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// TA: the A operand is TRANSPOSE(a) with a (k, m) column-major (k fastest); TB: the B operand
// is TRANSPOSE(b) with b (n, k).  The boxes then carry the k index along their 16-element
// rows instead of across them, and the fragment addresses swap roles (same bank analysis).
template <bool TA, bool TB>
__global__ void __launch_bounds__(THREADS, 1)
    dmma_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const __grid_constant__ MParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], MMA_WARPS);
    }
    dev::fence_barrier_init();
  }
  __syncthreads();

  int m0 = 0, n0 = 0;  // origin of the current tile
  // grouped raster for L2 reuse of A row-panels and B column-panels
  auto set_tile = [&](int tile) {
    const int per_group = GROUP_M * (int)p.tiles_n;
    const int first_m = (tile / per_group) * GROUP_M;
    const int gsz = min(GROUP_M, (int)p.tiles_m - first_m);
    const int tm = first_m + (tile % per_group) % gsz;
    const int tn = (tile % per_group) / gsz;
    m0 = tm * BM;
    n0 = tn * BN;
  };

  // TMA producer: lane 0 of warp 0.  k-step kk of the current tile into pipeline slot it
  // (it counts this CTA's k-steps over all its tiles: stage it % STAGES, phase it / STAGES).
  auto issue = [&](int kk, uint32_t it) {
    const int s = it % STAGES;
    if (it >= STAGES) dev::mbar_wait_idle(&empty[s], ((it / STAGES) - 1) & 1);
    uint8_t* st = smem + s * STAGE_BYTES;
    dev::mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
    const int k0 = kk * BK;
    if constexpr (!TA) {
#pragma unroll
      for (int a = 0; a < BM / 16; ++a) dev::tma_load_2d(st + a * A_BOX_BYTES, &map_a, &full[s], m0 + 16 * a, k0);
    } else {
#pragma unroll
      for (int h = 0; h < BK / 16; ++h) dev::tma_load_2d(st + h * B_BOX_BYTES, &map_a, &full[s], k0 + 16 * h, m0);
    }
    if constexpr (!TB) {
#pragma unroll
      for (int h = 0; h < BK / 16; ++h)
        dev::tma_load_2d(st + A_STAGE + h * B_BOX_BYTES, &map_b, &full[s], k0 + 16 * h, n0);
    } else {
#pragma unroll
      for (int a = 0; a < BN / 16; ++a)
        dev::tma_load_2d(st + A_STAGE + a * A_BOX_BYTES, &map_b, &full[s], n0 + 16 * a, k0);
    }
  };
  const bool producer = (warp == 0 && lane == 0);
  if (producer) {
    dev::prefetch_tma(&map_a);
    dev::prefetch_tma(&map_b);
  }

  // ---------------- MMA warps
  const int wm = warp >> 2;  // 0..1 -> rows wm*64
  const int wn = warp & 3;   // 0..3 -> cols wn*32
  const int g = lane >> 2, t = lane & 3;
  double acc[4][4][4];

  // fragment loads index the __shared__ array directly so the compiler emits LDS and
  // may schedule them early (the mbarrier waits are compiler memory barriers)
  const uint32_t smem_base = (uint32_t)(smem - smem_raw);
  const uint32_t tphys = (uint32_t)((t >> 1) + ((t & 1) << 2));  // {0,4,1,5}
  // per-thread constant parts of the fragment addresses
  uint32_t a_off[2][4][2];  // [q][mt][half]: offset within the A stage for kb = 0
  uint32_t b_off[2][4];     // [q][nt]: offset within the B stage for kb = 0
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const uint32_t l = tphys + 2 * q;  // row within an 8-block
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      if constexpr (!TA) {  // boxes of 16 rows (i) x 32 (l): row = l, element = i
        const uint32_t box = wm * 4 + mt;
        a_off[q][mt][0] = box * A_BOX_BYTES + swz(l, g);
        a_off[q][mt][1] = box * A_BOX_BYTES + swz(l, g + 8);
      } else {              // boxes of 16 (l) x 128 (i): row = i, element = l
        const uint32_t i = wm * 64 + mt * 16 + g;
        a_off[q][mt][0] = swz(i, l);
        a_off[q][mt][1] = swz(i + 8, l);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      if constexpr (!TB) {  // boxes of 16 (l) x 128 (j): row = j, element = l
        b_off[q][nt] = A_STAGE + swz(wn * 32 + nt * 8 + g, l);
      } else {              // boxes of 16 (j) x 32 (l): row = l, element = j
        const uint32_t box = wn * 2 + (nt >> 1);
        b_off[q][nt] = A_STAGE + box * A_BOX_BYTES + swz(l, (nt & 1) * 8 + g);
      }
    }
  }

  uint32_t it = 0;  // k-steps consumed by this CTA
  // acc = sum over k-steps [k_lo, k_hi) of the current tile
  auto run = [&](int k_lo, int k_hi) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;
    if (producer)
      for (int kk = k_lo; kk < k_lo + STAGES - 1 && kk < k_hi; ++kk) issue(kk, it + (uint32_t)(kk - k_lo));
    __syncwarp();
    for (int kk = k_lo; kk < k_hi; ++kk, ++it) {
      const int s = it % STAGES;
      if (producer && kk + STAGES - 1 < k_hi) issue(kk + STAGES - 1, it + STAGES - 1);  // the stage freed at it-1
      __syncwarp();
      dev::mbar_wait(&full[s], (it / STAGES) & 1);
      const uint32_t st = smem_base + s * STAGE_BYTES;
#pragma unroll
      for (int kb = 0; kb < BK / 8; ++kb) {
        // A: row l = kb*8 + phys -> +kb*8 rows (the swizzle phase (row & 7) is unchanged)
        // B: x = (kb & 1) * 8 + phys in box kb >> 1 -> +8 doubles = +4 chunks: XOR by 4 commutes
        // rows carry l (MK / NK layouts): +kb*8 rows; elements carry l (KM / KN): box kb>>1, chunk ^ 4
        const uint32_t a_kb = TA ? (kb >> 1) * B_BOX_BYTES : kb * 8 * 128;
        const uint32_t a_x = TA ? ((kb & 1) ? 64u : 0u) : 0u;
        const uint32_t b_kb = TB ? kb * 8 * 128 : (kb >> 1) * B_BOX_BYTES;
        const uint32_t b_x = TB ? 0u : ((kb & 1) ? 64u : 0u);  // chunk index ^ 4 == byte offset ^ 64
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          double af[4][2], bf[4];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            af[mt][0] = *reinterpret_cast<const double*>(smem_raw + st + a_kb + (a_off[q][mt][0] ^ a_x));
            af[mt][1] = *reinterpret_cast<const double*>(smem_raw + st + a_kb + (a_off[q][mt][1] ^ a_x));
          }
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
            bf[nt] = *reinterpret_cast<const double*>(smem_raw + st + b_kb + (b_off[q][nt] ^ b_x));
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], af[mt][0], af[mt][1], bf[nt]);
        }
      }
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&empty[s]);
    }
  };

  // ---------------- epilogue: c(i, j) through the descriptor strides
  auto store = [&]() {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t i = m0 + wm * 64 + mt * 16 + g + ((r >> 1) << 3);
          const int64_t j = n0 + wn * 32 + nt * 8 + 2 * t + (r & 1);
          if (i < p.M && j < p.N) *reinterpret_cast<double*>(p.c + i * p.c_sm0 + j * p.c_sm1) = acc[mt][nt][r];
        }
  };

  // Work items of this CTA: whole tiles blockIdx.x, +G, ... below dp_tiles, then (stream-K)
  // its share [lo, hi) of the tail's k-steps, tile by tile.  One call site of run() keeps the
  // register allocation of the single-tile kernel.
  __shared__ int sk_last;
  // 32-bit work cursors (tiles < 2^31; the tail's k-steps I < 2^31, checked on the host)
  const int G = (int)gridDim.x, b = (int)blockIdx.x, kt = p.kt, dpt = (int)p.dp_tiles;
  const int I = (int)(p.sk_tiles * kt);
  const int hi = p.sk_tiles ? (int)((int64_t)(b + 1) * I / G) : 0;
  int dp_t = b, a = p.sk_tiles ? (int)((int64_t)b * I / G) : 0;
  for (;;) {
    int tt, k_lo, k_hi;
    if (dp_t < dpt) {
      tt = dp_t;
      dp_t += G;
      k_lo = 0;
      k_hi = kt;
    } else if (a < hi) {
      k_lo = a % kt;
      k_hi = min(kt, k_lo + (hi - a));
      tt = dpt + a / kt;
      a += k_hi - k_lo;
    } else {
      break;
    }
    set_tile(tt);
    run(k_lo, k_hi);
    if (k_lo == 0 && k_hi == kt) {
      store();
      continue;
    }
    // a partial tile of the stream-K tail: publish it; the CTA that completes the tile
    // combines the partial sums in k order (CTA order), so the bits do not depend on which
    // CTA finishes last
    const int ts = tt - dpt;
    auto start_of = [&](int cb) { return (int)((int64_t)cb * I / G); };
    auto cta_of = [&](int x) {  // the CTA whose share holds tail k-step x
      int c = (int)((int64_t)x * G / I);
      while (c + 1 < G && start_of(c + 1) <= x) ++c;
      while (c > 0 && start_of(c) > x) --c;
      return c;
    };
    const int b_lo = cta_of(ts * kt), b_hi = cta_of((ts + 1) * kt - 1);
    auto slot_of = [&](int cb) { return 2 * cb + (start_of(cb) >= ts * kt ? 0 : 1); };
    double* mine = p.sk_part + (size_t)slot_of(b) * (BM * BN) + (size_t)threadIdx.x * 64;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
        *reinterpret_cast<double4*>(mine + (mt * 4 + nt) * 4) =
            make_double4(acc[mt][nt][0], acc[mt][nt][1], acc[mt][nt][2], acc[mt][nt][3]);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const int prev = atomicAdd(&p.sk_cnt[ts], 1);
      sk_last = prev == (int)(b_hi - b_lo);
      if (sk_last) p.sk_cnt[ts] = 0;  // left zero for the next launch
    }
    __syncthreads();
    if (!sk_last) continue;
    __threadfence();
    // every segment (this CTA's too) is in its slot: c = ((p_lo + p_lo+1) + ...) per element,
    // streamed from the slots (acc is dead here, so the fixup needs few registers)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const size_t off = (size_t)threadIdx.x * 64 + (mt * 4 + nt) * 4;
        const double* s0 = p.sk_part + (size_t)slot_of(b_lo) * (BM * BN) + off;
        double2 v01 = __ldcg(reinterpret_cast<const double2*>(s0));
        double2 v23 = __ldcg(reinterpret_cast<const double2*>(s0 + 2));
#pragma unroll 1
        for (int cb = b_lo + 1; cb <= b_hi; ++cb) {
          const double* sc = p.sk_part + (size_t)slot_of(cb) * (BM * BN) + off;
          const double2 w01 = __ldcg(reinterpret_cast<const double2*>(sc));
          const double2 w23 = __ldcg(reinterpret_cast<const double2*>(sc + 2));
          v01.x = v01.x + w01.x;
          v01.y = v01.y + w01.y;
          v23.x = v23.x + w23.x;
          v23.y = v23.y + w23.y;
        }
        const double v[4] = {v01.x, v01.y, v23.x, v23.y};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t i = m0 + wm * 64 + mt * 16 + g + ((r >> 1) << 3);
          const int64_t j = n0 + wn * 32 + nt * 8 + 2 * t + (r & 1);
          if (i < p.M && j < p.N) *reinterpret_cast<double*>(p.c + i * p.c_sm0 + j * p.c_sm1) = v[r];
        }
      }
  }
}

bool tma_able(const ftn_desc_t* d) {
  return d->type == FTN_F64 && (d->dim[0].sm == 8 || d->dim[0].extent <= 1) && d->dim[1].sm > 0 &&
         (d->dim[1].sm % 16) == 0 && ((uintptr_t)d->base_addr % 16) == 0 && d->dim[0].extent < (1ll << 32) &&
         d->dim[1].extent < (1ll << 32) && d->dim[1].sm < (1ll << 40);
}

int64_t packed_ld(int64_t rows) { return (rows + 3) / 4 * 4; }  // 32-byte aligned columns

size_t pack_bytes(const ftn_desc_t* d) {
  return tma_able(d) ? 0 : (size_t)(packed_ld(d->dim[0].extent) * d->dim[1].extent * 8 + 256);
}

ftn_status_t pack(const ftn_desc_t* d, char* ws, ftn_desc_t* out, cudaStream_t s) {
  ftn_desc_t p = *d;
  p.base_addr = ws;
  p.dim[0].sm = 8;
  p.dim[1].sm = packed_ld(d->dim[0].extent) * 8;
  p.dim[0].lower_bound = p.dim[1].lower_bound = 1;
  FTN_CHECK(launch_copy(&p, d, s));
  *out = p;
  return FTN_OK;
}

ftn_status_t make_map(CUtensorMap* map, const ftn_desc_t* d, uint32_t box0, uint32_t box1) {
  uint64_t dims[2] = {(uint64_t)d->dim[0].extent, (uint64_t)d->dim[1].extent};
  uint64_t strides[1] = {(uint64_t)d->dim[1].sm};
  uint32_t box[2] = {box0, box1};
  return encode_tma(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d->base_addr, dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B);
}

template <bool TA, bool TB>
ftn_status_t launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const MParams& p, cudaStream_t s) {
  static std::atomic<bool> attr_set[64] = {};  // per device (idempotent)
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    FTN_CUDA(cudaFuncSetAttribute(dmma_gemm_kernel<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  SMEM_BYTES));
    attr_set[dev & 63] = true;
  }
  const int64_t tiles = p.tiles_m * p.tiles_n;
  const int64_t grid = p.sk_tiles ? (int64_t)num_sms() : tiles;
  dmma_gemm_kernel<TA, TB><<<(unsigned)grid, THREADS, SMEM_BYTES, s>>>(ma, mb, p);
  return after_launch("dmma_gemm_kernel");
}

// Stream-K for the tail (FTN_MATMUL_SK=0 disables): when whole tiles would leave the last
// wave of one-CTA-per-SM tiles less than ~93 % full (e.g. MATMUL of a p = 8 column block of C3:
// 512 tiles on 148 SMs = 3.46 waves), all but one full wave stay whole tiles and the rest is
// split evenly by k-steps over one persistent wave.
bool use_stream_k(int64_t tiles, int kt) {
  static const bool on = !getenv("FTN_MATMUL_SK") || atoi(getenv("FTN_MATMUL_SK")) != 0;
  const int64_t G = num_sms();
  if (!on || tiles < G || kt < 8) return false;
  const int64_t waves = (tiles + G - 1) / G;
  return (double)tiles / (double)(waves * G) < 0.93;
}

size_t sk_ws_bytes(int64_t tiles_bound) {
  return (size_t)2 * num_sms() * BM * BN * 8 + (size_t)tiles_bound * 4 + 512;
}

// Small products (M*N*K <= 2^21, e.g. C1's 48 x 48 x 32): one thread per c(i, j) folding
// l = 1..K in ascending order with one rounding per product and per sum -- the literal
// definition (F2018 16.9.124) and therefore bit-identical to the oracle's
// sequential fold; no packing, any strides (op = TRANSPOSE by swapping a's or b's strides).
// A DMMA tile pipeline has nothing to amortise its TMA / mbarrier latency over at this size.
struct SmallMM {
  const char* a;
  int64_t a_si, a_sl;  // byte strides of op(a) along i and l
  const char* b;
  int64_t b_sl, b_sj;  // byte strides of op(b) along l and j
  char* c;
  int64_t c_si, c_sj;
  int64_t M, N, K;
};

__global__ void __launch_bounds__(256) small_matmul_kernel(const __grid_constant__ SmallMM p) {
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (t >= p.M * p.N) return;
  const int64_t i = t % p.M, j = t / p.M;
  const char* ap = p.a + i * p.a_si;
  const char* bp = p.b + j * p.b_sj;
  double s = 0.0;
#pragma unroll 8
  for (int64_t l = 0; l < p.K; ++l)
    s = __dadd_rn(s, __dmul_rn(*reinterpret_cast<const double*>(ap + l * p.a_sl),
                               *reinterpret_cast<const double*>(bp + l * p.b_sl)));
  *reinterpret_cast<double*>(p.c + i * p.c_si + j * p.c_sj) = s;
}

bool small_matmul(int64_t M, int64_t N, int64_t K) { return M * N * K <= (1ll << 21) && K <= 4096; }

ftn_status_t run_small_matmul(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, bool ta, bool tb,
                              int64_t M, int64_t N, int64_t K, cudaStream_t s) {
  SmallMM p;
  p.a = (const char*)a->base_addr;
  p.a_si = ta ? a->dim[1].sm : a->dim[0].sm;
  p.a_sl = ta ? a->dim[0].sm : a->dim[1].sm;
  p.b = (const char*)b->base_addr;
  p.b_sl = tb ? b->dim[1].sm : b->dim[0].sm;
  p.b_sj = tb ? b->dim[0].sm : b->dim[1].sm;
  p.c = (char*)c->base_addr;
  p.c_si = c->dim[0].sm;
  p.c_sj = c->dim[1].sm;
  p.M = M;
  p.N = N;
  p.K = K;
  small_matmul_kernel<<<(unsigned)((M * N + 255) / 256), 256, 0, s>>>(p);
  return after_launch("small_matmul_kernel");
}

// c = MATMUL(op(a), op(b)), op = TRANSPOSE when ta / tb.  op(a) is (M, K), op(b) is (K, N).
ftn_status_t run_matmul(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, bool ta, bool tb, char* ws,
                        size_t ws_bytes, cudaStream_t s, bool force_dmma = false) {
  const int64_t M = ta ? a->dim[1].extent : a->dim[0].extent;
  const int64_t K = ta ? a->dim[0].extent : a->dim[1].extent;
  const int64_t N = tb ? b->dim[0].extent : b->dim[1].extent;
  if (M == 0 || N == 0) return FTN_OK;
  if (K == 0) {
    const double zero = 0.0;
    return ftn_fill(c, &zero, s);
  }
  if (!force_dmma && small_matmul(M, N, K)) return run_small_matmul(c, a, b, ta, tb, M, N, K, s);
  ftn_desc_t ap = *a, bp = *b;
  char* w = ws;
  if (!tma_able(a)) {
    w = (char*)(((uintptr_t)w + 255) & ~uintptr_t(255));
    FTN_CHECK(pack(a, w, &ap, s));
    w += pack_bytes(a);
  }
  if (!tma_able(b)) {
    w = (char*)(((uintptr_t)w + 255) & ~uintptr_t(255));
    FTN_CHECK(pack(b, w, &bp, s));
  }
  // boxes: A (M,K) {16 (i), BK}; TRANSPOSE(a) from a (K,M) {16 (l), BM};
  //        B (K,N) {16 (l), BN}; TRANSPOSE(b) from b (N,K) {16 (j), BK}
  CUtensorMap ma, mb;
  FTN_CHECK(make_map(&ma, &ap, 16, ta ? BM : BK));
  FTN_CHECK(make_map(&mb, &bp, 16, tb ? BK : BN));
  MParams p;
  p.c = (char*)c->base_addr;
  p.c_sm0 = c->dim[0].sm;
  p.c_sm1 = c->dim[1].sm;
  p.M = M;
  p.N = N;
  p.K = K;
  p.tiles_m = (M + BM - 1) / BM;
  p.tiles_n = (N + BN - 1) / BN;
  p.kt = (int)((K + BK - 1) / BK);
  const int64_t tiles = p.tiles_m * p.tiles_n;
  p.dp_tiles = tiles;
  p.sk_tiles = 0;
  p.sk_part = nullptr;
  p.sk_cnt = nullptr;
  char* sk = ws ? (char*)(((uintptr_t)w + 255) & ~uintptr_t(255)) : nullptr;
  if (sk && !tma_able(b)) sk += pack_bytes(b);  // after the packed b
  sk = sk ? (char*)(((uintptr_t)sk + 255) & ~uintptr_t(255)) : nullptr;
  const int64_t G = num_sms();
  if (sk && use_stream_k(tiles, p.kt) &&
      (size_t)(sk - ws) + (size_t)2 * G * BM * BN * 8 + (size_t)tiles * 4 <= ws_bytes) {
    p.dp_tiles = (tiles / G - 1) * G;
    p.sk_tiles = tiles - p.dp_tiles;
    p.sk_part = reinterpret_cast<double*>(sk);
    p.sk_cnt = reinterpret_cast<int*>(sk + (size_t)2 * G * BM * BN * 8);
    FTN_CUDA(cudaMemsetAsync(p.sk_cnt, 0, (size_t)p.sk_tiles * 4, s));
  }
  if (!ta && !tb) return launch_gemm<false, false>(ma, mb, p, s);
  if (ta && !tb) return launch_gemm<true, false>(ma, mb, p, s);
  if (!ta && tb) return launch_gemm<false, true>(ma, mb, p, s);
  return launch_gemm<true, true>(ma, mb, p, s);
}

// ---------------------------------------------------------------- rank-1 forms
// y(i) = sum_l a(i,l) x(l): blocks of 256 rows x LC columns; each thread folds its row
// over the column chunk in l order (coalesced over i), partials per chunk go to ws and are
// added in chunk order by a second kernel.  HBM-bound on a: 8 B per element.
constexpr int MV_ROWS = 256;
constexpr int MV_MAXLC = 2048;

struct MVParams {
  const char* a;
  int64_t a_sm0, a_sm1;
  const char* x;
  int64_t x_sm;
  char* y;
  int64_t y_sm;
  double* part;  // [nch][m]
  int64_t m, k, lc, nch;
};

__global__ void __launch_bounds__(MV_ROWS) matvec_kernel(const __grid_constant__ MVParams p) {
  __shared__ double xs[MV_MAXLC];
  const int64_t rb = blockIdx.x, ch = blockIdx.y;
  const int64_t l0 = ch * p.lc, l1 = min(l0 + p.lc, p.k);
  for (int64_t l = l0 + threadIdx.x; l < l1; l += blockDim.x) xs[l - l0] = *reinterpret_cast<const double*>(p.x + l * p.x_sm);
  __syncthreads();
  const int64_t i = rb * MV_ROWS + threadIdx.x;
  if (i >= p.m) return;
  const char* ap = p.a + i * p.a_sm0;
  double acc = 0.0;
  int64_t l = l0;
  for (; l + 8 <= l1; l += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const double*>(ap + (l + u) * p.a_sm1);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double prod = v[u] * xs[l + u - l0];
      acc = acc + prod;
    }
  }
  for (; l < l1; ++l) {
    const double prod = *reinterpret_cast<const double*>(ap + l * p.a_sm1) * xs[l - l0];
    acc = acc + prod;
  }
  if (p.nch == 1) *reinterpret_cast<double*>(p.y + i * p.y_sm) = acc;
  else p.part[ch * p.m + i] = acc;
}

// Packed, 32-byte aligned a with m % 4 == 0: thread owns 4 consecutive rows (one 256-bit
// load per column, a warp covers 128 rows = 1 KB), MV_U columns in flight; every row is
// folded over the chunk in l order exactly as in matvec_kernel (same bits).
#ifndef FTN_MV_U
#define FTN_MV_U 8
#endif
#ifndef FTN_MV4_THREADS
#define FTN_MV4_THREADS 256  // 8192^2: 256 -> 5590, 128 -> 5000-5270, 512 -> 5130 GB/s
#endif
constexpr int MV4_THREADS = FTN_MV4_THREADS, MV4_ROWS = 4 * MV4_THREADS, MV_U = FTN_MV_U;

__global__ void __launch_bounds__(MV4_THREADS) matvec_v4_kernel(const __grid_constant__ MVParams p) {
  __shared__ double xs[MV_MAXLC];
  const int64_t rb = blockIdx.x, ch = blockIdx.y;
  const int64_t l0 = ch * p.lc, l1 = min(l0 + p.lc, p.k);
  for (int64_t l = l0 + threadIdx.x; l < l1; l += blockDim.x) xs[l - l0] = *reinterpret_cast<const double*>(p.x + l * p.x_sm);
  __syncthreads();
  const int64_t i = rb * MV4_ROWS + 4 * threadIdx.x;
  if (i >= p.m) return;
  const double* ap = reinterpret_cast<const double*>(p.a) + i;
  const int64_t ld = p.a_sm1 / 8;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t l = l0;
  for (; l + MV_U <= l1; l += MV_U) {
    double v[MV_U][4];
#pragma unroll
    for (int u = 0; u < MV_U; ++u) dev::ld_v4(ap + (l + u) * ld, v[u][0], v[u][1], v[u][2], v[u][3]);
#pragma unroll
    for (int u = 0; u < MV_U; ++u) {
      const double xv = xs[l + u - l0];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = acc[r] + v[u][r] * xv;
    }
  }
  for (; l < l1; ++l) {
    double v0, v1, v2, v3;
    dev::ld_v4(ap + l * ld, v0, v1, v2, v3);
    const double xv = xs[l - l0];
    acc[0] = acc[0] + v0 * xv;
    acc[1] = acc[1] + v1 * xv;
    acc[2] = acc[2] + v2 * xv;
    acc[3] = acc[3] + v3 * xv;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if (p.nch == 1) *reinterpret_cast<double*>(p.y + (i + r) * p.y_sm) = acc[r];
    else p.part[ch * p.m + i + r] = acc[r];
  }
}

// y(i) = ((part(0,i) + part(1,i)) + part(2,i)) + ...: chunk order; the loads of 8 chunks are
// issued together (they are independent), the additions stay in order.
__global__ void __launch_bounds__(64) matvec_combine(const __grid_constant__ MVParams p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.m; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    int64_t c = 0;
    for (; c + 8 <= p.nch; c += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = p.part[(c + u) * p.m + i];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = acc + v[u];
    }
    for (; c < p.nch; ++c) acc = acc + p.part[c * p.m + i];
    *reinterpret_cast<double*>(p.y + i * p.y_sm) = acc;
  }
}

// Launch plan of the matrix x vector form: the 256-bit path when a is packed, 32-byte aligned
// and m % 4 == 0; column chunks chosen so that the (row block, chunk) blocks spread evenly
// over the SMs (the kernel time is that of the busiest SM) with >= 4 blocks per SM, at a cost
// of 16 B per row and chunk for the partials.
struct MVPlan {
  bool v4;
  int64_t nch, lc, rows_per_block;
};

MVPlan matvec_plan(const ftn_desc_t* a) {
  MVPlan pl;
  const int64_t m = a->dim[0].extent > 0 ? a->dim[0].extent : 1, k = a->dim[1].extent > 0 ? a->dim[1].extent : 1;
  pl.v4 = a->dim[0].sm == 8 && (m % 4) == 0 && (a->dim[1].sm % 32) == 0 && ((uintptr_t)a->base_addr % 32) == 0;
  pl.rows_per_block = pl.v4 ? MV4_ROWS : MV_ROWS;
  const int64_t rblocks = (m + pl.rows_per_block - 1) / pl.rows_per_block;
  const int64_t nsm = 148;
  int64_t best_n = (k + MV_MAXLC - 1) / MV_MAXLC;
  double best = 1e30;
  for (int64_t n = (k + MV_MAXLC - 1) / MV_MAXLC; n <= k; ++n) {
    const int64_t lc = (k + n - 1) / n;
    const int64_t ne = (k + lc - 1) / lc;
    if (ne != n) continue;
    if (lc < 32 && n > 1) break;
    const int64_t units = rblocks * n;
    const int64_t per_sm = (units + nsm - 1) / nsm;
    if (per_sm < 4 && lc > 64) continue;   // too few blocks to hide latency: more chunks
    const double eff = (double)units / (double)(per_sm * nsm);
    const double cost = (1.0 / eff) * (1.0 + (n > 1 ? 2.0 * (double)n / (double)k : 0.0));
    if (cost < best - 1e-9) {
      best = cost;
      best_n = n;
    }
    if (per_sm > 64) break;
  }
  pl.lc = (k + best_n - 1) / best_n;
  pl.nch = (k + pl.lc - 1) / pl.lc;
  return pl;
}

ftn_status_t run_matvec(const ftn_desc_t* y, const ftn_desc_t* a, const ftn_desc_t* x, char* ws, cudaStream_t s) {
  MVParams p;
  p.a = (const char*)a->base_addr;
  p.a_sm0 = a->dim[0].sm;
  p.a_sm1 = a->dim[1].sm;
  p.x = (const char*)x->base_addr;
  p.x_sm = x->dim[0].sm;
  p.y = (char*)y->base_addr;
  p.y_sm = y->dim[0].sm;
  p.m = a->dim[0].extent;
  p.k = a->dim[1].extent;
  if (p.m == 0) return FTN_OK;
  if (p.k == 0) {
    const double zero = 0.0;
    return ftn_fill(y, &zero, s);
  }
  const MVPlan pl = matvec_plan(a);
  p.nch = pl.nch;
  p.lc = pl.lc;
  p.part = reinterpret_cast<double*>(((uintptr_t)ws + 255) & ~uintptr_t(255));
  if (pl.v4) {
    dim3 grid((unsigned)((p.m + MV4_ROWS - 1) / MV4_ROWS), (unsigned)p.nch);
    matvec_v4_kernel<<<grid, MV4_THREADS, 0, s>>>(p);
    FTN_CHECK(after_launch("matvec_v4_kernel"));
  } else {
    dim3 grid((unsigned)((p.m + MV_ROWS - 1) / MV_ROWS), (unsigned)p.nch);
    matvec_kernel<<<grid, MV_ROWS, 0, s>>>(p);
    FTN_CHECK(after_launch("matvec_kernel"));
  }
  if (p.nch > 1) {
    matvec_combine<<<(unsigned)((p.m + 63) / 64), 64, 0, s>>>(p);
    FTN_CHECK(after_launch("matvec_combine"));
  }
  return FTN_OK;
}

// y(j) = sum_l x(l) b(l,j): one warp per column of b (contiguous in l), lanes stride over l,
// then a fixed shfl.xor butterfly.
struct VMParams {
  const char* x;
  int64_t x_sm;
  const char* b;
  int64_t b_sm0, b_sm1;
  char* y;
  int64_t y_sm;
  int64_t k, n;
};

__global__ void __launch_bounds__(256) vecmat_kernel(const __grid_constant__ VMParams p) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < p.n;
       j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const char* bp = p.b + j * p.b_sm1;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t l = lane;
    for (; l + 224 < p.k; l += 256) {  // 8 independent loads of b in flight per lane
      double bv[8], xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        bv[u] = *reinterpret_cast<const double*>(bp + (l + 32 * u) * p.b_sm0);
        xv[u] = __ldg(reinterpret_cast<const double*>(p.x + (l + 32 * u) * p.x_sm));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double prod = xv[u] * bv[u];
        acc[u & 3] = acc[u & 3] + prod;
      }
    }
    for (; l < p.k; l += 32) {
      const double prod = *reinterpret_cast<const double*>(p.x + l * p.x_sm) *
                          *reinterpret_cast<const double*>(bp + l * p.b_sm0);
      acc[0] = acc[0] + prod;
    }
    double v = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int mask = 16; mask >= 1; mask >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, mask);
    if (lane == 0) *reinterpret_cast<double*>(p.y + j * p.y_sm) = v;
  }
}

// Packed, 32-byte aligned operands: lane loads 4 consecutive elements with one 256-bit
// access (a warp covers 1 KB of the column per load), 4 loads in flight per lane;
// accumulator v of a lane takes the elements l = 128 m + 4 lane + v (m = 0, 1, ...), the tail
// elements beyond the last full 128-element block go to accumulator 0 of lane (l / 4) mod 32 in
// order; (a0 + a1) + (a2 + a3), then the fixed xor butterfly.
template <int VU>
__global__ void __launch_bounds__(256) vecmat_v4_kernel(const __grid_constant__ VMParams p) {
  const int lane = threadIdx.x & 31;
  const double* x = reinterpret_cast<const double*>(p.x);
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < p.n;
       j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double* bp = reinterpret_cast<const double*>(p.b + j * p.b_sm1);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const int64_t kfull = p.k / 128 * 128;
    int64_t l = 4 * lane;
    for (; l + 128 * (VU - 1) < kfull; l += 128 * VU) {
      double b[VU][4], xv[VU][4];
#pragma unroll
      for (int u = 0; u < VU; ++u) dev::ld_v4(bp + l + 128 * u, b[u][0], b[u][1], b[u][2], b[u][3]);
#pragma unroll
      for (int u = 0; u < VU; ++u) dev::ldg_v4(x + l + 128 * u, xv[u][0], xv[u][1], xv[u][2], xv[u][3]);
#pragma unroll
      for (int u = 0; u < VU; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[v] = acc[v] + xv[u][v] * b[u][v];
    }
    for (; l < kfull; l += 128) {
      double b0, b1, b2, b3, x0, x1, x2, x3;
      dev::ld_v4(bp + l, b0, b1, b2, b3);
      dev::ldg_v4(x + l, x0, x1, x2, x3);
      acc[0] = acc[0] + x0 * b0;
      acc[1] = acc[1] + x1 * b1;
      acc[2] = acc[2] + x2 * b2;
      acc[3] = acc[3] + x3 * b3;
    }
    for (int64_t e = kfull + 4 * lane; e < p.k; e += 128)
      for (int v = 0; v < 4 && e + v < p.k; ++v) acc[0] = acc[0] + x[e + v] * bp[e + v];
    double s = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int mask = 16; mask >= 1; mask >>= 1) s = s + __shfl_xor_sync(0xffffffffu, s, mask);
    if (lane == 0) *reinterpret_cast<double*>(p.y + j * p.y_sm) = s;
  }
}

// Column per block (default): the 8 warps of a block split one column of b into 8 contiguous
// l ranges (multiples of 128), each folds its range as vecmat_v4_kernel does, and the 8
// partials are combined in a fixed tree -- ~1 K concurrent 64 KB streams instead of one per
// warp.  Deterministic; a different (bound-only) order than vecmat_v4_kernel.
template <int VU>
__global__ void __launch_bounds__(256) vecmat_blk_kernel(const __grid_constant__ VMParams p) {
  __shared__ double part[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* x = reinterpret_cast<const double*>(p.x);
  const int64_t kfull = p.k / 128 * 128;
  const int64_t seg = (kfull / 128 + 7) / 8 * 128;
  const int64_t la = min(kfull, warp * seg), lz = min(kfull, la + seg);
  for (int64_t j = blockIdx.x; j < p.n; j += gridDim.x) {
    const double* bp = reinterpret_cast<const double*>(p.b + j * p.b_sm1);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t l = la + 4 * lane;
    for (; l + 128 * (VU - 1) < lz; l += 128 * VU) {
      double bv[VU][4], xv[VU][4];
#pragma unroll
      for (int u = 0; u < VU; ++u) dev::ld_v4(bp + l + 128 * u, bv[u][0], bv[u][1], bv[u][2], bv[u][3]);
#pragma unroll
      for (int u = 0; u < VU; ++u) dev::ldg_v4(x + l + 128 * u, xv[u][0], xv[u][1], xv[u][2], xv[u][3]);
#pragma unroll
      for (int u = 0; u < VU; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[v] = acc[v] + xv[u][v] * bv[u][v];
    }
    for (; l < lz; l += 128) {
      double b0, b1, b2, b3, x0, x1, x2, x3;
      dev::ld_v4(bp + l, b0, b1, b2, b3);
      dev::ldg_v4(x + l, x0, x1, x2, x3);
      acc[0] = acc[0] + x0 * b0;
      acc[1] = acc[1] + x1 * b1;
      acc[2] = acc[2] + x2 * b2;
      acc[3] = acc[3] + x3 * b3;
    }
    if (warp == 7)
      for (int64_t e = kfull + 4 * lane; e < p.k; e += 128)
        for (int v = 0; v < 4 && e + v < p.k; ++v) acc[0] = acc[0] + x[e + v] * bp[e + v];
    double sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int mask = 16; mask >= 1; mask >>= 1) sum = sum + __shfl_xor_sync(0xffffffffu, sum, mask);
    if (lane == 0) part[warp] = sum;
    __syncthreads();
    if (threadIdx.x == 0)
      *reinterpret_cast<double*>(p.y + j * p.y_sm) =
          ((part[0] + part[1]) + (part[2] + part[3])) + ((part[4] + part[5]) + (part[6] + part[7]));
    __syncthreads();
  }
}

ftn_status_t run_vecmat(const ftn_desc_t* y, const ftn_desc_t* x, const ftn_desc_t* b, cudaStream_t s) {
  VMParams p;
  p.x = (const char*)x->base_addr;
  p.x_sm = x->dim[0].sm;
  p.b = (const char*)b->base_addr;
  p.b_sm0 = b->dim[0].sm;
  p.b_sm1 = b->dim[1].sm;
  p.y = (char*)y->base_addr;
  p.y_sm = y->dim[0].sm;
  p.k = b->dim[0].extent;
  p.n = b->dim[1].extent;
  if (p.n == 0) return FTN_OK;
  int64_t blocks = (p.n * 32 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  const bool v4 = p.b_sm0 == 8 && p.x_sm == 8 && (p.b_sm1 % 32) == 0 && ((uintptr_t)p.b % 32) == 0 &&
                  ((uintptr_t)p.x % 32) == 0;
  static const int vu = getenv("FTN_VM_UNROLL") ? atoi(getenv("FTN_VM_UNROLL")) : 16;  // 8192^2: 16 -> 5650, 8 -> 5190, 4 -> 4510 GB/s
  static const int blk = getenv("FTN_VM_BLK") ? atoi(getenv("FTN_VM_BLK")) : 8;  // 8192^2: 5.95-6.0 vs 5.72 TB/s (one warp per column)
  if (v4 && blk) {
    static const int gm = getenv("FTN_VM_GRIDM") ? atoi(getenv("FTN_VM_GRIDM")) : 8;
    const unsigned g = (unsigned)std::min<int64_t>(p.n, (int64_t)num_sms() * gm);
    if (blk == 4)
      vecmat_blk_kernel<4><<<g, 256, 0, s>>>(p);
    else if (blk == 16)
      vecmat_blk_kernel<16><<<g, 256, 0, s>>>(p);
    else
      vecmat_blk_kernel<8><<<g, 256, 0, s>>>(p);
    return after_launch("vecmat_blk_kernel");
  }
  if (v4) {
    if (vu == 8)
      vecmat_v4_kernel<8><<<(unsigned)blocks, 256, 0, s>>>(p);
    else if (vu == 12)
      vecmat_v4_kernel<12><<<(unsigned)blocks, 256, 0, s>>>(p);
    else if (vu == 16)
      vecmat_v4_kernel<16><<<(unsigned)blocks, 256, 0, s>>>(p);
    else if (vu == 32)
      vecmat_v4_kernel<32><<<(unsigned)blocks, 256, 0, s>>>(p);
    else if (vu == 2)
      vecmat_v4_kernel<2><<<(unsigned)blocks, 256, 0, s>>>(p);
    else
      vecmat_v4_kernel<4><<<(unsigned)blocks, 256, 0, s>>>(p);
    return after_launch("vecmat_v4_kernel");
  }
  vecmat_kernel<<<(unsigned)blocks, 256, 0, s>>>(p);
  return after_launch("vecmat_kernel");
}

// forms: 0 = matrix x matrix, 1 = matrix x vector, 2 = vector x matrix
int form_of(const ftn_desc_t* a, const ftn_desc_t* b) {
  if (a->rank == 2 && b->rank == 2) return 0;
  if (a->rank == 2 && b->rank == 1) return 1;
  return 2;
}

size_t ws_bytes_for(const ftn_desc_t* a, const ftn_desc_t* b) {
  switch (form_of(a, b)) {
    case 1: {
      const int64_t m = a->dim[0].extent, k = a->dim[1].extent;
      return (size_t)(matvec_plan(a).nch * (m > 0 ? m : 1) * 8 + 512);
    }
    case 2: return 0;
  }
  {
    // stream-K partial tiles (either orientation of the operands)
    const int64_t mm = std::max(a->dim[0].extent, a->dim[1].extent), nn = std::max(b->dim[0].extent, b->dim[1].extent);
    const int64_t tiles = ((mm + BM - 1) / BM) * ((nn + BN - 1) / BN);
    const int64_t kk = std::max(a->dim[0].extent, a->dim[1].extent);
    const size_t sk = tiles >= num_sms() && !small_matmul(mm, nn, kk) ? sk_ws_bytes(tiles) : 0;
    return pack_bytes(a) + pack_bytes(b) + 512 + sk;
  }
}

ftn_status_t dispatch(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, bool ta, bool tb, char* ws,
                      size_t ws_bytes, cudaStream_t s, bool force_dmma = false) {
  switch (form_of(a, b)) {
    case 1: return run_matvec(c, a, b, ws, s);
    case 2: return run_vecmat(c, a, b, s);
  }
  return run_matmul(c, a, b, ta, tb, ws, ws_bytes, s, force_dmma);
}

}  // namespace

size_t matmul_ws(const ftn_desc_t* a, const ftn_desc_t* b) { return ws_bytes_for(a, b); }

ftn_status_t matmul_local_ex(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, uint32_t flags, void* ws,
                             size_t ws_bytes, cudaStream_t s) {
  NvtxRange nvtx_("ftn_matmul");
  const bool ta = flags & FTN_MATMUL_TRANSPOSE_A, tb = flags & FTN_MATMUL_TRANSPOSE_B;
  const bool force = flags & FTN_MATMUL_FORCE_DMMA;
  const size_t need = ws_bytes_for(a, b);
  if (need > 512 && (!ws || ws_bytes < need))
    return fail(FTN_ERR_WORKSPACE, "ftn_matmul: workspace too small (see ftn_matmul_workspace_size)");
  if (!desc_overlap(c, a) && !desc_overlap(c, b)) return dispatch(c, a, b, ta, tb, (char*)ws, ws_bytes, s, force);
  StreamTemp tmp;  // R#5: the product is formed before c is defined
  FTN_CHECK(tmp.alloc((size_t)desc_size(c) * 8, s));
  ftn_desc_t t;
  FTN_CHECK(make_packed(&t, tmp.ptr, c));
  FTN_CHECK(dispatch(&t, a, b, ta, tb, (char*)ws, ws_bytes, s, force));
  return launch_copy(c, &t, s);
}

ftn_status_t matmul_local(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, void* ws, size_t ws_bytes,
                          cudaStream_t s) {
  return matmul_local_ex(c, a, b, 0, ws, ws_bytes, s);
}

// F2018 16.9.124: MATMUL(matrix(m,k), matrix(k,n)) -> (m,n); (m,k) x vector(k) -> (m);
// vector(k) x (k,n) -> (n).  TRANSPOSE flags apply to rank-2 operands only.
ftn_status_t check_matmul(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, uint32_t flags = 0) {
  FTN_CHECK(check_desc(c, "ftn_matmul(c)", 1, 2));
  FTN_CHECK(check_desc(a, "ftn_matmul(a)", 1, 2));
  FTN_CHECK(check_desc(b, "ftn_matmul(b)", 1, 2));
  if (a->type != FTN_F64 || b->type != FTN_F64 || c->type != FTN_F64)
    return fail(FTN_ERR_TYPE, "ftn_matmul: real(8) operands only");
  if (flags & ~(uint32_t)(FTN_MATMUL_TRANSPOSE_A | FTN_MATMUL_TRANSPOSE_B | FTN_MATMUL_FORCE_DMMA))
    return fail(FTN_ERR_UNSUPPORTED, "ftn_matmul: unknown flags");
  const bool ta = flags & FTN_MATMUL_TRANSPOSE_A, tb = flags & FTN_MATMUL_TRANSPOSE_B;
  if ((ta && a->rank != 2) || (tb && b->rank != 2))
    return fail(FTN_ERR_RANK, "ftn_matmul: TRANSPOSE needs a rank-2 operand");
  if (a->rank == 1 && b->rank == 1) return fail(FTN_ERR_RANK, "ftn_matmul: at least one operand must be rank 2");
  const int64_t am = a->rank == 2 ? (ta ? a->dim[1].extent : a->dim[0].extent) : -1;
  const int64_t ak = a->rank == 2 ? (ta ? a->dim[0].extent : a->dim[1].extent) : a->dim[0].extent;
  const int64_t bk = b->rank == 2 ? (tb ? b->dim[1].extent : b->dim[0].extent) : b->dim[0].extent;
  const int64_t bn = b->rank == 2 ? (tb ? b->dim[0].extent : b->dim[1].extent) : -1;
  if (ak != bk) return fail(FTN_ERR_SHAPE, "ftn_matmul: inner extents differ");
  if (a->rank == 2 && b->rank == 2) {
    if (c->rank != 2 || c->dim[0].extent != am || c->dim[1].extent != bn)
      return fail(FTN_ERR_SHAPE, "ftn_matmul: c must be (m, n)");
  } else if (a->rank == 2) {
    if (c->rank != 1 || c->dim[0].extent != am) return fail(FTN_ERR_SHAPE, "ftn_matmul: c must be (m)");
  } else {
    if (c->rank != 1 || c->dim[0].extent != bn) return fail(FTN_ERR_SHAPE, "ftn_matmul: c must be (n)");
  }
  return FTN_OK;
}

}  // namespace ftn

using namespace ftn;

extern "C" {

ftn_status_t ftn_matmul_workspace_size(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b,
                                       size_t* bytes) {
  FTN_CHECK(check_matmul(c, a, b));
  if (!bytes) return fail(FTN_ERR_NULL, "ftn_matmul_workspace_size: bytes NULL");
  *bytes = matmul_ws(a, b);
  return FTN_OK;
}

ftn_status_t ftn_matmul(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, void* ws, size_t ws_bytes,
                        ftn_stream_t stream) {
  FTN_CHECK(check_matmul(c, a, b));
  FTN_CHECK(require_sm100());
  return matmul_local(c, a, b, ws, ws_bytes, (cudaStream_t)stream);
}

ftn_status_t ftn_matmul_ex_workspace_size(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b,
                                          uint32_t flags, size_t* bytes) {
  FTN_CHECK(check_matmul(c, a, b, flags));
  if (!bytes) return fail(FTN_ERR_NULL, "ftn_matmul_ex_workspace_size: bytes NULL");
  *bytes = matmul_ws(a, b);
  return FTN_OK;
}

ftn_status_t ftn_matmul_ex(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, uint32_t flags, void* ws,
                           size_t ws_bytes, ftn_stream_t stream) {
  FTN_CHECK(check_matmul(c, a, b, flags));
  FTN_CHECK(require_sm100());
  return matmul_local_ex(c, a, b, flags, ws, ws_bytes, (cudaStream_t)stream);
}

}  // extern "C"
