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
// Shared-memory layout (conflict-free fragment loads):
//   A stage = 8 TMA boxes {16 (i), 32 (l)}, B stage = 2 boxes {16 (l), 128 (j)},
//   all with the 128-byte swizzle.  Fortran A is i-fastest, but the m16n8k4 A
//   fragment puts k across lanes; the MMA's k index t is therefore mapped to the
//   physical l offset {0,4,1,5} (first k4 of each 8) and {2,6,3,7} (second),
//   which with the swizzle spreads the four t-rows over all 32 banks.  The same
//   permutation is applied to B, so each product a(i,l) b(l,j) is still formed
//   for every l exactly once.
#include "ftn_internal.cuh"

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

__global__ void __launch_bounds__(THREADS, 1)
    dmma_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const __grid_constant__ MParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // grouped raster for L2 reuse of A row-panels and B column-panels
  const int64_t b = blockIdx.x;
  const int64_t per_group = GROUP_M * p.tiles_n;
  const int64_t first_m = (b / per_group) * GROUP_M;
  const int64_t gsz = min((int64_t)GROUP_M, p.tiles_m - first_m);
  const int64_t tm = first_m + (b % per_group) % gsz;
  const int64_t tn = (b % per_group) / gsz;
  const int m0 = (int)(tm * BM), n0 = (int)(tn * BN);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], MMA_WARPS);
    }
    dev::fence_barrier_init();
  }
  __syncthreads();

  // TMA producer: lane 0 of warp 0
  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    if (kt >= STAGES) dev::mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
    uint8_t* st = smem + s * STAGE_BYTES;
    dev::mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
    const int k0 = kt * BK;
#pragma unroll
    for (int a = 0; a < BM / 16; ++a) dev::tma_load_2d(st + a * A_BOX_BYTES, &map_a, &full[s], m0 + 16 * a, k0);
#pragma unroll
    for (int h = 0; h < BK / 16; ++h)
      dev::tma_load_2d(st + A_STAGE + h * B_BOX_BYTES, &map_b, &full[s], k0 + 16 * h, n0);
  };
  const bool producer = (warp == 0 && lane == 0);
  if (producer) {
    dev::prefetch_tma(&map_a);
    dev::prefetch_tma(&map_b);
    for (int kt = 0; kt < STAGES - 1 && kt < p.kt; ++kt) issue(kt);
  }
  __syncwarp();

  // ---------------- MMA warps
  const int wm = warp >> 2;  // 0..1 -> rows wm*64
  const int wn = warp & 3;   // 0..3 -> cols wn*32
  const int g = lane >> 2, t = lane & 3;
  double acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

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
      const uint32_t box = wm * 4 + mt;
      a_off[q][mt][0] = box * A_BOX_BYTES + swz(l, g);
      a_off[q][mt][1] = box * A_BOX_BYTES + swz(l, g + 8);
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) b_off[q][nt] = A_STAGE + swz(wn * 32 + nt * 8 + g, l);
  }

  for (int kt = 0; kt < p.kt; ++kt) {
    const int s = kt % STAGES;
    if (producer && kt + STAGES - 1 < p.kt) issue(kt + STAGES - 1);  // refills the stage freed at kt-1
    __syncwarp();
    dev::mbar_wait(&full[s], (kt / STAGES) & 1);
    const uint32_t st = smem_base + s * STAGE_BYTES;
#pragma unroll
    for (int kb = 0; kb < BK / 8; ++kb) {
      // A: row l = kb*8 + phys -> +kb*8 rows (the swizzle phase (row & 7) is unchanged)
      // B: x = (kb & 1) * 8 + phys in box kb >> 1 -> +8 doubles = +4 chunks: XOR by 4 commutes
      const uint32_t a_kb = kb * 8 * 128;
      const uint32_t b_kb = (kb >> 1) * B_BOX_BYTES;
      const uint32_t b_x = (kb & 1) ? 64u : 0u;  // chunk index ^ 4 == byte offset ^ 64
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        double af[4][2], bf[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          af[mt][0] = *reinterpret_cast<const double*>(smem_raw + st + a_kb + a_off[q][mt][0]);
          af[mt][1] = *reinterpret_cast<const double*>(smem_raw + st + a_kb + a_off[q][mt][1]);
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

  // ---------------- epilogue: c(i, j) through the descriptor strides
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

ftn_status_t run_matmul(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, char* ws, cudaStream_t s) {
  const int64_t M = a->dim[0].extent, K = a->dim[1].extent, N = b->dim[1].extent;
  if (M == 0 || N == 0) return FTN_OK;
  if (K == 0) {
    const double zero = 0.0;
    return ftn_fill(c, &zero, s);
  }
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
  CUtensorMap ma, mb;
  FTN_CHECK(make_map(&ma, &ap, 16, BK));
  FTN_CHECK(make_map(&mb, &bp, 16, BN));
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
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    FTN_CUDA(cudaFuncSetAttribute(dmma_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    attr_set[dev & 63] = true;
  }
  const int64_t tiles = p.tiles_m * p.tiles_n;
  dmma_gemm_kernel<<<(unsigned)tiles, THREADS, SMEM_BYTES, s>>>(ma, mb, p);
  return after_launch("dmma_gemm_kernel");
}

}  // namespace

size_t matmul_ws(const ftn_desc_t* a, const ftn_desc_t* b) { return pack_bytes(a) + pack_bytes(b) + 512; }

ftn_status_t matmul_local(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, void* ws, size_t ws_bytes,
                          cudaStream_t s) {
  const size_t need = pack_bytes(a) + pack_bytes(b);
  if (need && (!ws || ws_bytes < matmul_ws(a, b)))
    return fail(FTN_ERR_WORKSPACE, "ftn_matmul: workspace too small (see ftn_matmul_workspace_size)");
  if (!desc_overlap(c, a) && !desc_overlap(c, b)) return run_matmul(c, a, b, (char*)ws, s);
  StreamTemp tmp;  // R#5: the product is formed before c is defined
  FTN_CHECK(tmp.alloc((size_t)desc_size(c) * 8, s));
  ftn_desc_t t;
  FTN_CHECK(make_packed(&t, tmp.ptr, c));
  FTN_CHECK(run_matmul(&t, a, b, (char*)ws, s));
  return launch_copy(c, &t, s);
}

ftn_status_t check_matmul(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b) {
  FTN_CHECK(check_desc(c, "ftn_matmul(c)", 1, 2));
  FTN_CHECK(check_desc(a, "ftn_matmul(a)", 1, 2));
  FTN_CHECK(check_desc(b, "ftn_matmul(b)", 1, 2));
  if (a->rank != 2 || b->rank != 2 || c->rank != 2)
    return fail(FTN_ERR_UNSUPPORTED, "ftn_matmul: rank-1 (matrix-vector) forms are not implemented yet");
  if (a->type != FTN_F64 || b->type != FTN_F64 || c->type != FTN_F64)
    return fail(FTN_ERR_TYPE, "ftn_matmul: real(8) operands only");
  if (b->dim[0].extent != a->dim[1].extent || c->dim[0].extent != a->dim[0].extent ||
      c->dim[1].extent != b->dim[1].extent)
    return fail(FTN_ERR_SHAPE, "ftn_matmul: shapes (m,k) x (k,n) -> (m,n) do not match");
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

}  // extern "C"
