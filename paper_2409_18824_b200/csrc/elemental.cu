// Element-wise array expressions: dst = src, dst = s,
// dst = a op b, dst = a*b + c, plus the seeded input generator.
//
// The paper's story for these loops: Flang's code did not vectorise;
// the fix was affine loops + `affine-super-vectorize{virtual-vector-size=4}`.
// The B200 counterpart: every thread moves groups of 4 consecutive elements with
// one 256-bit (fp64) / 128-bit (fp32, int32) access when the fast-path
// predicate holds, and the dimensions that are contiguous in every operand are
// merged on the host first (P:281's "static shapes unlock the optimisations",
// done at call time).  HBM-bound: 32 B/element for b*c+d in fp64.
//
// Fortran assignment semantics (R#5): when dst overlaps an operand through any
// mapping other than the identical one, the RHS is evaluated into a temporary.
#include "ftn_internal.cuh"

#include <cstring>
#include <type_traits>

namespace ftn {
namespace {

constexpr int EW_THREADS = 256;
constexpr int EW_GROUP = 4;
constexpr int EW_GROUPS_PER_THREAD = 1;  // + 6 CTAs/SM (<= 40 registers): 1536 threads x 96 B in flight per SM
constexpr int64_t EW_CHUNK = (int64_t)EW_THREADS * EW_GROUP * EW_GROUPS_PER_THREAD;  // 1024

enum { OP_COPY = 0, OP_GEN = 9 };
enum { SC_NONE = 0, SC_DEVICE = 1, SC_VALUE = 2 };

struct EwParams {
  KDesc d[4];          // 0 = dst, 1..3 = operands
  int32_t sc[4];       // scalar kind of each operand
  uint64_t sval[4];    // SC_VALUE bits
  int64_t e0, e1, e2;  // merged extents
  int64_t nchunk0;     // chunks per row
  int64_t items;       // nchunk0 * e1 * e2
  // generator
  uint64_t key;
  uint64_t t0;         // index of the first element in the generator's sequence
  int32_t mode;
};

template <typename T> struct Bits;
template <> struct Bits<double> { typedef unsigned long long U; };
template <> struct Bits<int64_t> { typedef unsigned long long U; };
template <> struct Bits<float> { typedef unsigned int U; };
template <> struct Bits<int32_t> { typedef unsigned int U; };

template <typename T>
__device__ __forceinline__ void ld4(const char* p, T* v) {
  if constexpr (sizeof(T) == 8) {
    unsigned long long a, b, c, d;
    asm volatile("ld.global.L1::no_allocate.v4.b64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
    unsigned long long t[4] = {a, b, c, d};
    memcpy(v, t, 32);
  } else {
    unsigned int a, b, c, d;
    asm volatile("ld.global.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "l"(p));
    unsigned int t[4] = {a, b, c, d};
    memcpy(v, t, 16);
  }
}
template <typename T>
__device__ __forceinline__ void st4(char* p, const T* v) {
  if constexpr (sizeof(T) == 8) {
    unsigned long long t[4];
    memcpy(t, v, 32);
    asm volatile("st.global.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(t[0]), "l"(t[1]), "l"(t[2]), "l"(t[3])
                 : "memory");
  } else {
    unsigned int t[4];
    memcpy(t, v, 16);
    asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3])
                 : "memory");
  }
}

// ---- the operation on one element (IEEE RN; -fmad=false: no contraction unless CONTRACT)
template <typename T, int OP, bool CONTRACT>
__device__ __forceinline__ T apply(T a, T b, T c) {
  if constexpr (OP == OP_COPY) {
    return a;
  } else if constexpr (std::is_floating_point<T>::value) {
    if constexpr (OP == FTN_ADD) return a + b;
    if constexpr (OP == FTN_SUB) return a - b;
    if constexpr (OP == FTN_MUL) return a * b;
    if constexpr (OP == FTN_DIV) return a / b;
    if constexpr (OP == FTN_MULADD) {
      if constexpr (CONTRACT) return fma(a, b, c);
      T p = a * b;
      return p + c;
    }
  } else {
    typedef typename Bits<T>::U U;  // modulo 2^w
    if constexpr (OP == FTN_ADD) return (T)((U)a + (U)b);
    if constexpr (OP == FTN_SUB) return (T)((U)a - (U)b);
    if constexpr (OP == FTN_MUL) return (T)((U)a * (U)b);
    if constexpr (OP == FTN_DIV) return a / b;  // truncating toward zero
    if constexpr (OP == FTN_MULADD) return (T)((U)a * (U)b + (U)c);
  }
  return a;
}

// ---- splitmix64 generator, independent of synth/ (numpy)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
template <typename T>
__device__ __forceinline__ T gen_value(uint64_t key, int mode, uint64_t t) {
  if (mode == FTN_GEN_LINEAR) return (T)(int64_t)t;
  if (mode == FTN_GEN_MOD1024) return (T)(int64_t)(t & 1023u);
  const uint64_t h = splitmix64(key ^ t);
  if constexpr (std::is_floating_point<T>::value) {
    const double u = (double)(h >> 11) * 0x1.0p-53;
    if (mode == FTN_GEN_U01) return (T)u;
    if (mode == FTN_GEN_U11) return (T)(2.0 * u - 1.0);
    if (mode == FTN_GEN_INT8) return (T)((int64_t)((h >> 11) % 17u) - 8);
    return (T)0;
  } else {
    if (mode == FTN_GEN_INT8) return (T)((int64_t)((h >> 11) % 17u) - 8);
    if (mode == FTN_GEN_RAW) return (T)h;
    return (T)(h >> 11);
  }
}

template <typename T>
__device__ __forceinline__ T load_scalar(const EwParams& p, int a) {
  if (p.sc[a] == SC_VALUE) {
    T v;
    memcpy(&v, &p.sval[a], sizeof(T));
    return v;
  }
  return *reinterpret_cast<const T*>(p.d[a].base);
}

// One work item = EW_CHUNK consecutive elements of one merged "row" (dim 0).
// Thread tau handles the group at offset 4*tau.
template <typename T, int OP, bool CONTRACT, bool VEC, int NOPS>
__global__ void __launch_bounds__(EW_THREADS, 6) ew_kernel(const __grid_constant__ EwParams p) {
  const int64_t G = gridDim.x;
  int64_t c = blockIdx.x % p.nchunk0;
  int64_t r = blockIdx.x / p.nchunk0;
  int64_t i1 = r % p.e1, i2 = r / p.e1;
  const int64_t dc = G % p.nchunk0, dr = G / p.nchunk0;
  const int64_t dr1 = dr % p.e1, dr2 = dr / p.e1;

  T s[4];
#pragma unroll
  for (int a = 1; a <= NOPS; ++a) s[a] = p.sc[a] != SC_NONE ? load_scalar<T>(p, a) : T(0);

  for (int64_t w = blockIdx.x; w < p.items; w += G) {
    const int64_t base0 = c * EW_CHUNK;
    char* rowp[4];
#pragma unroll
    for (int a = 0; a <= NOPS; ++a) rowp[a] = p.d[a].base + i1 * p.d[a].sm[1] + i2 * p.d[a].sm[2];

    T v[EW_GROUPS_PER_THREAD][4][EW_GROUP];  // [group][operand][elem]
#pragma unroll
    for (int g = 0; g < EW_GROUPS_PER_THREAD; ++g) {
      const int64_t i0 = base0 + g * (EW_THREADS * EW_GROUP) + EW_GROUP * threadIdx.x;
      if (i0 >= p.e0) continue;
      const bool full = VEC && (i0 + EW_GROUP <= p.e0);
#pragma unroll
      for (int a = 1; a <= NOPS; ++a) {
        if (p.sc[a] != SC_NONE) {
#pragma unroll
          for (int e = 0; e < EW_GROUP; ++e) v[g][a][e] = s[a];
        } else if (full) {
          ld4<T>(rowp[a] + i0 * p.d[a].sm[0], v[g][a]);
        } else {
#pragma unroll
          for (int e = 0; e < EW_GROUP; ++e)
            if (i0 + e < p.e0) v[g][a][e] = *reinterpret_cast<const T*>(rowp[a] + (i0 + e) * p.d[a].sm[0]);
        }
      }
    }
#pragma unroll
    for (int g = 0; g < EW_GROUPS_PER_THREAD; ++g) {
      const int64_t i0 = base0 + g * (EW_THREADS * EW_GROUP) + EW_GROUP * threadIdx.x;
      if (i0 >= p.e0) continue;
      T out[EW_GROUP];
#pragma unroll
      for (int e = 0; e < EW_GROUP; ++e) {
        if constexpr (OP == OP_GEN) {
          const uint64_t t = p.t0 + (uint64_t)(i0 + e) + (uint64_t)p.e0 * (uint64_t)(i1 + p.e1 * i2);
          out[e] = gen_value<T>(p.key, p.mode, t);
        } else {
          out[e] = apply<T, OP, CONTRACT>(v[g][1][e], NOPS >= 2 ? v[g][2][e] : T(0), NOPS >= 3 ? v[g][3][e] : T(0));
        }
      }
      if (VEC && i0 + EW_GROUP <= p.e0) {
        st4<T>(rowp[0] + i0 * p.d[0].sm[0], out);
      } else {
#pragma unroll
        for (int e = 0; e < EW_GROUP; ++e)
          if (i0 + e < p.e0) *reinterpret_cast<T*>(rowp[0] + (i0 + e) * p.d[0].sm[0]) = out[e];
      }
    }
    // advance (c, i1, i2) by G items without dividing
    c += dc;
    i1 += dr1;
    i2 += dr2;
    if (c >= p.nchunk0) { c -= p.nchunk0; ++i1; }
    if (i1 >= p.e1) { i1 -= p.e1; ++i2; }
  }
}

template <typename T, int OP, bool CONTRACT, int NOPS>
ftn_status_t launch_t(const EwParams& p, bool vec, cudaStream_t stream) {
  if (p.items == 0) return FTN_OK;
  const int64_t max_blocks = (int64_t)num_sms() * (2048 / EW_THREADS) * 8;
  const int blocks = (int)(p.items < max_blocks ? p.items : max_blocks);
  if (vec)
    ew_kernel<T, OP, CONTRACT, true, NOPS><<<blocks, EW_THREADS, 0, stream>>>(p);
  else
    ew_kernel<T, OP, CONTRACT, false, NOPS><<<blocks, EW_THREADS, 0, stream>>>(p);
  return after_launch("ew_kernel");
}

template <typename T>
ftn_status_t dispatch_op(int op, bool contract, const EwParams& p, bool vec, cudaStream_t s) {
  switch (op) {
    case OP_COPY: return launch_t<T, OP_COPY, false, 1>(p, vec, s);
    case OP_GEN: return launch_t<T, OP_GEN, false, 0>(p, vec, s);
    case FTN_ADD: return launch_t<T, FTN_ADD, false, 2>(p, vec, s);
    case FTN_SUB: return launch_t<T, FTN_SUB, false, 2>(p, vec, s);
    case FTN_MUL: return launch_t<T, FTN_MUL, false, 2>(p, vec, s);
    case FTN_DIV: return launch_t<T, FTN_DIV, false, 2>(p, vec, s);
    case FTN_MULADD:
      if (contract) return launch_t<T, FTN_MULADD, true, 3>(p, vec, s);
      return launch_t<T, FTN_MULADD, false, 3>(p, vec, s);
  }
  return fail(FTN_ERR_UNSUPPORTED, "elemental: unknown op");
}

// Build params from dst + operands (operands may be rank 0 = device scalar or
// value scalars passed via sval/sc) and launch.
ftn_status_t run(int op, bool contract, const ftn_desc_t* dst, const ftn_desc_t* const* ops, int nops,
                 const uint64_t* svals, const int* sc_override, uint64_t key, int mode, cudaStream_t stream,
                 uint64_t t0 = 0) {
  EwParams p;
  memset(&p, 0, sizeof(p));
  const ftn_desc_t* arrays[4] = {dst, nullptr, nullptr, nullptr};
  ftn_desc_t scalar_stub;
  memset(&scalar_stub, 0, sizeof(scalar_stub));
  for (int a = 0; a < nops; ++a) {
    if (sc_override && sc_override[a] == SC_VALUE) {
      scalar_stub.rank = 0;
      arrays[a + 1] = &scalar_stub;
    } else {
      arrays[a + 1] = ops[a];
    }
  }
  KDesc kd[4];
  collapse(arrays, nops + 1, kd);
  for (int a = 0; a <= nops; ++a) p.d[a] = kd[a];
  for (int a = 0; a < nops; ++a) {
    if (sc_override && sc_override[a] == SC_VALUE) {
      p.sc[a + 1] = SC_VALUE;
      p.sval[a + 1] = svals[a];
    } else if (ops[a]->rank == 0) {
      p.sc[a + 1] = SC_DEVICE;
      p.d[a + 1].base = (char*)ops[a]->base_addr;
    }
  }
  p.e0 = kd[0].ext[0];
  p.e1 = kd[0].ext[1];
  p.e2 = kd[0].ext[2];
  p.nchunk0 = (p.e0 + EW_CHUNK - 1) / EW_CHUNK;
  p.items = p.nchunk0 * p.e1 * p.e2;
  if (desc_size(dst) == 0) p.items = 0;
  p.key = key;
  p.t0 = t0;
  p.mode = mode;
  // vector fast path: every array has unit-stride dim 0 and group-aligned rows
  const int64_t el = dst->elem_len, va = EW_GROUP * el;
  bool vec = true;
  for (int a = 0; a <= nops; ++a) {
    if (a > 0 && p.sc[a] != SC_NONE) continue;
    const KDesc& k = p.d[a];
    if (k.ext[0] > 1 && k.sm[0] != el) vec = false;
    if (((uintptr_t)k.base) % va) vec = false;
    if (k.sm[1] % va || k.sm[2] % va) vec = false;
  }
  switch (dst->type) {
    case FTN_F64: return dispatch_op<double>(op, contract, p, vec, stream);
    case FTN_F32: return dispatch_op<float>(op, contract, p, vec, stream);
    case FTN_I32: return dispatch_op<int32_t>(op, contract, p, vec, stream);
    case FTN_I64: return dispatch_op<int64_t>(op, contract, p, vec, stream);
  }
  return fail(FTN_ERR_TYPE, "elemental: type");
}

ftn_status_t check_operand(const ftn_desc_t* dst, const ftn_desc_t* x, const char* name) {
  FTN_CHECK(check_desc(x, name, 0, FTN_MAX_RANK));
  if (x->type != dst->type) return fail(FTN_ERR_TYPE, std::string(name) + ": type differs from dst");
  if (x->rank == 0) {
    if (!x->base_addr) return fail(FTN_ERR_NULL, std::string(name) + ": scalar base NULL");
    return FTN_OK;
  }
  if (!same_shape(dst, x)) return fail(FTN_ERR_SHAPE, std::string(name) + ": not conformable with dst");
  return FTN_OK;
}

bool needs_temp(const ftn_desc_t* dst, const ftn_desc_t* const* ops, int nops) {
  for (int a = 0; a < nops; ++a) {
    const ftn_desc_t* x = ops[a];
    if (x->rank == 0) {
      uintptr_t lo, hi;
      desc_byte_range(dst, &lo, &hi);
      uintptr_t s = (uintptr_t)x->base_addr;
      if (desc_size(dst) > 0 && s + x->elem_len > lo && s < hi) return true;
      continue;
    }
    if (desc_overlap(dst, x) && !desc_identical(dst, x)) return true;
  }
  return false;
}

}  // namespace

ftn_status_t launch_elementwise(int32_t op, const ftn_desc_t* dst, const ftn_desc_t* a, const ftn_desc_t* b,
                                const ftn_desc_t* c, uint32_t flags, cudaStream_t stream) {
  const ftn_desc_t* ops[3] = {a, b, c};
  const int nops = op == OP_COPY ? 1 : (op == FTN_MULADD ? 3 : 2);
  if (!needs_temp(dst, ops, nops))
    return run(op, flags & FTN_CONTRACT, dst, ops, nops, nullptr, nullptr, 0, 0, stream);
  // R#5: evaluate the RHS into a packed temporary, then store it
  StreamTemp tmp;
  FTN_CHECK(tmp.alloc((size_t)desc_size(dst) * dst->elem_len, stream));
  ftn_desc_t t;
  FTN_CHECK(make_packed(&t, tmp.ptr, dst));
  FTN_CHECK(run(op, flags & FTN_CONTRACT, &t, ops, nops, nullptr, nullptr, 0, 0, stream));
  const ftn_desc_t* src[1] = {&t};
  return run(OP_COPY, false, dst, src, 1, nullptr, nullptr, 0, 0, stream);
}

ftn_status_t launch_copy(const ftn_desc_t* dst, const ftn_desc_t* src, cudaStream_t stream) {
  return launch_elementwise(OP_COPY, dst, src, nullptr, nullptr, 0, stream);
}

}  // namespace ftn

using namespace ftn;

extern "C" {

ftn_status_t ftn_assign(const ftn_desc_t* dst, const ftn_desc_t* src, ftn_stream_t stream) {
  FTN_CHECK(check_desc(dst, "ftn_assign(dst)", 1, FTN_MAX_RANK));
  FTN_CHECK(check_operand(dst, src, "ftn_assign(src)"));
  FTN_CHECK(require_sm100());
  return launch_copy(dst, src, (cudaStream_t)stream);
}

ftn_status_t ftn_fill(const ftn_desc_t* dst, const void* scalar_host, ftn_stream_t stream) {
  FTN_CHECK(check_desc(dst, "ftn_fill(dst)", 1, FTN_MAX_RANK));
  if (!scalar_host) return fail(FTN_ERR_NULL, "ftn_fill: scalar_host NULL");
  FTN_CHECK(require_sm100());
  uint64_t v = 0;
  memcpy(&v, scalar_host, (size_t)dst->elem_len);
  int sc = SC_VALUE;
  const ftn_desc_t* ops[1] = {nullptr};
  return run(OP_COPY, false, dst, ops, 1, &v, &sc, 0, 0, (cudaStream_t)stream);
}

ftn_status_t ftn_elemental(int32_t op, const ftn_desc_t* dst, const ftn_desc_t* a, const ftn_desc_t* b,
                           const ftn_desc_t* c, uint32_t flags, ftn_stream_t stream) {
  FTN_CHECK(check_desc(dst, "ftn_elemental(dst)", 1, FTN_MAX_RANK));
  if (op < FTN_ADD || op > FTN_MULADD) return fail(FTN_ERR_UNSUPPORTED, "ftn_elemental: unknown op");
  FTN_CHECK(check_operand(dst, a, "ftn_elemental(a)"));
  FTN_CHECK(check_operand(dst, b, "ftn_elemental(b)"));
  if (op == FTN_MULADD) FTN_CHECK(check_operand(dst, c, "ftn_elemental(c)"));
  if ((flags & ~FTN_CONTRACT) != 0) return fail(FTN_ERR_UNSUPPORTED, "ftn_elemental: unknown flags");
  FTN_CHECK(require_sm100());
  return launch_elementwise(op, dst, a, b, c, flags, (cudaStream_t)stream);
}

ftn_status_t ftn_gen_fill(const ftn_desc_t* dst, uint64_t seed, uint64_t array_id, int32_t mode,
                          ftn_stream_t stream) {
  return ftn_gen_fill_at(dst, seed, array_id, mode, 0, stream);
}

ftn_status_t ftn_gen_fill_at(const ftn_desc_t* dst, uint64_t seed, uint64_t array_id, int32_t mode, uint64_t t0,
                             ftn_stream_t stream) {
  FTN_CHECK(check_desc(dst, "ftn_gen_fill(dst)", 1, FTN_MAX_RANK));
  if (mode < FTN_GEN_U01 || mode > FTN_GEN_RAW) return fail(FTN_ERR_UNSUPPORTED, "ftn_gen_fill: mode");
  const bool is_real = dst->type == FTN_F32 || dst->type == FTN_F64;
  if (mode == FTN_GEN_RAW && is_real) return fail(FTN_ERR_TYPE, "ftn_gen_fill: RAW is for integer types");
  if ((mode == FTN_GEN_U01 || mode == FTN_GEN_U11) && !is_real)
    return fail(FTN_ERR_TYPE, "ftn_gen_fill: U01/U11 are for real types");
  FTN_CHECK(require_sm100());
  const ftn_desc_t* ops[1] = {nullptr};
  return run(OP_GEN, false, dst, ops, 0, nullptr, nullptr, seed ^ (array_id << 56), mode, (cudaStream_t)stream, t0);
}

}  // extern "C"
