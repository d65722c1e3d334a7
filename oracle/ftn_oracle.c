/*
 * oracle/ftn_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, sequential CPU evaluation of the Fortran array statements that
 * arXiv 2409.18824 ("Fully integrating the Flang Fortran compiler with standard
 * MLIR") lowers to memref/scf/affine/linalg.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA library
 * (paper_2409_18824_b200/csrc, include/ftn.h) and neither side includes the other.
 *
 * Citation keys: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n,
 * "R#n" = reading n of DESIGN.md section 3 (ambiguities resolved there).
 *
 * Conventions (all from the paper's statement of the lowering):
 *   - An array is a descriptor {base, type, rank, dim[d] = {lb, ext, sm}}.
 *     base is the address of element (lb_1, ..., lb_r); sm is a signed byte
 *     stride.  Element (j_1..j_r) lives at base + sum_d (j_d - lb_d) * sm_d:
 *     the origin subtraction of P:233 done once per access.
 *   - Array element order is column-major: the first subscript varies fastest
 *     (R#1).  Every loop below walks that order with an explicit odometer.
 *   - Floating point: built with -O2 -ffp-contract=off, never -ffast-math, so
 *     every + and * below is one IEEE-754 binary64/binary32 operation rounded to
 *     nearest-even, exactly as written (R#19).  Integer arithmetic wraps modulo
 *     2^w (R#9) -- done in unsigned types so C has no UB.
 *
 * Parity status: every exported function is pinned by tests/test_oracle_*.py
 * (closed forms, brute force, math.fsum, numpy routines, invariants).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAXRANK 3

enum { ORC_I32 = 1, ORC_I64 = 2, ORC_F32 = 3, ORC_F64 = 4 };
enum { ORC_OK = 0, ORC_EBOUNDS = 5, ORC_ESHAPE = 4, ORC_ERANK = 2, ORC_ETYPE = 3, ORC_ESTEP = 6 };
enum { ORC_ADD = 1, ORC_SUB = 2, ORC_MUL = 3, ORC_DIV = 4, ORC_MULADD = 5 };

typedef struct { int64_t lb, ext, sm; } orc_dim;
typedef struct {
  char* base;      /* address of element (lb_1, ..., lb_r) */
  int32_t type;
  int32_t rank;    /* 0 = scalar */
  orc_dim dim[ORC_MAXRANK];
} orc_array;

static int64_t elem_len(int32_t type) { return (type == ORC_I32 || type == ORC_F32) ? 4 : 8; }

static int64_t total_size(const orc_array* a) {
  int64_t n = 1;
  for (int d = 0; d < a->rank; ++d) n *= a->dim[d].ext;
  return n;
}

/* Address of the element whose 0-based position in dimension d is k[d]
 * (k[d] = j_d - lb_d): P:233's "subtraction of the index from its starting index". */
static char* addr_of(const orc_array* a, const int64_t* k) {
  char* p = a->base;
  for (int d = 0; d < a->rank; ++d) p += k[d] * a->dim[d].sm;
  return p;
}

/* Advance a column-major odometer over extents ext[0..rank-1]. */
static void odometer_next(int64_t* k, const orc_array* a) {
  for (int d = 0; d < a->rank; ++d) {
    if (++k[d] < a->dim[d].ext) return;
    k[d] = 0;
  }
}

/* Address of the t-th element in array element order (0-based t). */
static char* addr_linear(const orc_array* a, int64_t t) {
  int64_t k[ORC_MAXRANK] = {0, 0, 0};
  for (int d = 0; d < a->rank; ++d) { k[d] = t % a->dim[d].ext; t /= a->dim[d].ext; }
  return addr_of(a, k);
}

/* ------------------------------------------------------------------------ */
/* Sections: x(lo:hi:step, ...)                                              */
/* P:237 (slices are memref subviews: same memory, new offsets/sizes/strides), */
/* P:191 (Fortran DO/triplet semantics with negative steps).    */
/* Extent = max(0, (hi - lo + step) / step); the section's lbounds are 1 (R#2); */
/* zero step or an out-of-parent selected element is an error. */
/* ------------------------------------------------------------------------ */
int orc_section(const orc_array* parent, const int64_t* lo, const int64_t* hi,
                const int64_t* step, orc_array* out) {
  orc_array r = *parent;
  char* base = parent->base;
  for (int d = 0; d < parent->rank; ++d) {
    if (step[d] == 0) return ORC_ESTEP;
    int64_t n = (hi[d] - lo[d] + step[d]) / step[d];
    if (n < 0) n = 0;
    const int64_t lb = parent->dim[d].lb, ub = parent->dim[d].lb + parent->dim[d].ext - 1;
    if (n > 0) {
      const int64_t first = lo[d], last = lo[d] + (n - 1) * step[d];
      if (first < lb || first > ub || last < lb || last > ub) return ORC_EBOUNDS;
      base += (first - lb) * parent->dim[d].sm;
    }
    r.dim[d].lb = 1;
    r.dim[d].ext = n;
    r.dim[d].sm = step[d] * parent->dim[d].sm;
  }
  r.base = base;
  *out = r;
  return ORC_OK;
}

/* Enumerate the parent subscripts a triplet selects, in order:
 * writes up to cap values into idx and returns the count. */
int64_t orc_triplet_indices(int64_t lo, int64_t hi, int64_t step, int64_t* idx, int64_t cap) {
  if (step == 0) return -1;
  int64_t n = 0;
  if (step > 0) {
    for (int64_t i = lo; i <= hi; i += step) { if (n < cap) idx[n] = i; ++n; }
  } else {
    for (int64_t i = lo; i >= hi; i += step) { if (n < cap) idx[n] = i; ++n; }
  }
  return n;
}

/* Byte offset of element (j_1..j_r) from base (P:233 worked example: data(2) with
 * lbound 1 -> index 1). */
int64_t orc_element_offset(const orc_array* a, const int64_t* j) {
  int64_t off = 0;
  for (int d = 0; d < a->rank; ++d) off += (j[d] - a->dim[d].lb) * a->dim[d].sm;
  return off;
}

/* ------------------------------------------------------------------------ */
/* Assignment and element-wise expressions.                                 */
/* Fortran assignment: the whole right-hand side is evaluated before any    */
/* element of the left-hand side is defined (R#5), so we evaluate into a    */
/* fresh temporary in array element order, then store in that order.        */
/* Scalars (rank 0) broadcast.                                               */
/* ------------------------------------------------------------------------ */
static int conformable(const orc_array* dst, const orc_array* s) {
  if (s->rank == 0) return 1;
  if (s->rank != dst->rank) return 0;
  for (int d = 0; d < dst->rank; ++d) if (s->dim[d].ext != dst->dim[d].ext) return 0;
  return 1;
}

static char* operand_addr(const orc_array* s, const int64_t* k) {
  return s->rank == 0 ? s->base : addr_of(s, k);
}

/* dst = a op b   (op in ADD SUB MUL DIV)   or   dst = a*b + c  (MULADD).
 * contract != 0 -> MULADD is one fused multiply-add, single rounding (P:152
 * lists math-uplift-to-fma; R#6).  Default: fl(fl(a*b) + c). */
int orc_elemental(int32_t op, const orc_array* dst, const orc_array* a, const orc_array* b,
                  const orc_array* c, int32_t contract) {
  if (dst->rank < 1 || dst->rank > ORC_MAXRANK) return ORC_ERANK;
  const orc_array* ops[3] = {a, b, c};
  const int nops = (op == ORC_MULADD) ? 3 : 2;
  for (int i = 0; i < nops; ++i) {
    if (ops[i]->type != dst->type) return ORC_ETYPE;
    if (!conformable(dst, ops[i])) return ORC_ESHAPE;
  }
  const int64_t n = total_size(dst), el = elem_len(dst->type);
  char* tmp = (char*)malloc((size_t)(n > 0 ? n : 1) * (size_t)el);
  int64_t k[ORC_MAXRANK] = {0, 0, 0};
  for (int64_t t = 0; t < n; ++t, odometer_next(k, dst)) {
    const char* pa = operand_addr(a, k);
    const char* pb = operand_addr(b, k);
    const char* pc = nops == 3 ? operand_addr(c, k) : NULL;
    char* pt = tmp + t * el;
    switch (dst->type) {
      case ORC_F64: {
        double x = *(const double*)pa, y = *(const double*)pb, r = 0;
        if (op == ORC_ADD) r = x + y;
        else if (op == ORC_SUB) r = x - y;
        else if (op == ORC_MUL) r = x * y;
        else if (op == ORC_DIV) r = x / y;
        else { double z = *(const double*)pc; if (contract) r = fma(x, y, z); else { double p = x * y; r = p + z; } }
        *(double*)pt = r; break;
      }
      case ORC_F32: {
        float x = *(const float*)pa, y = *(const float*)pb, r = 0;
        if (op == ORC_ADD) r = x + y;
        else if (op == ORC_SUB) r = x - y;
        else if (op == ORC_MUL) r = x * y;
        else if (op == ORC_DIV) r = x / y;
        else { float z = *(const float*)pc; if (contract) r = fmaf(x, y, z); else { float p = x * y; r = p + z; } }
        *(float*)pt = r; break;
      }
      case ORC_I32: {
        uint32_t x = *(const uint32_t*)pa, y = *(const uint32_t*)pb, r = 0;
        if (op == ORC_ADD) r = x + y;
        else if (op == ORC_SUB) r = x - y;
        else if (op == ORC_MUL) r = x * y;
        else if (op == ORC_DIV) r = (uint32_t)((int32_t)x / (int32_t)y);  /* truncating; y != 0 */
        else r = x * y + *(const uint32_t*)pc;
        *(uint32_t*)pt = r; break;
      }
      case ORC_I64: {
        uint64_t x = *(const uint64_t*)pa, y = *(const uint64_t*)pb, r = 0;
        if (op == ORC_ADD) r = x + y;
        else if (op == ORC_SUB) r = x - y;
        else if (op == ORC_MUL) r = x * y;
        else if (op == ORC_DIV) r = (uint64_t)((int64_t)x / (int64_t)y);
        else r = x * y + *(const uint64_t*)pc;
        *(uint64_t*)pt = r; break;
      }
      default: free(tmp); return ORC_ETYPE;
    }
  }
  int64_t k2[ORC_MAXRANK] = {0, 0, 0};
  for (int64_t t = 0; t < n; ++t, odometer_next(k2, dst)) memcpy(addr_of(dst, k2), tmp + t * el, (size_t)el);
  free(tmp);
  return ORC_OK;
}

/* dst = src (R#5: RHS first).  A rank-0 src is "dst = scalar" (fill). */
int orc_assign(const orc_array* dst, const orc_array* src) {
  if (dst->rank < 1 || dst->rank > ORC_MAXRANK) return ORC_ERANK;
  if (src->type != dst->type) return ORC_ETYPE;
  if (!conformable(dst, src)) return ORC_ESHAPE;
  const int64_t n = total_size(dst), el = elem_len(dst->type);
  char* tmp = (char*)malloc((size_t)(n > 0 ? n : 1) * (size_t)el);
  int64_t k[ORC_MAXRANK] = {0, 0, 0};
  for (int64_t t = 0; t < n; ++t, odometer_next(k, dst)) memcpy(tmp + t * el, operand_addr(src, k), (size_t)el);
  int64_t k2[ORC_MAXRANK] = {0, 0, 0};
  for (int64_t t = 0; t < n; ++t, odometer_next(k2, dst)) memcpy(addr_of(dst, k2), tmp + t * el, (size_t)el);
  free(tmp);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Reductions.  P:243: SUM lowers to a zero-initialised rank-0 output and a  */
/* linalg.reduce whose body adds each element to the running value; MAXVAL  */
/* and PRODUCT "are also implemented" the same way.                          */
/* ------------------------------------------------------------------------ */

/* (1) The literal sequential fold of P:243:  s = 0;  s = s + x(t)  in element order. */
double orc_sum_seq_f64(const orc_array* x) {
  const int64_t n = total_size(x);
  double s = 0.0;
  for (int64_t t = 0; t < n; ++t) s = s + *(const double*)addr_linear(x, t);
  return s;
}

/* Integer SUM: the sum modulo 2^w, two's complement (R#9). */
int64_t orc_sum_i64(const orc_array* x) {
  const int64_t n = total_size(x);
  uint64_t s = 0;
  for (int64_t t = 0; t < n; ++t) s += *(const uint64_t*)addr_linear(x, t);
  return (int64_t)s;
}
int32_t orc_sum_i32(const orc_array* x) {
  const int64_t n = total_size(x);
  uint32_t s = 0;
  for (int64_t t = 0; t < n; ++t) s += *(const uint32_t*)addr_linear(x, t);
  return (int32_t)s;
}

/* (2) The exactly rounded sum: a superaccumulator, i.e. a fixed-point integer
 * wide enough for every binary64 value (2^-1074 .. 2^1024) plus 64 bits of
 * headroom, stored as 32-bit digits in int64 limbs.  The final conversion is
 * round-to-nearest-even of the exact integer.  This is the plain definition of
 * "the exact sum" against which R#8's bound is stated. */
#define SA_LIMBS 72                   /* 72 * 32 = 2304 bits >= 1074 + 1024 + 64 */
#define SA_BIAS 1074                  /* bit 0 of limb 0 has weight 2^-1074 */
typedef struct { int64_t limb[SA_LIMBS]; int64_t adds; int special; double special_val; } superacc;

static void sa_init(superacc* s) { memset(s, 0, sizeof(*s)); }

static void sa_normalize(superacc* s) {
  for (int i = 0; i < SA_LIMBS - 1; ++i) {
    int64_t carry = s->limb[i] >> 32;         /* arithmetic shift: floor division */
    s->limb[i] -= carry * ((int64_t)1 << 32);
    s->limb[i + 1] += carry;
  }
}

static void sa_add(superacc* s, double v) {
  if (v == 0.0) return;
  if (!isfinite(v)) {
    s->special_val = s->special ? s->special_val + v : v;
    s->special = 1;
    return;
  }
  int e;
  double m = frexp(fabs(v), &e);              /* |v| = m * 2^e, m in [0.5, 1) */
  uint64_t mant = (uint64_t)ldexp(m, 53);     /* exact: 53-bit integer */
  int64_t shift = (int64_t)e - 53 + SA_BIAS;  /* |v| = mant * 2^(e-53) */
  if (shift < 0) { mant >>= -shift; shift = 0; }  /* only subnormal-range bits, exact */
  const int limb = (int)(shift / 32), off = (int)(shift % 32);
  /* mant < 2^53, spread over up to 3 limbs of 32 bits */
  unsigned __int128 w = (unsigned __int128)mant << off;
  const int sign = v < 0 ? -1 : 1;
  for (int i = 0; i < 3 && limb + i < SA_LIMBS; ++i) {
    s->limb[limb + i] += sign * (int64_t)(uint32_t)(w & 0xffffffffu);
    w >>= 32;
  }
  /* each add moves a limb by < 2^32: normalise long before an int64 can overflow */
  if (++s->adds % (1 << 20) == 0) sa_normalize(s);
}

/* Round the exact value to the nearest binary64 (ties to even). */
static double sa_round(superacc* s) {
  if (s->special) return s->special_val;
  sa_normalize(s);
  /* after normalising, limbs 0..L-2 are in [0, 2^32) and the top limb carries the sign */
  int negative = s->limb[SA_LIMBS - 1] < 0;
  if (negative) {                 /* |value|: negate every limb and renormalise */
    for (int i = 0; i < SA_LIMBS; ++i) s->limb[i] = -s->limb[i];
    sa_normalize(s);
  }
  uint32_t mag[SA_LIMBS];
  for (int i = 0; i < SA_LIMBS; ++i) mag[i] = (uint32_t)s->limb[i];
  int top = -1;
  for (int i = SA_LIMBS - 1; i >= 0; --i) if (mag[i]) { top = i; break; }
  if (top < 0) return 0.0;
  int hb = 31;
  while (!(mag[top] >> hb & 1u)) --hb;
  const int64_t msb = (int64_t)top * 32 + hb;          /* weight 2^(msb - 1074) */
  /* keep 53 significant bits, but never below bit 0 (subnormals) */
  int64_t lsb = msb - 52;
  if (lsb < 0) lsb = 0;
  uint64_t q = 0;
  for (int64_t b = msb; b >= lsb; --b) q = (q << 1) | (uint64_t)(mag[b / 32] >> (b % 32) & 1u);
  int round_bit = 0, sticky = 0;
  if (lsb > 0) {
    round_bit = (int)(mag[(lsb - 1) / 32] >> ((lsb - 1) % 32) & 1u);
    const int64_t bhi = lsb - 2;                       /* sticky = any bit in [0, bhi] */
    if (bhi >= 0) {
      for (int64_t i = 0; i < bhi / 32; ++i) if (mag[i]) sticky = 1;
      const int r = (int)(bhi % 32);
      const uint32_t mask = r == 31 ? 0xffffffffu : ((1u << (r + 1)) - 1u);
      if (mag[bhi / 32] & mask) sticky = 1;
    }
  }
  if (round_bit && (sticky || (q & 1u))) q += 1;      /* may carry to 2^53: ldexp handles it */
  double r = ldexp((double)q, (int)(lsb - SA_BIAS));   /* exact unless it overflows to inf */
  return negative ? -r : r;
}

double orc_sum_exact_f64(const orc_array* x) {
  superacc s; sa_init(&s);
  const int64_t n = total_size(x);
  for (int64_t t = 0; t < n; ++t) sa_add(&s, *(const double*)addr_linear(x, t));
  return sa_round(&s);
}

/* (3) sum of |x|, rounded once (the scale of R#8's error bound). */
double orc_sum_abs_f64(const orc_array* x) {
  superacc s; sa_init(&s);
  const int64_t n = total_size(x);
  for (int64_t t = 0; t < n; ++t) sa_add(&s, fabs(*(const double*)addr_linear(x, t)));
  return sa_round(&s);
}

/* Exactly rounded sum of an explicit list (used by the pins). */
double orc_fsum(const double* v, int64_t n) {
  superacc s; sa_init(&s);
  for (int64_t i = 0; i < n; ++i) sa_add(&s, v[i]);
  return sa_round(&s);
}

/* ---- order R: the documented combine order of DESIGN.md section 4.2 ----
 * Written from that text, step by step:
 *  1. elements in array element order t = 0..N-1;
 *  2. chunks of C = 65536 consecutive elements;
 *  3. in a chunk, thread tau (0..255) owns the 4-groups starting at
 *     cC + 1024*m + 4*tau (m ascending); accumulator acc_v (v = position in the
 *     group) starts at +0.0 and adds its present elements in m order; the thread
 *     value is (acc_0 + acc_1) + (acc_2 + acc_3);
 *  4. each warp of 32 threads combines by a butterfly: for mask 16,8,4,2,1 every
 *     lane l replaces its value by value[l] + value[l ^ mask];
 *  5. the 8 warp values combine as ((w0+w1)+(w2+w3)) + ((w4+w5)+(w6+w7));
 *  6. the chunk partials are combined by a balanced adjacent-pair tree padded
 *     with +0.0 to the next power of two (no chunks: +0.0).
 * MAXVAL/MINVAL use the same shape with max/min (order-free up to ties of +-0).
 */
#define R_CHUNK 65536
#define R_THREADS 256
#define R_GROUP 4

typedef double (*combine_fn)(double, double);
static double add_f(double a, double b) { return a + b; }
/* maxNum/minNum: a NaN operand is ignored unless both are NaN (R#11). */
static double max_f(double a, double b) { if (isnan(a)) return b; if (isnan(b)) return a; return a > b ? a : b; }
static double min_f(double a, double b) { if (isnan(a)) return b; if (isnan(b)) return a; return a < b ? a : b; }
static double mul_f(double a, double b) { return a * b; }

/* kind: 0 SUM, 1 MAXVAL, 2 MINVAL, 3 PRODUCT */
static combine_fn kind_fn(int32_t kind) {
  return kind == 0 ? add_f : (kind == 1 ? max_f : (kind == 2 ? min_f : mul_f));
}
static double kind_neutral(int32_t kind) {
  return kind == 0 ? 0.0 : (kind == 1 ? -INFINITY : (kind == 2 ? INFINITY : 1.0));
}

static double chunk_partial(const double* v, int64_t n, int64_t c, combine_fn f, double neutral) {
  double thread_val[R_THREADS];
  const int64_t start = c * R_CHUNK;
  int64_t end = start + R_CHUNK;
  if (end > n) end = n;
  for (int tau = 0; tau < R_THREADS; ++tau) {
    double acc[R_GROUP];
    for (int q = 0; q < R_GROUP; ++q) acc[q] = neutral;
    for (int64_t m = 0; m < R_CHUNK / (R_THREADS * R_GROUP); ++m) {
      const int64_t g = start + 1024 * m + R_GROUP * tau;
      for (int q = 0; q < R_GROUP; ++q)
        if (g + q < end) acc[q] = f(acc[q], v[g + q]);
    }
    thread_val[tau] = f(f(acc[0], acc[1]), f(acc[2], acc[3]));
  }
  double warp_val[R_THREADS / 32];
  for (int w = 0; w < R_THREADS / 32; ++w) {
    double lane[32], next[32];
    for (int l = 0; l < 32; ++l) lane[l] = thread_val[32 * w + l];
    for (int mask = 16; mask >= 1; mask /= 2) {
      for (int l = 0; l < 32; ++l) next[l] = f(lane[l], lane[l ^ mask]);
      for (int l = 0; l < 32; ++l) lane[l] = next[l];
    }
    warp_val[w] = lane[0];
  }
  return f(f(f(warp_val[0], warp_val[1]), f(warp_val[2], warp_val[3])),
           f(f(warp_val[4], warp_val[5]), f(warp_val[6], warp_val[7])));
}

/* Balanced adjacent-pair tree over p[0..n-1], padded with pad to a power of two. */
double orc_tree_combine(const double* p, int64_t n, int32_t kind) {
  combine_fn f = kind_fn(kind);
  const double pad = kind_neutral(kind);
  if (n <= 0) return pad;
  int64_t m = 1;
  while (m < n) m *= 2;
  double* buf = (double*)malloc((size_t)m * sizeof(double));
  for (int64_t i = 0; i < m; ++i) buf[i] = i < n ? p[i] : pad;
  while (m > 1) {
    for (int64_t i = 0; i < m / 2; ++i) buf[i] = f(buf[2 * i], buf[2 * i + 1]);
    m /= 2;
  }
  double r = buf[0];
  free(buf);
  return r;
}

/* Chunk partials of order R (steps 1-5) over a packed vector. */
void orc_orderR_partials(const double* v, int64_t n, int32_t kind, double* partials) {
  combine_fn f = kind_fn(kind);
  const double neutral = kind_neutral(kind);
  const int64_t nc = (n + R_CHUNK - 1) / R_CHUNK;
  for (int64_t c = 0; c < nc; ++c) partials[c] = chunk_partial(v, n, c, f, neutral);
}

static double* pack_f64(const orc_array* x, int64_t* n_out) {
  const int64_t n = total_size(x);
  double* v = (double*)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  for (int64_t t = 0; t < n; ++t) v[t] = *(const double*)addr_linear(x, t);
  *n_out = n;
  return v;
}

/* kind: 0 = SUM, 1 = MAXVAL, 2 = MINVAL, 3 = PRODUCT ("a range of other Fortran
 * array intrinsics such as maxval and product are also implemented" the same way) */
double orc_reduce_orderR_f64(const orc_array* x, int32_t kind) {
  int64_t n;
  double* v = pack_f64(x, &n);
  const int64_t nc = (n + R_CHUNK - 1) / R_CHUNK;
  double* part = (double*)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(double));
  orc_orderR_partials(v, n, kind, part);
  double r = orc_tree_combine(part, nc, kind);
  free(part);
  free(v);
  return r;
}

/* MAXVAL / MINVAL by the definition: the largest / smallest element; empty
 * arrays give -inf / +inf for reals, INT_MIN / INT_MAX for integers (R#10);
 * NaN elements are ignored unless all are NaN (R#11).  P:243. */
double orc_maxval_f64(const orc_array* x) {
  const int64_t n = total_size(x);
  double r = -INFINITY;
  int seen = 0;
  for (int64_t t = 0; t < n; ++t) {
    double v = *(const double*)addr_linear(x, t);
    if (isnan(v)) { if (!seen) r = v; continue; }
    if (!seen || isnan(r) || v > r) r = v;
    seen = 1;
  }
  return r;
}
double orc_minval_f64(const orc_array* x) {
  const int64_t n = total_size(x);
  double r = INFINITY;
  int seen = 0;
  for (int64_t t = 0; t < n; ++t) {
    double v = *(const double*)addr_linear(x, t);
    if (isnan(v)) { if (!seen) r = v; continue; }
    if (!seen || isnan(r) || v < r) r = v;
    seen = 1;
  }
  return r;
}
int64_t orc_maxval_int(const orc_array* x) {
  const int64_t n = total_size(x);
  int64_t r = x->type == ORC_I32 ? INT32_MIN : INT64_MIN;
  for (int64_t t = 0; t < n; ++t) {
    const char* p = addr_linear(x, t);
    int64_t v = x->type == ORC_I32 ? (int64_t)*(const int32_t*)p : *(const int64_t*)p;
    if (v > r) r = v;
  }
  return r;
}
int64_t orc_minval_int(const orc_array* x) {
  const int64_t n = total_size(x);
  int64_t r = x->type == ORC_I32 ? INT32_MAX : INT64_MAX;
  for (int64_t t = 0; t < n; ++t) {
    const char* p = addr_linear(x, t);
    int64_t v = x->type == ORC_I32 ? (int64_t)*(const int32_t*)p : *(const int64_t*)p;
    if (v < r) r = v;
  }
  return r;
}

/* DOT_PRODUCT of two rank-1 real vectors = SUM(x*y) (R#12):
 *   products[t] = fl(x(t) * y(t)) in element order. */
int orc_dot_products_f64(const orc_array* x, const orc_array* y, double* products) {
  if (x->rank != 1 || y->rank != 1) return ORC_ERANK;
  if (x->dim[0].ext != y->dim[0].ext) return ORC_ESHAPE;
  for (int64_t t = 0; t < x->dim[0].ext; ++t) {
    double a = *(const double*)(x->base + t * x->dim[0].sm);
    double b = *(const double*)(y->base + t * y->dim[0].sm);
    products[t] = a * b;
  }
  return ORC_OK;
}

/* The exact dot product sum_t x(t)*y(t) with unrounded products: each product is
 * split exactly as p + e with p = fl(x*y), e = fma(x, y, -p) (exact), and both
 * are accumulated in the superaccumulator, then rounded once.  Also returns
 * sum |x(t) y(t)|.  R#8. */
int orc_dot_exact_f64(const orc_array* x, const orc_array* y, double* exact, double* absum) {
  if (x->rank != 1 || y->rank != 1) return ORC_ERANK;
  if (x->dim[0].ext != y->dim[0].ext) return ORC_ESHAPE;
  superacc s, a;
  sa_init(&s); sa_init(&a);
  for (int64_t t = 0; t < x->dim[0].ext; ++t) {
    double u = *(const double*)(x->base + t * x->dim[0].sm);
    double w = *(const double*)(y->base + t * y->dim[0].sm);
    double p = u * w;
    double e = fma(u, w, -p);
    sa_add(&s, p); sa_add(&s, e);
    sa_add(&a, fabs(p)); sa_add(&a, p < 0 ? -e : e);   /* |p + e| = |p| + sign(p) e */
  }
  *exact = sa_round(&s);
  *absum = sa_round(&a);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* TRANSPOSE: r(j, i) = a(lb1 + i - 1, lb2 + j - 1), shape (n2, n1).   */
/* ------------------------------------------------------------------------ */
int orc_transpose(const orc_array* dst, const orc_array* src) {
  if (src->rank != 2 || dst->rank != 2) return ORC_ERANK;
  if (src->type != dst->type) return ORC_ETYPE;
  if (dst->dim[0].ext != src->dim[1].ext || dst->dim[1].ext != src->dim[0].ext) return ORC_ESHAPE;
  const int64_t el = elem_len(src->type);
  for (int64_t i = 0; i < src->dim[0].ext; ++i)
    for (int64_t j = 0; j < src->dim[1].ext; ++j)
      memcpy(dst->base + j * dst->dim[0].sm + i * dst->dim[1].sm,
             src->base + i * src->dim[0].sm + j * src->dim[1].sm, (size_t)el);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* MATMUL: c(i,j) = sum_{l=1..K} a(i,l) * b(l,j), l ascending, */
/* starting from 0, each product rounded then added (R#14: the oracle's order; */
/* the GPU is held to R#8's bound).  Written as the column-major j, l, i       */
/* update loop, which visits l in the same ascending order for every (i,j).    */
/* absum (optional) receives sum_l |a(i,l)| |b(l,j)| for the bound.            */
/* ------------------------------------------------------------------------ */
#define AT(arr, i, j) (*(double*)((arr)->base + (i) * (arr)->dim[0].sm + (j) * (arr)->dim[1].sm))
int orc_matmul_f64(const orc_array* c, const orc_array* a, const orc_array* b, const orc_array* absum) {
  if (a->rank != 2 || b->rank != 2 || c->rank != 2) return ORC_ERANK;
  if (a->type != ORC_F64 || b->type != ORC_F64 || c->type != ORC_F64) return ORC_ETYPE;
  const int64_t m = a->dim[0].ext, k = a->dim[1].ext, n = b->dim[1].ext;
  if (b->dim[0].ext != k || c->dim[0].ext != m || c->dim[1].ext != n) return ORC_ESHAPE;
  double* col = (double*)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
  double* acol = (double*)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = 0; i < m; ++i) { col[i] = 0.0; acol[i] = 0.0; }
    for (int64_t l = 0; l < k; ++l) {
      const double blj = AT(b, l, j);
      for (int64_t i = 0; i < m; ++i) {
        const double p = AT(a, i, l) * blj;
        col[i] = col[i] + p;
        acol[i] = acol[i] + fabs(p);
      }
    }
    for (int64_t i = 0; i < m; ++i) {
      AT(c, i, j) = col[i];
      if (absum) AT(absum, i, j) = acol[i];
    }
  }
  free(col);
  free(acol);
  return ORC_OK;
}

/* One element of MATMUL, same order as orc_matmul_f64 (for sampled checks at
 * sizes where the full product is out of reach). */
double orc_matmul_element_f64(const orc_array* a, const orc_array* b, int64_t i, int64_t j, double* absum) {
  const int64_t k = a->dim[1].ext;
  double s = 0.0, t = 0.0;
  for (int64_t l = 0; l < k; ++l) {
    const double p = AT(a, i, l) * AT(b, l, j);
    s = s + p;
    t = t + fabs(p);
  }
  if (absum) *absum = t;
  return s;
}

/* ------------------------------------------------------------------------ */
/* Jacobi ("a Jacobi iteration solving Laplace's equation ... over a    */
/* single two dimensional grid"; the source is not printed, R#16):            */
/*   do sweep = 1, sweeps                                                     */
/*     do j = lb2+1, ub2-1;  do i = lb1+1, ub1-1                              */
/*       unew(i,j) = c * (((u(i-1,j) + u(i+1,j)) + u(i,j-1)) + u(i,j+1))      */
/*     swap(u, unew)        ! "u = unew" realised as a swap (same values)     */
/* 3-D: unew = c * (((((u(i-1)+u(i+1)) + u(j-1)) + u(j+1)) + u(k-1)) + u(k+1)) */
/* The boundary of unew is left as the caller set it.  Returns, in           */
/* *result_in_unew, whether the last sweep wrote the array passed as unew.   */
/* ------------------------------------------------------------------------ */
static double ld3(const orc_array* a, int64_t i, int64_t j, int64_t k) {
  return *(const double*)(a->base + i * a->dim[0].sm + j * a->dim[1].sm + k * a->dim[2].sm);
}
static void st3(const orc_array* a, int64_t i, int64_t j, int64_t k, double v) {
  *(double*)(a->base + i * a->dim[0].sm + j * a->dim[1].sm + k * a->dim[2].sm) = v;
}

int orc_jacobi_f64(const orc_array* u0, const orc_array* unew0, int64_t sweeps, double coeff,
                   int32_t* result_in_unew) {
  if (u0->rank != unew0->rank || (u0->rank != 2 && u0->rank != 3)) return ORC_ERANK;
  for (int d = 0; d < u0->rank; ++d) if (u0->dim[d].ext != unew0->dim[d].ext) return ORC_ESHAPE;
  const orc_array* u = u0;
  const orc_array* w = unew0;
  const int64_t n1 = u0->dim[0].ext, n2 = u0->dim[1].ext, n3 = u0->rank == 3 ? u0->dim[2].ext : 1;
  for (int64_t s = 0; s < sweeps; ++s) {
    if (u0->rank == 2) {
#pragma omp parallel for schedule(static)
      for (int64_t j = 1; j < n2 - 1; ++j)
        for (int64_t i = 1; i < n1 - 1; ++i) {
          double t = ld3(u, i - 1, j, 0) + ld3(u, i + 1, j, 0);
          t = t + ld3(u, i, j - 1, 0);
          t = t + ld3(u, i, j + 1, 0);
          st3(w, i, j, 0, coeff * t);
        }
    } else {
#pragma omp parallel for schedule(static)
      for (int64_t k = 1; k < n3 - 1; ++k)
        for (int64_t j = 1; j < n2 - 1; ++j)
          for (int64_t i = 1; i < n1 - 1; ++i) {
            double t = ld3(u, i - 1, j, k) + ld3(u, i + 1, j, k);
            t = t + ld3(u, i, j - 1, k);
            t = t + ld3(u, i, j + 1, k);
            t = t + ld3(u, i, j, k - 1);
            t = t + ld3(u, i, j, k + 1);
            st3(w, i, j, k, coeff * t);
          }
    }
    const orc_array* tmp = u; u = w; w = tmp;   /* u = unew */
  }
  *result_in_unew = (int32_t)(sweeps % 2 == 1);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* PRODUCT by definition: the sequential fold p = 1; p = p * x(t) in element */
/* order (reals); integers modulo 2^w.                                      */
/* ------------------------------------------------------------------------ */
double orc_product_seq_f64(const orc_array* x) {
  const int64_t n = total_size(x);
  double p = 1.0;
  for (int64_t t = 0; t < n; ++t) p = p * *(const double*)addr_linear(x, t);
  return p;
}
int64_t orc_product_int(const orc_array* x) {
  const int64_t n = total_size(x);
  if (x->type == ORC_I32) {
    uint32_t p = 1;
    for (int64_t t = 0; t < n; ++t) p *= *(const uint32_t*)addr_linear(x, t);
    return (int64_t)(int32_t)p;
  }
  uint64_t p = 1;
  for (int64_t t = 0; t < n; ++t) p *= *(const uint64_t*)addr_linear(x, t);
  return (int64_t)p;
}

/* ------------------------------------------------------------------------ */
/* SUM / MAXVAL / MINVAL / PRODUCT (x, DIM=dim)  (linalg.reduce with a    */
/* `dimensions` attribute).  The result has x's shape with       */
/* dimension dim (1-based) removed; result element o is the sequential fold over   */
/* the reduced subscript in ascending order, starting from the neutral element     */
/* (R#24).  MAXVAL/MINVAL: NaN ignored unless all are NaN; an empty reduced        */
/* dimension gives the R#10 value.  result: rank(x)-1 (rank 0 = one element).      */
/* ------------------------------------------------------------------------ */
int orc_reduce_dim(const orc_array* x, int32_t dim, int32_t kind, const orc_array* result) {
  if (x->rank < 1 || dim < 1 || dim > x->rank) return ORC_ERANK;
  if (result->rank != x->rank - 1 || result->type != x->type) return ORC_ESHAPE;
  int64_t kept_ext[ORC_MAXRANK] = {1, 1, 1}, kept_sm[ORC_MAXRANK] = {0, 0, 0};
  int nk = 0;
  for (int d = 0; d < x->rank; ++d) {
    if (d == dim - 1) continue;
    if (result->dim[nk].ext != x->dim[d].ext) return ORC_ESHAPE;
    kept_ext[nk] = x->dim[d].ext;
    kept_sm[nk] = x->dim[d].sm;
    ++nk;
  }
  const int64_t n = x->dim[dim - 1].ext, step = x->dim[dim - 1].sm;
  int64_t nout = 1;
  for (int d = 0; d < nk; ++d) nout *= kept_ext[d];
  int64_t k[ORC_MAXRANK] = {0, 0, 0};
  for (int64_t o = 0; o < nout; ++o) {
    const char* xp = x->base;
    char* rp = result->base;
    for (int d = 0; d < nk; ++d) { xp += k[d] * kept_sm[d]; rp += k[d] * result->dim[d].sm; }
    if (x->type == ORC_F64) {
      double acc;
      if (kind == 1 || kind == 2) {
        if (n == 0) acc = kind == 1 ? -INFINITY : INFINITY;
        else {
          acc = NAN;
          combine_fn f = kind_fn(kind);
          for (int64_t j = 0; j < n; ++j) acc = f(acc, *(const double*)(xp + j * step));
        }
      } else {
        acc = kind_neutral(kind);
        combine_fn f = kind_fn(kind);
        for (int64_t j = 0; j < n; ++j) acc = f(acc, *(const double*)(xp + j * step));
      }
      *(double*)rp = acc;
    } else if (x->type == ORC_I32 || x->type == ORC_I64) {
      const int w32 = x->type == ORC_I32;
      uint64_t acc = kind == 0 ? 0 : (kind == 3 ? 1 : 0);
      int64_t best = kind == 1 ? (w32 ? INT32_MIN : INT64_MIN) : (w32 ? INT32_MAX : INT64_MAX);
      for (int64_t j = 0; j < n; ++j) {
        const char* e = xp + j * step;
        const int64_t v = w32 ? (int64_t)*(const int32_t*)e : *(const int64_t*)e;
        if (kind == 0) acc += (uint64_t)v;
        else if (kind == 3) acc *= (uint64_t)v;
        else if (kind == 1) { if (v > best) best = v; }
        else { if (v < best) best = v; }
      }
      const int64_t r = (kind == 0 || kind == 3) ? (int64_t)acc : best;
      if (w32) *(int32_t*)rp = (int32_t)(uint32_t)(uint64_t)r;
      else *(int64_t*)rp = r;
    } else {
      return ORC_ETYPE;
    }
    for (int d = 0; d < nk; ++d) { if (++k[d] < kept_ext[d]) break; k[d] = 0; }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* MATMUL rank-1 forms (F2018: MATMUL(matrix_a(m,k), vector_b(k)) has shape  */
/* (m) and MATMUL(vector_a(k), matrix_b(k,n)) has shape (n)):      */
/*   y(i) = sum_{l=1..k} a(i,l) x(l)      y(j) = sum_{l=1..k} x(l) b(l,j)            */
/* l ascending from 0, each product rounded then added; absum = sum |products|.     */
/* ------------------------------------------------------------------------ */
int orc_matvec_f64(const orc_array* y, const orc_array* a, const orc_array* x, const orc_array* absum) {
  if (a->rank != 2 || x->rank != 1 || y->rank != 1) return ORC_ERANK;
  const int64_t m = a->dim[0].ext, k = a->dim[1].ext;
  if (x->dim[0].ext != k || y->dim[0].ext != m) return ORC_ESHAPE;
  for (int64_t i = 0; i < m; ++i) {
    double s = 0.0, t = 0.0;
    for (int64_t l = 0; l < k; ++l) {
      const double p = AT(a, i, l) * *(const double*)(x->base + l * x->dim[0].sm);
      s = s + p;
      t = t + fabs(p);
    }
    *(double*)(y->base + i * y->dim[0].sm) = s;
    if (absum) *(double*)(absum->base + i * absum->dim[0].sm) = t;
  }
  return ORC_OK;
}

int orc_vecmat_f64(const orc_array* y, const orc_array* x, const orc_array* b, const orc_array* absum) {
  if (b->rank != 2 || x->rank != 1 || y->rank != 1) return ORC_ERANK;
  const int64_t k = b->dim[0].ext, n = b->dim[1].ext;
  if (x->dim[0].ext != k || y->dim[0].ext != n) return ORC_ESHAPE;
  for (int64_t j = 0; j < n; ++j) {
    double s = 0.0, t = 0.0;
    for (int64_t l = 0; l < k; ++l) {
      const double p = *(const double*)(x->base + l * x->dim[0].sm) * AT(b, l, j);
      s = s + p;
      t = t + fabs(p);
    }
    *(double*)(y->base + j * y->dim[0].sm) = s;
    if (absum) *(double*)(absum->base + j * absum->dim[0].sm) = t;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* MAXVAL(ABS(x - y)) by the definition (R#10/R#11 rules; empty -> -inf).          */
/* ------------------------------------------------------------------------ */
double orc_maxabsdiff_f64(const orc_array* x, const orc_array* y) {
  const int64_t n = total_size(x);
  double r = -INFINITY;
  int seen = 0;
  for (int64_t t = 0; t < n; ++t) {
    const double d = fabs(*(const double*)addr_linear(x, t) - *(const double*)addr_linear(y, t));
    if (isnan(d)) { if (!seen) r = d; continue; }
    if (!seen || isnan(r) || d > r) r = d;
    seen = 1;
  }
  return r;
}

/* max |x - y| over the interior points of two conformable arrays (the section
 * (lb+1 : ub-1) in every dimension): the points a Jacobi sweep updates (R#16, R#25).
 * An empty interior gives -inf (R#10). */
static double interior_maxabsdiff(const orc_array* x, const orc_array* y) {
  int64_t lo[ORC_MAXRANK], hi[ORC_MAXRANK], st[ORC_MAXRANK];
  orc_array ix, iy;
  for (int d = 0; d < x->rank; ++d) {
    lo[d] = x->dim[d].lb + 1;
    hi[d] = x->dim[d].lb + x->dim[d].ext - 2;
    st[d] = 1;
  }
  orc_section(x, lo, hi, st, &ix);
  for (int d = 0; d < y->rank; ++d) {
    lo[d] = y->dim[d].lb + 1;
    hi[d] = y->dim[d].lb + y->dim[d].ext - 2;
  }
  orc_section(y, lo, hi, st, &iy);
  return orc_maxabsdiff_f64(&ix, &iy);
}

/* Jacobi to convergence (R#25): the DO nest of orc_jacobi_f64 one sweep at a time; after
 * every check_every-th sweep (and after max_sweeps) res = max |u_s - u_{s-1}| over the
 * interior points (the points the sweep updates; the boundary rings are never changed);
 * stop when res <= tol. */
int orc_jacobi_solve_f64(const orc_array* u, const orc_array* unew, int64_t max_sweeps, int64_t check_every,
                         double tol, double coeff, int64_t* sweeps_done, double* residual, int32_t* in_unew) {
  const orc_array* a = u;
  const orc_array* b = unew;
  int64_t s = 0;
  double res = 0.0;
  int32_t dummy;
  while (s < max_sweeps) {
    int rc = orc_jacobi_f64(a, b, 1, coeff, &dummy);
    if (rc) return rc;
    const orc_array* t = a; a = b; b = t;   /* a holds u_s */
    ++s;
    if (s % check_every == 0 || s == max_sweeps) {
      res = interior_maxabsdiff(a, b);
      if (res <= tol) break;
    }
  }
  *sweeps_done = s;
  *residual = res;
  *in_unew = (int32_t)(a == unew);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* pw-advection (R#26): the 3-field advection stencil of the  */
/* paper's pw-advection benchmark.  Its body is NOT in the paper;    */
/* this is the MONC pw_advection kernel (advect_flow_fields) as reproduced in DESIGN.md   */
/* R#26, written as the Fortran DO nest with the fields indexed (k, j, i) = dims (1, 2, 3), */
/* k contiguous.  Every tendency is built in the same order: the x term (tcx), the y term  */
/* (tcy), then the vertical term, whose two fluxes are differenced inside one parenthesis:  */
/*   do i = 2, nx-1; do j = 2, ny-1; do k = 2, nz-1                                      */
/*     su = tcx*(u(k,j,i-1)*(u(k,j,i)+u(k,j,i-1)) - u(k,j,i+1)*(u(k,j,i)+u(k,j,i+1)))    */
/*     su = su + tcy*(u(k,j-1,i)*(v(k,j-1,i)+v(k,j-1,i+1)) - u(k,j+1,i)*(v(k,j,i)+v(k,j,i+1))) */
/*     su = su + (tzc1(k)*u(k-1,j,i)*(w(k-1,j,i)+w(k-1,j,i+1))                            */
/*              - tzc2(k)*u(k+1,j,i)*(w(k,j,i)+w(k,j,i+1)))                               */
/*     sv = tcx*(v(k,j,i-1)*(u(k,j,i-1)+u(k,j+1,i-1)) - v(k,j,i+1)*(u(k,j,i)+u(k,j+1,i))) */
/*     sv = sv + tcy*(v(k,j-1,i)*(v(k,j,i)+v(k,j-1,i)) - v(k,j+1,i)*(v(k,j,i)+v(k,j+1,i))) */
/*     sv = sv + (tzc1(k)*v(k-1,j,i)*(w(k-1,j,i)+w(k-1,j+1,i))                            */
/*              - tzc2(k)*v(k+1,j,i)*(w(k,j,i)+w(k,j+1,i)))                               */
/*     sw = tcx*(w(k,j,i-1)*(u(k,j,i-1)+u(k+1,j,i-1)) - w(k,j,i+1)*(u(k,j,i)+u(k+1,j,i))) */
/*     sw = sw + tcy*(w(k,j-1,i)*(v(k,j-1,i)+v(k+1,j-1,i)) - w(k,j+1,i)*(v(k,j,i)+v(k+1,j,i))) */
/*     sw = sw + (tzd1(k)*w(k-1,j,i)*(w(k,j,i)+w(k-1,j,i))                                */
/*              - tzd2(k)*w(k+1,j,i)*(w(k,j,i)+w(k+1,j,i)))                               */
/* Fortran evaluation: a*b*c = (a*b)*c, x + (a - b) as parenthesised; one rounding per op. */
/* Boundary points of su, sv, sw are not written.                                          */
/* ------------------------------------------------------------------------ */
int orc_pw_advection_f64(const orc_array* su, const orc_array* sv, const orc_array* sw, const orc_array* u,
                         const orc_array* v, const orc_array* w, const double* tzc1, const double* tzc2,
                         const double* tzd1, const double* tzd2, double tcx, double tcy) {
  const orc_array* all[6] = {su, sv, sw, u, v, w};
  for (int q = 0; q < 6; ++q) {
    if (all[q]->rank != 3) return ORC_ERANK;
    if (all[q]->type != ORC_F64) return ORC_ETYPE;
    for (int d = 0; d < 3; ++d) if (all[q]->dim[d].ext != u->dim[d].ext) return ORC_ESHAPE;
  }
  const int64_t nz = u->dim[0].ext, ny = u->dim[1].ext, nx = u->dim[2].ext;
#pragma omp parallel for schedule(static)
  for (int64_t i = 1; i < nx - 1; ++i)
    for (int64_t j = 1; j < ny - 1; ++j)
      for (int64_t k = 1; k < nz - 1; ++k) {
        double a, b, s;
        /* su(k,j,i) = tcx*(u(k,j,i-1)*(u(k,j,i)+u(k,j,i-1)) - u(k,j,i+1)*(u(k,j,i)+u(k,j,i+1))) */
        a = ld3(u, k, j, i - 1) * (ld3(u, k, j, i) + ld3(u, k, j, i - 1));
        b = ld3(u, k, j, i + 1) * (ld3(u, k, j, i) + ld3(u, k, j, i + 1));
        s = tcx * (a - b);
        /* su = su + tcy*(u(k,j-1,i)*(v(k,j-1,i)+v(k,j-1,i+1)) - u(k,j+1,i)*(v(k,j,i)+v(k,j,i+1))) */
        a = ld3(u, k, j - 1, i) * (ld3(v, k, j - 1, i) + ld3(v, k, j - 1, i + 1));
        b = ld3(u, k, j + 1, i) * (ld3(v, k, j, i) + ld3(v, k, j, i + 1));
        s = s + tcy * (a - b);
        /* su = su + (tzc1(k)*u(k-1,j,i)*(w(k-1,j,i)+w(k-1,j,i+1)) - tzc2(k)*u(k+1,j,i)*(w(k,j,i)+w(k,j,i+1))) */
        a = (tzc1[k] * ld3(u, k - 1, j, i)) * (ld3(w, k - 1, j, i) + ld3(w, k - 1, j, i + 1));
        b = (tzc2[k] * ld3(u, k + 1, j, i)) * (ld3(w, k, j, i) + ld3(w, k, j, i + 1));
        s = s + (a - b);
        st3(su, k, j, i, s);
        /* sv(k,j,i) = tcx*(v(k,j,i-1)*(u(k,j,i-1)+u(k,j+1,i-1)) - v(k,j,i+1)*(u(k,j,i)+u(k,j+1,i))) */
        a = ld3(v, k, j, i - 1) * (ld3(u, k, j, i - 1) + ld3(u, k, j + 1, i - 1));
        b = ld3(v, k, j, i + 1) * (ld3(u, k, j, i) + ld3(u, k, j + 1, i));
        s = tcx * (a - b);
        /* sv = sv + tcy*(v(k,j-1,i)*(v(k,j,i)+v(k,j-1,i)) - v(k,j+1,i)*(v(k,j,i)+v(k,j+1,i))) */
        a = ld3(v, k, j - 1, i) * (ld3(v, k, j, i) + ld3(v, k, j - 1, i));
        b = ld3(v, k, j + 1, i) * (ld3(v, k, j, i) + ld3(v, k, j + 1, i));
        s = s + tcy * (a - b);
        /* sv = sv + (tzc1(k)*v(k-1,j,i)*(w(k-1,j,i)+w(k-1,j+1,i)) - tzc2(k)*v(k+1,j,i)*(w(k,j,i)+w(k,j+1,i))) */
        a = (tzc1[k] * ld3(v, k - 1, j, i)) * (ld3(w, k - 1, j, i) + ld3(w, k - 1, j + 1, i));
        b = (tzc2[k] * ld3(v, k + 1, j, i)) * (ld3(w, k, j, i) + ld3(w, k, j + 1, i));
        s = s + (a - b);
        st3(sv, k, j, i, s);
        /* sw(k,j,i) = tcx*(w(k,j,i-1)*(u(k,j,i-1)+u(k+1,j,i-1)) - w(k,j,i+1)*(u(k,j,i)+u(k+1,j,i))) */
        a = ld3(w, k, j, i - 1) * (ld3(u, k, j, i - 1) + ld3(u, k + 1, j, i - 1));
        b = ld3(w, k, j, i + 1) * (ld3(u, k, j, i) + ld3(u, k + 1, j, i));
        s = tcx * (a - b);
        /* sw = sw + tcy*(w(k,j-1,i)*(v(k,j-1,i)+v(k+1,j-1,i)) - w(k,j+1,i)*(v(k,j,i)+v(k+1,j,i))) */
        a = ld3(w, k, j - 1, i) * (ld3(v, k, j - 1, i) + ld3(v, k + 1, j - 1, i));
        b = ld3(w, k, j + 1, i) * (ld3(v, k, j, i) + ld3(v, k + 1, j, i));
        s = s + tcy * (a - b);
        /* sw = sw + (tzd1(k)*w(k-1,j,i)*(w(k,j,i)+w(k-1,j,i)) - tzd2(k)*w(k+1,j,i)*(w(k,j,i)+w(k+1,j,i))) */
        a = (tzd1[k] * ld3(w, k - 1, j, i)) * (ld3(w, k, j, i) + ld3(w, k - 1, j, i));
        b = (tzd2[k] * ld3(w, k + 1, j, i)) * (ld3(w, k, j, i) + ld3(w, k + 1, j, i));
        s = s + (a - b);
        st3(sw, k, j, i, s);
      }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* tra-adv (R#28): the NEMO tracer-advection benchmark the paper   */
/* runs ("tra-adv": "a tracer advection scheme from the NEMO ocean model benchmarking  */
/* suite ... six fields on a three dimensional grid of size 1024 by 512 by 512, running over */
/* 20 iterations").  Its body is NOT in the paper; this is the PSyclone NEMO benchmark's     */
/* tra_adv loop nest as recalled in DESIGN.md R#28 (not checked against the source), written */
/* as the Fortran DO nests in their order, fields indexed (ji, jj, jk), ji contiguous.        */
/* Temporaries zind, zwx, zwy, zslpx, zslpy are zero at the start of the call (R#28) and keep */
/* their values from one iteration to the next; zdt = zbtr = 1.                              */
/*   do jt = 1, iters                                                                        */
/*    (1) zind = 1 - MAX(rnfmsk*rnfmsk_z, upsmsk, zice) * tmask, zice = tsn <= ztfreez+0.1    */
/*    (2) zwx(:,:,jpk) = 0; zwy(:,:,jpk) = 0                                                 */
/*        jk<jpk, jj<jpj, ji<jpi: zwx = umask*(md(ji+1)-md); zwy = vmask*(md(jj+1)-md)        */
/*    (3) zslpx(:,:,jpk) = 0; zslpy(:,:,jpk) = 0                                              */
/*        jk<jpk, jj>=2, ji>=2: zslpx = (zwx + zwx(ji-1)) * (0.25 + SIGN(0.25, zwx*zwx(ji-1))) */
/*                              zslpy = (zwy + zwy(jj-1)) * (0.25 + SIGN(0.25, zwy*zwy(jj-1))) */
/*    (4) same range: zslpx = SIGN(1, zslpx) * MIN(ABS(zslpx), 2*ABS(zwx(ji-1)), 2*ABS(zwx))  */
/*                    zslpy = SIGN(1, zslpy) * MIN(ABS(zslpy), 2*ABS(zwy(jj-1)), 2*ABS(zwy))  */
/*    (5) jk<jpk, 2<=jj<jpj, 2<=ji<jpi:                                                       */
/*          z0u = SIGN(0.5, pun); zalpha = 0.5 - z0u; zu = z0u - 0.5*pun*zdt                  */
/*          zzwx = md(ji+1) + zind*(zu*zslpx(ji+1)); zzwy = md + zind*(zu*zslpx)              */
/*          zwx = pun*(zalpha*zzwx + (1-zalpha)*zzwy)                                         */
/*          z0v = SIGN(0.5, pvn); zalpha = 0.5 - z0v; zv = z0v - 0.5*pvn*zdt                  */
/*          zzwx = md(jj+1) + zind*(zv*zslpy(jj+1)); zzwy = md + zind*(zv*zslpy)              */
/*          zwy = pvn*(zalpha*zzwx + (1-zalpha)*zzwy)                                         */
/*    (6) same range: md = md + (-zbtr*(zwx - zwx(ji-1) + zwy - zwy(jj-1)))                  */
/*    (7) zwx(:,:,1) = 0; zwx(:,:,jpk) = 0; 2<=jk<jpk: zwx = tmask*(md(jk-1) - md)            */
/*    (8) zslpx(:,:,1) = 0; 2<=jk<jpk, all ji, jj:                                            */
/*          zslpx = (zwx + zwx(jk+1)) * (0.25 + SIGN(0.25, zwx*zwx(jk+1)))                    */
/*    (9) same: zslpx = SIGN(1, zslpx) * MIN(ABS(zslpx), 2*ABS(zwx(jk+1)), 2*ABS(zwx))        */
/*   (10) zwx(:,:,1) = pwn(:,:,1)*md(:,:,1)                                                   */
/*   (11) jk<jpk, 2<=jj<jpj, 2<=ji<jpi:                                                       */
/*          z0w = SIGN(0.5, pwn(jk+1)); zalpha = 0.5 + z0w; zw = z0w - 0.5*pwn(jk+1)*zdt*zbtr */
/*          zzwx = md(jk+1) + zind*(zw*zslpx(jk+1)); zzwy = md + zind*(zw*zslpx)              */
/*          zwx(jk+1) = pwn(jk+1)*(zalpha*zzwx + (1-zalpha)*zzwy)                             */
/*   (12) same range: md = -zbtr*(zwx - zwx(jk+1))                                            */
/* Fortran evaluation: left to right for * and -, parentheses as written; SIGN(a,b) = |a| with */
/* the sign of b (a -0 b gives -|a|); MIN/MAX/ABS exact.  One rounding per operation.        */
/* ------------------------------------------------------------------------ */
#define TA(a, i, j, k) (*(double*)((a)->base + (i) * (a)->dim[0].sm + (j) * (a)->dim[1].sm + (k) * (a)->dim[2].sm))
#define TA2(a, i, j) (*(const double*)((a)->base + (i) * (a)->dim[0].sm + (j) * (a)->dim[1].sm))
static double f_sign(double a, double b) { return copysign(fabs(a), b); }

int orc_tra_adv_f64(const orc_array* md, const orc_array* tsn, const orc_array* pun, const orc_array* pvn,
                    const orc_array* pwn, const orc_array* umask, const orc_array* vmask, const orc_array* tmask,
                    const orc_array* ztfreez, const orc_array* rnfmsk, const orc_array* upsmsk,
                    const double* rnfmsk_z, int64_t iters) {
  const orc_array* f3[8] = {md, tsn, pun, pvn, pwn, umask, vmask, tmask};
  for (int q = 0; q < 8; ++q) {
    if (f3[q]->rank != 3) return ORC_ERANK;
    if (f3[q]->type != ORC_F64) return ORC_ETYPE;
    for (int d = 0; d < 3; ++d) if (f3[q]->dim[d].ext != md->dim[d].ext) return ORC_ESHAPE;
  }
  const orc_array* f2[3] = {ztfreez, rnfmsk, upsmsk};
  for (int q = 0; q < 3; ++q) {
    if (f2[q]->rank != 2) return ORC_ERANK;
    if (f2[q]->type != ORC_F64) return ORC_ETYPE;
    for (int d = 0; d < 2; ++d) if (f2[q]->dim[d].ext != md->dim[d].ext) return ORC_ESHAPE;
  }
  if (iters < 0) return ORC_ESHAPE;
  const int64_t ni = md->dim[0].ext, nj = md->dim[1].ext, nk = md->dim[2].ext, n = ni * nj * nk;
  if (n == 0 || iters == 0) return ORC_OK;
  /* temporaries: zero at the start of the call (R#28), packed (ji, jj, jk) */
  double* buf = (double*)calloc((size_t)(5 * n), sizeof(double));
  if (!buf) return ORC_ESHAPE;
  orc_array tmp[5];
  for (int q = 0; q < 5; ++q) {
    tmp[q].base = (char*)(buf + q * n);
    tmp[q].type = ORC_F64;
    tmp[q].rank = 3;
    tmp[q].dim[0] = (orc_dim){1, ni, 8};
    tmp[q].dim[1] = (orc_dim){1, nj, 8 * ni};
    tmp[q].dim[2] = (orc_dim){1, nk, 8 * ni * nj};
  }
  const orc_array *zind = &tmp[0], *zwx = &tmp[1], *zwy = &tmp[2], *zslpx = &tmp[3], *zslpy = &tmp[4];
  const double zdt = 1.0, zbtr = 1.0;
  for (int64_t jt = 0; jt < iters; ++jt) {
    /* (1) */
    for (int64_t k = 0; k < nk; ++k)
      for (int64_t j = 0; j < nj; ++j)
        for (int64_t i = 0; i < ni; ++i) {
          const double zice = TA(tsn, i, j, k) <= TA2(ztfreez, i, j) + 0.1 ? 1.0 : 0.0;
          double m = TA2(rnfmsk, i, j) * rnfmsk_z[k];
          m = fmax(fmax(m, TA2(upsmsk, i, j)), zice);
          TA(zind, i, j, k) = 1.0 - m * TA(tmask, i, j, k);
        }
    /* (2) */
    for (int64_t j = 0; j < nj; ++j)
      for (int64_t i = 0; i < ni; ++i) TA(zwx, i, j, nk - 1) = TA(zwy, i, j, nk - 1) = 0.0;
    for (int64_t k = 0; k < nk - 1; ++k)
      for (int64_t j = 0; j < nj - 1; ++j)
        for (int64_t i = 0; i < ni - 1; ++i) {
          TA(zwx, i, j, k) = TA(umask, i, j, k) * (TA(md, i + 1, j, k) - TA(md, i, j, k));
          TA(zwy, i, j, k) = TA(vmask, i, j, k) * (TA(md, i, j + 1, k) - TA(md, i, j, k));
        }
    /* (3) */
    for (int64_t j = 0; j < nj; ++j)
      for (int64_t i = 0; i < ni; ++i) TA(zslpx, i, j, nk - 1) = TA(zslpy, i, j, nk - 1) = 0.0;
    for (int64_t k = 0; k < nk - 1; ++k)
      for (int64_t j = 1; j < nj; ++j)
        for (int64_t i = 1; i < ni; ++i) {
          const double ax = TA(zwx, i, j, k), bx = TA(zwx, i - 1, j, k);
          TA(zslpx, i, j, k) = (ax + bx) * (0.25 + f_sign(0.25, ax * bx));
          const double ay = TA(zwy, i, j, k), by = TA(zwy, i, j - 1, k);
          TA(zslpy, i, j, k) = (ay + by) * (0.25 + f_sign(0.25, ay * by));
        }
    /* (4) */
    for (int64_t k = 0; k < nk - 1; ++k)
      for (int64_t j = 1; j < nj; ++j)
        for (int64_t i = 1; i < ni; ++i) {
          const double sx = TA(zslpx, i, j, k);
          TA(zslpx, i, j, k) = f_sign(1.0, sx) * fmin(fmin(fabs(sx), 2.0 * fabs(TA(zwx, i - 1, j, k))),
                                                      2.0 * fabs(TA(zwx, i, j, k)));
          const double sy = TA(zslpy, i, j, k);
          TA(zslpy, i, j, k) = f_sign(1.0, sy) * fmin(fmin(fabs(sy), 2.0 * fabs(TA(zwy, i, j - 1, k))),
                                                      2.0 * fabs(TA(zwy, i, j, k)));
        }
    /* (5) */
    for (int64_t k = 0; k < nk - 1; ++k)
      for (int64_t j = 1; j < nj - 1; ++j)
        for (int64_t i = 1; i < ni - 1; ++i) {
          const double zi = TA(zind, i, j, k), u = TA(pun, i, j, k), v = TA(pvn, i, j, k);
          const double z0u = f_sign(0.5, u);
          double zalpha = 0.5 - z0u;
          const double zu = z0u - (0.5 * u) * zdt;
          double zzwx = TA(md, i + 1, j, k) + zi * (zu * TA(zslpx, i + 1, j, k));
          double zzwy = TA(md, i, j, k) + zi * (zu * TA(zslpx, i, j, k));
          TA(zwx, i, j, k) = u * (zalpha * zzwx + (1.0 - zalpha) * zzwy);
          const double z0v = f_sign(0.5, v);
          zalpha = 0.5 - z0v;
          const double zv = z0v - (0.5 * v) * zdt;
          zzwx = TA(md, i, j + 1, k) + zi * (zv * TA(zslpy, i, j + 1, k));
          zzwy = TA(md, i, j, k) + zi * (zv * TA(zslpy, i, j, k));
          TA(zwy, i, j, k) = v * (zalpha * zzwx + (1.0 - zalpha) * zzwy);
        }
    /* (6) */
    for (int64_t k = 0; k < nk - 1; ++k)
      for (int64_t j = 1; j < nj - 1; ++j)
        for (int64_t i = 1; i < ni - 1; ++i) {
          const double ztra = -(zbtr * (((TA(zwx, i, j, k) - TA(zwx, i - 1, j, k)) + TA(zwy, i, j, k)) -
                                        TA(zwy, i, j - 1, k)));
          TA(md, i, j, k) = TA(md, i, j, k) + ztra;
        }
    /* (7) */
    for (int64_t j = 0; j < nj; ++j)
      for (int64_t i = 0; i < ni; ++i) TA(zwx, i, j, 0) = TA(zwx, i, j, nk - 1) = 0.0;
    for (int64_t k = 1; k < nk - 1; ++k)
      for (int64_t j = 0; j < nj; ++j)
        for (int64_t i = 0; i < ni; ++i)
          TA(zwx, i, j, k) = TA(tmask, i, j, k) * (TA(md, i, j, k - 1) - TA(md, i, j, k));
    /* (8) */
    for (int64_t j = 0; j < nj; ++j)
      for (int64_t i = 0; i < ni; ++i) TA(zslpx, i, j, 0) = 0.0;
    for (int64_t k = 1; k < nk - 1; ++k)
      for (int64_t j = 0; j < nj; ++j)
        for (int64_t i = 0; i < ni; ++i) {
          const double a = TA(zwx, i, j, k), b = TA(zwx, i, j, k + 1);
          TA(zslpx, i, j, k) = (a + b) * (0.25 + f_sign(0.25, a * b));
        }
    /* (9) */
    for (int64_t k = 1; k < nk - 1; ++k)
      for (int64_t j = 0; j < nj; ++j)
        for (int64_t i = 0; i < ni; ++i) {
          const double sx = TA(zslpx, i, j, k);
          TA(zslpx, i, j, k) = f_sign(1.0, sx) * fmin(fmin(fabs(sx), 2.0 * fabs(TA(zwx, i, j, k + 1))),
                                                      2.0 * fabs(TA(zwx, i, j, k)));
        }
    /* (10) */
    for (int64_t j = 0; j < nj; ++j)
      for (int64_t i = 0; i < ni; ++i) TA(zwx, i, j, 0) = TA(pwn, i, j, 0) * TA(md, i, j, 0);
    /* (11) */
    for (int64_t k = 0; k < nk - 1; ++k)
      for (int64_t j = 1; j < nj - 1; ++j)
        for (int64_t i = 1; i < ni - 1; ++i) {
          const double w1 = TA(pwn, i, j, k + 1), zi = TA(zind, i, j, k);
          const double z0w = f_sign(0.5, w1);
          const double zalpha = 0.5 + z0w;
          const double zw = z0w - ((0.5 * w1) * zdt) * zbtr;
          const double zzwx = TA(md, i, j, k + 1) + zi * (zw * TA(zslpx, i, j, k + 1));
          const double zzwy = TA(md, i, j, k) + zi * (zw * TA(zslpx, i, j, k));
          TA(zwx, i, j, k + 1) = w1 * (zalpha * zzwx + (1.0 - zalpha) * zzwy);
        }
    /* (12) */
    for (int64_t k = 0; k < nk - 1; ++k)
      for (int64_t j = 1; j < nj - 1; ++j)
        for (int64_t i = 1; i < ni - 1; ++i)
          TA(md, i, j, k) = -(zbtr * (TA(zwx, i, j, k) - TA(zwx, i, j, k + 1)));
  }
  free(buf);
  return ORC_OK;
}
#undef TA
#undef TA2

/* Timing helper for bench.py's cpu_baseline (not part of any computed result): the number of
 * OpenMP threads the parallel loops above use; returns the previous setting (1 without OpenMP). */
int orc_set_threads(int n) {
#ifdef _OPENMP
  const int prev = omp_get_max_threads();
  if (n > 0) omp_set_num_threads(n);
  return prev;
#else
  (void)n;
  return 1;
#endif
}
