/*
 * ftn.h -- the C ABI of libftn, a B200 (sm_100a) library that executes the
 * Fortran array statements arXiv 2409.18824 ("Fully integrating the Flang
 * Fortran compiler with standard MLIR", N. Brown) lowers from Flang's
 * HLFIR/FIR to standard MLIR (memref / scf / affine / linalg).
 *
 * Citation keys: P:n = the paper line n; S:n = SPEC.md line n;
 * R#n = reading n listed in DESIGN.md section 3 (where the paper is silent).
 *
 * Conventions for every call
 *   - Plain C: no C++ or CUDA types.  A stream is a cudaStream_t passed as
 *     ftn_stream_t (void*); NULL is the legacy default stream.
 *   - Memory: the CALLER owns every buffer, on the device, and every
 *     workspace; the library never frees caller memory.  Descriptors
 *     (ftn_desc_t) live in host memory and are copied by value into kernel
 *     parameters; the array elements they describe live in device memory.
 *   - Validation: every argument is checked on the host before anything is
 *     launched; on error nothing is launched and no output is touched
 *     (no partial output).  The status tells what failed;
 *     ftn_last_error() gives thread-local detail text.
 *   - Asynchrony: compute calls enqueue kernels on `stream` and return; a
 *     device fault surfaces at the caller's next synchronisation.  Scalar
 *     results are written to DEVICE memory.
 *   - No CPU fallback: on a device that is not sm_100 the calls return
 *     FTN_ERR_DEVICE.
 *   - Calls on distinct streams are thread-safe; an ftn_comm_t is used by one
 *     thread at a time.
 */
#ifndef FTN_H
#define FTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FTN_MAX_RANK 3

/* Element types: Fortran real(8), real(4), integer(4) (default kind, R#20),
 * integer(8).  elem_len 8/4/4/8 bytes. */
typedef enum { FTN_I32 = 1, FTN_I64 = 2, FTN_F32 = 3, FTN_F64 = 4 } ftn_type_t;

/* One dimension of a Fortran array ("tracks the starting location of
 * each dimension"; P:237 subviews carry "offsets, sizes and strides").
 * sm is the signed distance in BYTES between consecutive elements of the
 * dimension (it may be negative for a section with a negative step). */
typedef struct {
  int64_t lower_bound;
  int64_t extent;
  int64_t sm;
} ftn_dim_t;

/* A fir.box-like descriptor.  base_addr is the device address of element
 * (lower_bound_1, ..., lower_bound_rank); element (j_1..j_r) is at
 *   base_addr + sum_d (j_d - lower_bound_d) * dim[d].sm
 * i.e. the origin subtraction of P:233 folded into each access.  Array
 * element order is column-major: dim[0] varies fastest (R#1).
 * rank 0 describes a scalar operand at base_addr (device memory). */
typedef struct {
  void* base_addr;
  int64_t elem_len;
  int32_t rank;
  int32_t type; /* ftn_type_t */
  ftn_dim_t dim[FTN_MAX_RANK];
} ftn_desc_t;

typedef enum {
  FTN_OK = 0,
  FTN_ERR_NULL = 1,        /* a required pointer is NULL */
  FTN_ERR_RANK = 2,        /* rank outside what the call accepts */
  FTN_ERR_TYPE = 3,        /* element type mismatch / unsupported type */
  FTN_ERR_SHAPE = 4,       /* operands are not conformable */
  FTN_ERR_BOUNDS = 5,      /* section outside its parent, zero step */
  FTN_ERR_DIM = 6,         /* bad DIM argument of an inquiry */
  FTN_ERR_ALIGN = 7,       /* an entry point that requires alignment did not get it */
  FTN_ERR_UNSUPPORTED = 8, /* a valid Fortran form this library does not implement (MASK=, rank > 3) */
  FTN_ERR_WORKSPACE = 9,   /* workspace NULL or smaller than *_workspace_size */
  FTN_ERR_DEVICE = 10,     /* current device is not sm_100 */
  FTN_ERR_CUDA = 11,       /* a CUDA launch / API error */
  FTN_ERR_NCCL = 12        /* an NCCL error */
} ftn_status_t;

typedef void* ftn_stream_t; /* cudaStream_t */

/* ---------------------------------------------------------------- a1 / a2
 * Descriptors and inquiry (host only, pure; no device access). */

/* Declaration `T :: x(lb(1):lb(1)+ext(1)-1, ...)` of a contiguous array at
 * base (P:217 allocatables; P:233 lower bounds).  Strides are the packed
 * column-major ones: sm_1 = elem_len, sm_{d+1} = sm_d * ext_d.  rank 0..3;
 * ext >= 0. */
ftn_status_t ftn_desc_contiguous(ftn_desc_t* out, void* base, int32_t type, int32_t rank,
                                 const int64_t* lower_bounds, const int64_t* extents);

/* Section `parent(lo(1):hi(1):step(1), ...)` (a subview -- same memory,
 * new offsets/sizes/strides, no copy).  Per dimension the extent is
 * max(0, (hi - lo + step) / step) (P:191 negative steps); the section's
 * lower bounds are 1 (R#2); sm = step * parent sm; base = &parent(lo...).
 * FTN_ERR_BOUNDS if a step is 0 or a selected element lies outside the parent
 * (checked only when the extent is > 0).  *out is written only on FTN_OK. */
ftn_status_t ftn_desc_section(ftn_desc_t* out, const ftn_desc_t* parent, const int64_t* lo,
                              const int64_t* hi, const int64_t* step);

/* LBOUND / UBOUND / SIZE / SHAPE ("SIZE corresponds directly to
 * memref.dim").  dim is 1-based; ftn_size with dim == 0 is SIZE(x). */
ftn_status_t ftn_lbound(const ftn_desc_t* x, int32_t dim, int64_t* out);
ftn_status_t ftn_ubound(const ftn_desc_t* x, int32_t dim, int64_t* out);
ftn_status_t ftn_size(const ftn_desc_t* x, int32_t dim, int64_t* out);
ftn_status_t ftn_shape(const ftn_desc_t* x, int64_t* out /* [rank] */);

/* May a and b share a byte of memory?  The alias test behind R#5's temporaries.
 * *out = 0 only when they provably do not: empty, disjoint byte ranges, or
 * element addresses that fall in disjoint residue classes modulo the gcd of all
 * strides (e.g. a(1::2,:) and a(2::2,:) of an array with an even leading
 * extent); otherwise 1 (conservative: never 0 for sections that share a byte).
 * Host-only. */
ftn_status_t ftn_desc_may_overlap(const ftn_desc_t* a, const ftn_desc_t* b, int32_t* out);

/* ---------------------------------------------------------------- a3
 * Element-wise array expressions.  Fortran assignment semantics: the whole
 * right-hand side is evaluated before the left-hand side is defined (R#5);
 * when dst shares memory with an operand through any mapping other than the
 * identical one, the library evaluates into a temporary that it allocates on
 * the stream (cudaMallocAsync) and frees after the store.  Operands must be
 * conformable with dst (same rank and extents; lower bounds are ignored) or
 * rank 0 (a scalar in device memory, broadcast).  All operands share dst's
 * type. */

typedef enum { FTN_ADD = 1, FTN_SUB = 2, FTN_MUL = 3, FTN_DIV = 4, FTN_MULADD = 5 } ftn_op_t;
#define FTN_CONTRACT 1u /* MULADD as one fused multiply-add (single rounding), R#6 */

/* dst = src.  rank 1..3. */
ftn_status_t ftn_assign(const ftn_desc_t* dst, const ftn_desc_t* src, ftn_stream_t stream);

/* dst = s, with s one element of dst's type read from HOST memory. */
ftn_status_t ftn_fill(const ftn_desc_t* dst, const void* scalar_host, ftn_stream_t stream);

/* dst = a op b (ADD/SUB/MUL/DIV) or dst = a*b + c (MULADD; c ignored otherwise).
 * Reals: IEEE binary64/32 round-to-nearest-even, no contraction unless
 * flags & FTN_CONTRACT (then MULADD is fma(a,b,c)).  Integers: modulo 2^w
 * (R#9); DIV truncates toward zero and a zero divisor is undefined. */
ftn_status_t ftn_elemental(int32_t op, const ftn_desc_t* dst, const ftn_desc_t* a,
                           const ftn_desc_t* b, const ftn_desc_t* c, uint32_t flags,
                           ftn_stream_t stream);

/* ---------------------------------------------------------------- a4
 * Reductions to a scalar (a zero-initialised rank-0 output and a
 * linalg.reduce over the array; MAXVAL and PRODUCT "are also implemented").
 * x: rank 1..3, any strides.  result_dev: device pointer to one element of
 * x's type.  ws: device workspace of at least ftn_reduce_workspace_size()
 * bytes (8-byte aligned), not used concurrently by another call.
 * Real SUM is combined in the documented order R, so results
 * are deterministic, identical for a section and its packed copy, and within
 * 4*n*2^-53*sum|x| of the exact sum (R#8).  Integer SUM wraps (exact).
 * Empty arrays: SUM = 0, MAXVAL = -inf / most negative integer, MINVAL = +inf
 * / most positive integer (R#10).  NaN is ignored by MAXVAL/MINVAL unless all
 * elements are NaN (R#11). */
ftn_status_t ftn_reduce_workspace_size(const ftn_desc_t* x, size_t* bytes);
ftn_status_t ftn_sum(const ftn_desc_t* x, void* result_dev, void* ws, size_t ws_bytes,
                     ftn_stream_t stream);
ftn_status_t ftn_maxval(const ftn_desc_t* x, void* result_dev, void* ws, size_t ws_bytes,
                        ftn_stream_t stream);
ftn_status_t ftn_minval(const ftn_desc_t* x, void* result_dev, void* ws, size_t ws_bytes,
                        ftn_stream_t stream);
/* PRODUCT(x) ("product ... also implemented"): order R with
 * multiplication, neutral 1 (empty -> 1); reals within (n-1)*2^-53 relative of the exact
 * product (each multiply rounds once); integers modulo 2^w.  Workspace as for ftn_sum. */
ftn_status_t ftn_product(const ftn_desc_t* x, void* result_dev, void* ws, size_t ws_bytes,
                         ftn_stream_t stream);

/* SUM / PRODUCT / MAXVAL / MINVAL (x, DIM=dim) (linalg.reduce with `dimensions`;
 * SURVEY §8(f) f1).  x: rank 1..3, any strides; dim 1-based.  result: rank(x)-1 descriptor
 * (rank 0 = one element at base_addr) whose extents are x's without dimension dim, same
 * type, not overlapping x.  Each result element is the sequential fold over the reduced
 * subscript in ascending order from the neutral element (R#24), so results are exact
 * replicas of the paper's loop; MAXVAL/MINVAL NaN and empty rules as above.  No workspace. */
ftn_status_t ftn_sum_dim(const ftn_desc_t* x, int32_t dim, const ftn_desc_t* result, ftn_stream_t stream);
ftn_status_t ftn_product_dim(const ftn_desc_t* x, int32_t dim, const ftn_desc_t* result, ftn_stream_t stream);
ftn_status_t ftn_maxval_dim(const ftn_desc_t* x, int32_t dim, const ftn_desc_t* result, ftn_stream_t stream);
ftn_status_t ftn_minval_dim(const ftn_desc_t* x, int32_t dim, const ftn_desc_t* result, ftn_stream_t stream);

/* DOT_PRODUCT(x, y) = SUM(x*y) for rank-1 real vectors of equal size (P:298,
 * R#12); each product is rounded, then summed in order R, so the result is
 * bit-identical to ftn_sum of the packed product vector.  Workspace as for
 * ftn_sum(x). */
ftn_status_t ftn_dot_product(const ftn_desc_t* x, const ftn_desc_t* y, void* result_dev,
                             void* ws, size_t ws_bytes, ftn_stream_t stream);

/* ---------------------------------------------------------------- a5
 * dst = TRANSPOSE(src): dst(j,i) = src(i,j); src rank 2 with shape
 * (n1,n2), dst rank 2 with shape (n2,n1), same type, any strides, no overlap
 * (an overlapping dst is evaluated through a temporary). */
ftn_status_t ftn_transpose(const ftn_desc_t* dst, const ftn_desc_t* src, ftn_stream_t stream);

/* ---------------------------------------------------------------- a6
 * c = MATMUL(a, b) for real(8) operands (F2018 16.9.124):
 *   rank 2 x rank 2: c(i,j) = sum_l a(i,l) b(l,j), a (m,k), b (k,n), c (m,n), computed on the
 *     fp64 tensor cores (DMMA); the per-element summation order inside a tensor-core step is
 *     the hardware's, so c is within 4*k*2^-53*sum|a||b| of the exact value (R#8, R#14) and
 *     exact when all partial sums are representable (integer-valued data);
 *   rank 2 x rank 1: c(i) = sum_l a(i,l) b(l) (m);  rank 1 x rank 2: c(j) = sum_l a(l) b(l,j)
 *     (n) -- HBM-bound kernels, same bound.
 * Rank-2 operands that are not TMA-able (dim-1 stride != 8 bytes, a column stride that is
 * not a multiple of 16 bytes, a base that is not 16-byte aligned) are first packed into ws.
 * An overlapping c is computed through a temporary (R#5). */
ftn_status_t ftn_matmul_workspace_size(const ftn_desc_t* c, const ftn_desc_t* a,
                                       const ftn_desc_t* b, size_t* bytes);
ftn_status_t ftn_matmul(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, void* ws,
                        size_t ws_bytes, ftn_stream_t stream);

/* c = MATMUL(op(a), op(b)) with op = TRANSPOSE when the flag is set, for rank-2 operands,
 * without materialising the transpose (the TMA boxes and fragment addressing swap roles;
 * SURVEY §8(f) f3).  Workspace: ftn_matmul_ex_workspace_size. */
#define FTN_MATMUL_TRANSPOSE_A 1u
#define FTN_MATMUL_TRANSPOSE_B 2u
/* Small rank-2 products (M*N*K <= 2^21, K <= 4096, e.g. C1's 48 x 48 x 32) run one thread per
 * c(i,j) folding l = 1..K in order with one rounding per product and per sum (the literal
 * definition: bit-identical to a sequential fold; no packing, any strides); the DMMA path
 * serves the rest.  FTN_MATMUL_FORCE_DMMA (tuning / testing) takes the DMMA path always. */
#define FTN_MATMUL_FORCE_DMMA 4u
ftn_status_t ftn_matmul_ex_workspace_size(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b,
                                          uint32_t flags, size_t* bytes);
ftn_status_t ftn_matmul_ex(const ftn_desc_t* c, const ftn_desc_t* a, const ftn_desc_t* b, uint32_t flags,
                           void* ws, size_t ws_bytes, ftn_stream_t stream);

/* ---------------------------------------------------------------- a7
 * Jacobi sweeps ("a Jacobi iteration solving Laplace's equation"; the
 * DO-nest of R#16):
 *   do s = 1, sweeps
 *     unew(i,j) = coeff * (((u(i-1,j) + u(i+1,j)) + u(i,j-1)) + u(i,j+1))
 *   (3-D: coeff * (((((u(i-1)+u(i+1)) + u(j-1)) + u(j+1)) + u(k-1)) + u(k+1)))
 *   for every interior point, then swap(u, unew).
 * u, unew: real(8), rank 2 (5-point) or rank 3 (7-point), conformable, not
 * overlapping.  Only interior points are written: the caller presets the
 * boundary of both arrays to the SAME values (R#16: then the swap equals u = unew; the
 * fused kernels carry the source's ring through their intermediate sweeps).  *result_in_unew (host) receives 1 when the final
 * values are in unew (odd sweeps), else 0.  Bit-exact vs the oracle.
 * Allocates nothing: arrays the TMA kernels cannot address (odd leading dimension, strided
 * or reversed sections) run the generic one-point-per-thread kernel (see ftn_jacobi_ws for
 * the faster path with a caller workspace).  Results are identical either way. */
ftn_status_t ftn_jacobi(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t sweeps, double coeff,
                        int32_t* result_in_unew, ftn_stream_t stream);

/* Bytes of caller workspace with which ftn_jacobi_ws runs `sweeps` sweeps of these arrays
 * through the temporally blocked kernels: 0 when u / unew are TMA-able (or sweeps < 8, or
 * an extent is < 3), else two padded packed copies (even leading dimension).  Host-only. */
ftn_status_t ftn_jacobi_workspace_size(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t sweeps,
                                       size_t* bytes);

/* ftn_jacobi with a caller workspace ws (256-byte aligned, or NULL): when ws_bytes >=
 * ftn_jacobi_workspace_size(u, unew, sweeps) > 0, both arrays are copied into padded packed
 * copies in ws, advanced there by the temporally blocked kernels and copied back (4 extra
 * passes instead of `sweeps` passes of the generic kernel); otherwise as ftn_jacobi.  Same
 * results and result array either way.  FTN_ERR_WORKSPACE for a misaligned ws. */
ftn_status_t ftn_jacobi_ws(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t sweeps, double coeff,
                           void* ws, size_t ws_bytes, int32_t* result_in_unew, ftn_stream_t stream);

/* Tuning (not semantics): rank-2 sweeps are executed up to T at a time by one kernel that
 * keeps the intermediate iterates in registers (temporal blocking, SURVEY §8(f) f2,
 * DESIGN.md §4.3), rank-3 sweeps up to min(T, 3) at a time (§4.4).  Results are
 * bit-identical for every T; the array that does not hold the result holds an earlier
 * iterate.  T in 1..12 (1 = one sweep per launch; the kernels fuse up to 8 and a larger T
 * runs launches of 8, except in -DFTN_WQ_BIG_T tuning builds); default 8 or the FTN_JACOBI_FUSE environment variable; unless T is set
 * explicitly, rank-2 grids of <= 2^22 points use 6 and of < 2^24 points 7 (measured best;
 * small launches are latency bound).  ftn_jacobi_get_fusion returns
 * the process-wide T (8 by default).  ftn_jacobi_set_fusion(0) restores the default.
 * Process-wide. */
ftn_status_t ftn_jacobi_set_fusion(int32_t sweeps_per_launch);
int32_t ftn_jacobi_get_fusion(void);
/* The sweeps per launch ftn_jacobi uses for this array (at most ftn_jacobi_get_fusion(); the
 * size-dependent rank-2 default; min(T, 3) for rank 3 -- jacobi3d_wr / jacobi3d_tb2; 1 for
 * arrays the fused kernels cannot address); 0 for an invalid descriptor.  Host-only. */
int32_t ftn_jacobi_fusion_for(const ftn_desc_t* u);

/* ftn_jacobi with the data on the host: host_u -> u (host-to-device copy), u -> unew
 * (device copy, presets the boundary of unew), `sweeps` sweeps, then the result -> host_result
 * (device-to-host copy), all enqueued on `stream` in that order.  host_u and host_result are
 * packed column-major real(8) arrays of u's shape (host pointers; pinned memory makes the
 * call asynchronous and lets calls on different streams overlap their copies and kernels);
 * u and unew are packed device arrays (desc contiguous).  host_result may alias host_u.
 * *result_in_unew as for ftn_jacobi.  FTN_ERR_SHAPE for non-packed device arrays. */
ftn_status_t ftn_jacobi_host(const double* host_u, double* host_result, const ftn_desc_t* u,
                             const ftn_desc_t* unew, int64_t sweeps, double coeff, int32_t* result_in_unew,
                             ftn_stream_t stream);

/* The launch plan ftn_jacobi / ftn_jacobi_dist use for `sweeps` sweeps with at most T per
 * launch: floor(S/T) launches of T and one of S mod T, with one launch split k -> (k-1)+1
 * when needed so that the launch count has the parity of S (the result then lands in unew
 * iff S is odd).  Writes up to cap sweep counts to sizes (may be NULL); returns the count. */
int64_t ftn_jacobi_plan(int64_t sweeps, int32_t T, int32_t* sizes, int64_t cap);

/* Jacobi iteration to convergence (R#25): sweeps in blocks of
 * check_every (the last block may be shorter); after each block the residual
 * res = MAXVAL(ABS(u_s - u_{s-1})) of the last two iterates over the INTERIOR points (the
 * points a sweep updates; -inf when there are none) is computed on the device and read back
 * (one stream synchronisation per block); stop when res <= tol or after max_sweeps.  For
 * rank-2 TMA-able arrays the residual is fused into the block's last launch (no extra pass
 * over the arrays).  *sweeps_done, *residual (0 when no sweep ran) and *result_in_unew are
 * written on the host; the result is in unew iff sweeps_done is odd (as for ftn_jacobi).
 * ws: 256-byte aligned, at least ftn_reduce_workspace_size(u) + 16 bytes; with
 * ftn_jacobi_solve_workspace_size bytes, arrays the TMA kernels cannot address run on padded
 * copies in ws (as ftn_jacobi_ws). */
ftn_status_t ftn_jacobi_solve_workspace_size(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t max_sweeps,
                                             int64_t check_every, size_t* bytes);
ftn_status_t ftn_jacobi_solve(const ftn_desc_t* u, const ftn_desc_t* unew, int64_t max_sweeps,
                              int64_t check_every, double tol, double coeff, void* ws, size_t ws_bytes,
                              int64_t* sweeps_done, double* residual, int32_t* result_in_unew,
                              ftn_stream_t stream);

/* MAXVAL(ABS(x - y)) of conformable real(8) arrays without forming x - y (a fused
 * reduction of an element-wise expression; exact).  Workspace as for ftn_sum(x). */
ftn_status_t ftn_maxval_absdiff(const ftn_desc_t* x, const ftn_desc_t* y, void* result_dev, void* ws,
                                size_t ws_bytes, ftn_stream_t stream);

/* ---------------------------------------------------------------- f4
 * pw-advection (the paper's pw-advection benchmark, P:92-93, P:345-366 —
 * its body is not in the paper; R#26 gives the DO nest this implements):
 *   do i = 2, nx-1; do j = 2, ny-1; do k = 2, nz-1
 *     su(k,j,i) = tcx*(u(k,j,i-1)*(u(k,j,i)+u(k,j,i-1)) - u(k,j,i+1)*(u(k,j,i)+u(k,j,i+1)))
 *               + tcy*(...) + tzc1(k)*u(k-1,j,i)*(...) - tzc2(k)*u(k+1,j,i)*(...)   (and sv, sw)
 * u, v, w, su, sv, sw: real(8) rank-3 conformable arrays indexed (k, j, i) (dim 1 = k);
 * tzc1, tzc2, tzd1, tzd2: real(8) rank-1 of extent size(u, 1); tcx, tcy: scalars.  Only
 * interior points of su, sv, sw are written (boundaries are the caller's).  Outputs must
 * not overlap inputs or each other (FTN_ERR_SHAPE).  Bit-exact vs the oracle (one rounding
 * per operation, Fortran evaluation order).  Any strides; the fast path needs TMA-able
 * inputs (unit stride in dim 1, 16-byte aligned base and dim-2/3 strides). */
ftn_status_t ftn_pw_advection(const ftn_desc_t* su, const ftn_desc_t* sv, const ftn_desc_t* sw,
                              const ftn_desc_t* u, const ftn_desc_t* v, const ftn_desc_t* w,
                              const ftn_desc_t* tzc1, const ftn_desc_t* tzc2, const ftn_desc_t* tzd1,
                              const ftn_desc_t* tzd2, double tcx, double tcy, ftn_stream_t stream);

/* tra-adv (the paper's NEMO tracer-advection benchmark, P:92 -- its body is
 * not in the paper; R#28 gives the recalled loop nests this implements, identical
 * to oracle/ftn_oracle.c's orc_tra_adv_f64): `iters` iterations updating the tracer md in
 * place from the velocities pun, pvn, pwn, the masks umask, vmask, tmask, the temperature
 * tsn (3-D, real(8), conformable, indexed (ji, jj, jk)), ztfreez, rnfmsk, upsmsk (2-D, extents
 * (jpi, jpj)) and rnfmsk_z (1-D, extent jpk).  Any strides.  The temporaries zind, zwx, zwy,
 * zslpx, zslpy live in the caller's workspace (ftn_tra_adv_workspace_size bytes, 256-byte
 * aligned), are zeroed at the start of the call and carry over between iterations (R#28).
 * md must not overlap an input (FTN_ERR_SHAPE); jpj, jpk <= 65535.  Bit-exact vs the oracle. */
ftn_status_t ftn_tra_adv_workspace_size(const ftn_desc_t* md, size_t* bytes);
ftn_status_t ftn_tra_adv(const ftn_desc_t* md, const ftn_desc_t* tsn, const ftn_desc_t* pun, const ftn_desc_t* pvn,
                         const ftn_desc_t* pwn, const ftn_desc_t* umask, const ftn_desc_t* vmask,
                         const ftn_desc_t* tmask, const ftn_desc_t* ztfreez, const ftn_desc_t* rnfmsk,
                         const ftn_desc_t* upsmsk, const ftn_desc_t* rnfmsk_z, int64_t iters, void* ws,
                         size_t ws_bytes, ftn_stream_t stream);

/* ---------------------------------------------------------------- a8
 * Multi-GPU (one process per GPU, NCCL over NVLink).  The id travels between
 * processes through the caller's own channel (torch.distributed store). */
typedef struct ftn_comm_s* ftn_comm_t;
#define FTN_COMM_ID_BYTES 128
ftn_status_t ftn_comm_unique_id(uint8_t id[FTN_COMM_ID_BYTES]);
ftn_status_t ftn_comm_init(ftn_comm_t* comm, int32_t nranks, int32_t rank,
                           const uint8_t id[FTN_COMM_ID_BYTES], int32_t device);
/* nranks communicators of ONE process ("virtual ranks"): comms[r] is rank r, on device
 * devices[r] (all ranks may share one GPU).  Each rank must be driven by its own host thread
 * (its calls block until the matching calls of its peers arrive, at most 300 s, then
 * FTN_ERR_NCCL).  Every message is one cudaMemcpyAsync on the receiver's stream, ordered by
 * CUDA events after the sender's stream; a send completes, in stream order, once the
 * receiver's copy has (the semantics of grouped ncclSend/ncclRecv).  The distributed calls
 * below run exactly the same loops as over NCCL: this is how their p > 1 paths are tested on
 * one GPU.  Destroy each comm with ftn_comm_destroy. */
ftn_status_t ftn_comm_init_virtual(ftn_comm_t* comms, int32_t nranks, const int32_t* devices);
ftn_status_t ftn_comm_destroy(ftn_comm_t comm);
/* Overlap of the Jacobi halo exchange with the interior sweeps in ftn_jacobi_dist: the owned
 * planes whose dependence cone stays inside the owned planes are advanced on a side stream
 * of the communicator while ncclSend/ncclRecv run on the caller's stream; the planes next to
 * the halos follow the exchange.  mode 0 = off, 1 = when nranks > 1 (default), 2 = always
 * (also at nranks = 1, for testing).  Results are identical in every mode. */
ftn_status_t ftn_comm_set_overlap(ftn_comm_t comm, int32_t mode);
/* SMs the interior sweeps on the side stream leave free for the exchange's kernels while
 * the overlap runs (persistent grids are sized for num_SMs - sms); 0..64, default 8. */
ftn_status_t ftn_comm_set_sm_reserve(ftn_comm_t comm, int32_t sms);

/* Global reductions of an array slab-distributed over the ranks along its
 * last dimension (x_local is this rank's slab).  The result, identical on
 * every rank, goes to result_dev.  Real SUM / DOT: each rank reduces its slab
 * in order R, the p rank partials are all-gathered and combined by the same
 * balanced tree, so the result equals the single-GPU one bit for bit when
 * every slab holds the same power-of-two number of R chunks; otherwise it is
 * within the bound of R#8.  MAX/MIN and integer(8) SUM use the same all-gather +
 * tree (exact).  real(8) and integer(8) only.  ws: ftn_reduce_workspace_size of
 * x_local plus 8*(nranks+1) bytes, 8-byte aligned. */
ftn_status_t ftn_sum_global(ftn_comm_t comm, const ftn_desc_t* x_local, void* result_dev, void* ws,
                            size_t ws_bytes, ftn_stream_t stream);
ftn_status_t ftn_maxval_global(ftn_comm_t comm, const ftn_desc_t* x_local, void* result_dev,
                               void* ws, size_t ws_bytes, ftn_stream_t stream);
ftn_status_t ftn_minval_global(ftn_comm_t comm, const ftn_desc_t* x_local, void* result_dev,
                               void* ws, size_t ws_bytes, ftn_stream_t stream);
ftn_status_t ftn_dot_product_global(ftn_comm_t comm, const ftn_desc_t* x_local,
                                    const ftn_desc_t* y_local, void* result_dev, void* ws,
                                    size_t ws_bytes, ftn_stream_t stream);

/* Distributed Jacobi: u_local / unew_local are this rank's slab of the global array
 * along the last dimension with `halo` planes on each side: local planes
 * [halo, n_last - halo) are owned, rank r's first owned plane follows rank r-1's last,
 * and on the first (last) rank local plane halo-1 (n_last-halo) is the global boundary
 * plane.  Per step the k owned planes next to each neighbour are exchanged with
 * ncclSend/ncclRecv (k = 1, or k = T sweeps fused per step for TMA-able slabs,
 * T = min(halo, ftn_jacobi_fusion_for(u_local)): for rank 3 at most FTN_J3_T, default 3)
 * and ftn_jacobi_slab advances the owned planes by k sweeps.  Results are bit-identical to ftn_jacobi on the undivided array;
 * *result_in_unew as for ftn_jacobi. */
ftn_status_t ftn_jacobi_dist(ftn_comm_t comm, const ftn_desc_t* u_local, const ftn_desc_t* unew_local,
                             int64_t sweeps, double coeff, int32_t halo, int32_t* result_in_unew,
                             ftn_stream_t stream);

/* Distributed Jacobi to convergence (SURVEY §8(f) f2 with the a8 exchange; R#25): slabs as
 * for ftn_jacobi_dist; blocks of check_every sweeps by its plan; each rank's residual
 * MAXVAL(ABS(u_s - u_{s-1})) over its owned interior points (fused into the block's last
 * launch for rank-2 TMA-able slabs), all-gathered; the global residual is the maximum of the
 * p values (exact, so identical on every rank and equal to ftn_jacobi_solve's on the
 * undivided array).  Stops when it is <= tol or after max_sweeps; one stream synchronisation
 * per block.  ws: 8*(nranks+2) + ftn_reduce_workspace_size(u_local) bytes, 16-byte aligned.
 * Outputs as for ftn_jacobi_solve; results bit-identical to it on the undivided array. */
ftn_status_t ftn_jacobi_solve_dist(ftn_comm_t comm, const ftn_desc_t* u_local, const ftn_desc_t* unew_local,
                                   int32_t halo, int64_t max_sweeps, int64_t check_every, double tol,
                                   double coeff, void* ws, size_t ws_bytes, int64_t* sweeps_done,
                                   double* residual, int32_t* result_in_unew, ftn_stream_t stream);

/* One local step of the distributed Jacobi without communication (for callers with their
 * own exchange, e.g. MPI): `sweeps` (1 <= sweeps <= halo) sweeps of the owned planes of a
 * slab laid out as for ftn_jacobi_dist whose halo planes are current, src -> dst.  Reads src
 * planes [halo - sweeps, n_last - halo + sweeps); writes only the owned interior of dst.
 * first / last: this slab holds the global lower / upper boundary plane.  sweeps > 1 needs
 * a TMA-able slab: rank 2 up to 8 sweeps, rank 3 up to 4 (FTN_ERR_UNSUPPORTED otherwise). */
ftn_status_t ftn_jacobi_slab(const ftn_desc_t* src, const ftn_desc_t* dst, int32_t sweeps, double coeff,
                             int32_t halo, int32_t first, int32_t last, ftn_stream_t stream);

/* c(:, J_r) = MATMUL(a, b(:, J_r)): b_local / c_local are this rank's column
 * block, a is replicated (see ftn_bcast).  No communication. */
ftn_status_t ftn_matmul_colsharded(ftn_comm_t comm, const ftn_desc_t* c_local, const ftn_desc_t* a_full,
                                   const ftn_desc_t* b_local, void* ws, size_t ws_bytes,
                                   ftn_stream_t stream);
/* Broadcast a contiguous array from root to every rank (ncclBroadcast). */
ftn_status_t ftn_bcast(ftn_comm_t comm, const ftn_desc_t* x, int32_t root, ftn_stream_t stream);

/* ---------------------------------------------------------------- support */

/* Seeded synthetic inputs (not part of the method):
 * element t (array element order) of dst gets a value derived from
 *   h = splitmix64(seed ^ (array_id << 56) ^ t)
 * mode 1 U[0,1) = (h >> 11) * 2^-53; 2 U[-1,1) = 2*U[0,1) - 1;
 * 3 integer in [-8, 8] = (h >> 11) % 17 - 8; 4 t; 5 t mod 1024;
 * 6 (integer types) the low bits of h. */
typedef enum { FTN_GEN_U01 = 1, FTN_GEN_U11 = 2, FTN_GEN_INT8 = 3, FTN_GEN_LINEAR = 4,
               FTN_GEN_MOD1024 = 5, FTN_GEN_RAW = 6 } ftn_gen_mode_t;
ftn_status_t ftn_gen_fill(const ftn_desc_t* dst, uint64_t seed, uint64_t array_id, int32_t mode,
                          ftn_stream_t stream);
/* ftn_gen_fill with the sequence starting at element t0: element t of dst gets the value of
 * element t0 + t (a slab of a larger array generated where it lives; mode 4/5 use t0 + t too). */
ftn_status_t ftn_gen_fill_at(const ftn_desc_t* dst, uint64_t seed, uint64_t array_id, int32_t mode, uint64_t t0,
                             ftn_stream_t stream);

/* Number of kernels this library has launched in this process (all devices). */
uint64_t ftn_launch_count(void);

const char* ftn_status_string(ftn_status_t s);
const char* ftn_last_error(void); /* thread-local detail of the last failure */

#ifdef __cplusplus
}
#endif
#endif /* FTN_H */
