/*
 * Plain-C use of the library through include/ftn.h (no Python): the Fortran program
 *
 *   real(8), allocatable :: u(:,:), unew(:,:)
 *   allocate(u(0:n1-1, -5:n2-6), unew(0:n1-1, -5:n2-6))
 *   u = <seeded U[0,1)>;  u(:, -5) = 1;  unew = u
 *   do s = 1, 10  (5-point Jacobi, swap)              ->  ftn_jacobi
 *   total = sum(u_result(::2, :))                       ->  ftn_sum on a section
 *
 * Writes the result array (column-major doubles) and the sum to the file given as argv[1]
 * (tests/test_gpu_c_api.py checks both against the oracle).
 * Build: gcc examples/c_api_demo.c -Iinclude -I/usr/local/cuda/include \
 *          -Lpaper_2409_18824_b200 -lftn -L/usr/local/cuda/lib64 -lcudart \
 *          -Wl,-rpath,$PWD/paper_2409_18824_b200 -o c_api_demo
 */
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime_api.h>

#include "ftn.h"

#define CHECK(call)                                                                  \
  do {                                                                               \
    ftn_status_t st_ = (call);                                                       \
    if (st_ != FTN_OK) {                                                             \
      fprintf(stderr, "%s failed: %s (%s)\n", #call, ftn_status_string(st_), ftn_last_error()); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: %s out.bin\n", argv[0]);
    return 2;
  }
  const int64_t n1 = 300, n2 = 200;
  const int64_t lb[2] = {0, -5}, ext[2] = {n1, n2};
  double *du = NULL, *dw = NULL, *dsum = NULL;
  if (cudaMalloc((void**)&du, n1 * n2 * 8) || cudaMalloc((void**)&dw, n1 * n2 * 8) || cudaMalloc((void**)&dsum, 8)) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  ftn_desc_t u, w;
  CHECK(ftn_desc_contiguous(&u, du, FTN_F64, 2, lb, ext));
  CHECK(ftn_desc_contiguous(&w, dw, FTN_F64, 2, lb, ext));
  /* u = U[0,1) (seed 18824, array id 0), boundary faces 0, the face j = lbound(2) = 1 */
  CHECK(ftn_gen_fill(&u, 18824, 0, FTN_GEN_U01, 0));
  const double zero = 0.0, one = 1.0;
  ftn_desc_t face;
  {
    const int64_t lo[2] = {0, n2 - 6}, hi[2] = {n1 - 1, n2 - 6}, st[2] = {1, 1};   /* j = ubound */
    CHECK(ftn_desc_section(&face, &u, lo, hi, st));
    CHECK(ftn_fill(&face, &zero, 0));
  }
  {
    const int64_t lo[2] = {0, -5}, hi[2] = {0, n2 - 6}, st[2] = {1, 1};            /* i = lbound */
    CHECK(ftn_desc_section(&face, &u, lo, hi, st));
    CHECK(ftn_fill(&face, &zero, 0));
  }
  {
    const int64_t lo[2] = {n1 - 1, -5}, hi[2] = {n1 - 1, n2 - 6}, st[2] = {1, 1};  /* i = ubound */
    CHECK(ftn_desc_section(&face, &u, lo, hi, st));
    CHECK(ftn_fill(&face, &zero, 0));
  }
  {
    const int64_t lo[2] = {0, -5}, hi[2] = {n1 - 1, -5}, st[2] = {1, 1};           /* j = lbound */
    CHECK(ftn_desc_section(&face, &u, lo, hi, st));
    CHECK(ftn_fill(&face, &one, 0));
  }
  CHECK(ftn_assign(&w, &u, 0));
  int32_t in_unew = 0;
  CHECK(ftn_jacobi(&u, &w, 10, 0.25, &in_unew, 0));
  const ftn_desc_t* res = in_unew ? &w : &u;
  ftn_desc_t sec;
  const int64_t lo[2] = {0, -5}, hi[2] = {n1 - 1, n2 - 6}, st[2] = {2, 1};
  CHECK(ftn_desc_section(&sec, res, lo, hi, st));
  size_t ws_bytes = 0;
  CHECK(ftn_reduce_workspace_size(&sec, &ws_bytes));
  void* ws = NULL;
  if (cudaMalloc(&ws, ws_bytes ? ws_bytes : 16)) return 1;
  CHECK(ftn_sum(&sec, dsum, ws, ws_bytes, 0));
  double* host = (double*)malloc(n1 * n2 * 8);
  double total = 0.0;
  if (cudaMemcpy(host, res->base_addr, n1 * n2 * 8, cudaMemcpyDeviceToHost) ||
      cudaMemcpy(&total, dsum, 8, cudaMemcpyDeviceToHost)) {
    fprintf(stderr, "cudaMemcpy failed\n");
    return 1;
  }
  FILE* f = fopen(argv[1], "wb");
  if (!f) return 1;
  fwrite(&total, 8, 1, f);
  fwrite(&in_unew, 4, 1, f);
  fwrite(host, 8, (size_t)(n1 * n2), f);
  fclose(f);
  printf("sum(u(::2,:)) = %.17g  result in unew: %d  launches: %llu\n", total, in_unew,
         (unsigned long long)ftn_launch_count());
  cudaFree(du);
  cudaFree(dw);
  cudaFree(dsum);
  cudaFree(ws);
  free(host);
  return 0;
}
