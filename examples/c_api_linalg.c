/*
 * MATMUL, TRANSPOSE and Jacobi-to-convergence from plain C through include/ftn.h:
 *
 *   real(8) :: a(64, 80), b(80, 48), c(64, 48), at(80, 64)
 *   a = <seeded U[-1,1), id 1>;  b = <seeded U[-1,1), id 2>
 *   c = matmul(a, b)                      ->  ftn_matmul (caller workspace)
 *   at = transpose(a)                     ->  ftn_transpose
 *   real(8) :: u(130, 90), unew(130, 90)  (u = seeded U[0,1) interior, faces 0, u(:,1) = 1)
 *   sweep until maxval(abs(u_s - u_(s-1))) <= 1e-6, checked every 10 sweeps, at most 3000
 *                                         ->  ftn_jacobi_solve
 *
 * Writes c, at, the solve's (sweeps, residual, result-in-unew) and its result array to argv[1]
 * (tests/test_gpu_c_api.py checks them against the oracle).
 */
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime_api.h>

#include "ftn.h"

#define CHECK(call)                                                                                 \
  do {                                                                                              \
    ftn_status_t st_ = (call);                                                                      \
    if (st_ != FTN_OK) {                                                                            \
      fprintf(stderr, "%s failed: %s (%s)\n", #call, ftn_status_string(st_), ftn_last_error());    \
      return 1;                                                                                     \
    }                                                                                               \
  } while (0)

static double* dalloc(size_t n) {
  double* p = NULL;
  return cudaMalloc((void**)&p, n * sizeof(double)) == cudaSuccess ? p : NULL;
}

static int face(const ftn_desc_t* u, int64_t i0, int64_t i1, int64_t j0, int64_t j1, double v) {
  const int64_t lo[2] = {i0, j0}, hi[2] = {i1, j1}, st[2] = {1, 1};
  ftn_desc_t f;
  CHECK(ftn_desc_section(&f, u, lo, hi, st));
  CHECK(ftn_fill(&f, &v, 0));
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: %s out.bin\n", argv[0]);
    return 2;
  }
  const int64_t m = 64, k = 80, n = 48, lb[2] = {1, 1};
  const int64_t ea[2] = {m, k}, eb[2] = {k, n}, ec[2] = {m, n}, et[2] = {k, m};
  double *da = dalloc(m * k), *db = dalloc(k * n), *dc = dalloc(m * n), *dt = dalloc(k * m);
  if (!da || !db || !dc || !dt) return 1;
  ftn_desc_t a, b, c, at;
  CHECK(ftn_desc_contiguous(&a, da, FTN_F64, 2, lb, ea));
  CHECK(ftn_desc_contiguous(&b, db, FTN_F64, 2, lb, eb));
  CHECK(ftn_desc_contiguous(&c, dc, FTN_F64, 2, lb, ec));
  CHECK(ftn_desc_contiguous(&at, dt, FTN_F64, 2, lb, et));
  CHECK(ftn_gen_fill(&a, 18824, 1, FTN_GEN_U11, 0));
  CHECK(ftn_gen_fill(&b, 18824, 2, FTN_GEN_U11, 0));
  size_t ws_bytes = 0;
  CHECK(ftn_matmul_workspace_size(&c, &a, &b, &ws_bytes));
  void* ws = NULL;
  if (cudaMalloc(&ws, ws_bytes ? ws_bytes : 16)) return 1;
  CHECK(ftn_matmul(&c, &a, &b, ws, ws_bytes, 0));
  CHECK(ftn_transpose(&at, &a, 0));

  const int64_t n1 = 130, n2 = 90, eu[2] = {n1, n2};
  double *du = dalloc(n1 * n2), *dw = dalloc(n1 * n2);
  if (!du || !dw) return 1;
  ftn_desc_t u, w;
  CHECK(ftn_desc_contiguous(&u, du, FTN_F64, 2, lb, eu));
  CHECK(ftn_desc_contiguous(&w, dw, FTN_F64, 2, lb, eu));
  CHECK(ftn_gen_fill(&u, 18824, 0, FTN_GEN_U01, 0));
  if (face(&u, 1, n1, n2, n2, 0.0) || face(&u, 1, 1, 1, n2, 0.0) || face(&u, n1, n1, 1, n2, 0.0) ||
      face(&u, 1, n1, 1, 1, 1.0))
    return 1;
  CHECK(ftn_assign(&w, &u, 0));
  size_t sws_bytes = 0;
  CHECK(ftn_jacobi_solve_workspace_size(&u, &w, 3000, 10, &sws_bytes));
  void* sws = NULL;
  if (cudaMalloc(&sws, sws_bytes ? sws_bytes : 256)) return 1;
  int64_t sweeps = 0;
  double residual = 0.0;
  int32_t in_unew = 0;
  CHECK(ftn_jacobi_solve(&u, &w, 3000, 10, 1e-6, 0.25, sws, sws_bytes, &sweeps, &residual, &in_unew, 0));

  double* host = (double*)malloc((size_t)(m * n + k * m + n1 * n2) * sizeof(double));
  if (!host || cudaMemcpy(host, dc, m * n * 8, cudaMemcpyDeviceToHost) ||
      cudaMemcpy(host + m * n, dt, k * m * 8, cudaMemcpyDeviceToHost) ||
      cudaMemcpy(host + m * n + k * m, in_unew ? dw : du, n1 * n2 * 8, cudaMemcpyDeviceToHost)) {
    fprintf(stderr, "cudaMemcpy failed\n");
    return 1;
  }
  FILE* f = fopen(argv[1], "wb");
  if (!f) return 1;
  fwrite(&sweeps, 8, 1, f);
  fwrite(&residual, 8, 1, f);
  fwrite(&in_unew, 4, 1, f);
  fwrite(host, 8, (size_t)(m * n + k * m + n1 * n2), f);
  fclose(f);
  printf("matmul %lldx%lldx%lld, transpose, jacobi_solve: %lld sweeps, residual %.3e, in unew %d\n",
         (long long)m, (long long)k, (long long)n, (long long)sweeps, residual, in_unew);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dc);
  cudaFree(dt);
  cudaFree(du);
  cudaFree(dw);
  cudaFree(ws);
  cudaFree(sws);
  free(host);
  return 0;
}
