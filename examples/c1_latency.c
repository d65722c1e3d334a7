/*
 * C1 latency through the C ABI (no Python in the loop): real(8) a(0:63,1:48) with
 * a(i,j) = i + 64(j-1), s = a(::2,:), c = a(1::2,:), d(-5:26,10:57).  For each call, the
 * median over 1000 calls of (call + cudaStreamSynchronize) on the host clock, and the mean
 * per call of 1000 calls issued back to back then synchronised once.  Prints one JSON object.
 * Build: gcc -O2 examples/c1_latency.c -Iinclude -I/usr/local/cuda/include \
 *          -Lpaper_2409_18824_b200 -lftn -L/usr/local/cuda/lib64 -lcudart \
 *          -Wl,-rpath,$PWD/paper_2409_18824_b200 -o c1_latency
 */
#include <stdio.h>
#include <stdlib.h>
#include <time.h>
#include <cuda_runtime_api.h>

#include "ftn.h"

#define CHECK(call)                                                                             \
  do {                                                                                          \
    ftn_status_t st_ = (call);                                                                  \
    if (st_ != FTN_OK) {                                                                        \
      fprintf(stderr, "%s failed: %s (%s)\n", #call, ftn_status_string(st_), ftn_last_error()); \
      exit(1);                                                                                  \
    }                                                                                           \
  } while (0)

enum { N = 1000 };

static double now_us(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}

static int cmp(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

static ftn_desc_t a, s, c, d, r, st, m48, b1, b2;
static void* ws;
static size_t ws_bytes;
static double* res;

static void op(int k) {
  switch (k) {
    case 0: CHECK(ftn_elemental(FTN_MULADD, &r, &s, &c, &d, 0, 0)); break;
    case 1: CHECK(ftn_sum(&s, res, ws, ws_bytes, 0)); break;
    case 2: CHECK(ftn_maxval(&s, res, ws, ws_bytes, 0)); break;
    case 3: CHECK(ftn_transpose(&st, &s, 0)); break;
    case 4: CHECK(ftn_matmul_ex(&m48, &s, &s, FTN_MATMUL_TRANSPOSE_A, ws, ws_bytes, 0)); break;
    case 5: CHECK(ftn_matmul(&m48, &b1, &b2, ws, ws_bytes, 0)); break;
  }
}

int main(void) {
  static const char* names[] = {"muladd_r=s*c+d", "sum_s", "maxval_s", "transpose_s",
                                "matmul_transpose(s)_s_48x48x32", "matmul_48^3"};
  double *pa, *pd, *pr, *pst, *pm, *pb1, *pb2;
  if (cudaMalloc((void**)&pa, 64 * 48 * 8) || cudaMalloc((void**)&pd, 32 * 48 * 8) ||
      cudaMalloc((void**)&pr, 32 * 48 * 8) || cudaMalloc((void**)&pst, 48 * 32 * 8) ||
      cudaMalloc((void**)&pm, 48 * 48 * 8) || cudaMalloc((void**)&pb1, 48 * 48 * 8) ||
      cudaMalloc((void**)&pb2, 48 * 48 * 8) || cudaMalloc((void**)&res, 8))
    return 1;
  const int64_t lba[2] = {0, 1}, exa[2] = {64, 48}, lbd[2] = {-5, 10}, ex32[2] = {32, 48};
  const int64_t one[2] = {1, 1}, ex48t[2] = {48, 32}, ex48[2] = {48, 48};
  CHECK(ftn_desc_contiguous(&a, pa, FTN_F64, 2, lba, exa));
  CHECK(ftn_desc_contiguous(&d, pd, FTN_F64, 2, lbd, ex32));
  CHECK(ftn_desc_contiguous(&r, pr, FTN_F64, 2, one, ex32));
  CHECK(ftn_desc_contiguous(&st, pst, FTN_F64, 2, one, ex48t));
  CHECK(ftn_desc_contiguous(&m48, pm, FTN_F64, 2, one, ex48));
  CHECK(ftn_desc_contiguous(&b1, pb1, FTN_F64, 2, one, ex48));
  CHECK(ftn_desc_contiguous(&b2, pb2, FTN_F64, 2, one, ex48));
  CHECK(ftn_gen_fill(&a, 18824, 0, FTN_GEN_LINEAR, 0));
  CHECK(ftn_gen_fill(&d, 18824, 1, FTN_GEN_U01, 0));
  CHECK(ftn_gen_fill(&b1, 18824, 2, FTN_GEN_U11, 0));
  CHECK(ftn_gen_fill(&b2, 18824, 3, FTN_GEN_U11, 0));
  const int64_t lo_s[2] = {0, 1}, hi_s[2] = {63, 48}, step[2] = {2, 1}, lo_c[2] = {1, 1};
  CHECK(ftn_desc_section(&s, &a, lo_s, hi_s, step));
  CHECK(ftn_desc_section(&c, &a, lo_c, hi_s, step));
  size_t w1 = 0, w2 = 0, w3 = 0;
  CHECK(ftn_reduce_workspace_size(&s, &w1));
  CHECK(ftn_matmul_ex_workspace_size(&m48, &s, &s, FTN_MATMUL_TRANSPOSE_A, &w2));
  CHECK(ftn_matmul_workspace_size(&m48, &b1, &b2, &w3));
  ws_bytes = w1 > w2 ? w1 : w2;
  ws_bytes = ws_bytes > w3 ? ws_bytes : w3;
  if (cudaMalloc(&ws, ws_bytes ? ws_bytes : 16)) return 1;
  /* closed form check: SUM(s) = 2357760 */
  double h = 0;
  CHECK(ftn_sum(&s, res, ws, ws_bytes, 0));
  cudaMemcpy(&h, res, 8, cudaMemcpyDeviceToHost);
  printf("{\"sum_closed_form_ok\": %s", h == 2357760.0 ? "true" : "false");
  static double t[N];
  printf(", \"sync_median_us\": {");
  for (int k = 0; k < 6; ++k) {
    for (int i = 0; i < 20; ++i) op(k);
    cudaStreamSynchronize(0);
    for (int i = 0; i < N; ++i) {
      const double t0 = now_us();
      op(k);
      cudaStreamSynchronize(0);
      t[i] = now_us() - t0;
    }
    qsort(t, N, sizeof(double), cmp);
    printf("%s\"%s\": %.2f", k ? ", " : "", names[k], t[N / 2]);
  }
  printf("}, \"back_to_back_mean_us\": {");
  for (int k = 0; k < 6; ++k) {
    cudaStreamSynchronize(0);
    const double t0 = now_us();
    for (int i = 0; i < N; ++i) op(k);
    cudaStreamSynchronize(0);
    printf("%s\"%s\": %.2f", k ? ", " : "", names[k], (now_us() - t0) / N);
  }
  printf("}}\n");
  return 0;
}
