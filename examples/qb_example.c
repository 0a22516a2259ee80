/* Minimal C client of the C ABI (include/qb.h): factor a synthetic low-rank matrix with host
 * buffers (qb_factor_host), then finish to a partial SVD on the device factors.
 *
 *   gcc -O2 -std=c99 -I include examples/qb_example.c -L paper_1503_07157_b200 -lqb \
 *       -Wl,-rpath,$PWD/paper_1503_07157_b200 -lm -o qb_example && ./qb_example
 *
 * Prints k, the reported residual, a host-side check of ||A - QB||_F and the leading singular
 * values; exits non-zero on any failure.  No CUDA headers are needed: the ABI has plain types. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "qb.h"

#define CHECK(call)                                                                     \
  do {                                                                                  \
    qb_status s_ = (call);                                                              \
    if (s_ != QB_OK && s_ != QB_NOT_CONVERGED) {                                        \
      fprintf(stderr, "%s: %s (%s)\n", #call, qb_status_string(s_), qb_last_error(ctx)); \
      return 1;                                                                         \
    }                                                                                   \
  } while (0)

int main(void) {
  const int64_t m = 600, n = 400, r = 40;
  /* A = U diag(s) V^T with U, V of random +-1/sqrt(.) entries (not orthonormal: fine for a demo),
   * column-major; s_j = 2^-j */
  double* A = calloc((size_t)(m * n), sizeof(double));
  double* U = malloc(sizeof(double) * (size_t)(m * r));
  double* V = malloc(sizeof(double) * (size_t)(n * r));
  unsigned x = 12345u;
  for (int64_t i = 0; i < m * r; ++i) { x = x * 1664525u + 1013904223u; U[i] = ((x >> 31) ? 1.0 : -1.0) / sqrt((double)m); }
  for (int64_t i = 0; i < n * r; ++i) { x = x * 1664525u + 1013904223u; V[i] = ((x >> 31) ? 1.0 : -1.0) / sqrt((double)n); }
  for (int64_t t = 0; t < r; ++t) {
    const double s = ldexp(1.0, -(int)t);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < m; ++i) A[i + j * m] += U[i + t * m] * s * V[j + t * n];
  }
  const int64_t kcap = 400;
  double* Q = malloc(sizeof(double) * (size_t)(m * kcap));
  double* B = malloc(sizeof(double) * (size_t)(n * kcap)); /* row-major k x n, ld n */
  qb_ctx ctx = NULL;
  CHECK(qb_create(&ctx, 0, QB_F64, NULL));
  int64_t k = 0;
  double resid = 0.0;
  const double eps = 1e-8;
  CHECK(qb_factor_host(ctx, A, m, n, m, eps, 16, 0, 7, 0, &k, Q, m, B, n, kcap, &resid));
  /* host check of ||A - QB||_F */
  double err2 = 0.0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      double v = A[i + j * m];
      for (int64_t t = 0; t < k; ++t) v -= Q[i + t * m] * B[t * n + j];
      err2 += v * v;
    }
  printf("k = %lld, reported residual = %.3e, host ||A - QB||_F = %.3e (eps = %.1e)\n", (long long)k, resid,
         sqrt(err2), eps);
  if (!(sqrt(err2) <= eps * (1 + 1e-6)) || fabs(sqrt(err2) - resid) > 1e-10) return 2;
  const void *Ud = NULL, *Sd = NULL, *Vd = NULL;
  int64_t ldu = 0, ldv = 0, kk = 0;
  CHECK(rqb_svd(ctx, 0.0, 5, &kk, &Ud, &ldu, &Sd, &Vd, &ldv));
  printf("rqb_svd: leading singular values live on the device at %p (k' = %lld); kernel launches so far: %lld\n", Sd,
         (long long)kk, (long long)qb_kernel_launches(ctx));
  qb_destroy(ctx);
  free(A); free(U); free(V); free(Q); free(B);
  return 0;
}
