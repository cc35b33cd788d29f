/* A compiled C consumer of the drop-in ABI: includes only include/bandsolve.h,
 * links against the library through its reference SONAME (libbandsolve.so.1),
 * and checks the behaviours the reference's own C-API suite asserts
 * (test_capi.cpp:21-141: statuses, version, threads, batch lifecycle, factor
 * error codes, tri / pent / uniform solves with residuals, shape mismatch,
 * periodic handles).
 *
 *   capi_consumer gpu     solves must succeed (B200 present)
 *   capi_consumer nogpu   solves must fail with BANDSOLVE_ERR_INTERNAL (no CPU fallback)
 *
 * Exit status 0 when every check passed; prints the failures otherwise. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "bandsolve.h"

static int g_checks = 0, g_failed = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(cond)) {                                                       \
      ++g_failed;                                                        \
      fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                    \
  } while (0)

static int g_gpu = 0;
/* a solve's status: OK with a device, ERR_INTERNAL without one */
static int solved(bandsolve_status st) {
  return g_gpu ? st == BANDSOLVE_OK : st == BANDSOLVE_ERR_INTERNAL;
}

static bandsolve_batch* batch_of(size_t n, size_t m, double (*f)(double), double w) {
  bandsolve_batch* b = NULL;
  if (bandsolve_batch_create(n, m, &b) != BANDSOLVE_OK) return NULL;
  double* d = bandsolve_batch_data(b);
  for (size_t k = 0; k < n * m; ++k) d[k] = f(w * (double)k);
  return b;
}

static bandsolve_batch* copy_of(const bandsolve_batch* src) {
  bandsolve_batch* b = NULL;
  const size_t n = bandsolve_batch_rows(src), m = bandsolve_batch_systems(src);
  if (bandsolve_batch_create(n, m, &b) != BANDSOLVE_OK) return NULL;
  memcpy(bandsolve_batch_data(b), bandsolve_batch_data_const(src), n * m * sizeof(double));
  return b;
}

static void statuses_and_threads(void) {
  CHECK(strcmp(bandsolve_status_string(BANDSOLVE_OK), "ok") == 0);
  CHECK(strcmp(bandsolve_status_string(BANDSOLVE_ERR_FACTORIZATION_BREAKDOWN), "factorization breakdown") == 0);
  CHECK(bandsolve_version() != NULL && strcmp(bandsolve_version(), "1.0.0") == 0);
  bandsolve_set_threads(3);
  CHECK(bandsolve_get_threads() == 3);
  bandsolve_set_threads(0);
  CHECK(bandsolve_get_threads() >= 1);
}

static void batches(void) {
  bandsolve_batch* b = NULL;
  CHECK(bandsolve_batch_create(4, 3, &b) == BANDSOLVE_OK);
  CHECK(bandsolve_batch_rows(b) == 4 && bandsolve_batch_systems(b) == 3);
  const double* d = bandsolve_batch_data_const(b);
  int zero = d != NULL;
  for (int k = 0; d && k < 12; ++k) zero = zero && d[k] == 0.0;
  CHECK(zero);
  bandsolve_batch* other = NULL;
  CHECK(bandsolve_batch_create(0, 3, &other) == BANDSOLVE_ERR_BAD_ARG && other == NULL);
  CHECK(bandsolve_batch_create(4, 3, NULL) == BANDSOLVE_ERR_BAD_ARG);
  CHECK(bandsolve_batch_rows(NULL) == 0 && bandsolve_batch_systems(NULL) == 0);
  bandsolve_batch_destroy(b);
  bandsolve_batch_destroy(NULL);
}

static void tridiagonal(void) {
  enum { n = 8 };
  double sub[n], diag[n], sup[n];
  for (int i = 0; i < n; ++i) sub[i] = sup[i] = -0.5, diag[i] = 2.0;
  sub[0] = sup[n - 1] = 0.0;
  bandsolve_tri_factor* f = NULL;
  CHECK(bandsolve_tri_factor_create(sub, diag, sup, n, &f) == BANDSOLVE_OK);
  bandsolve_batch* rhs = batch_of(n, 2, sin, 0.7);
  bandsolve_batch* x = copy_of(rhs);
  CHECK(solved(bandsolve_tri_solve_shared(f, x)));
  if (g_gpu) {
    double r = -1.0;
    CHECK(bandsolve_tri_residual(sub, diag, sup, n, 0, x, rhs, &r) == BANDSOLVE_OK && r >= 0.0 && r <= 1e-12);
  }
  bandsolve_batch* wrong = NULL;
  CHECK(bandsolve_batch_create(n + 1, 2, &wrong) == BANDSOLVE_OK);
  CHECK(bandsolve_tri_solve_shared(f, wrong) == BANDSOLVE_ERR_SHAPE_MISMATCH);
  CHECK(bandsolve_tri_solve_shared(NULL, x) == BANDSOLVE_ERR_BAD_ARG);
  bandsolve_batch_destroy(wrong);
  bandsolve_batch_destroy(x);
  bandsolve_batch_destroy(rhs);
  bandsolve_tri_factor_destroy(f);
  bandsolve_tri_factor_destroy(NULL);

  /* error codes: breakdown, nonzero structural slot, NULL band; *out stays NULL */
  double zero[4] = {0, 0, 0, 0}, ones[4] = {1, 1, 1, 1};
  f = NULL;
  CHECK(bandsolve_tri_factor_create(zero, zero, zero, 4, &f) == BANDSOLVE_ERR_FACTORIZATION_BREAKDOWN && f == NULL);
  CHECK(bandsolve_tri_factor_create(ones, ones, zero, 4, &f) == BANDSOLVE_ERR_BAD_ARG && f == NULL);
  CHECK(bandsolve_tri_factor_create(NULL, ones, zero, 4, &f) == BANDSOLVE_ERR_BAD_ARG && f == NULL);
}

static void pentadiagonal(void) {
  enum { n = 12 };
  double a[n], b[n], c[n], d[n], e[n];
  for (int i = 0; i < n; ++i) a[i] = e[i] = 0.25, b[i] = d[i] = -1.0, c[i] = 2.5;
  a[0] = a[1] = b[0] = 0.0;
  d[n - 1] = e[n - 1] = e[n - 2] = 0.0;
  bandsolve_pent_factor* f = NULL;
  bandsolve_uniform_pent_factor* u = NULL;
  CHECK(bandsolve_pent_factor_create(a, b, c, d, e, n, &f) == BANDSOLVE_OK);
  CHECK(bandsolve_uniform_pent_factor_create(0.25, -1.0, 2.5, -1.0, 0.25, n, &u) == BANDSOLVE_OK);
  bandsolve_batch* rhs = batch_of(n, 3, cos, 0.3);
  bandsolve_batch* xs = copy_of(rhs);
  bandsolve_batch* xu = copy_of(rhs);
  CHECK(solved(bandsolve_pent_solve_shared(f, xs)));
  CHECK(solved(bandsolve_pent_solve_uniform(u, xu)));
  if (g_gpu) {
    /* uniform is bitwise the shared solve (test_pent_solver.cpp:165-177) */
    CHECK(memcmp(bandsolve_batch_data(xs), bandsolve_batch_data(xu), 3 * n * sizeof(double)) == 0);
    double r = -1.0;
    CHECK(bandsolve_pent_residual(a, b, c, d, e, n, 0, xs, rhs, &r) == BANDSOLVE_OK && r <= 1e-12);
  }
  bandsolve_batch_destroy(xu);
  bandsolve_batch_destroy(xs);
  bandsolve_batch_destroy(rhs);
  bandsolve_pent_factor_destroy(f);
  bandsolve_uniform_pent_factor_destroy(u);
  bandsolve_pent_factor* g = NULL;
  CHECK(bandsolve_pent_factor_create(a, b, c, d, e, 4, &g) == BANDSOLVE_ERR_BAD_ARG && g == NULL);  /* n >= 5 */
}

static void periodic(void) {
  enum { n = 16 };
  bandsolve_periodic_tri* t = NULL;
  CHECK(bandsolve_periodic_tri_create(-0.5, 2.0, -0.5, n, &t) == BANDSOLVE_OK);
  bandsolve_batch* x = batch_of(n, 2, sin, 1.1);
  bandsolve_batch* rhs = copy_of(x);
  CHECK(solved(bandsolve_periodic_tri_solve(t, x)));
  double sub[n], diag[n], sup[n];
  for (int i = 0; i < n; ++i) sub[i] = sup[i] = -0.5, diag[i] = 2.0;
  sub[0] = sup[n - 1] = 0.0;
  if (g_gpu) {
    double r = -1.0;
    CHECK(bandsolve_tri_residual(sub, diag, sup, n, 1, x, rhs, &r) == BANDSOLVE_OK && r <= 1e-10);
  }
  double ms[n], md[n], mu[n];
  CHECK(bandsolve_periodic_tri_modified_bands(t, ms, md, mu) == BANDSOLVE_OK);
  CHECK(fabs(md[0] - 4.0) <= 1e-12 && fabs(md[n - 1] - (2.0 + 0.25 / 2.0)) <= 1e-12 && ms[1] == -0.5);
  bandsolve_periodic_tri_destroy(t);
  bandsolve_batch_destroy(rhs);
  bandsolve_batch_destroy(x);

  t = NULL;
  CHECK(bandsolve_periodic_tri_create(1.0, 0.0, 1.0, 8, &t) == BANDSOLVE_ERR_DIVISION_BY_ZERO && t == NULL);
  CHECK(bandsolve_periodic_tri_create(-1.0, 1.0, 0.0, 3, &t) == BANDSOLVE_ERR_SINGULAR_CORRECTION);

  bandsolve_periodic_pent* p = NULL;
  CHECK(bandsolve_periodic_pent_create(0.25, -1.0, 2.5, -1.0, 0.25, n, &p) == BANDSOLVE_OK);
  bandsolve_batch* px = batch_of(n, 2, cos, 0.9);
  bandsolve_batch* prhs = copy_of(px);
  CHECK(solved(bandsolve_periodic_pent_solve(p, px)));
  if (g_gpu) {
    double a[n], b[n], c[n], d[n], e[n], r = -1.0;
    for (int i = 0; i < n; ++i) a[i] = e[i] = 0.25, b[i] = d[i] = -1.0, c[i] = 2.5;
    a[0] = a[1] = b[0] = 0.0;
    d[n - 1] = e[n - 1] = e[n - 2] = 0.0;
    CHECK(bandsolve_pent_residual(a, b, c, d, e, n, 1, px, prhs, &r) == BANDSOLVE_OK && r <= 1e-10);
  }
  bandsolve_periodic_pent_destroy(p);
  bandsolve_batch_destroy(prhs);
  bandsolve_batch_destroy(px);
}

int main(int argc, char** argv) {
  if (argc != 2 || (strcmp(argv[1], "gpu") != 0 && strcmp(argv[1], "nogpu") != 0)) {
    fprintf(stderr, "usage: %s gpu|nogpu\n", argv[0]);
    return 2;
  }
  g_gpu = strcmp(argv[1], "gpu") == 0;
  statuses_and_threads();
  batches();
  tridiagonal();
  pentadiagonal();
  periodic();
  printf("%d checks, %d failed\n", g_checks, g_failed);
  return g_failed == 0 ? 0 : 1;
}
