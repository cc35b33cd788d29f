/*
 * TEST INFRASTRUCTURE ONLY — see bandsolve_oracle.h. Plain-C restatement of
 * the reference hot path, pinned bit-for-bit against the reference build in
 * oracle/_ref/ by tests/test_oracle.py. Compile with -ffp-contract=off.
 */
#include "bandsolve_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum {
  ST_OK = 0,
  ST_BAD_ARG = 1,
  ST_SHAPE = 2,
  ST_BREAKDOWN = 3,
  ST_DIV_ZERO = 4,
  ST_SINGULAR_CORRECTION = 5,
  ST_SINGULAR_MATRIX = 6,
  ST_INTERNAL = 9
};

/* common.hpp:17 */
static const double k_breakdown_eps = 1e-300;

/* banded.cpp:32-36 — the negated >= also rejects NaN pivots */
static int denom_ok(double denom) { return fabs(denom) >= k_breakdown_eps; }

static int all_finite(const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

int oracle_tri_prefactor(const double* sub, const double* diag,
                         const double* sup, size_t n, double* chat,
                         double* inv_denom, double* sub_out) {
  /* tri_lhs validation, banded.cpp:40-57 */
  if (!sub || !diag || !sup || !chat || !inv_denom || !sub_out) return ST_BAD_ARG;
  if (n < 2) return ST_BAD_ARG;
  if (!all_finite(sub, n) || !all_finite(diag, n) || !all_finite(sup, n))
    return ST_BAD_ARG;
  if (sub[0] != 0.0 || sup[n - 1] != 0.0) return ST_BAD_ARG;

  /* banded.cpp:75-84; chat divides by denom (not sup * inv) */
  memcpy(sub_out, sub, n * sizeof(double));
  double denom = diag[0];
  if (!denom_ok(denom)) return ST_BREAKDOWN;
  inv_denom[0] = 1.0 / denom;
  chat[0] = sup[0] / denom;
  for (size_t i = 1; i < n; ++i) {
    denom = diag[i] - sub[i] * chat[i - 1];
    if (!denom_ok(denom)) return ST_BREAKDOWN;
    inv_denom[i] = 1.0 / denom;
    chat[i] = (i + 1 < n) ? sup[i] / denom : 0.0;
  }
  return ST_OK;
}

void oracle_tri_solve_shared(const double* chat, const double* inv_denom,
                             const double* sub, size_t n, size_t m, size_t ld,
                             double* x) {
  /* forward, tri_solver.cpp:24-38 */
  for (size_t j = 0; j < m; ++j) x[j] *= inv_denom[0];
  for (size_t i = 1; i < n; ++i) {
    const double ai = sub[i], mi = inv_denom[i];
    double* row = x + i * ld;
    const double* prev = row - ld;
    for (size_t j = 0; j < m; ++j) row[j] = (row[j] - ai * prev[j]) * mi;
  }
  /* backward, tri_solver.cpp:39-47 */
  for (size_t i = n - 1; i-- > 0;) {
    const double ci = chat[i];
    double* row = x + i * ld;
    const double* next = row + ld;
    for (size_t j = 0; j < m; ++j) row[j] -= ci * next[j];
  }
}

int oracle_pent_prefactor(const double* a, const double* b, const double* c,
                          const double* d, const double* e, size_t n,
                          double* inv_alpha, double* beta, double* gamma,
                          double* delta, double* epsilon) {
  /* pent_lhs validation, banded.cpp:88-116 */
  if (!a || !b || !c || !d || !e || !inv_alpha || !beta || !gamma || !delta ||
      !epsilon)
    return ST_BAD_ARG;
  if (n < 5) return ST_BAD_ARG;
  if (!all_finite(a, n) || !all_finite(b, n) || !all_finite(c, n) ||
      !all_finite(d, n) || !all_finite(e, n))
    return ST_BAD_ARG;
  if (a[0] != 0.0 || a[1] != 0.0 || b[0] != 0.0 || d[n - 1] != 0.0 ||
      e[n - 1] != 0.0 || e[n - 2] != 0.0)
    return ST_BAD_ARG;

  double* alpha = (double*)malloc(n * sizeof(double));
  if (!alpha) return ST_INTERNAL;
  int st = ST_OK;
  memset(beta, 0, n * sizeof(double));
  memset(gamma, 0, n * sizeof(double));
  memset(delta, 0, n * sizeof(double));
  memcpy(epsilon, a, n * sizeof(double));

  /* banded.cpp:141-150 */
  alpha[0] = c[0];
  if (!denom_ok(alpha[0])) { st = ST_BREAKDOWN; goto done; }
  gamma[0] = d[0] / alpha[0];
  delta[0] = e[0] / alpha[0];
  beta[1] = b[1];
  alpha[1] = c[1] - beta[1] * gamma[0];
  if (!denom_ok(alpha[1])) { st = ST_BREAKDOWN; goto done; }
  gamma[1] = (d[1] - beta[1] * delta[0]) / alpha[1];
  delta[1] = e[1] / alpha[1];
  /* banded.cpp:152-158; alpha is (c - a*delta) - beta*gamma, left to right */
  for (size_t i = 2; i + 2 < n; ++i) {
    beta[i] = b[i] - a[i] * gamma[i - 2];
    alpha[i] = c[i] - a[i] * delta[i - 2] - beta[i] * gamma[i - 1];
    if (!denom_ok(alpha[i])) { st = ST_BREAKDOWN; goto done; }
    gamma[i] = (d[i] - beta[i] * delta[i - 1]) / alpha[i];
    delta[i] = e[i] / alpha[i];
  }
  /* banded.cpp:160-172 */
  {
    const size_t i = n - 2;
    beta[i] = b[i] - a[i] * gamma[i - 2];
    alpha[i] = c[i] - a[i] * delta[i - 2] - beta[i] * gamma[i - 1];
    if (!denom_ok(alpha[i])) { st = ST_BREAKDOWN; goto done; }
    gamma[i] = (d[i] - beta[i] * delta[i - 1]) / alpha[i];
  }
  {
    const size_t i = n - 1;
    beta[i] = b[i] - a[i] * gamma[i - 2];
    alpha[i] = c[i] - a[i] * delta[i - 2] - beta[i] * gamma[i - 1];
    if (!denom_ok(alpha[i])) { st = ST_BREAKDOWN; goto done; }
  }
  /* banded.cpp:174 */
  for (size_t i = 0; i < n; ++i) inv_alpha[i] = 1.0 / alpha[i];
done:
  free(alpha);
  return st;
}

void oracle_pent_solve(const double* inv_alpha, const double* beta,
                       const double* gamma, const double* delta,
                       const double* eps, double eps_scalar, size_t n,
                       size_t m, size_t ld, double* x) {
  /* g over f, pent_solver.cpp:19-43 */
  for (size_t j = 0; j < m; ++j) x[j] *= inv_alpha[0];
  {
    const double b1 = beta[1], ia1 = inv_alpha[1];
    double* row = x + ld;
    for (size_t j = 0; j < m; ++j) row[j] = (row[j] - b1 * x[j]) * ia1;
  }
  for (size_t i = 2; i < n; ++i) {
    const double ei = eps ? eps[i] : eps_scalar;
    const double bi = beta[i], iai = inv_alpha[i];
    double* row = x + i * ld;
    const double* p1 = row - ld;
    const double* p2 = row - 2 * ld;
    for (size_t j = 0; j < m; ++j)
      row[j] = (row[j] - ei * p2[j] - bi * p1[j]) * iai;
  }
  /* x over g, pent_solver.cpp:44-62 */
  {
    const double gn2 = gamma[n - 2];
    double* row = x + (n - 2) * ld;
    const double* next = row + ld;
    for (size_t j = 0; j < m; ++j) row[j] -= gn2 * next[j];
  }
  for (size_t i = n - 2; i-- > 0;) {
    const double gi = gamma[i], di = delta[i];
    double* row = x + i * ld;
    const double* n1 = row + ld;
    const double* n2 = row + 2 * ld;
    for (size_t j = 0; j < m; ++j) row[j] -= gi * n1[j] + di * n2[j];
  }
}

int oracle_uniform_pent_prefactor(double a, double b, double c, double d,
                                  double e, size_t n, double* inv_alpha,
                                  double* beta, double* gamma, double* delta,
                                  double* eps_scalar) {
  if (n < 5) return ST_BAD_ARG; /* banded.cpp:120 */
  double* bands = (double*)malloc(6 * n * sizeof(double));
  if (!bands) return ST_INTERNAL;
  double *av = bands, *bv = bands + n, *cv = bands + 2 * n, *dv = bands + 3 * n,
         *ev = bands + 4 * n, *eps = bands + 5 * n;
  for (size_t i = 0; i < n; ++i) {
    av[i] = a; bv[i] = b; cv[i] = c; dv[i] = d; ev[i] = e;
  }
  av[0] = av[1] = bv[0] = 0.0; /* banded.cpp:122-123 */
  dv[n - 1] = ev[n - 1] = ev[n - 2] = 0.0;
  int st = oracle_pent_prefactor(av, bv, cv, dv, ev, n, inv_alpha, beta, gamma,
                                 delta, eps);
  if (st == ST_OK && eps_scalar) *eps_scalar = a; /* pent_solver.cpp:109 */
  free(bands);
  return st;
}

static double residual_pass_tri(size_t n, size_t m, const double* x,
                                const double* rhs, const double* sub,
                                const double* diag, const double* sup,
                                double corner_tr, double corner_bl) {
  /* tri_solver.cpp:116-136 */
  double worst = 0.0;
  for (size_t j = 0; j < m; ++j) {
    double rmax = 0.0, dmax = 0.0;
    for (size_t i = 0; i < n; ++i) {
      double acc = diag[i] * x[i * m + j];
      if (i > 0) acc += sub[i] * x[(i - 1) * m + j];
      if (i + 1 < n) acc += sup[i] * x[(i + 1) * m + j];
      if (i == 0) acc += corner_tr * x[(n - 1) * m + j];
      if (i == n - 1) acc += corner_bl * x[j];
      double r = fabs(acc - rhs[i * m + j]);
      if (r > rmax) rmax = r;
      double dv = fabs(rhs[i * m + j]);
      if (dv > dmax) dmax = dv;
    }
    double w = dmax > 0.0 ? rmax / dmax : rmax;
    if (w > worst) worst = w;
  }
  return worst;
}

int oracle_tri_residual(const double* sub, const double* diag,
                        const double* sup, size_t n, int cyclic, size_t m,
                        const double* x, const double* rhs, double* out) {
  if (!sub || !diag || !sup || !x || !rhs || !out) return ST_BAD_ARG;
  if (cyclic) {
    /* capi.cpp:336-339, tri_solver.cpp:149-156 */
    if (n < 3) return ST_BAD_ARG;
    const double a = sub[1], b = diag[0], c = sup[0];
    double* bands = (double*)malloc(3 * n * sizeof(double));
    if (!bands) return ST_INTERNAL;
    double *sv = bands, *dv = bands + n, *uv = bands + 2 * n;
    for (size_t i = 0; i < n; ++i) { sv[i] = a; dv[i] = b; uv[i] = c; }
    sv[0] = 0.0;
    uv[n - 1] = 0.0;
    if (!all_finite(bands, 3 * n)) { free(bands); return ST_BAD_ARG; }
    *out = residual_pass_tri(n, m, x, rhs, sv, dv, uv, a, c);
    free(bands);
    return ST_OK;
  }
  if (n < 2 || !all_finite(sub, n) || !all_finite(diag, n) ||
      !all_finite(sup, n) || sub[0] != 0.0 || sup[n - 1] != 0.0)
    return ST_BAD_ARG;
  *out = residual_pass_tri(n, m, x, rhs, sub, diag, sup, 0.0, 0.0);
  return ST_OK;
}

static double residual_pass_pent(size_t n, size_t m, const double* x,
                                 const double* rhs, const double* a,
                                 const double* b, const double* c,
                                 const double* d, const double* e, int cyclic,
                                 double ca, double cb, double cd, double ce) {
  /* pent_solver.cpp:223-251 */
  double worst = 0.0;
  for (size_t j = 0; j < m; ++j) {
    double rmax = 0.0, dmax = 0.0;
#define X(r) x[(r) * m + j]
    for (size_t i = 0; i < n; ++i) {
      double acc = c[i] * X(i);
      if (i >= 2) acc += a[i] * X(i - 2);
      if (i >= 1) acc += b[i] * X(i - 1);
      if (i + 1 < n) acc += d[i] * X(i + 1);
      if (i + 2 < n) acc += e[i] * X(i + 2);
      if (cyclic) {
        if (i == 0) acc += ca * X(n - 2) + cb * X(n - 1);
        if (i == 1) acc += ca * X(n - 1);
        if (i == n - 2) acc += ce * X(0);
        if (i == n - 1) acc += cd * X(0) + ce * X(1);
      }
      double r = fabs(acc - rhs[i * m + j]);
      if (r > rmax) rmax = r;
      double dv = fabs(rhs[i * m + j]);
      if (dv > dmax) dmax = dv;
    }
#undef X
    double w = dmax > 0.0 ? rmax / dmax : rmax;
    if (w > worst) worst = w;
  }
  return worst;
}

int oracle_pent_residual(const double* a, const double* b, const double* c,
                         const double* d, const double* e, size_t n,
                         int cyclic, size_t m, const double* x,
                         const double* rhs, double* out) {
  if (!a || !b || !c || !d || !e || !x || !rhs || !out) return ST_BAD_ARG;
  if (cyclic) {
    /* capi.cpp:357-360, pent_solver.cpp:265-273 */
    if (n < 6) return ST_BAD_ARG;
    const double ca = a[2], cb = b[1], cc = c[0], cd = d[0], ce = e[0];
    double* bands = (double*)malloc(5 * n * sizeof(double));
    if (!bands) return ST_INTERNAL;
    double *av = bands, *bv = bands + n, *cv = bands + 2 * n, *dv = bands + 3 * n,
           *ev = bands + 4 * n;
    for (size_t i = 0; i < n; ++i) {
      av[i] = ca; bv[i] = cb; cv[i] = cc; dv[i] = cd; ev[i] = ce;
    }
    av[0] = av[1] = bv[0] = 0.0;
    dv[n - 1] = ev[n - 1] = ev[n - 2] = 0.0;
    if (!all_finite(bands, 5 * n)) { free(bands); return ST_BAD_ARG; }
    *out = residual_pass_pent(n, m, x, rhs, av, bv, cv, dv, ev, 1, ca, cb, cd,
                              ce);
    free(bands);
    return ST_OK;
  }
  if (n < 5 || !all_finite(a, n) || !all_finite(b, n) || !all_finite(c, n) ||
      !all_finite(d, n) || !all_finite(e, n) || a[0] != 0.0 || a[1] != 0.0 ||
      b[0] != 0.0 || d[n - 1] != 0.0 || e[n - 1] != 0.0 || e[n - 2] != 0.0)
    return ST_BAD_ARG;
  *out = residual_pass_pent(n, m, x, rhs, a, b, c, d, e, 0, 0, 0, 0, 0);
  return ST_OK;
}

int oracle_max_error_vs_dense(const double* a, size_t n, size_t m,
                              const double* x, const double* rhs,
                              double* out) {
  /* dense.cpp:15-48 (partial-pivot LU with row permutation), :50-71
   * (solve_in_place), oracles.cpp:104-122 (metric). */
  if (!a || !x || !rhs || !out || n == 0) return ST_BAD_ARG;
  double* lu = (double*)malloc(n * n * sizeof(double));
  size_t* perm = (size_t*)malloc(n * sizeof(size_t));
  double* col = (double*)malloc(n * sizeof(double));
  double* y = (double*)malloc(n * sizeof(double));
  int st = ST_OK;
  if (!lu || !perm || !col || !y) { st = ST_INTERNAL; goto done; }
  memcpy(lu, a, n * n * sizeof(double));
  for (size_t i = 0; i < n; ++i) perm[i] = i;
  for (size_t k = 0; k < n; ++k) {
    size_t piv = k;
    double best = fabs(lu[perm[k] * n + k]);
    for (size_t i = k + 1; i < n; ++i) {
      double mag = fabs(lu[perm[i] * n + k]);
      if (mag > best) { best = mag; piv = i; }
    }
    if (!(best > 1e-14)) { st = ST_SINGULAR_MATRIX; goto done; }
    size_t t = perm[k]; perm[k] = perm[piv]; perm[piv] = t;
    const double* prow = lu + perm[k] * n;
    const double inv_piv = 1.0 / prow[k];
    for (size_t i = k + 1; i < n; ++i) {
      double* row = lu + perm[i] * n;
      const double l = row[k] * inv_piv;
      row[k] = l;
      if (l != 0.0)
        for (size_t jj = k + 1; jj < n; ++jj) row[jj] -= l * prow[jj];
    }
  }
  double worst = 0.0;
  for (size_t j = 0; j < m; ++j) {
    for (size_t i = 0; i < n; ++i) col[i] = rhs[i * m + j];
    for (size_t i = 0; i < n; ++i) {
      double s = col[perm[i]];
      const double* row = lu + perm[i] * n;
      for (size_t q = 0; q < i; ++q) s -= row[q] * y[q];
      y[i] = s;
    }
    for (size_t ii = n; ii-- > 0;) {
      double s = y[ii];
      const double* row = lu + perm[ii] * n;
      for (size_t q = ii + 1; q < n; ++q) s -= row[q] * y[q];
      y[ii] = s / row[ii];
    }
    double err = 0.0, scale = 0.0;
    for (size_t i = 0; i < n; ++i) {
      double e = fabs(x[i * m + j] - y[i]);
      if (e > err) err = e;
      double s = fabs(y[i]);
      if (s > scale) scale = s;
    }
    double w = scale > 0.0 ? err / scale : err;
    if (w > worst) worst = w;
  }
  *out = worst;
done:
  free(lu); free(perm); free(col); free(y);
  return st;
}

static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double oracle_rhs_value(uint64_t seed, uint64_t i, uint64_t j) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ i);
  h = splitmix64(h ^ j);
  /* (k - 2^52) / 2^52 with k < 2^53: exact in binary64, range [-1, 1) */
  return (double)(h >> 11) * 0x1.0p-52 - 1.0;
}

void oracle_fill_rhs(uint64_t seed, size_t n, size_t m, size_t j_offset,
                     size_t m_total, double* x) {
  (void)m_total;
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < m; ++j)
      x[i * m + j] = oracle_rhs_value(seed, i, j_offset + j);
}

/* ---- periodic wrap correction (reference periodic.cpp) ------------------ */

int oracle_periodic_tri_prepare(double a, double b, double c, size_t n,
                                double* chat, double* inv_denom,
                                double* sub, double* z, double* v_last,
                                double* scale) {
  /* periodic_tri_splitting, periodic.cpp:11-31 */
  if (n < 3) return ST_BAD_ARG;
  if (!(isfinite(a) && isfinite(b) && isfinite(c))) return ST_BAD_ARG;
  if (b == 0.0) return ST_DIV_ZERO;
  double* sb = malloc(3 * n * sizeof(double));
  if (!sb) return ST_INTERNAL;
  double *s_sub = sb, *s_diag = sb + n, *s_sup = sb + 2 * n;
  for (size_t i = 0; i < n; ++i) {
    s_sub[i] = a;
    s_diag[i] = b;
    s_sup[i] = c;
  }
  s_sub[0] = 0.0;
  s_sup[n - 1] = 0.0;
  s_diag[0] = 2.0 * b;
  s_diag[n - 1] = b + a * c / b;
  /* u = (-b, 0, ..., 0, c); v = (1, 0, ..., 0, -a/b) */
  const double vl = -a / b;
  /* periodic_tri_prepare, periodic.cpp:33-55 */
  int st = oracle_tri_prefactor(s_sub, s_diag, s_sup, n, chat, inv_denom, sub);
  free(sb);
  if (st) return st;
  for (size_t i = 0; i < n; ++i) z[i] = 0.0;
  z[0] = -b;
  z[n - 1] = c;
  oracle_tri_solve_shared(chat, inv_denom, sub, n, 1, 1, z);
  const double vdotz = z[0] + vl * z[n - 1];
  const double denom = 1.0 + vdotz;
  if (!(fabs(denom) > 1e-300)) return ST_SINGULAR_CORRECTION;
  *v_last = vl;
  *scale = 1.0 / denom; /* periodic.cpp:67 inv_denom_scale */
  return ST_OK;
}

void oracle_periodic_tri_apply(const double* z, double v_last, double scale,
                               size_t n, size_t m, double* x) {
  /* periodic.cpp:57-89: w = (y_0 + v_last y_{n-1}) * scale; y_i -= w z_i */
  for (size_t j = 0; j < m; ++j) {
    const double w = (x[j] + v_last * x[(n - 1) * m + j]) * scale;
    for (size_t i = 0; i < n; ++i) x[i * m + j] -= w * z[i];
  }
}

int oracle_periodic_pent_prepare(double a, double b, double c, double d,
                                 double e, size_t n, double* inv_alpha,
                                 double* beta, double* gamma, double* delta,
                                 double* epsilon, double* z1, double* z2,
                                 double* cap_inv) {
  /* periodic_pent_splitting, periodic.cpp:97-129 */
  if (n < 6) return ST_BAD_ARG;
  if (!(isfinite(a) && isfinite(b) && isfinite(c) && isfinite(d) && isfinite(e))) return ST_BAD_ARG;
  double* bb = malloc(5 * n * sizeof(double));
  if (!bb) return ST_INTERNAL;
  double *av = bb, *bv = bb + n, *cv = bb + 2 * n, *dv = bb + 3 * n, *ev = bb + 4 * n;
  for (size_t i = 0; i < n; ++i) {
    av[i] = a;
    bv[i] = b;
    cv[i] = c;
    dv[i] = d;
    ev[i] = e;
  }
  av[0] = av[1] = bv[0] = 0.0;
  dv[n - 1] = ev[n - 1] = ev[n - 2] = 0.0;
  cv[0] = c + b;
  dv[0] = d + a;
  bv[1] = b + a;
  dv[n - 2] = d + e;
  bv[n - 1] = b + e;
  cv[n - 1] = c + d;
  /* periodic_pent_prepare, periodic.cpp:131-170 */
  int st = oracle_pent_prefactor(av, bv, cv, dv, ev, n, inv_alpha, beta, gamma, delta, epsilon);
  free(bb);
  if (st) return st;
  /* u1 = (-b, -a, 0, ..., 0, e, d), u2 = (-a, 0, ..., 0, e); solved as the two
   * columns of one interleaved batch (identical per-column arithmetic) */
  for (size_t i = 0; i < n; ++i) z1[i] = z2[i] = 0.0;
  z1[0] = -b;
  z1[1] = -a;
  z1[n - 2] = e;
  z1[n - 1] = d;
  z2[0] = -a;
  z2[n - 1] = e;
  oracle_pent_solve(inv_alpha, beta, gamma, delta, epsilon, 0.0, n, 1, 1, z1);
  oracle_pent_solve(inv_alpha, beta, gamma, delta, epsilon, 0.0, n, 1, 1, z2);
  double cap[2][2];
  cap[0][0] = 1.0 + z1[0] - z1[n - 1];
  cap[0][1] = z2[0] - z2[n - 1];
  cap[1][0] = z1[1] - z1[n - 2];
  cap[1][1] = 1.0 + z2[1] - z2[n - 2];
  const double det = cap[0][0] * cap[1][1] - cap[0][1] * cap[1][0];
  if (!(fabs(det) > 1e-300)) return ST_SINGULAR_CORRECTION;
  const double inv_det = 1.0 / det;
  cap_inv[0] = cap[1][1] * inv_det;
  cap_inv[1] = -cap[0][1] * inv_det;
  cap_inv[2] = -cap[1][0] * inv_det;
  cap_inv[3] = cap[0][0] * inv_det;
  return ST_OK;
}

void oracle_periodic_pent_apply(const double* z1, const double* z2,
                                const double* cap_inv, size_t n, size_t m,
                                double* x) {
  /* periodic.cpp:172-208 */
  for (size_t j = 0; j < m; ++j) {
    const double w1 = x[j] - x[(n - 1) * m + j];
    const double w2 = x[m + j] - x[(n - 2) * m + j];
    const double t1 = cap_inv[0] * w1 + cap_inv[1] * w2;
    const double t2 = cap_inv[2] * w1 + cap_inv[3] * w2;
    for (size_t i = 0; i < n; ++i) x[i * m + j] -= z1[i] * t1 + z2[i] * t2;
  }
}

/* ---- Crank-Nicolson pieces (reference pde.cpp) ------------------------------ */

void oracle_default_mode_initial(size_t n, size_t m, double* out) {
  /* pde.cpp:48-58 */
  const size_t mode_span = n / 4 > 0 ? n / 4 : 1;
  const double pi = 3.141592653589793238462643383279502884; /* std::numbers::pi */
  for (size_t j = 0; j < m; ++j) {
    const double k = (double)(1 + (j % mode_span));
    for (size_t i = 0; i < n; ++i) {
      const double x = (double)(i + 1) / (double)n;
      out[i * m + j] = sin(2.0 * pi * k * x);
    }
  }
}

void oracle_cn_rhs(int problem, double sigma_x, size_t n, size_t m,
                   const double* u, double* out) {
  if (problem == 0) { /* diffusion_rhs_into, pde.cpp:73-91 */
    const double s = sigma_x;
    const double mid = 1.0 - 2.0 * sigma_x;
    for (size_t i = 0; i < n; ++i) {
      const double* up = u + (i == 0 ? n - 1 : i - 1) * m;
      const double* mi = u + i * m;
      const double* dn = u + (i + 1 == n ? 0 : i + 1) * m;
      for (size_t j = 0; j < m; ++j) out[i * m + j] = s * (up[j] + dn[j]) + mid * mi[j];
    }
  } else { /* hyper_rhs_into, pde.cpp:93-114 */
    const double s = sigma_x;
    const double s4 = 4.0 * sigma_x;
    const double mid = 1.0 - 6.0 * sigma_x;
    for (size_t i = 0; i < n; ++i) {
      const double* u2 = u + ((i + n - 2) % n) * m;
      const double* u1 = u + (i == 0 ? n - 1 : i - 1) * m;
      const double* mi = u + i * m;
      const double* d1 = u + (i + 1 == n ? 0 : i + 1) * m;
      const double* d2 = u + ((i + 2) % n) * m;
      for (size_t j = 0; j < m; ++j)
        out[i * m + j] = -s * (u2[j] + d2[j]) + s4 * (u1[j] + d1[j]) + mid * mi[j];
    }
  }
}

/* ---- per-system baselines ------------------------------------------------ */
/* tri_solver.cpp:51-112: reciprocals over b, chat over c, dhat over d, then
 * the backward sweep in place over d. */
int oracle_tri_per_system(const double* a, double* b, double* c, double* d, size_t n, size_t m) {
  if (n < 2) return ST_BAD_ARG;
  int broke = 0;
  for (size_t j = 0; j < m; ++j) {
    double denom = b[j];
    if (!denom_ok(denom)) { broke = 1; continue; }
    double r = 1.0 / denom;
    b[j] = r;
    double cg = c[j] * r;
    c[j] = cg;
    double dg = d[j] * r;
    d[j] = dg;
    int ok = 1;
    for (size_t i = 1; i < n; ++i) {
      const size_t k = i * m + j;
      denom = b[k] - a[k] * cg;
      if (!denom_ok(denom)) { broke = 1; ok = 0; break; }
      r = 1.0 / denom;
      b[k] = r;
      cg = c[k] * r;
      c[k] = cg;
      dg = (d[k] - a[k] * dg) * r;
      d[k] = dg;
    }
    if (!ok) continue;
    double xnext = d[(n - 1) * m + j];
    for (size_t i = n - 1; i-- > 0;) {
      const size_t k = i * m + j;
      const double xi = d[k] - c[k] * xnext;
      d[k] = xi;
      xnext = xi;
    }
  }
  return broke ? ST_BREAKDOWN : ST_OK;
}

/* pent_solver.cpp:131-219: beta over b, alpha over c, gamma over d, delta
 * over e (a doubles as epsilon), g then x over f. */
int oracle_pent_per_system(const double* a, double* b, double* c, double* d, double* e, double* f,
                           size_t n, size_t m) {
  if (n < 5) return ST_BAD_ARG;
  int broke = 0;
#define AT(i) ((size_t)(i) * m + j)
  for (size_t j = 0; j < m; ++j) {
    double alpha = c[AT(0)];
    if (!denom_ok(alpha)) { broke = 1; continue; }
    d[AT(0)] /= alpha;
    e[AT(0)] /= alpha;
    alpha = c[AT(1)] - b[AT(1)] * d[AT(0)];
    if (!denom_ok(alpha)) { broke = 1; continue; }
    c[AT(1)] = alpha;
    d[AT(1)] = (d[AT(1)] - b[AT(1)] * e[AT(0)]) / alpha;
    e[AT(1)] /= alpha;
    int ok = 1;
    for (size_t i = 2; i < n; ++i) {
      const double beta = b[AT(i)] - a[AT(i)] * d[AT(i - 2)];
      b[AT(i)] = beta;
      alpha = c[AT(i)] - a[AT(i)] * e[AT(i - 2)] - beta * d[AT(i - 1)];
      if (!denom_ok(alpha)) { ok = 0; break; }
      c[AT(i)] = alpha;
      if (i + 1 < n) d[AT(i)] = (d[AT(i)] - beta * e[AT(i - 1)]) / alpha;
      if (i + 2 < n) e[AT(i)] /= alpha;
    }
    if (!ok) { broke = 1; continue; }
    f[AT(0)] /= c[AT(0)];
    f[AT(1)] = (f[AT(1)] - b[AT(1)] * f[AT(0)]) / c[AT(1)];
    for (size_t i = 2; i < n; ++i)
      f[AT(i)] = (f[AT(i)] - a[AT(i)] * f[AT(i - 2)] - b[AT(i)] * f[AT(i - 1)]) / c[AT(i)];
    f[AT(n - 2)] -= d[AT(n - 2)] * f[AT(n - 1)];
    for (size_t i = n - 2; i-- > 0;) f[AT(i)] -= d[AT(i)] * f[AT(i + 1)] + e[AT(i)] * f[AT(i + 2)];
  }
#undef AT
  return broke ? ST_BREAKDOWN : ST_OK;
}
