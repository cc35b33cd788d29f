// Host-side LHS validation and one-time prefactorisation.
//
// This is the "factorise once on the host" half of the hot path
// (SURVEY.md §8a rows a1/a2/a4/a5/a7). It must reproduce the reference's
// factor arrays bit for bit, so it follows the reference's evaluation order
// exactly and this translation unit is compiled with -ffp-contract=off and
// without -march (no FMA contraction): every expression below is one
// IEEE-754 binary64 rounding per operator, left to right.
#include <cmath>
#include <cstring>

#include "internal.hpp"

namespace bsb {

namespace {

bool all_finite(const double* v, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

// banded.cpp:32-36: the negated comparison also rejects NaN pivots.
bool pivot_ok(double denom) { return std::abs(denom) >= kBreakdownEps; }

}  // namespace

bandsolve_status validate_tri_bands(const double* sub, const double* diag,
                                    const double* sup, std::size_t n) {
  // tri_lhs::tri_lhs, banded.cpp:40-57
  if (n < 2) return fail(BANDSOLVE_ERR_BAD_ARG, "tridiagonal system needs n >= 2");
  if (!all_finite(sub, n) || !all_finite(diag, n) || !all_finite(sup, n))
    return fail(BANDSOLVE_ERR_BAD_ARG, "non-finite entry in a tridiagonal band");
  if (sub[0] != 0.0 || sup[n - 1] != 0.0)
    return fail(BANDSOLVE_ERR_BAD_ARG, "structural band slot must be zero: sub[0] / sup[n-1]");
  return BANDSOLVE_OK;
}

bandsolve_status validate_pent_bands(const double* a, const double* b,
                                     const double* c, const double* d,
                                     const double* e, std::size_t n) {
  // pent_lhs::pent_lhs, banded.cpp:88-116
  if (n < 5) return fail(BANDSOLVE_ERR_BAD_ARG, "pentadiagonal system needs n >= 5");
  if (!all_finite(a, n) || !all_finite(b, n) || !all_finite(c, n) ||
      !all_finite(d, n) || !all_finite(e, n))
    return fail(BANDSOLVE_ERR_BAD_ARG, "non-finite entry in a pentadiagonal band");
  if (a[0] != 0.0 || a[1] != 0.0 || b[0] != 0.0 || d[n - 1] != 0.0 ||
      e[n - 1] != 0.0 || e[n - 2] != 0.0)
    return fail(BANDSOLVE_ERR_BAD_ARG,
                "structural band slot must be zero: a[0], a[1], b[0], d[n-1], e[n-1], e[n-2]");
  return BANDSOLVE_OK;
}

bandsolve_status make_tri_factor(const double* sub, const double* diag,
                                 const double* sup, std::size_t n,
                                 std::unique_ptr<Factor>& out) {
  bandsolve_status st = validate_tri_bands(sub, diag, sup, n);
  if (st != BANDSOLVE_OK) return st;
  auto f = std::make_unique<Factor>();
  f->kind = Kind::Tri;
  f->n = n;
  f->chat.assign(n, 0.0);
  f->inv_denom.assign(n, 0.0);
  f->sub.assign(sub, sub + n);  // banded.cpp:73: the factor keeps a copy of a_i
  f->bands.reserve(3 * n);
  for (const double* v : {sub, diag, sup}) f->bands.insert(f->bands.end(), v, v + n);

  // banded.cpp:75-84. chat is sup / denom (a division, not sup * inv), and
  // the last chat slot stays zero.
  double denom = diag[0];
  if (!pivot_ok(denom))
    return fail(BANDSOLVE_ERR_FACTORIZATION_BREAKDOWN, "zero pivot at row 0");
  f->inv_denom[0] = 1.0 / denom;
  f->chat[0] = sup[0] / denom;
  for (std::size_t i = 1; i < n; ++i) {
    denom = diag[i] - sub[i] * f->chat[i - 1];
    if (!pivot_ok(denom))
      return fail(BANDSOLVE_ERR_FACTORIZATION_BREAKDOWN,
                  "zero pivot at row " + std::to_string(i));
    f->inv_denom[i] = 1.0 / denom;
    if (i + 1 < n) f->chat[i] = sup[i] / denom;
  }
  out = std::move(f);
  return BANDSOLVE_OK;
}

bandsolve_status make_pent_factor(const double* a, const double* b,
                                  const double* c, const double* d,
                                  const double* e, std::size_t n,
                                  std::unique_ptr<Factor>& out) {
  bandsolve_status st = validate_pent_bands(a, b, c, d, e, n);
  if (st != BANDSOLVE_OK) return st;
  auto f = std::make_unique<Factor>();
  f->kind = Kind::Pent;
  f->n = n;
  f->inv_alpha.assign(n, 0.0);
  f->beta.assign(n, 0.0);
  f->gamma.assign(n, 0.0);
  f->delta.assign(n, 0.0);
  f->epsilon.assign(a, a + n);  // banded.cpp:137: epsilon is a verbatim copy of a
  f->bands.reserve(5 * n);
  for (const double* v : {a, b, c, d, e}) f->bands.insert(f->bands.end(), v, v + n);
  std::vector<double> alpha(n, 0.0);
  auto& be = f->beta;
  auto& ga = f->gamma;
  auto& de = f->delta;

  auto breakdown = [](std::size_t row) {
    return fail(BANDSOLVE_ERR_FACTORIZATION_BREAKDOWN,
                "zero alpha at row " + std::to_string(row));
  };

  // The fourteen steps of PAPER.md:461-482 as banded.cpp:141-172 orders them.
  alpha[0] = c[0];
  if (!pivot_ok(alpha[0])) return breakdown(0);
  ga[0] = d[0] / alpha[0];
  de[0] = e[0] / alpha[0];

  be[1] = b[1];
  alpha[1] = c[1] - be[1] * ga[0];
  if (!pivot_ok(alpha[1])) return breakdown(1);
  ga[1] = (d[1] - be[1] * de[0]) / alpha[1];
  de[1] = e[1] / alpha[1];

  for (std::size_t i = 2; i + 2 < n; ++i) {
    be[i] = b[i] - a[i] * ga[i - 2];
    alpha[i] = c[i] - a[i] * de[i - 2] - be[i] * ga[i - 1];
    if (!pivot_ok(alpha[i])) return breakdown(i);
    ga[i] = (d[i] - be[i] * de[i - 1]) / alpha[i];
    de[i] = e[i] / alpha[i];
  }
  {
    const std::size_t i = n - 2;  // no delta in the second-to-last row
    be[i] = b[i] - a[i] * ga[i - 2];
    alpha[i] = c[i] - a[i] * de[i - 2] - be[i] * ga[i - 1];
    if (!pivot_ok(alpha[i])) return breakdown(i);
    ga[i] = (d[i] - be[i] * de[i - 1]) / alpha[i];
  }
  {
    const std::size_t i = n - 1;  // neither gamma nor delta in the last row
    be[i] = b[i] - a[i] * ga[i - 2];
    alpha[i] = c[i] - a[i] * de[i - 2] - be[i] * ga[i - 1];
    if (!pivot_ok(alpha[i])) return breakdown(i);
  }
  // banded.cpp:174: only the reciprocal of alpha is stored.
  for (std::size_t i = 0; i < n; ++i) f->inv_alpha[i] = 1.0 / alpha[i];
  out = std::move(f);
  return BANDSOLVE_OK;
}

bandsolve_status make_uniform_factor(double a, double b, double c, double d,
                                     double e, std::size_t n,
                                     std::unique_ptr<Factor>& out) {
  // pent_solver.cpp:99-111: expand to constant bands with the structural
  // zeros of constant_pent_lhs (banded.cpp:118-125), factor, keep a scalar.
  if (n < 5) return fail(BANDSOLVE_ERR_BAD_ARG, "pentadiagonal system needs n >= 5");
  std::vector<double> av(n, a), bv(n, b), cv(n, c), dv(n, d), ev(n, e);
  av[0] = av[1] = bv[0] = 0.0;
  dv[n - 1] = ev[n - 1] = ev[n - 2] = 0.0;
  std::unique_ptr<Factor> f;
  bandsolve_status st =
      make_pent_factor(av.data(), bv.data(), cv.data(), dv.data(), ev.data(), n, f);
  if (st != BANDSOLVE_OK) return st;
  f->kind = Kind::Uniform;
  f->eps_scalar = a;
  f->epsilon.clear();  // 4N + 1 stored reals (pent_solver.hpp:29-38)
  out = std::move(f);
  return BANDSOLVE_OK;
}

// ---- periodic wrap correction (reference periodic.cpp) -------------------
namespace {

// One column of the shared sweeps in the reference order
// (tri_solver.cpp:25-47, pent_solver.cpp:19-62); used once per periodic
// preparation for A' z = u, exactly as periodic.cpp:41-44 / :139-142 do.
void tri_sweep_column(const Factor& f, double* x) {
  const std::size_t n = f.n;
  x[0] = x[0] * f.inv_denom[0];
  for (std::size_t i = 1; i < n; ++i) x[i] = (x[i] - f.sub[i] * x[i - 1]) * f.inv_denom[i];
  for (std::size_t i = n - 1; i-- > 0;) x[i] = x[i] - f.chat[i] * x[i + 1];
}

void pent_sweep_column(const Factor& f, double* x) {
  const std::size_t n = f.n;
  const double* ia = f.inv_alpha.data();
  const double* be = f.beta.data();
  const double* ga = f.gamma.data();
  const double* de = f.delta.data();
  const double* ep = f.epsilon.data();
  x[0] = x[0] * ia[0];
  x[1] = (x[1] - be[1] * x[0]) * ia[1];
  for (std::size_t i = 2; i < n; ++i) x[i] = ((x[i] - ep[i] * x[i - 2]) - be[i] * x[i - 1]) * ia[i];
  x[n - 2] = x[n - 2] - ga[n - 2] * x[n - 1];
  for (std::size_t i = n - 2; i-- > 0;) x[i] = x[i] - (ga[i] * x[i + 1] + de[i] * x[i + 2]);
}

}  // namespace

bandsolve_status make_periodic_tri(double a, double b, double c, std::size_t n,
                                   std::unique_ptr<Periodic>& out) {
  // periodic_tri_splitting, periodic.cpp:11-31
  if (n < 3) return fail(BANDSOLVE_ERR_BAD_ARG, "periodic tridiagonal wrap needs n >= 3");
  if (!(std::isfinite(a) && std::isfinite(b) && std::isfinite(c)))
    return fail(BANDSOLVE_ERR_BAD_ARG, "non-finite band value");
  if (b == 0.0) return fail(BANDSOLVE_ERR_DIVISION_BY_ZERO, "zero diagonal in periodic splitting");
  std::vector<double> sub(n, a), diag(n, b), sup(n, c);
  sub[0] = 0.0;
  sup[n - 1] = 0.0;
  diag[0] = 2.0 * b;
  diag[n - 1] = b + a * c / b;
  auto p = std::make_unique<Periodic>();
  p->kind = Kind::Tri;
  p->n = n;
  // periodic_tri_prepare, periodic.cpp:33-55
  bandsolve_status st = make_tri_factor(sub.data(), diag.data(), sup.data(), n, p->factor);
  if (st != BANDSOLVE_OK) return st;
  p->z1.assign(n, 0.0);
  p->z1[0] = -b;  // u = (-b, 0, ..., 0, c)
  p->z1[n - 1] = c;
  tri_sweep_column(*p->factor, p->z1.data());
  p->v_last = -a / b;  // v = (1, 0, ..., 0, -a/b)
  const double vdotz = p->z1[0] + p->v_last * p->z1[n - 1];
  const double denom = 1.0 + vdotz;
  if (!(std::abs(denom) > kBreakdownEps))
    return fail(BANDSOLVE_ERR_SINGULAR_CORRECTION, "cyclic system is singular: 1 + v.z vanishes");
  p->scale = 1.0 / denom;  // periodic.cpp:67 inv_denom_scale
  // fused fast path: y_0 = sum_k r0_k dhat_k with U^T r0 = e_0 (U = I + chat superdiagonal)
  p->fused.assign(2 * n, 0.0);
  double* r0 = p->fused.data();
  r0[0] = 1.0;
  for (std::size_t k = 1; k < n; ++k) r0[k] = -p->factor->chat[k - 1] * r0[k - 1];
  std::memcpy(p->fused.data() + n, p->z1.data(), n * sizeof(double));
  out = std::move(p);
  return BANDSOLVE_OK;
}

bandsolve_status make_periodic_pent(double a, double b, double c, double d,
                                    double e, std::size_t n,
                                    std::unique_ptr<Periodic>& out) {
  // periodic_pent_splitting, periodic.cpp:97-129
  if (n < 6) return fail(BANDSOLVE_ERR_BAD_ARG, "periodic pentadiagonal wrap needs n >= 6");
  if (!(std::isfinite(a) && std::isfinite(b) && std::isfinite(c) && std::isfinite(d) && std::isfinite(e)))
    return fail(BANDSOLVE_ERR_BAD_ARG, "non-finite band value");
  std::vector<double> av(n, a), bv(n, b), cv(n, c), dv(n, d), ev(n, e);
  av[0] = av[1] = bv[0] = 0.0;
  dv[n - 1] = ev[n - 1] = ev[n - 2] = 0.0;
  cv[0] = c + b;
  dv[0] = d + a;
  bv[1] = b + a;
  dv[n - 2] = d + e;
  bv[n - 1] = b + e;
  cv[n - 1] = c + d;
  auto p = std::make_unique<Periodic>();
  p->kind = Kind::Pent;
  p->n = n;
  // periodic_pent_prepare, periodic.cpp:131-170
  bandsolve_status st = make_pent_factor(av.data(), bv.data(), cv.data(), dv.data(), ev.data(), n, p->factor);
  if (st != BANDSOLVE_OK) return st;
  p->z1.assign(n, 0.0);
  p->z2.assign(n, 0.0);
  p->z1[0] = -b;  // u1 = (-b, -a, 0, ..., 0, e, d)
  p->z1[1] = -a;
  p->z1[n - 2] = e;
  p->z1[n - 1] = d;
  p->z2[0] = -a;  // u2 = (-a, 0, ..., 0, e)
  p->z2[n - 1] = e;
  pent_sweep_column(*p->factor, p->z1.data());
  pent_sweep_column(*p->factor, p->z2.data());
  const std::vector<double>& z1 = p->z1;
  const std::vector<double>& z2 = p->z2;
  double cap[2][2];  // I + V^T Z, v1 = e_1 - e_N, v2 = e_2 - e_{N-1}
  cap[0][0] = 1.0 + z1[0] - z1[n - 1];
  cap[0][1] = z2[0] - z2[n - 1];
  cap[1][0] = z1[1] - z1[n - 2];
  cap[1][1] = 1.0 + z2[1] - z2[n - 2];
  const double det = cap[0][0] * cap[1][1] - cap[0][1] * cap[1][0];
  if (!(std::abs(det) > kBreakdownEps))
    return fail(BANDSOLVE_ERR_SINGULAR_CORRECTION, "cyclic system is singular: capacitance");
  const double inv_det = 1.0 / det;
  p->cap_inv[0] = cap[1][1] * inv_det;
  p->cap_inv[1] = -cap[0][1] * inv_det;
  p->cap_inv[2] = -cap[1][0] * inv_det;
  p->cap_inv[3] = cap[0][0] * inv_det;
  // fused fast path: y_0, y_1 = r0.g, r1.g with U^T r = e_0, e_1
  // (U = I + gamma superdiagonal + delta second superdiagonal)
  p->fused.assign(4 * n, 0.0);
  double* r0 = p->fused.data();
  double* r1 = r0 + n;
  const Factor& f = *p->factor;
  r0[0] = 1.0;
  r0[1] = -f.gamma[0] * r0[0];
  r1[0] = 0.0;
  r1[1] = 1.0;
  for (std::size_t k = 2; k < n; ++k) {
    r0[k] = -f.gamma[k - 1] * r0[k - 1] - f.delta[k - 2] * r0[k - 2];
    r1[k] = -f.gamma[k - 1] * r1[k - 1] - f.delta[k - 2] * r1[k - 2];
  }
  std::memcpy(r1 + n, p->z1.data(), n * sizeof(double));
  std::memcpy(r1 + 2 * n, p->z2.data(), n * sizeof(double));
  out = std::move(p);
  return BANDSOLVE_OK;
}

void periodic_tri_modified_bands(const Periodic& p, double* sub, double* diag, double* sup) {
  // capi.cpp:249-262
  const Factor& f = *p.factor;
  const std::size_t n = f.n;
  for (std::size_t i = 0; i < n; ++i) {
    const double denom = 1.0 / f.inv_denom[i];
    if (sub) sub[i] = f.sub[i];
    if (diag) diag[i] = i == 0 ? denom : denom + f.sub[i] * f.chat[i - 1];
    if (sup) sup[i] = i + 1 < n ? f.chat[i] * denom : 0.0;
  }
}

void periodic_pent_modified_bands(const Periodic& p, double* a, double* b, double* c, double* d, double* e) {
  // capi.cpp:414-446: A' = L R reassembled band by band
  const Factor& f = *p.factor;
  const std::size_t n = f.n;
  std::vector<double> alpha(n), gamma(n, 0.0), delta(n, 0.0);
  for (std::size_t i = 0; i < n; ++i) alpha[i] = 1.0 / f.inv_alpha[i];
  for (std::size_t i = 0; i + 1 < n; ++i) gamma[i] = f.gamma[i];
  for (std::size_t i = 0; i + 2 < n; ++i) delta[i] = f.delta[i];
  for (std::size_t i = 0; i < n; ++i) {
    const double eps = f.epsilon[i];
    const double beta = f.beta[i];
    if (a) a[i] = i >= 2 ? eps : 0.0;
    if (b) b[i] = i >= 1 ? beta + (i >= 2 ? eps * gamma[i - 2] : 0.0) : 0.0;
    if (c) {
      double v = alpha[i];
      if (i >= 1) v += beta * gamma[i - 1];
      if (i >= 2) v += eps * delta[i - 2];
      c[i] = v;
    }
    if (d) {
      double v = i + 1 < n ? alpha[i] * gamma[i] : 0.0;
      if (i >= 1 && i + 1 < n) v += beta * delta[i - 1];
      d[i] = v;
    }
    if (e) e[i] = i + 2 < n ? alpha[i] * delta[i] : 0.0;
  }
}

}  // namespace bsb
