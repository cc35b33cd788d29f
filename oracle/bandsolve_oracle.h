/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the shared-LHS batch solvers.
 *
 * A plain-C restatement of the reference `bandsolve` hot path
 * (/root/reference/proj). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this; the product library
 * (paper_1909_04539_b200/) never links or calls it.
 *
 * Parity pin: every function is checked bit-for-bit against the reference
 * itself (oracle/_ref/libbandsolve_ref.so, compiled from the reference's own
 * sources by oracle/Makefile) on the golden fixtures in tests/golden/, and
 * against the reference's hand-written known-answer tables
 * (proj/tests/test_banded_core.cpp:35-55, :111-148).
 *
 * Arithmetic contract: compiled with -ffp-contract=off and no -march, so each
 * C operator is one IEEE-754 binary64 rounding, in the reference's order.
 * Status codes are the reference's bandsolve_status values
 * (proj/include/bandsolve.h:22-33).
 */
#ifndef BANDSOLVE_ORACLE_H
#define BANDSOLVE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Reference banded.cpp:67-86 (tri_prefactor) plus tri_lhs validation
 * banded.cpp:40-57. Outputs: chat[n], inv_denom[n], sub copy in sub_out[n]. */
int oracle_tri_prefactor(const double* sub, const double* diag,
                         const double* sup, size_t n, double* chat,
                         double* inv_denom, double* sub_out);

/* Reference tri_solver.cpp:11-49, one worker: in place over x[i*ld + j],
 * j in [0, m). */
void oracle_tri_solve_shared(const double* chat, const double* inv_denom,
                             const double* sub, size_t n, size_t m, size_t ld,
                             double* x);

/* Reference banded.cpp:127-176 (pent_prefactor) plus pent_lhs validation
 * banded.cpp:88-116. epsilon is a verbatim copy of a. */
int oracle_pent_prefactor(const double* a, const double* b, const double* c,
                          const double* d, const double* e, size_t n,
                          double* inv_alpha, double* beta, double* gamma,
                          double* delta, double* epsilon);

/* Reference pent_solver.cpp:15-63 (pent_sweep) with the vector epsilon of
 * pent_solve_shared_batch (:67-81) when eps != NULL, else the scalar of
 * pent_solve_uniform_batch (:83-97). */
void oracle_pent_solve(const double* inv_alpha, const double* beta,
                       const double* gamma, const double* delta,
                       const double* eps, double eps_scalar, size_t n,
                       size_t m, size_t ld, double* x);

/* Reference pent_solver.cpp:99-111 (uniform_prefactor via constant_pent_lhs
 * banded.cpp:118-125). */
int oracle_uniform_pent_prefactor(double a, double b, double c, double d,
                                  double e, size_t n, double* inv_alpha,
                                  double* beta, double* gamma, double* delta,
                                  double* eps_scalar);

/* Reference tri_solver.cpp:116-156 (residual_pass): max over systems of
 * ||A x - rhs||_inf / ||rhs||_inf; cyclic corners read sub[1], sup[0]. */
int oracle_tri_residual(const double* sub, const double* diag,
                        const double* sup, size_t n, int cyclic, size_t m,
                        const double* x, const double* rhs, double* out);

/* Reference pent_solver.cpp:223-273 (pent_residual_pass). */
int oracle_pent_residual(const double* a, const double* b, const double* c,
                         const double* d, const double* e, size_t n,
                         int cyclic, size_t m, const double* x,
                         const double* rhs, double* out);

/* Dense partial-pivot LU oracle, reference src/dense.cpp:15-76, used by the
 * per-system max-norm metric of tests/support/oracles.cpp:104-122.
 * a is row-major n x n. Returns max_j ||x_j - xref_j|| / ||xref_j||. */
int oracle_max_error_vs_dense(const double* a, size_t n, size_t m,
                              const double* x, const double* rhs,
                              double* out);

/* Periodic (cyclic, constant bands) wrap correction, reference
 * periodic.cpp. tri: splitting :11-31, prepare :33-55 (factor of A' into
 * chat/inv_denom/sub, z = A'^-1 u, v_last = -a/b, scale = 1/(1 + v.z));
 * apply :57-89 (x = y - ((y_0 + v_last y_{n-1}) * scale) z). */
int oracle_periodic_tri_prepare(double a, double b, double c, size_t n,
                                double* chat, double* inv_denom,
                                double* sub, double* z, double* v_last,
                                double* scale);
void oracle_periodic_tri_apply(const double* z, double v_last, double scale,
                               size_t n, size_t m, double* x);
/* pent: splitting :97-129, prepare :131-170 (Woodbury: z1, z2, the 2x2
 * capacitance inverse cap_inv[4] row-major); apply :172-208. */
int oracle_periodic_pent_prepare(double a, double b, double c, double d,
                                 double e, size_t n, double* inv_alpha,
                                 double* beta, double* gamma, double* delta,
                                 double* epsilon, double* z1, double* z2,
                                 double* cap_inv);
void oracle_periodic_pent_apply(const double* z1, const double* z2,
                                const double* cap_inv, size_t n, size_t m,
                                double* x);

/* Crank-Nicolson pieces of reference pde.cpp: default_mode_initial
 * (:48-58) and the periodic explicit stencils diffusion_rhs_into (:73-91,
 * problem 0) / hyper_rhs_into (:93-114, problem 1), out = B u. */
void oracle_default_mode_initial(size_t n, size_t m, double* out);
void oracle_cn_rhs(int problem, double sigma_x, size_t n, size_t m,
                   const double* u, double* out);

/* Counter-based synthetic RHS shared with the device generator:
 * U(-1, 1) from SplitMix64 of (seed, i, j), 53-bit mantissa. */
double oracle_rhs_value(uint64_t seed, uint64_t i, uint64_t j);
void oracle_fill_rhs(uint64_t seed, size_t n, size_t m, size_t j_offset,
                     size_t m_total, double* x);

/* Per-system baselines, reference tri_solver.cpp:51-112 and
 * pent_solver.cpp:131-219: one band copy per system, interleaved (n, m),
 * destroyed in place exactly as the reference leaves them (tri: b, c, d;
 * pent: b, c, d, e, f); d (tri) / f (pent) holds the solutions. Returns 0,
 * 1 (n too small) or 3 (zero pivot in some column; the other columns are
 * still solved, outputs unspecified, as in the reference). */
int oracle_tri_per_system(const double* a, double* b, double* c, double* d, size_t n, size_t m);
int oracle_pent_per_system(const double* a, double* b, double* c, double* d, double* e, double* f,
                           size_t n, size_t m);

#ifdef __cplusplus
}
#endif

#endif
