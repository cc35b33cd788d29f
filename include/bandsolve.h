/*
 * bandsolve (B200) — shared-LHS interleaved batch tridiagonal / pentadiagonal
 * solvers for NVIDIA B200 (sm_100a), drop-in for the reference C ABI.
 *
 * Every declaration in the first part carries the same name, arguments,
 * ownership and status semantics as the reference header
 * /root/reference/proj/include/bandsolve.h (cited per entry point as
 * "ref bandsolve.h:<line>", with the implementing reference source). A
 * caller linked against libbandsolve.so.1 runs unchanged against this
 * library: all 37 reference entry points are implemented (shared, uniform and
 * per-system solves, periodic corrections, IBAT I/O, footprint, the
 * Crank-Nicolson benchmark driver and the residuals). The build also installs
 * the reference SONAME alias libbandsolve.so.1.
 *
 * The second part ("B200 extensions") adds device-resident entry points for
 * callers that keep their batch in HBM: they take a device pointer, a row
 * pitch and a CUDA stream, enqueue the solve and return without
 * synchronising.
 *
 * Layout contract (ref batch.hpp:13-16): element (row i, system j) of an
 * n x m batch lives at data[i*m + j] (device variants: data[i*ld + j]).
 *
 * Solves run on the GPU only. Without a usable CUDA device every solve
 * returns BANDSOLVE_ERR_INTERNAL and bandsolve_last_error() says why; there
 * is no CPU fallback.
 */
#ifndef BANDSOLVE_H
#define BANDSOLVE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ref bandsolve.h:22-33 — identical values. */
typedef enum bandsolve_status {
  BANDSOLVE_OK = 0,
  BANDSOLVE_ERR_BAD_ARG = 1,
  BANDSOLVE_ERR_SHAPE_MISMATCH = 2,
  BANDSOLVE_ERR_FACTORIZATION_BREAKDOWN = 3,
  BANDSOLVE_ERR_DIVISION_BY_ZERO = 4,
  BANDSOLVE_ERR_SINGULAR_CORRECTION = 5,
  BANDSOLVE_ERR_SINGULAR_MATRIX = 6,
  BANDSOLVE_ERR_BAD_FORMAT = 7,
  BANDSOLVE_ERR_IO = 8,
  BANDSOLVE_ERR_INTERNAL = 9
} bandsolve_status;

/* ref bandsolve.h:35 (capi.cpp:82-97) — same strings. */
const char* bandsolve_status_string(bandsolve_status status);
/* ref bandsolve.h:36 (capi.cpp:99) — the ABI version, "1.0.0". */
const char* bandsolve_version(void);

/* ref bandsolve.h:41-42 (parallel.cpp:30-37). The count is recorded and
 * reported with the reference's resolution order (set value >
 * BANDSOLVE_THREADS > hardware concurrency); it does not change the GPU
 * solve, whose results are bitwise independent of it, as in the reference. */
int bandsolve_get_threads(void);
void bandsolve_set_threads(int threads);

/* ---- Interleaved batch (ref bandsolve.h:47-55, capi.cpp:105-128) ---------
 * Host storage, zero-filled, page-locked when a CUDA driver is present so
 * the staged solves copy at full PCIe rate. n == 0 or m == 0 -> BAD_ARG. */
typedef struct bandsolve_batch bandsolve_batch;

bandsolve_status bandsolve_batch_create(size_t n, size_t m,
                                        bandsolve_batch** out);
void bandsolve_batch_destroy(bandsolve_batch* batch);
size_t bandsolve_batch_rows(const bandsolve_batch* batch);
size_t bandsolve_batch_systems(const bandsolve_batch* batch);
double* bandsolve_batch_data(bandsolve_batch* batch);
const double* bandsolve_batch_data_const(const bandsolve_batch* batch);

/* ref bandsolve.h:57-62 (capi.cpp:130-141 -> batch.cpp:146-218). IBAT file:
 * little-endian "IBAT" magic, u32 version = 1, u64 n, u64 m, then n*m
 * binary64 values in interleaved order; byte-exact round trip. Open/seek/
 * write failures -> BANDSOLVE_ERR_IO; truncated header, bad magic, version
 * != 1, n or m of 0 or > 2^28, payload size mismatch -> BAD_FORMAT. */
bandsolve_status bandsolve_batch_read_ibat(const char* path,
                                           bandsolve_batch** out);
bandsolve_status bandsolve_batch_write_ibat(const bandsolve_batch* batch,
                                            const char* path);

/* ---- Tridiagonal (ref bandsolve.h:67-78) ---------------------------------
 * sub/diag/sup of length n >= 2, finite, sub[0] = sup[n-1] = 0
 * (banded.cpp:40-57). The factor (banded.cpp:67-86) is computed on the host
 * in the reference's operation order and uploaded to each device on first
 * use; the handle is immutable and may be shared across threads. */
typedef struct bandsolve_tri_factor bandsolve_tri_factor;

bandsolve_status bandsolve_tri_factor_create(const double* sub,
                                             const double* diag,
                                             const double* sup, size_t n,
                                             bandsolve_tri_factor** out);
void bandsolve_tri_factor_destroy(bandsolve_tri_factor* factor);

/* ref bandsolve.h:77-78 (capi.cpp:159-163 -> tri_solver.cpp:11-49).
 * Overwrites every system of the host batch with its solution: pinned
 * host -> device copies, sweep kernel, device -> host copies, pipelined over
 * column chunks, synchronous on return. rows != n -> SHAPE_MISMATCH. */
bandsolve_status bandsolve_tri_solve_shared(const bandsolve_tri_factor* factor,
                                            bandsolve_batch* batch);

/* ref bandsolve.h:80-85 (capi.cpp:165-172 -> tri_solver.cpp:51-112).
 * Baseline with one band copy per system: a/b/c are consumed (b holds the
 * pivot reciprocals, c the scaled super-diagonal on return, as in the
 * reference), d holds the solutions. Shapes differ -> SHAPE_MISMATCH; n < 2
 * -> BAD_ARG; a zero pivot -> FACTORIZATION_BREAKDOWN (outputs unspecified).
 * Runs on the GPU (thread per system, the reference's operation order:
 * bitwise equal), staged over column chunks, synchronous. */
bandsolve_status bandsolve_tri_solve_per_system(bandsolve_batch* a,
                                                bandsolve_batch* b,
                                                bandsolve_batch* c,
                                                bandsolve_batch* d);

/* ---- Pentadiagonal (ref bandsolve.h:91-113) ------------------------------
 * Bands a..e of length n >= 5, main diagonal c, structural zeros
 * a[0] = a[1] = b[0] = d[n-1] = e[n-1] = e[n-2] = 0 (banded.cpp:88-116). */
typedef struct bandsolve_pent_factor bandsolve_pent_factor;
typedef struct bandsolve_uniform_pent_factor bandsolve_uniform_pent_factor;

bandsolve_status bandsolve_pent_factor_create(const double* a, const double* b,
                                              const double* c, const double* d,
                                              const double* e, size_t n,
                                              bandsolve_pent_factor** out);
void bandsolve_pent_factor_destroy(bandsolve_pent_factor* factor);
/* ref bandsolve.h:99-100 (capi.cpp:191-195 -> pent_solver.cpp:67-81). */
bandsolve_status bandsolve_pent_solve_shared(
    const bandsolve_pent_factor* factor, bandsolve_batch* batch);

/* ref bandsolve.h:101-103 (capi.cpp:197-205 -> pent_solver.cpp:131-219).
 * Per-system baseline: b..e are consumed (beta, alpha, gamma, delta as the
 * reference leaves them), f holds the solutions; a is read only. n < 5 ->
 * BAD_ARG; zero alpha -> FACTORIZATION_BREAKDOWN. GPU, bitwise, synchronous. */
bandsolve_status bandsolve_pent_solve_per_system(
    bandsolve_batch* a, bandsolve_batch* b, bandsolve_batch* c,
    bandsolve_batch* d, bandsolve_batch* e, bandsolve_batch* f);

/* ref bandsolve.h:107-113 (capi.cpp:207-227 -> pent_solver.cpp:83-111):
 * constant bands, epsilon kept as one scalar; bitwise equal to the shared
 * solve of the expanded matrix. */
bandsolve_status bandsolve_uniform_pent_factor_create(
    double a, double b, double c, double d, double e, size_t n,
    bandsolve_uniform_pent_factor** out);
void bandsolve_uniform_pent_factor_destroy(
    bandsolve_uniform_pent_factor* factor);
bandsolve_status bandsolve_pent_solve_uniform(
    const bandsolve_uniform_pent_factor* factor, bandsolve_batch* batch);

/* ---- Periodic (cyclic) systems with constant bands (ref bandsolve.h:115-146,
 * periodic.cpp, capi.cpp:229-298, :414-446). The cyclic matrix is split into
 * a strictly banded A' (factorised once on the host, reference order) plus
 * a rank-1 (tri) / rank-2 (pent, Woodbury) wrap; a solve is the shared A'
 * sweep followed by the correction x = y - Z t(y), both on the GPU.
 * create: BAD_ARG for n < 3 (tri) / n < 6 (pent) or non-finite bands,
 * DIVISION_BY_ZERO for b == 0 (tri), SINGULAR_CORRECTION when the cyclic
 * matrix is singular; *out is NULL on failure. */
typedef struct bandsolve_periodic_tri bandsolve_periodic_tri;
typedef struct bandsolve_periodic_pent bandsolve_periodic_pent;

bandsolve_status bandsolve_periodic_tri_create(double a, double b, double c,
                                               size_t n,
                                               bandsolve_periodic_tri** out);
void bandsolve_periodic_tri_destroy(bandsolve_periodic_tri* corr);
bandsolve_status bandsolve_periodic_tri_solve(
    const bandsolve_periodic_tri* corr, bandsolve_batch* batch);
bandsolve_status bandsolve_periodic_tri_modified_bands(
    const bandsolve_periodic_tri* corr, double* sub, double* diag,
    double* sup);
bandsolve_status bandsolve_periodic_tri_correct(
    const bandsolve_periodic_tri* corr, bandsolve_batch* batch);

bandsolve_status bandsolve_periodic_pent_create(double a, double b, double c,
                                                double d, double e, size_t n,
                                                bandsolve_periodic_pent** out);
void bandsolve_periodic_pent_destroy(bandsolve_periodic_pent* corr);
bandsolve_status bandsolve_periodic_pent_solve(
    const bandsolve_periodic_pent* corr, bandsolve_batch* batch);
bandsolve_status bandsolve_periodic_pent_modified_bands(
    const bandsolve_periodic_pent* corr, double* a, double* b, double* c,
    double* d, double* e);
bandsolve_status bandsolve_periodic_pent_correct(
    const bandsolve_periodic_pent* corr, bandsolve_batch* batch);

/* ---- Storage accounting (ref bandsolve.h:148-163, batch.cpp:72-105) -------- */
typedef enum bandsolve_storage_variant {
  BANDSOLVE_STORAGE_TRI_PER_SYSTEM = 0,
  BANDSOLVE_STORAGE_TRI_SHARED = 1,
  BANDSOLVE_STORAGE_PENT_PER_SYSTEM = 2,
  BANDSOLVE_STORAGE_PENT_SHARED = 3,
  BANDSOLVE_STORAGE_PENT_UNIFORM = 4
} bandsolve_storage_variant;

bandsolve_status bandsolve_footprint(bandsolve_storage_variant variant,
                                     size_t n, size_t m, uint64_t* elements,
                                     double* reduction_vs_baseline);

/* ---- Crank-Nicolson driver (ref bandsolve.h:182-220, capi.cpp:369-411,
 * pde.cpp run_benchmark). Periodic diffusion through the tridiagonal path,
 * periodic hyperdiffusion through the pentadiagonal path, from the
 * reference's default initial field. Same parameters, checks, statuses and
 * IBAT dumps; the stepping loop (RHS assembly + cyclic solve per step) runs
 * on the GPU and each step is timed with CUDA events. The uniform variant
 * is the shared one (bitwise identical, pent_solver.cpp:83-97); the
 * per-system variant rewrites replicated band copies every step and runs
 * the per-system kernels, as the reference's engine (pde.cpp:168-221). */
typedef enum bandsolve_problem {
  BANDSOLVE_PROBLEM_DIFFUSION = 0,
  BANDSOLVE_PROBLEM_HYPERDIFFUSION = 1
} bandsolve_problem;

typedef enum bandsolve_variant {
  BANDSOLVE_VARIANT_SHARED = 0,
  BANDSOLVE_VARIANT_PER_SYSTEM = 1,
  BANDSOLVE_VARIANT_UNIFORM = 2, /* hyperdiffusion only */
  /* extension: the per-system step with cuSPARSE's gtsvInterleavedBatch
   * (Thomas) / gpsvInterleavedBatch as the solver, the paper's cuThomasBatch
   * comparator; ERR_INTERNAL when cuSPARSE is absent */
  BANDSOLVE_VARIANT_CUSPARSE = 3
} bandsolve_variant;

typedef struct bandsolve_bench_params {
  size_t n;
  size_t m;
  long steps;
  double dt; /* <= 0 selects the default with sigma_x = 1 */
  int problem; /* bandsolve_problem */
  int variant; /* bandsolve_variant */
  long dump_every; /* 0 disables IBAT field dumps */
  const char* dump_prefix; /* may be NULL when dump_every is 0 */
} bandsolve_bench_params;

typedef struct bandsolve_bench_result {
  double wall_s;
  double per_step_mean_s;
  double per_step_std_s;
  uint64_t elements; /* storage footprint of the variant */
  int threads;
  long steps;
} bandsolve_bench_result;

bandsolve_status bandsolve_bench_run(const bandsolve_bench_params* params,
                                     bandsolve_bench_result* result);

/* ---- Residuals (ref bandsolve.h:165-179, tri_solver.cpp:116-156,
 * pent_solver.cpp:223-273) — max over systems of ||A x - rhs||_inf /
 * ||rhs||_inf, evaluated on the GPU in the reference's operation order.
 * cyclic != 0 reads the wrap corners from the interior band entries. */
bandsolve_status bandsolve_tri_residual(const double* sub, const double* diag,
                                        const double* sup, size_t n,
                                        int cyclic,
                                        const bandsolve_batch* x,
                                        const bandsolve_batch* rhs,
                                        double* out);
bandsolve_status bandsolve_pent_residual(const double* a, const double* b,
                                         const double* c, const double* d,
                                         const double* e, size_t n, int cyclic,
                                         const bandsolve_batch* x,
                                         const bandsolve_batch* rhs,
                                         double* out);

/* ======================================================================== */
/* B200 extensions                                                          */
/* ======================================================================== */

/* Arithmetic mode of the sweep kernels.
 *   EXACT (default): the reference's operation order with every product and
 *     difference rounded separately (no FMA contraction): fp64 results are
 *     bitwise identical to the reference CPU solver.
 *   FAST: fused multiply-adds over host-prescaled factors (tri: p_i = a_i m_i;
 *     pent: beta_i/alpha_i, eps_i/alpha_i) — one dependent DFMA per row and
 *     sweep. Differs from the reference by rounding only (per-system
 *     max-norm relative gap <= 1e-12 on the conditioned systems tested).
 * Process-global; the environment variable BANDSOLVE_MODE=exact|fast sets
 * the initial value. */
typedef enum bandsolve_mode {
  BANDSOLVE_MODE_EXACT = 0,
  BANDSOLVE_MODE_FAST = 1
} bandsolve_mode;
bandsolve_status bandsolve_set_mode(int mode);
int bandsolve_get_mode(void);

/* Device-resident solves. x points to an n x m interleaved array in device
 * memory of the current CUDA device, row pitch ld >= m elements; stream is a
 * cudaStream_t (NULL = legacy default stream). The call validates, enqueues
 * and returns; it does not synchronise. n must equal the factor's order.
 * The f32 variants round the fp64 factor once and sweep in binary32. */
bandsolve_status bandsolve_tri_solve_shared_dev(
    const bandsolve_tri_factor* factor, double* x, size_t n, size_t m,
    size_t ld, void* stream);
bandsolve_status bandsolve_tri_solve_shared_dev_f32(
    const bandsolve_tri_factor* factor, float* x, size_t n, size_t m,
    size_t ld, void* stream);
bandsolve_status bandsolve_pent_solve_shared_dev(
    const bandsolve_pent_factor* factor, double* x, size_t n, size_t m,
    size_t ld, void* stream);
bandsolve_status bandsolve_pent_solve_shared_dev_f32(
    const bandsolve_pent_factor* factor, float* x, size_t n, size_t m,
    size_t ld, void* stream);
/* Device-resident per-system baselines (extension): the same arrays as the
 * host calls, each n x m with row pitch ld, in device memory. Synchronises
 * `stream` to report breakdown. */
bandsolve_status bandsolve_tri_solve_per_system_dev(double* a, double* b,
                                                    double* c, double* d,
                                                    size_t n, size_t m,
                                                    size_t ld, void* stream);
bandsolve_status bandsolve_pent_solve_per_system_dev(
    double* a, double* b, double* c, double* d, double* e, double* f,
    size_t n, size_t m, size_t ld, void* stream);
/* cuSPARSE comparators (extension): the library
 * per-system batch solvers the paper benchmarks against, on the same
 * interleaved layout with pitch m (cuSPARSE takes none). Bands are per-system
 * copies, n x m each, device memory: tri dl (sub, dl[0] = 0), d, du (sup,
 * du[n-1] = 0); pent ds, dl, d, du, dw (the a..e bands). x (n x m) is
 * overwritten with the solution; the bands may be overwritten. tri algo:
 * 0 Thomas (cuThomasBatch), 1 LU with partial pivoting, 2 QR; pent: 0 (QR).
 * cuSPARSE is loaded at first use (dlopen libcusparse.so.12); absent ->
 * BANDSOLVE_ERR_INTERNAL. Stream-ordered, no synchronisation. */
int bandsolve_cusparse_available(void);
bandsolve_status bandsolve_tri_solve_cusparse_dev(double* dl, double* d,
                                                  double* du, double* x,
                                                  size_t n, size_t m, int algo,
                                                  void* stream);
bandsolve_status bandsolve_pent_solve_cusparse_dev(double* ds, double* dl,
                                                   double* d, double* du,
                                                   double* dw, double* x,
                                                   size_t n, size_t m,
                                                   void* stream);
bandsolve_status bandsolve_pent_solve_uniform_dev(
    const bandsolve_uniform_pent_factor* factor, double* x, size_t n,
    size_t m, size_t ld, void* stream);
bandsolve_status bandsolve_pent_solve_uniform_dev_f32(
    const bandsolve_uniform_pent_factor* factor, float* x, size_t n, size_t m,
    size_t ld, void* stream);

/* Periodic solves / corrections of a device-resident batch (same contract
 * as the *_dev solves above; correct_only = the wrap correction alone, for
 * callers that solved A' y = d themselves). */
bandsolve_status bandsolve_periodic_tri_solve_dev(
    const bandsolve_periodic_tri* corr, double* x, size_t n, size_t m,
    size_t ld, void* stream);
bandsolve_status bandsolve_periodic_tri_correct_dev(
    const bandsolve_periodic_tri* corr, double* x, size_t n, size_t m,
    size_t ld, void* stream);
bandsolve_status bandsolve_periodic_pent_solve_dev(
    const bandsolve_periodic_pent* corr, double* x, size_t n, size_t m,
    size_t ld, void* stream);
bandsolve_status bandsolve_periodic_pent_correct_dev(
    const bandsolve_periodic_pent* corr, double* x, size_t n, size_t m,
    size_t ld, void* stream);

/* One Crank-Nicolson step on device arrays: out = A^-1 (B u) with B the
 * explicit periodic stencil of pde.cpp:73-114 for sigma_x (diffusion:
 * s (u[i-1] + u[i+1]) + (1 - 2s) u[i]; hyperdiffusion: -s (u[i-2] + u[i+2])
 * + 4s (u[i-1] + u[i+1]) + (1 - 6s) u[i], indices mod n) and A the cyclic
 * LHS held by the handle. u and out must not alias (pitch ld, stream-ordered). */
bandsolve_status bandsolve_periodic_tri_cn_step_dev(
    const bandsolve_periodic_tri* lhs, double sigma_x, const double* u,
    double* out, size_t n, size_t m, size_t ld, void* stream);
bandsolve_status bandsolve_periodic_pent_cn_step_dev(
    const bandsolve_periodic_pent* lhs, double sigma_x, const double* u,
    double* out, size_t n, size_t m, size_t ld, void* stream);

/* Two-dimensional ADI (BASELINE configs[3]; no reference counterpart). One
 * Peaceman-Rachford step of the periodic diffusion / hyperdiffusion problem
 * on an ny x nx field C[y*ld + x] (device, fp64):
 *   (I - s Lx) u* = (I + s Ly) u,   (I - s Ly) u' = (I + s Lx) u*
 * with the Crank-Nicolson bands and stencils of the 1D driver along each
 * axis. y-solves run on the interleaved layout directly (systems = x), x-solves
 * on a transposed copy (systems = y). work: an ny x ld scratch array, used
 * as the transposed field (pitch ny rounded up to even) when it is 16-byte
 * aligned and large enough, else the library takes a block from its pool for
 * the step; must not alias field. The call is stream-ordered. */
typedef struct bandsolve_adi bandsolve_adi;
bandsolve_status bandsolve_adi_create(int problem, double sigma_x, size_t nx,
                                      size_t ny, bandsolve_adi** out);
void bandsolve_adi_destroy(bandsolve_adi* adi);
bandsolve_status bandsolve_adi_step_dev(const bandsolve_adi* adi,
                                        double* field, double* work,
                                        size_t ld, void* stream);

/* Device residual of a device-resident solution against a device-resident
 * right-hand side (both n x m, pitch ld), bands on the host. Synchronous:
 * writes the max relative residual to *out. */
bandsolve_status bandsolve_tri_residual_dev(const double* sub,
                                            const double* diag,
                                            const double* sup, size_t n,
                                            int cyclic, const double* x,
                                            const double* rhs, size_t m,
                                            size_t ld, void* stream,
                                            double* out);
bandsolve_status bandsolve_pent_residual_dev(
    const double* a, const double* b, const double* c, const double* d,
    const double* e, size_t n, int cyclic, const double* x, const double* rhs,
    size_t m, size_t ld, void* stream, double* out);

/* Synthetic right-hand side on the device: x[i*ld + j] = U(-1, 1) drawn
 * from SplitMix64 of (seed, i, j_offset + j), identical bit for bit to the
 * host generator in oracle/ (so shards of one global batch agree). */
bandsolve_status bandsolve_fill_rhs_dev(double* x, size_t n, size_t m,
                                        size_t ld, uint64_t seed,
                                        uint64_t j_offset, void* stream);
bandsolve_status bandsolve_fill_rhs_dev_f32(float* x, size_t n, size_t m,
                                            size_t ld, uint64_t seed,
                                            uint64_t j_offset, void* stream);

/* Factor introspection: copies the host factor arrays (the reference's
 * tri_factor / pent_factor / uniform_pent_factor fields, banded.hpp:48-53,
 * :88-95, pent_solver.hpp:31-38). Any pointer may be NULL. */
size_t bandsolve_tri_factor_order(const bandsolve_tri_factor* factor);
bandsolve_status bandsolve_tri_factor_arrays(const bandsolve_tri_factor* f,
                                             double* chat, double* inv_denom,
                                             double* sub);
size_t bandsolve_pent_factor_order(const bandsolve_pent_factor* factor);
bandsolve_status bandsolve_pent_factor_arrays(const bandsolve_pent_factor* f,
                                              double* inv_alpha, double* beta,
                                              double* gamma, double* delta,
                                              double* epsilon);
size_t bandsolve_uniform_pent_factor_order(
    const bandsolve_uniform_pent_factor* factor);
bandsolve_status bandsolve_uniform_pent_factor_arrays(
    const bandsolve_uniform_pent_factor* f, double* inv_alpha, double* beta,
    double* gamma, double* delta, double* eps_scalar);

/* Kernel plan the sweep would use for (kind, n, m, dtype) on the current
 * device: writes a short human-readable description ("smem-tma W=16 ..."). */
typedef enum bandsolve_kind {
  BANDSOLVE_KIND_TRI = 0,
  BANDSOLVE_KIND_PENT = 1,
  BANDSOLVE_KIND_UNIFORM = 2
} bandsolve_kind;
bandsolve_status bandsolve_describe_plan(int kind, size_t n, size_t m,
                                         size_t ld, int f32, char* buf,
                                         size_t buflen);

/* Devices the host-batch solves (bandsolve_*_solve_shared, periodic solves
 * on a bandsolve_batch) spread over: the batch's m systems are split into
 * contiguous column ranges j0 = m*g/G, one per listed device (the
 * reference's worker split, parallel.cpp:53-54), each streamed through its
 * own device's copy/sweep pipeline, all in flight at once. count = 0 (the
 * default) uses the calling thread's current device. A device may be listed
 * more than once (independent pipelines on it). Results are bitwise
 * independent of the list. Ids are checked against the device count at
 * solve time (BANDSOLVE_ERR_BAD_ARG). Process-wide setting. */
bandsolve_status bandsolve_set_devices(const int* devices, int count);
/* Writes up to `capacity` ids to `devices` (may be NULL); returns the count. */
int bandsolve_get_devices(int* devices, int capacity);

/* Tuning overrides (plans, ring depths, fused/unfused variants; for tests
 * and tuning runs, never needed for correctness). The table is seeded once,
 * at first use, from the environment variables BANDSOLVE_<key>; after that
 * only these calls change it. Keys: PLAN (stream|global|persist|smem|smemW8|
 * smemW16|smemW32), PWARPS, PTAIL (persist plan); SWG, STAIL, SKB, SKR, SPD,
 * SV, SRC, SSEG, TM8, TMEM, SSTAG (stream plan: group width, smem tail rows,
 * b / reload ring slots, L2 prefetch distance, systems per lane, recomputed
 * rows, recompute segment chunks, TMEM with 5..8 warps, TMEM on/off, start
 * stagger); SPIKE (0|1: the one-pass partitioned kernel, fast mode),
 * SPIKE_K (its block count), NO_PDL (flag: no programmatic dependent
 * launch); PIPE (0|1: the pipelined on-chip sequential kernel), PKB (its
 * minimum ring slots), PIPE_MAX_N (its row limit, default 4096; beyond 512
 * rows with an L2 tier), PIPE_L2_P (compute warps with the L2 tier), PRT
 * (its register chunks), PIPE_CN (flag: the CN step through it),
 * SPIKE_F32_MIN_N (smallest n for the fp32 spike kernel); PARTITION (0|1), PART_K; CN_UNFUSED, PERIODIC_UNFUSED,
 * ADI_UNFUSED, ADI_FUSE_PENT (flags: set = on); HOST_CHUNK_MIB (host-batch
 * staging chunk); L2_SETASIDE (1: grow the device's persisting-L2 limit to
 * cover the spill scratch; process-wide state, off by default).
 * value NULL unsets the key. Unknown key -> BANDSOLVE_ERR_BAD_ARG. */
bandsolve_status bandsolve_tune_set(const char* key, const char* value);
/* Current value (copied into buf) or BANDSOLVE_ERR_BAD_ARG when unset. */
bandsolve_status bandsolve_tune_get(const char* key, char* buf, size_t buflen);
/* Clear every override (the environment is not re-read). */
void bandsolve_tune_reset(void);

/* Number of this library's kernels launched since load (all threads). */
uint64_t bandsolve_kernel_launches(void);

/* Thread-local description of the last non-OK status on this thread. */
const char* bandsolve_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* BANDSOLVE_H */
