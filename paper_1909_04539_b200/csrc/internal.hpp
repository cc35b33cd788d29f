// Internal interfaces of libbandsolve_b200: host factor objects, the device
// launch layer and the thread-local error channel. Nothing here is exported;
// the C ABI lives in capi.cpp.
#pragma once

#include <cstddef>
#include <cstdint>
#include <deque>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include <cuda_runtime_api.h>

#include "../../include/bandsolve.h"

namespace bsb {

// common.hpp:17 — pivots with |denom| < 1e-300 are a breakdown.
inline constexpr double kBreakdownEps = 1e-300;

enum class Kind { Tri = 0, Pent = 1, Uniform = 2 };

// Device copies of one factor on one device (see solve.cu for the packed
// record layouts). One allocation holds all four variants
// {exact, fast} x {f64, f32}.
struct DeviceFactor {
  int device = -1;
  void* base = nullptr;
  const void* fwd[2][2] = {};  // [f32][fast]
  const void* bwd[2][2] = {};
};

// Partitioned (SPIKE) solve plan for few long systems, cached per factor and
// block count (partition.cu).
struct PartPlan;
struct PartPlanDeleter {
  void operator()(PartPlan* p) const;
};

// Host factor: the reference's factor arrays, computed once on the host in
// the reference's operation order (banded.cpp:67-86, :127-176,
// pent_solver.cpp:99-111), plus a lazily filled per-device cache.
struct Factor {
  Kind kind = Kind::Tri;
  std::size_t n = 0;
  // tri_factor fields (banded.hpp:48-53)
  std::vector<double> chat, inv_denom, sub;
  // pent_factor / uniform_pent_factor fields (banded.hpp:88-95)
  std::vector<double> inv_alpha, beta, gamma, delta, epsilon;
  double eps_scalar = 0.0;
  // the bands the factor was built from (tri: sub|diag|sup, pent: a|b|c|d|e),
  // for the partitioned path's block factors
  std::vector<double> bands;

  mutable std::mutex mu;
  // one entry per touched device; a deque so that an entry handed out to one
  // thread never moves when another thread adds a device
  mutable std::deque<DeviceFactor> devices;
  mutable std::vector<std::unique_ptr<PartPlan, PartPlanDeleter>> parts;
  ~Factor();
};

// ---- host prefactor (host_factor.cpp) ------------------------------------
bandsolve_status make_tri_factor(const double* sub, const double* diag,
                                 const double* sup, std::size_t n,
                                 std::unique_ptr<Factor>& out);
bandsolve_status make_pent_factor(const double* a, const double* b,
                                  const double* c, const double* d,
                                  const double* e, std::size_t n,
                                  std::unique_ptr<Factor>& out);
bandsolve_status make_uniform_factor(double a, double b, double c, double d,
                                     double e, std::size_t n,
                                     std::unique_ptr<Factor>& out);
// Band validation shared with the residual entry points
// (banded.cpp:40-57, :88-116).
bandsolve_status validate_tri_bands(const double* sub, const double* diag,
                                    const double* sup, std::size_t n);
bandsolve_status validate_pent_bands(const double* a, const double* b,
                                     const double* c, const double* d,
                                     const double* e, std::size_t n);

// Periodic (cyclic, constant bands) systems: the strictly banded A' that
// backs them plus the low-rank wrap correction (reference periodic.hpp,
// periodic.cpp). kind Tri: rank 1, z1 = A'^-1 u, v_last = -a/b,
// scale = 1 / (1 + v.z). kind Pent: rank 2 (Woodbury), z1, z2 and the 2x2
// capacitance inverse, row-major.
struct Periodic {
  Kind kind = Kind::Tri;
  std::size_t n = 0;
  std::unique_ptr<Factor> factor;
  std::vector<double> z1, z2;
  double v_last = 0.0, scale = 0.0;
  double cap_inv[4] = {0.0, 0.0, 0.0, 0.0};
  // fused fast-mode sweep: rows 0 (and 1) of U^-1 of A' = L U, then z1 (z2):
  // r0 | z1 (tri) or r0 | r1 | z1 | z2 (pent), n each
  std::vector<double> fused;

  mutable std::mutex mu;
  mutable std::vector<std::pair<int, double*>> devices;  // z1 | z2 per device
  ~Periodic();
};

// periodic.cpp:11-55 / :97-170, in the reference's evaluation order.
bandsolve_status make_periodic_tri(double a, double b, double c, std::size_t n,
                                   std::unique_ptr<Periodic>& out);
bandsolve_status make_periodic_pent(double a, double b, double c, double d,
                                    double e, std::size_t n,
                                    std::unique_ptr<Periodic>& out);
// capi.cpp:249-262 / :414-446: A' reassembled from its factor.
void periodic_tri_modified_bands(const Periodic& p, double* sub, double* diag,
                                 double* sup);
void periodic_pent_modified_bands(const Periodic& p, double* a, double* b,
                                  double* c, double* d, double* e);

// ---- device layer (solve.cu) ---------------------------------------------
int current_mode();
void set_mode(int mode);

// Stream-ordered allocation from the library's own per-device pool (freed
// blocks stay mapped; the application's default pool is untouched). Free
// with cudaFreeAsync.
cudaError_t pool_malloc_async_raw(void** p, std::size_t bytes, cudaStream_t s);
template <typename T>
cudaError_t pool_malloc_async(T** p, std::size_t bytes, cudaStream_t s) {
  return pool_malloc_async_raw(reinterpret_cast<void**>(p), bytes, s);
}

// Tuning overrides (tuning.cpp): bandsolve_tune_set(), seeded once from the
// BANDSOLVE_<KEY> environment. tune_flag: the key is set (any value).
std::optional<std::string> tune_str(const char* key);
long long tune_int(const char* key, long long dflt);
bool tune_flag(const char* key);
bool tune_set(const char* key, const char* value);
void tune_reset();

// Enqueue an in-place solve of the n x m (pitch ld) device array x.
bandsolve_status solve_device(const Factor& f, void* x, bool f32,
                              std::size_t n, std::size_t m, std::size_t ld,
                              void* stream);
// Partitioned fast-mode solve (partition.cu) for the few-long-systems regime;
// BANDSOLVE_OK and *done = false when it does not apply (caller falls back).
// With `per`, the periodic (Woodbury) correction is fused into the last pass.
struct PartPeriodic {
  const double* z1;
  const double* z2;
  double c[4];  // tri: v_last, scale; pent: cap_inv
};
// With `st`, the RHS is the periodic CN stencil across systems of src, laid
// out src[j * lds + i] (system j, row i): the ADI explicit half + transpose
// fused into the first pass. x is then output only.
struct PartStencil {
  const double* src;
  std::size_t lds;
  double s, s4, mid;
};
int partition_blocks(std::size_t n, std::size_t m, int sms, bool pent);  // 0 = not used
// One-pass partitioned sweep for many long systems (sweep_spike.cuh), fast
// mode fp64: blocks per system, 0 when it does not apply.
int spike_blocks(std::size_t n, std::size_t m, std::size_t ld, const void* x, int sms, bool pent,
                 std::size_t elem = 8);
// Pipelined sequential sweep (sweep_pipe.cuh), fp64, n % 16 == 0: compute
// warps (0 = not used), ring slots, shared-memory chunks, and the launch.
struct PartPeriodic;
// Crank-Nicolson step through the spike kernel: b = the periodic stencil of
// u (read only), x receives u_new; c = s, 4s (pent), 1-2s / 1-6s
struct SpikeCN {
  const double* u;
  double c[3];
};
bandsolve_status spike_solve_device(const Factor& f, double* x, std::size_t n, std::size_t m, std::size_t ld,
                                    void* stream, int sms, bool* done, const PartPeriodic* per = nullptr,
                                    const SpikeCN* cn = nullptr);
bandsolve_status spike_solve_device_f32(const Factor& f, float* x, std::size_t n, std::size_t m, std::size_t ld,
                                        void* stream, int sms, bool* done);
int pipe_warps(std::size_t n, std::size_t m, std::size_t ld, const void* x, bool pent, int sms, int* kb, int* rt,
               int* st, bool per = false);
bandsolve_status pipe_solve_device(bool pent, bool fast, const void* fwd, const void* bwd, double* x, std::size_t n,
                                   std::size_t m, std::size_t ld, void* stream, int sms, bool* done,
                                   const PartPeriodic* per = nullptr, const SpikeCN* cn = nullptr,
                                   bool f32 = false);
bool partition_stencil_ok(std::size_t n, std::size_t m, int K, std::size_t lds);
bandsolve_status partition_solve_device(const Factor& f, double* x, std::size_t n,
                                        std::size_t m, std::size_t ld,
                                        void* stream, int sms, bool* done,
                                        const PartPeriodic* per = nullptr,
                                        const PartStencil* st = nullptr);
// Per-system baselines (per_system.cu): arr = a, b, c, d (tri) / a..f (pent),
// reference tri_solver.cpp:51-112, pent_solver.cpp:131-219. The device form
// synchronises `stream` to report breakdown.
bandsolve_status per_system_device(bool pent, double* const* arr, std::size_t n, std::size_t m, std::size_t ld,
                                   void* stream);
bandsolve_status per_system_host(bool pent, double* const* arr, std::size_t n, std::size_t m);
// cuSPARSE comparators (cusparse_cmp.cpp, dlopen'ed): gtsv/gpsvInterleavedBatch
// on per-system bands, n x m with pitch m; x overwritten, stream-ordered.
bool cusparse_available();
bandsolve_status cusparse_solve_device(bool pent, double* const* bands, double* x, std::size_t n, std::size_t m,
                                       int algo, void* stream);
// IBAT files (capi.cpp), reference batch.cpp:146-218
bandsolve_status ibat_write(const char* path, const double* data, std::size_t n, std::size_t m);
bandsolve_status ibat_read(const char* path, std::size_t* n, std::size_t* m, double** data, bool* pinned);

// Host batch: staged through the device, synchronous. With `per`, the
// periodic correction follows the sweep on each staged chunk; with
// `correct_only`, only the correction runs.
// Device list of the host-batch solves (empty: the caller's current device).
bandsolve_status set_devices(const int* ids, int count);
int get_devices(int* ids, int capacity);
bandsolve_status solve_host(const Factor& f, double* x, std::size_t n,
                            std::size_t m, const Periodic* per = nullptr,
                            bool correct_only = false);
// Crank-Nicolson explicit half B u with the periodic stencil of
// pde.cpp:73-114 (out must not alias u), stream-ordered.
bandsolve_status cn_rhs_device(bool pent, double sigma_x, const double* u,
                               double* out, std::size_t n, std::size_t m,
                               std::size_t ld, void* stream);
// One Peaceman-Rachford ADI step of a periodic ny x nx field (pitch ld).
bandsolve_status adi_step_device(const Periodic& px, const Periodic& py,
                                 double sigma, double* field, double* work,
                                 std::size_t nx, std::size_t ny,
                                 std::size_t ld, void* stream);
// One Crank-Nicolson step out = A^-1 (B u), stencil fused into the sweep.
bandsolve_status cn_step_device(const Periodic& p, double sigma_x,
                                const double* u, double* out, std::size_t n,
                                std::size_t m, std::size_t ld, void* stream);
// bandsolve_bench_run: the reference's Crank-Nicolson driver (capi.cpp:369,
// pde.cpp run_benchmark) with the stepping loop on the GPU.
bandsolve_status bench_run_device(const bandsolve_bench_params& prm,
                                  bandsolve_bench_result* res,
                                  int threads_report);
// Periodic solve / correction of a device array (pitch ld), stream-ordered.
bandsolve_status periodic_device(const Periodic& p, double* x, std::size_t n,
                                 std::size_t m, std::size_t ld, void* stream,
                                 bool correct_only);
// Residual kernels; bands are host arrays of length n (5 for pent).
bandsolve_status residual_device(Kind kind, const double* const* bands,
                                 std::size_t n, int cyclic, const double* x,
                                 const double* rhs, std::size_t m,
                                 std::size_t ld, void* stream, double* out);
bandsolve_status residual_host(Kind kind, const double* const* bands,
                               std::size_t n, int cyclic, const double* x,
                               const double* rhs, std::size_t m, double* out);
bandsolve_status fill_rhs_device(void* x, bool f32, std::size_t n,
                                 std::size_t m, std::size_t ld, uint64_t seed,
                                 uint64_t j_offset, void* stream);
bandsolve_status describe_plan(Kind kind, std::size_t n, std::size_t m,
                               std::size_t ld, bool f32, std::string& out);
void release_device_factor(DeviceFactor& d);
uint64_t kernel_launches();
void note_launches(int k);

// Page-locked host allocation when a driver is present, else calloc.
double* host_alloc_zeroed(std::size_t count, bool* pinned);
void host_free(double* p, bool pinned);

// ---- errors ----------------------------------------------------------------
bandsolve_status fail(bandsolve_status st, const std::string& msg);
const char* last_error();
void clear_error();

}  // namespace bsb
