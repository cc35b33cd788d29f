// extern "C" surface of libbandsolve_b200 — the drop-in for the reference's
// shared library (proj/src/capi.cpp, proj/include/bandsolve.h). Same entry
// points, argument checks, ownership and status codes; the solves run on
// the GPU (solve.cu). C++ exceptions never cross this boundary.
#include <atomic>
#include <cmath>
#include <vector>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <thread>

#include "internal.hpp"

#define BSB_API extern "C" __attribute__((visibility("default")))

// Opaque handles (ref capi.cpp:17-34).
struct bandsolve_batch {
  std::size_t n = 0, m = 0;
  double* data = nullptr;
  bool pinned = false;
  ~bandsolve_batch() { bsb::host_free(data, pinned); }
};
struct bandsolve_tri_factor {
  std::unique_ptr<bsb::Factor> impl;
};
struct bandsolve_pent_factor {
  std::unique_ptr<bsb::Factor> impl;
};
struct bandsolve_uniform_pent_factor {
  std::unique_ptr<bsb::Factor> impl;
};
struct bandsolve_periodic_tri {
  std::unique_ptr<bsb::Periodic> impl;
};
struct bandsolve_periodic_pent {
  std::unique_ptr<bsb::Periodic> impl;
};
struct bandsolve_adi {
  int problem = 0;
  double sigma = 0.0;
  std::size_t nx = 0, ny = 0;
  std::unique_ptr<bsb::Periodic> px, py;
};

namespace bsb {

namespace {
thread_local std::string t_last_error;
}

bandsolve_status fail(bandsolve_status st, const std::string& msg) {
  t_last_error = msg;
  return st;
}
const char* last_error() { return t_last_error.c_str(); }
void clear_error() { t_last_error.clear(); }

}  // namespace bsb

namespace {

// capi.cpp:64-72: every exception maps to a status; allocation failures and
// anything unexpected are INTERNAL.
template <typename Fn>
bandsolve_status guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const std::bad_alloc&) {
    return bsb::fail(BANDSOLVE_ERR_INTERNAL, "out of host memory");
  } catch (const std::exception& e) {
    return bsb::fail(BANDSOLVE_ERR_INTERNAL, e.what());
  } catch (...) {
    return bsb::fail(BANDSOLVE_ERR_INTERNAL, "unknown exception");
  }
}

// parallel.cpp:17-37: set value > BANDSOLVE_THREADS > hardware concurrency.
std::atomic<int> g_threads{0};
int default_threads() {
  if (const char* env = std::getenv("BANDSOLVE_THREADS")) {
    const int v = std::atoi(env);
    if (v >= 1) return v;
  }
  const unsigned hw = std::thread::hardware_concurrency();
  return hw ? static_cast<int>(hw) : 1;
}

bandsolve_status null_arg() { return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "null argument"); }

}  // namespace

BSB_API const char* bandsolve_status_string(bandsolve_status status) {
  switch (status) {  // capi.cpp:82-97
    case BANDSOLVE_OK: return "ok";
    case BANDSOLVE_ERR_BAD_ARG: return "bad argument";
    case BANDSOLVE_ERR_SHAPE_MISMATCH: return "shape mismatch";
    case BANDSOLVE_ERR_FACTORIZATION_BREAKDOWN: return "factorization breakdown";
    case BANDSOLVE_ERR_DIVISION_BY_ZERO: return "division by zero";
    case BANDSOLVE_ERR_SINGULAR_CORRECTION: return "singular correction";
    case BANDSOLVE_ERR_SINGULAR_MATRIX: return "singular matrix";
    case BANDSOLVE_ERR_BAD_FORMAT: return "malformed IBAT data";
    case BANDSOLVE_ERR_IO: return "I/O failure";
    case BANDSOLVE_ERR_INTERNAL: return "internal error";
  }
  return "unknown status";
}

BSB_API const char* bandsolve_version(void) { return "1.0.0"; }

BSB_API int bandsolve_get_threads(void) {
  const int pinned = g_threads.load(std::memory_order_relaxed);
  return pinned >= 1 ? pinned : default_threads();
}

BSB_API void bandsolve_set_threads(int threads) {
  g_threads.store(threads >= 1 ? threads : 0, std::memory_order_relaxed);
}

// ---- batch (capi.cpp:105-128; batch.cpp:10-13) ----------------------------
BSB_API bandsolve_status bandsolve_batch_create(size_t n, size_t m, bandsolve_batch** out) {
  if (!out) return null_arg();
  *out = nullptr;
  if (n == 0 || m == 0) return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "batch shape must be positive");
  return guarded([&] {
    if (m > SIZE_MAX / sizeof(double) / n) return bsb::fail(BANDSOLVE_ERR_INTERNAL, "batch too large");
    auto b = std::make_unique<bandsolve_batch>();
    b->n = n;
    b->m = m;
    b->data = bsb::host_alloc_zeroed(n * m, &b->pinned);
    if (!b->data) return bsb::fail(BANDSOLVE_ERR_INTERNAL, "out of host memory");
    *out = b.release();
    return BANDSOLVE_OK;
  });
}

BSB_API void bandsolve_batch_destroy(bandsolve_batch* batch) { delete batch; }
BSB_API size_t bandsolve_batch_rows(const bandsolve_batch* batch) { return batch ? batch->n : 0; }
BSB_API size_t bandsolve_batch_systems(const bandsolve_batch* batch) { return batch ? batch->m : 0; }
BSB_API double* bandsolve_batch_data(bandsolve_batch* batch) { return batch ? batch->data : nullptr; }
BSB_API const double* bandsolve_batch_data_const(const bandsolve_batch* batch) {
  return batch ? batch->data : nullptr;
}

// ---- IBAT files (capi.cpp:130-141; batch.cpp:146-218) -------------------------
BSB_API bandsolve_status bandsolve_batch_read_ibat(const char* path, bandsolve_batch** out) {
  if (!path || !out) return null_arg();
  *out = nullptr;
  return guarded([&] {
    auto b = std::make_unique<bandsolve_batch>();
    bandsolve_status st = bsb::ibat_read(path, &b->n, &b->m, &b->data, &b->pinned);
    if (st != BANDSOLVE_OK) return st;
    *out = b.release();
    return BANDSOLVE_OK;
  });
}

BSB_API bandsolve_status bandsolve_batch_write_ibat(const bandsolve_batch* batch, const char* path) {
  if (!batch || !path) return null_arg();
  return guarded([&] { return bsb::ibat_write(path, batch->data, batch->n, batch->m); });
}

// ---- per-system baselines (capi.cpp:165-172, :197-205) --------------------------
namespace {
bandsolve_status per_system_batches(bool pent, bandsolve_batch* const* v) {
  const int na = pent ? 6 : 4;
  for (int q = 0; q < na; ++q)
    if (!v[q]) return null_arg();
  return guarded([&] {
    for (int q = 1; q < na; ++q)
      if (v[q]->n != v[0]->n || v[q]->m != v[0]->m)
        return bsb::fail(BANDSOLVE_ERR_SHAPE_MISMATCH, "band/rhs buffers differ in shape");
    double* arr[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    for (int q = 0; q < na; ++q) arr[q] = v[q]->data;
    return bsb::per_system_host(pent, arr, v[0]->n, v[0]->m);
  });
}
}  // namespace

BSB_API bandsolve_status bandsolve_tri_solve_per_system(bandsolve_batch* a, bandsolve_batch* b, bandsolve_batch* c,
                                                        bandsolve_batch* d) {
  bandsolve_batch* v[4] = {a, b, c, d};
  return per_system_batches(false, v);
}

BSB_API bandsolve_status bandsolve_pent_solve_per_system(bandsolve_batch* a, bandsolve_batch* b, bandsolve_batch* c,
                                                         bandsolve_batch* d, bandsolve_batch* e, bandsolve_batch* f) {
  bandsolve_batch* v[6] = {a, b, c, d, e, f};
  return per_system_batches(true, v);
}

BSB_API bandsolve_status bandsolve_tri_solve_per_system_dev(double* a, double* b, double* c, double* d, size_t n,
                                                            size_t m, size_t ld, void* stream) {
  double* arr[4] = {a, b, c, d};
  return guarded([&] { return bsb::per_system_device(false, arr, n, m, ld, stream); });
}

BSB_API bandsolve_status bandsolve_pent_solve_per_system_dev(double* a, double* b, double* c, double* d, double* e,
                                                             double* f, size_t n, size_t m, size_t ld,
                                                             void* stream) {
  double* arr[6] = {a, b, c, d, e, f};
  return guarded([&] { return bsb::per_system_device(true, arr, n, m, ld, stream); });
}

BSB_API int bandsolve_cusparse_available(void) {
  try {
    return bsb::cusparse_available() ? 1 : 0;
  } catch (...) {
    return 0;
  }
}

BSB_API bandsolve_status bandsolve_tri_solve_cusparse_dev(double* dl, double* d, double* du, double* x, size_t n,
                                                          size_t m, int algo, void* stream) {
  double* arr[3] = {dl, d, du};
  return guarded([&] { return bsb::cusparse_solve_device(false, arr, x, n, m, algo, stream); });
}

BSB_API bandsolve_status bandsolve_pent_solve_cusparse_dev(double* ds, double* dl, double* d, double* du, double* dw,
                                                           double* x, size_t n, size_t m, void* stream) {
  double* arr[5] = {ds, dl, d, du, dw};
  return guarded([&] { return bsb::cusparse_solve_device(true, arr, x, n, m, 0, stream); });
}

// ---- tridiagonal (capi.cpp:143-163) ----------------------------------------
BSB_API bandsolve_status bandsolve_tri_factor_create(const double* sub, const double* diag, const double* sup,
                                                     size_t n, bandsolve_tri_factor** out) {
  if (!sub || !diag || !sup || !out) return null_arg();
  *out = nullptr;
  return guarded([&] {
    std::unique_ptr<bsb::Factor> f;
    bandsolve_status st = bsb::make_tri_factor(sub, diag, sup, n, f);
    if (st != BANDSOLVE_OK) return st;
    *out = new bandsolve_tri_factor{std::move(f)};
    return BANDSOLVE_OK;
  });
}

BSB_API void bandsolve_tri_factor_destroy(bandsolve_tri_factor* factor) { delete factor; }

BSB_API bandsolve_status bandsolve_tri_solve_shared(const bandsolve_tri_factor* factor, bandsolve_batch* batch) {
  if (!factor || !batch) return null_arg();
  return guarded([&] { return bsb::solve_host(*factor->impl, batch->data, batch->n, batch->m); });
}

// ---- pentadiagonal (capi.cpp:174-227) ----------------------------------------
BSB_API bandsolve_status bandsolve_pent_factor_create(const double* a, const double* b, const double* c,
                                                      const double* d, const double* e, size_t n,
                                                      bandsolve_pent_factor** out) {
  if (!a || !b || !c || !d || !e || !out) return null_arg();
  *out = nullptr;
  return guarded([&] {
    std::unique_ptr<bsb::Factor> f;
    bandsolve_status st = bsb::make_pent_factor(a, b, c, d, e, n, f);
    if (st != BANDSOLVE_OK) return st;
    *out = new bandsolve_pent_factor{std::move(f)};
    return BANDSOLVE_OK;
  });
}

BSB_API void bandsolve_pent_factor_destroy(bandsolve_pent_factor* factor) { delete factor; }

BSB_API bandsolve_status bandsolve_pent_solve_shared(const bandsolve_pent_factor* factor, bandsolve_batch* batch) {
  if (!factor || !batch) return null_arg();
  return guarded([&] { return bsb::solve_host(*factor->impl, batch->data, batch->n, batch->m); });
}

BSB_API bandsolve_status bandsolve_uniform_pent_factor_create(double a, double b, double c, double d, double e,
                                                              size_t n, bandsolve_uniform_pent_factor** out) {
  if (!out) return null_arg();
  *out = nullptr;
  return guarded([&] {
    std::unique_ptr<bsb::Factor> f;
    bandsolve_status st = bsb::make_uniform_factor(a, b, c, d, e, n, f);
    if (st != BANDSOLVE_OK) return st;
    *out = new bandsolve_uniform_pent_factor{std::move(f)};
    return BANDSOLVE_OK;
  });
}

BSB_API void bandsolve_uniform_pent_factor_destroy(bandsolve_uniform_pent_factor* factor) { delete factor; }

BSB_API bandsolve_status bandsolve_pent_solve_uniform(const bandsolve_uniform_pent_factor* factor,
                                                      bandsolve_batch* batch) {
  if (!factor || !batch) return null_arg();
  return guarded([&] { return bsb::solve_host(*factor->impl, batch->data, batch->n, batch->m); });
}

// ---- periodic (capi.cpp:229-298, :414-446) -----------------------------------
BSB_API bandsolve_status bandsolve_periodic_tri_create(double a, double b, double c, size_t n,
                                                       bandsolve_periodic_tri** out) {
  if (!out) return null_arg();
  *out = nullptr;
  return guarded([&] {
    std::unique_ptr<bsb::Periodic> p;
    bandsolve_status st = bsb::make_periodic_tri(a, b, c, n, p);
    if (st != BANDSOLVE_OK) return st;
    *out = new bandsolve_periodic_tri{std::move(p)};
    return BANDSOLVE_OK;
  });
}

BSB_API void bandsolve_periodic_tri_destroy(bandsolve_periodic_tri* corr) { delete corr; }

BSB_API bandsolve_status bandsolve_periodic_tri_solve(const bandsolve_periodic_tri* corr, bandsolve_batch* batch) {
  if (!corr || !batch) return null_arg();
  return guarded([&] {
    return bsb::solve_host(*corr->impl->factor, batch->data, batch->n, batch->m, corr->impl.get(), false);
  });
}

BSB_API bandsolve_status bandsolve_periodic_tri_correct(const bandsolve_periodic_tri* corr, bandsolve_batch* batch) {
  if (!corr || !batch) return null_arg();
  return guarded([&] {
    return bsb::solve_host(*corr->impl->factor, batch->data, batch->n, batch->m, corr->impl.get(), true);
  });
}

BSB_API bandsolve_status bandsolve_periodic_tri_modified_bands(const bandsolve_periodic_tri* corr, double* sub,
                                                               double* diag, double* sup) {
  if (!corr) return null_arg();
  return guarded([&] {
    bsb::periodic_tri_modified_bands(*corr->impl, sub, diag, sup);
    return BANDSOLVE_OK;
  });
}

BSB_API bandsolve_status bandsolve_periodic_pent_create(double a, double b, double c, double d, double e, size_t n,
                                                        bandsolve_periodic_pent** out) {
  if (!out) return null_arg();
  *out = nullptr;
  return guarded([&] {
    std::unique_ptr<bsb::Periodic> p;
    bandsolve_status st = bsb::make_periodic_pent(a, b, c, d, e, n, p);
    if (st != BANDSOLVE_OK) return st;
    *out = new bandsolve_periodic_pent{std::move(p)};
    return BANDSOLVE_OK;
  });
}

BSB_API void bandsolve_periodic_pent_destroy(bandsolve_periodic_pent* corr) { delete corr; }

BSB_API bandsolve_status bandsolve_periodic_pent_solve(const bandsolve_periodic_pent* corr, bandsolve_batch* batch) {
  if (!corr || !batch) return null_arg();
  return guarded([&] {
    return bsb::solve_host(*corr->impl->factor, batch->data, batch->n, batch->m, corr->impl.get(), false);
  });
}

BSB_API bandsolve_status bandsolve_periodic_pent_correct(const bandsolve_periodic_pent* corr, bandsolve_batch* batch) {
  if (!corr || !batch) return null_arg();
  return guarded([&] {
    return bsb::solve_host(*corr->impl->factor, batch->data, batch->n, batch->m, corr->impl.get(), true);
  });
}

BSB_API bandsolve_status bandsolve_periodic_pent_modified_bands(const bandsolve_periodic_pent* corr, double* a,
                                                                double* b, double* c, double* d, double* e) {
  if (!corr) return null_arg();
  return guarded([&] {
    bsb::periodic_pent_modified_bands(*corr->impl, a, b, c, d, e);
    return BANDSOLVE_OK;
  });
}

BSB_API bandsolve_status bandsolve_periodic_tri_solve_dev(const bandsolve_periodic_tri* corr, double* x, size_t n,
                                                          size_t m, size_t ld, void* stream) {
  if (!corr) return null_arg();
  return guarded([&] { return bsb::periodic_device(*corr->impl, x, n, m, ld, stream, false); });
}
BSB_API bandsolve_status bandsolve_periodic_tri_correct_dev(const bandsolve_periodic_tri* corr, double* x, size_t n,
                                                            size_t m, size_t ld, void* stream) {
  if (!corr) return null_arg();
  return guarded([&] { return bsb::periodic_device(*corr->impl, x, n, m, ld, stream, true); });
}
BSB_API bandsolve_status bandsolve_periodic_pent_solve_dev(const bandsolve_periodic_pent* corr, double* x, size_t n,
                                                           size_t m, size_t ld, void* stream) {
  if (!corr) return null_arg();
  return guarded([&] { return bsb::periodic_device(*corr->impl, x, n, m, ld, stream, false); });
}
BSB_API bandsolve_status bandsolve_periodic_pent_correct_dev(const bandsolve_periodic_pent* corr, double* x,
                                                             size_t n, size_t m, size_t ld, void* stream) {
  if (!corr) return null_arg();
  return guarded([&] { return bsb::periodic_device(*corr->impl, x, n, m, ld, stream, true); });
}

// ---- Crank-Nicolson (capi.cpp:300-411) ------------------------------------------
BSB_API bandsolve_status bandsolve_footprint(bandsolve_storage_variant variant, size_t n, size_t m,
                                             uint64_t* elements, double* reduction_vs_baseline) {
  // capi.cpp:300-325 -> batch.cpp:72-105: the variant is checked first, then
  // the shape; either out-parameter may be NULL (only the non-NULL ones are written)
  uint64_t count = 0, baseline = 0;
  const uint64_t un = n, um = m;
  switch (variant) {
    case BANDSOLVE_STORAGE_TRI_PER_SYSTEM: count = baseline = 4 * um * un; break;
    case BANDSOLVE_STORAGE_TRI_SHARED: count = 3 * un + un * um; baseline = 4 * um * un; break;
    case BANDSOLVE_STORAGE_PENT_PER_SYSTEM: count = baseline = 6 * um * un; break;
    case BANDSOLVE_STORAGE_PENT_SHARED: count = 5 * un + un * um; baseline = 6 * um * un; break;
    case BANDSOLVE_STORAGE_PENT_UNIFORM: count = 4 * un + un * um; baseline = 6 * um * un; break;
    default: return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "unknown storage variant");
  }
  if (n < 2 || m < 1) return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "footprint needs n >= 2, m >= 1");
  if (elements) *elements = count;
  if (reduction_vs_baseline)
    *reduction_vs_baseline = 1.0 - static_cast<double>(count) / static_cast<double>(baseline);
  return BANDSOLVE_OK;
}

BSB_API bandsolve_status bandsolve_bench_run(const bandsolve_bench_params* params, bandsolve_bench_result* result) {
  if (!params || !result) return null_arg();
  return guarded([&] { return bsb::bench_run_device(*params, result, bandsolve_get_threads()); });
}

BSB_API bandsolve_status bandsolve_periodic_tri_cn_step_dev(const bandsolve_periodic_tri* lhs, double sigma_x,
                                                            const double* u, double* out, size_t n, size_t m,
                                                            size_t ld, void* stream) {
  if (!lhs) return null_arg();
  return guarded([&] { return bsb::cn_step_device(*lhs->impl, sigma_x, u, out, n, m, ld, stream); });
}

BSB_API bandsolve_status bandsolve_periodic_pent_cn_step_dev(const bandsolve_periodic_pent* lhs, double sigma_x,
                                                             const double* u, double* out, size_t n, size_t m,
                                                             size_t ld, void* stream) {
  if (!lhs) return null_arg();
  return guarded([&] { return bsb::cn_step_device(*lhs->impl, sigma_x, u, out, n, m, ld, stream); });
}

// ---- 2D ADI (B200 extension; BASELINE configs[3]) -----------------------------
BSB_API bandsolve_status bandsolve_adi_create(int problem, double sigma_x, size_t nx, size_t ny, bandsolve_adi** out) {
  if (!out) return null_arg();
  *out = nullptr;
  if (problem != BANDSOLVE_PROBLEM_DIFFUSION && problem != BANDSOLVE_PROBLEM_HYPERDIFFUSION)
    return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "unknown problem");
  if (!(sigma_x > 0.0)) return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "sigma_x must be positive");
  return guarded([&] {
    auto h = std::make_unique<bandsolve_adi>();
    h->problem = problem;
    h->sigma = sigma_x;
    h->nx = nx;
    h->ny = ny;
    const double s = sigma_x;
    for (int axis = 0; axis < 2; ++axis) {
      const std::size_t n = axis == 0 ? nx : ny;
      std::unique_ptr<bsb::Periodic>& p = axis == 0 ? h->px : h->py;
      // pde.cpp:59-71: diffusion (-s, 1+2s, -s), hyperdiffusion (s, -4s, 1+6s, -4s, s)
      bandsolve_status st = problem == BANDSOLVE_PROBLEM_DIFFUSION
                                ? bsb::make_periodic_tri(-s, 1.0 + 2.0 * s, -s, n, p)
                                : bsb::make_periodic_pent(s, -4.0 * s, 1.0 + 6.0 * s, -4.0 * s, s, n, p);
      if (st != BANDSOLVE_OK) return st;
    }
    *out = h.release();
    return BANDSOLVE_OK;
  });
}

BSB_API void bandsolve_adi_destroy(bandsolve_adi* adi) { delete adi; }

BSB_API bandsolve_status bandsolve_adi_step_dev(const bandsolve_adi* adi, double* field, double* work, size_t ld,
                                                void* stream) {
  if (!adi) return null_arg();
  return guarded([&] {
    return bsb::adi_step_device(*adi->px, *adi->py, adi->sigma, field, work, adi->nx, adi->ny, ld, stream);
  });
}

// ---- residuals (capi.cpp:327-367) ----------------------------------------------
namespace {

bandsolve_status tri_residual_checks(const double* sub, const double* diag, const double* sup, size_t n,
                                     int cyclic, size_t rows) {
  if (cyclic) {
    if (n < 3) return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "cyclic residual needs n >= 3");
    // constant_tri_lhs (banded.cpp:59-65) validates the expanded bands
    const double v[3] = {sub[1], diag[0], sup[0]};
    for (double x : v)
      if (!std::isfinite(x)) return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "non-finite band value");
  } else {
    bandsolve_status st = bsb::validate_tri_bands(sub, diag, sup, n);
    if (st != BANDSOLVE_OK) return st;
  }
  if (rows != n) return bsb::fail(BANDSOLVE_ERR_SHAPE_MISMATCH, "residual shapes disagree");
  return BANDSOLVE_OK;
}

bandsolve_status pent_residual_checks(const double* const* bands, size_t n, int cyclic, size_t rows) {
  if (cyclic) {
    if (n < 6) return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "cyclic residual needs n >= 6");
    const double v[5] = {bands[0][2], bands[1][1], bands[2][0], bands[3][0], bands[4][0]};
    for (double x : v)
      if (!std::isfinite(x)) return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "non-finite band value");
  } else {
    bandsolve_status st = bsb::validate_pent_bands(bands[0], bands[1], bands[2], bands[3], bands[4], n);
    if (st != BANDSOLVE_OK) return st;
  }
  if (rows != n) return bsb::fail(BANDSOLVE_ERR_SHAPE_MISMATCH, "residual shapes disagree");
  return BANDSOLVE_OK;
}

}  // namespace

BSB_API bandsolve_status bandsolve_tri_residual(const double* sub, const double* diag, const double* sup, size_t n,
                                                int cyclic, const bandsolve_batch* x, const bandsolve_batch* rhs,
                                                double* out) {
  if (!sub || !diag || !sup || !x || !rhs || !out) return null_arg();
  return guarded([&] {
    if (x->n != rhs->n || x->m != rhs->m) return bsb::fail(BANDSOLVE_ERR_SHAPE_MISMATCH, "residual shapes disagree");
    bandsolve_status st = tri_residual_checks(sub, diag, sup, n, cyclic, x->n);
    if (st != BANDSOLVE_OK) return st;
    const double* bands[3] = {sub, diag, sup};
    return bsb::residual_host(bsb::Kind::Tri, bands, n, cyclic, x->data, rhs->data, x->m, out);
  });
}

BSB_API bandsolve_status bandsolve_pent_residual(const double* a, const double* b, const double* c, const double* d,
                                                 const double* e, size_t n, int cyclic, const bandsolve_batch* x,
                                                 const bandsolve_batch* rhs, double* out) {
  if (!a || !b || !c || !d || !e || !x || !rhs || !out) return null_arg();
  return guarded([&] {
    if (x->n != rhs->n || x->m != rhs->m) return bsb::fail(BANDSOLVE_ERR_SHAPE_MISMATCH, "residual shapes disagree");
    const double* bands[5] = {a, b, c, d, e};
    bandsolve_status st = pent_residual_checks(bands, n, cyclic, x->n);
    if (st != BANDSOLVE_OK) return st;
    return bsb::residual_host(bsb::Kind::Pent, bands, n, cyclic, x->data, rhs->data, x->m, out);
  });
}

// ---- B200 extensions -----------------------------------------------------------
BSB_API bandsolve_status bandsolve_set_mode(int mode) {
  if (mode != BANDSOLVE_MODE_EXACT && mode != BANDSOLVE_MODE_FAST)
    return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "unknown mode");
  bsb::set_mode(mode);
  return BANDSOLVE_OK;
}
BSB_API int bandsolve_get_mode(void) { return bsb::current_mode(); }

#define BSB_DEV_SOLVE(NAME, HANDLE, PTR_T, F32)                                                          \
  BSB_API bandsolve_status NAME(const HANDLE* factor, PTR_T* x, size_t n, size_t m, size_t ld, void* stream) { \
    if (!factor) return null_arg();                                                                      \
    return guarded([&] { return bsb::solve_device(*factor->impl, x, F32, n, m, ld, stream); });          \
  }
BSB_DEV_SOLVE(bandsolve_tri_solve_shared_dev, bandsolve_tri_factor, double, false)
BSB_DEV_SOLVE(bandsolve_tri_solve_shared_dev_f32, bandsolve_tri_factor, float, true)
BSB_DEV_SOLVE(bandsolve_pent_solve_shared_dev, bandsolve_pent_factor, double, false)
BSB_DEV_SOLVE(bandsolve_pent_solve_shared_dev_f32, bandsolve_pent_factor, float, true)
BSB_DEV_SOLVE(bandsolve_pent_solve_uniform_dev, bandsolve_uniform_pent_factor, double, false)
BSB_DEV_SOLVE(bandsolve_pent_solve_uniform_dev_f32, bandsolve_uniform_pent_factor, float, true)
#undef BSB_DEV_SOLVE

BSB_API bandsolve_status bandsolve_tri_residual_dev(const double* sub, const double* diag, const double* sup,
                                                    size_t n, int cyclic, const double* x, const double* rhs,
                                                    size_t m, size_t ld, void* stream, double* out) {
  if (!sub || !diag || !sup || !x || !rhs || !out) return null_arg();
  return guarded([&] {
    bandsolve_status st = tri_residual_checks(sub, diag, sup, n, cyclic, n);
    if (st != BANDSOLVE_OK) return st;
    const double* bands[3] = {sub, diag, sup};
    return bsb::residual_device(bsb::Kind::Tri, bands, n, cyclic, x, rhs, m, ld, stream, out);
  });
}

BSB_API bandsolve_status bandsolve_pent_residual_dev(const double* a, const double* b, const double* c,
                                                     const double* d, const double* e, size_t n, int cyclic,
                                                     const double* x, const double* rhs, size_t m, size_t ld,
                                                     void* stream, double* out) {
  if (!a || !b || !c || !d || !e || !x || !rhs || !out) return null_arg();
  return guarded([&] {
    const double* bands[5] = {a, b, c, d, e};
    bandsolve_status st = pent_residual_checks(bands, n, cyclic, n);
    if (st != BANDSOLVE_OK) return st;
    return bsb::residual_device(bsb::Kind::Pent, bands, n, cyclic, x, rhs, m, ld, stream, out);
  });
}

BSB_API bandsolve_status bandsolve_fill_rhs_dev(double* x, size_t n, size_t m, size_t ld, uint64_t seed,
                                                uint64_t j_offset, void* stream) {
  return guarded([&] { return bsb::fill_rhs_device(x, false, n, m, ld, seed, j_offset, stream); });
}
BSB_API bandsolve_status bandsolve_fill_rhs_dev_f32(float* x, size_t n, size_t m, size_t ld, uint64_t seed,
                                                    uint64_t j_offset, void* stream) {
  return guarded([&] { return bsb::fill_rhs_device(x, true, n, m, ld, seed, j_offset, stream); });
}

namespace {
void copy_opt(double* dst, const std::vector<double>& src) {
  if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(double));
}
}  // namespace

BSB_API size_t bandsolve_tri_factor_order(const bandsolve_tri_factor* f) { return f ? f->impl->n : 0; }
BSB_API bandsolve_status bandsolve_tri_factor_arrays(const bandsolve_tri_factor* f, double* chat, double* inv_denom,
                                                     double* sub) {
  if (!f) return null_arg();
  copy_opt(chat, f->impl->chat);
  copy_opt(inv_denom, f->impl->inv_denom);
  copy_opt(sub, f->impl->sub);
  return BANDSOLVE_OK;
}
BSB_API size_t bandsolve_pent_factor_order(const bandsolve_pent_factor* f) { return f ? f->impl->n : 0; }
BSB_API bandsolve_status bandsolve_pent_factor_arrays(const bandsolve_pent_factor* f, double* inv_alpha,
                                                      double* beta, double* gamma, double* delta, double* epsilon) {
  if (!f) return null_arg();
  copy_opt(inv_alpha, f->impl->inv_alpha);
  copy_opt(beta, f->impl->beta);
  copy_opt(gamma, f->impl->gamma);
  copy_opt(delta, f->impl->delta);
  copy_opt(epsilon, f->impl->epsilon);
  return BANDSOLVE_OK;
}
BSB_API size_t bandsolve_uniform_pent_factor_order(const bandsolve_uniform_pent_factor* f) {
  return f ? f->impl->n : 0;
}
BSB_API bandsolve_status bandsolve_uniform_pent_factor_arrays(const bandsolve_uniform_pent_factor* f,
                                                              double* inv_alpha, double* beta, double* gamma,
                                                              double* delta, double* eps_scalar) {
  if (!f) return null_arg();
  copy_opt(inv_alpha, f->impl->inv_alpha);
  copy_opt(beta, f->impl->beta);
  copy_opt(gamma, f->impl->gamma);
  copy_opt(delta, f->impl->delta);
  if (eps_scalar) *eps_scalar = f->impl->eps_scalar;
  return BANDSOLVE_OK;
}

BSB_API bandsolve_status bandsolve_describe_plan(int kind, size_t n, size_t m, size_t ld, int f32, char* buf,
                                                 size_t buflen) {
  if (!buf || buflen == 0) return null_arg();
  if (kind < 0 || kind > 2) return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "unknown kind");
  return guarded([&] {
    std::string s;
    bandsolve_status st = bsb::describe_plan(static_cast<bsb::Kind>(kind), n, m, ld, f32 != 0, s);
    std::strncpy(buf, s.c_str(), buflen - 1);
    buf[buflen - 1] = '\0';
    return st;
  });
}

BSB_API bandsolve_status bandsolve_set_devices(const int* devices, int count) {
  return guarded([&] { return bsb::set_devices(devices, count); });
}

BSB_API int bandsolve_get_devices(int* devices, int capacity) { return bsb::get_devices(devices, capacity); }

BSB_API bandsolve_status bandsolve_tune_set(const char* key, const char* value) {
  if (!key) return null_arg();
  if (!bsb::tune_set(key, value)) return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "unknown tuning key");
  return BANDSOLVE_OK;
}

BSB_API bandsolve_status bandsolve_tune_get(const char* key, char* buf, size_t buflen) {
  if (!key || !buf || buflen == 0) return null_arg();
  const auto v = bsb::tune_str(key);
  if (!v) return bsb::fail(BANDSOLVE_ERR_BAD_ARG, "tuning key not set");
  std::strncpy(buf, v->c_str(), buflen - 1);
  buf[buflen - 1] = '\0';
  return BANDSOLVE_OK;
}

BSB_API void bandsolve_tune_reset(void) { bsb::tune_reset(); }

BSB_API uint64_t bandsolve_kernel_launches(void) { return bsb::kernel_launches(); }

BSB_API const char* bandsolve_last_error(void) { return bsb::last_error(); }
