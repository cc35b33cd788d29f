// cuSPARSE comparators: the library batch solvers the
// paper measures its constant-LHS kernels against — cuThomasBatch is
// cusparseDgtsvInterleavedBatch ("Speedup of
// cuThomasConstantBatch versus cuThomasBatch (gtsvInterleavedBatch)"), and
// the pentadiagonal counterpart is cusparseDgpsvInterleavedBatch. Both take
// one band copy per system in the interleaved layout (element (i, j) at
// i*m + j, no pitch argument) and overwrite the right-hand side with x.
//
// The library is resolved with dlopen at first use, so libbandsolve_b200.so
// has no load-time dependency on cuSPARSE; without it the comparator entry
// points return BANDSOLVE_ERR_INTERNAL. This is a measurement baseline, not a
// product path: no shared-LHS solve ever routes through it.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "internal.hpp"

namespace bsb {
bandsolve_status cuda_fail(cudaError_t err, const char* what);        // solve.cu
cudaError_t pool_malloc_async_raw(void** p, std::size_t bytes, cudaStream_t s);  // solve.cu
int device_count_cached();                                             // solve.cu

namespace {

// the slice of cusparse.h the comparators use (ABI of libcusparse.so.12)
using Handle = void*;
using Status = int;
using FnCreate = Status (*)(Handle*);
using FnDestroy = Status (*)(Handle);
using FnSetStream = Status (*)(Handle, cudaStream_t);
using FnGtsvBuf = Status (*)(Handle, int, int, const double*, const double*, const double*, const double*, int,
                             std::size_t*);
using FnGtsv = Status (*)(Handle, int, int, double*, double*, double*, double*, int, void*);
using FnGpsvBuf = Status (*)(Handle, int, int, const double*, const double*, const double*, const double*,
                             const double*, const double*, int, std::size_t*);
using FnGpsv = Status (*)(Handle, int, int, double*, double*, double*, double*, double*, double*, int, void*);

struct Api {
  bool tried = false;
  void* so = nullptr;
  FnCreate create = nullptr;
  FnDestroy destroy = nullptr;
  FnSetStream set_stream = nullptr;
  FnGtsvBuf gtsv_buf = nullptr;
  FnGtsv gtsv = nullptr;
  FnGpsvBuf gpsv_buf = nullptr;
  FnGpsv gpsv = nullptr;
  std::string why;
};

Api& api() {
  static Api a;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (a.tried) return a;
  a.tried = true;
  for (const char* name : {"libcusparse.so.12", "libcusparse.so"}) {
    a.so = dlopen(name, RTLD_NOW | RTLD_LOCAL);
    if (a.so) break;
  }
  if (!a.so) {
    a.why = "libcusparse.so.12 not found";
    return a;
  }
  auto sym = [&](const char* s) { return dlsym(a.so, s); };
  a.create = reinterpret_cast<FnCreate>(sym("cusparseCreate"));
  a.destroy = reinterpret_cast<FnDestroy>(sym("cusparseDestroy"));
  a.set_stream = reinterpret_cast<FnSetStream>(sym("cusparseSetStream"));
  a.gtsv_buf = reinterpret_cast<FnGtsvBuf>(sym("cusparseDgtsvInterleavedBatch_bufferSizeExt"));
  a.gtsv = reinterpret_cast<FnGtsv>(sym("cusparseDgtsvInterleavedBatch"));
  a.gpsv_buf = reinterpret_cast<FnGpsvBuf>(sym("cusparseDgpsvInterleavedBatch_bufferSizeExt"));
  a.gpsv = reinterpret_cast<FnGpsv>(sym("cusparseDgpsvInterleavedBatch"));
  if (!a.create || !a.destroy || !a.set_stream || !a.gtsv_buf || !a.gtsv || !a.gpsv_buf || !a.gpsv) {
    a.why = "libcusparse.so.12 lacks the interleaved batch solvers";
    dlclose(a.so);
    a.so = nullptr;
  }
  return a;
}

// one handle per (thread, device); handles are not thread-safe to share
struct ThreadHandles {
  Handle h[64] = {};
  ~ThreadHandles() {
    Api& a = api();
    if (!a.so) return;
    for (Handle x : h)
      if (x) a.destroy(x);
  }
};

bandsolve_status handle_for(int device, Handle* out) {
  thread_local ThreadHandles th;
  if (device < 0 || device >= 64) return fail(BANDSOLVE_ERR_INTERNAL, "device id out of range");
  if (!th.h[device]) {
    if (api().create(&th.h[device]) != 0) {
      th.h[device] = nullptr;
      return fail(BANDSOLVE_ERR_INTERNAL, "cusparseCreate failed");
    }
  }
  *out = th.h[device];
  return BANDSOLVE_OK;
}

}  // namespace

bool cusparse_available() { return api().so != nullptr; }

// bands: dl, d, du (tri) / ds, dl, d, du, dw (pent), each n x m interleaved
// (pitch m), device memory; x: n x m right-hand sides, overwritten with the
// solution. algo: gtsv 0 = Thomas (cuThomasBatch), 1 = LU with pivoting,
// 2 = QR; gpsv 0 = QR (the only algorithm cuSPARSE offers). Stream-ordered.
bandsolve_status cusparse_solve_device(bool pent, double* const* bands, double* x, std::size_t n, std::size_t m,
                                       int algo, void* stream) {
  if (!x) return fail(BANDSOLVE_ERR_BAD_ARG, "null device pointer");
  for (int b = 0; b < (pent ? 5 : 3); ++b)
    if (!bands[b]) return fail(BANDSOLVE_ERR_BAD_ARG, "null device pointer");
  if (n < (pent ? 5u : 2u)) return fail(BANDSOLVE_ERR_BAD_ARG, pent ? "pentadiagonal system needs n >= 5"
                                                                     : "tridiagonal system needs n >= 2");
  if (m == 0) return BANDSOLVE_OK;
  if (n > 0x7fffffffu || m > 0x7fffffffu) return fail(BANDSOLVE_ERR_BAD_ARG, "shape beyond cuSPARSE's int sizes");
  if (pent ? algo != 0 : (algo < 0 || algo > 2)) return fail(BANDSOLVE_ERR_BAD_ARG, "unknown cuSPARSE algorithm");
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  Api& a = api();
  if (!a.so) return fail(BANDSOLVE_ERR_INTERNAL, a.why);
  int device = 0;
  if (cudaError_t e = cudaGetDevice(&device); e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  Handle h = nullptr;
  if (bandsolve_status st = handle_for(device, &h); st != BANDSOLVE_OK) return st;
  auto s = static_cast<cudaStream_t>(stream);
  if (a.set_stream(h, s) != 0) return fail(BANDSOLVE_ERR_INTERNAL, "cusparseSetStream failed");
  const int ni = static_cast<int>(n), mi = static_cast<int>(m);
  std::size_t bytes = 0;
  Status cs = pent ? a.gpsv_buf(h, algo, ni, bands[0], bands[1], bands[2], bands[3], bands[4], x, mi, &bytes)
                   : a.gtsv_buf(h, algo, ni, bands[0], bands[1], bands[2], x, mi, &bytes);
  if (cs != 0) return fail(BANDSOLVE_ERR_INTERNAL, "cuSPARSE bufferSizeExt failed (status " + std::to_string(cs) + ")");
  void* work = nullptr;
  if (bytes) {
    if (cudaError_t e = pool_malloc_async_raw(&work, bytes, s); e != cudaSuccess) return cuda_fail(e, "cuSPARSE workspace");
  }
  cs = pent ? a.gpsv(h, algo, ni, bands[0], bands[1], bands[2], bands[3], bands[4], x, mi, work)
            : a.gtsv(h, algo, ni, bands[0], bands[1], bands[2], x, mi, work);
  if (work) cudaFreeAsync(work, s);
  if (cs != 0) return fail(BANDSOLVE_ERR_INTERNAL, "cuSPARSE interleaved batch solve failed (status " +
                                                       std::to_string(cs) + ")");
  if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return cuda_fail(e, "cuSPARSE solve");
  return BANDSOLVE_OK;
}

}  // namespace bsb
