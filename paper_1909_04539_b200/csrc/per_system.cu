// Per-system baselines (one band copy per system; the paper's cuThomasBatch /
// cuPentBatch comparators): reference
// tri_solver.cpp:51-112 and pent_solver.cpp:131-219.
//
// Thread per system, interleaved (row i of system j at i*ld + j, coalesced
// across the warp), the reference's fused destructive factor + solve in its
// operation order with separately rounded operations (__dmul_rn/__dsub_rn/
// __ddiv_rn: nvcc cannot contract them), so every array the reference
// overwrites ends bitwise equal to the reference's. These kernels read and
// write 4 (tri) / 6 (pent) n x m arrays: they are the baseline the shared-LHS
// sweep is measured against, not a hot path.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>

#include "internal.hpp"
#include "sweep_kernels.cuh"

namespace bsb {
bandsolve_status cuda_fail(cudaError_t err, const char* what);  // solve.cu
int device_count_cached();                                     // solve.cu

#define BSB_CUDA(call)                                          \
  do {                                                          \
    cudaError_t err_ = (call);                                  \
    if (err_ != cudaSuccess) return cuda_fail(err_, #call);     \
  } while (0)

namespace {

using dev::add_rn;
using dev::mul_rn;
using dev::sub_rn;
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ bool pivot_ok(double v) { return fabs(v) >= kBreakdownEps; }

__global__ void tri_per_system_kernel(const double* __restrict__ pa, double* __restrict__ pb, double* __restrict__ pc,
                                      double* __restrict__ pd, int n, long long m, long long ld, int* broke) {
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  auto at = [&](int i) { return static_cast<long long>(i) * ld + j; };
  // tri_solver.cpp:71-96: reciprocals over b, chat over c, dhat over d
  double denom = pb[at(0)];
  if (!pivot_ok(denom)) {
    atomicExch(broke, 1);
    return;
  }
  double r = div_rn(1.0, denom);
  pb[at(0)] = r;
  double cg = mul_rn(pc[at(0)], r);
  pc[at(0)] = cg;
  double dg = mul_rn(pd[at(0)], r);
  pd[at(0)] = dg;
  for (int i = 1; i < n; ++i) {
    const long long k = at(i);
    const double a = pa[k];
    denom = sub_rn(pb[k], mul_rn(a, cg));
    if (!pivot_ok(denom)) {
      atomicExch(broke, 1);
      return;
    }
    r = div_rn(1.0, denom);
    pb[k] = r;
    cg = mul_rn(pc[k], r);
    pc[k] = cg;
    dg = mul_rn(sub_rn(pd[k], mul_rn(a, dg)), r);
    pd[k] = dg;
  }
  // tri_solver.cpp:99-105: backward in place over d
  double xnext = dg;
  for (int i = n - 2; i >= 0; --i) {
    const long long k = at(i);
    xnext = sub_rn(pd[k], mul_rn(pc[k], xnext));
    pd[k] = xnext;
  }
}

__global__ void pent_per_system_kernel(const double* __restrict__ pa, double* __restrict__ pb, double* __restrict__ pc,
                                       double* __restrict__ pd, double* __restrict__ pe, double* __restrict__ pf,
                                       int n, long long m, long long ld, int* broke) {
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  auto at = [&](int i) { return static_cast<long long>(i) * ld + j; };
  // pent_solver.cpp:156-196: beta over b, alpha over c, gamma over d, delta over e
  double alpha = pc[at(0)];
  if (!pivot_ok(alpha)) {
    atomicExch(broke, 1);
    return;
  }
  double d_prev2 = div_rn(pd[at(0)], alpha);  // gamma_0
  double e_prev2 = div_rn(pe[at(0)], alpha);  // delta_0
  pd[at(0)] = d_prev2;
  pe[at(0)] = e_prev2;
  const double b1 = pb[at(1)];
  alpha = sub_rn(pc[at(1)], mul_rn(b1, d_prev2));
  if (!pivot_ok(alpha)) {
    atomicExch(broke, 1);
    return;
  }
  pc[at(1)] = alpha;
  double d_prev1 = div_rn(sub_rn(pd[at(1)], mul_rn(b1, e_prev2)), alpha);
  double e_prev1 = div_rn(pe[at(1)], alpha);
  pd[at(1)] = d_prev1;
  pe[at(1)] = e_prev1;
  for (int i = 2; i < n; ++i) {
    const long long k = at(i);
    const double a = pa[k];
    const double beta = sub_rn(pb[k], mul_rn(a, d_prev2));
    pb[k] = beta;
    alpha = sub_rn(sub_rn(pc[k], mul_rn(a, e_prev2)), mul_rn(beta, d_prev1));
    if (!pivot_ok(alpha)) {
      atomicExch(broke, 1);
      return;
    }
    pc[k] = alpha;
    double dn = 0.0, en = 0.0;
    if (i + 1 < n) {  // rows n-2 (gamma only) and n-1 (neither) per :182-196
      dn = div_rn(sub_rn(pd[k], mul_rn(beta, e_prev1)), alpha);
      pd[k] = dn;
      if (i + 2 < n) {
        en = div_rn(pe[k], alpha);
        pe[k] = en;
      }
    }
    d_prev2 = d_prev1;
    e_prev2 = e_prev1;
    d_prev1 = dn;
    e_prev1 = en;
  }
  // pent_solver.cpp:199-206: g over f
  double g2 = div_rn(pf[at(0)], pc[at(0)]);
  pf[at(0)] = g2;
  double g1 = div_rn(sub_rn(pf[at(1)], mul_rn(pb[at(1)], g2)), pc[at(1)]);
  pf[at(1)] = g1;
  for (int i = 2; i < n; ++i) {
    const long long k = at(i);
    const double g = div_rn(sub_rn(sub_rn(pf[k], mul_rn(pa[k], g2)), mul_rn(pb[k], g1)), pc[k]);
    pf[k] = g;
    g2 = g1;
    g1 = g;
  }
  // :208-211: x over g
  double x1 = g1;                                                     // x_{n-1}
  double x0 = sub_rn(pf[at(n - 2)], mul_rn(pd[at(n - 2)], x1));  // x_{n-2}
  pf[at(n - 2)] = x0;
  for (int i = n - 3; i >= 0; --i) {
    const long long k = at(i);
    const double x = sub_rn(pf[k], add_rn(mul_rn(pd[k], x0), mul_rn(pe[k], x1)));
    pf[k] = x;
    x1 = x0;
    x0 = x;
  }
}

}  // namespace

bandsolve_status per_system_device(bool pent, double* const* arr, std::size_t n, std::size_t m, std::size_t ld,
                                   void* stream) {
  if (n < (pent ? 5u : 2u))
    return fail(BANDSOLVE_ERR_BAD_ARG, pent ? "pentadiagonal system needs n >= 5" : "tridiagonal system needs n >= 2");
  if (ld < m) return fail(BANDSOLVE_ERR_BAD_ARG, "row pitch ld < m");
  if (n > static_cast<std::size_t>(INT_MAX)) return fail(BANDSOLVE_ERR_BAD_ARG, "n too large");
  for (int q = 0; q < (pent ? 6 : 4); ++q)
    if (!arr[q]) return fail(BANDSOLVE_ERR_BAD_ARG, "null device pointer");
  if (m == 0) return BANDSOLVE_OK;
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  auto s = static_cast<cudaStream_t>(stream);
  int* flag = nullptr;
  BSB_CUDA(pool_malloc_async(reinterpret_cast<void**>(&flag), sizeof(int), s));
  cudaMemsetAsync(flag, 0, sizeof(int), s);
  const unsigned grid = static_cast<unsigned>((m + 127) / 128);
  if (pent)
    pent_per_system_kernel<<<grid, 128, 0, s>>>(arr[0], arr[1], arr[2], arr[3], arr[4], arr[5], static_cast<int>(n),
                                                static_cast<long long>(m), static_cast<long long>(ld), flag);
  else
    tri_per_system_kernel<<<grid, 128, 0, s>>>(arr[0], arr[1], arr[2], arr[3], static_cast<int>(n),
                                               static_cast<long long>(m), static_cast<long long>(ld), flag);
  note_launches(1);
  int broke = 0;
  cudaError_t err = cudaGetLastError();
  if (err == cudaSuccess) err = cudaMemcpyAsync(&broke, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(flag, s);
  if (err == cudaSuccess) err = cudaStreamSynchronize(s);
  if (err != cudaSuccess) return cuda_fail(err, "per-system solve");
  if (broke)
    return fail(BANDSOLVE_ERR_FACTORIZATION_BREAKDOWN,
                pent ? "zero alpha in per-system elimination; outputs are unspecified"
                     : "zero pivot in per-system elimination; outputs are unspecified");
  return BANDSOLVE_OK;
}

bandsolve_status per_system_host(bool pent, double* const* arr, std::size_t n, std::size_t m) {
  if (n < (pent ? 5u : 2u))
    return fail(BANDSOLVE_ERR_BAD_ARG, pent ? "pentadiagonal system needs n >= 5" : "tridiagonal system needs n >= 2");
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  const int na = pent ? 6 : 4;
  // column chunks bounded to ~4 GiB of device arrays; strided 2D copies
  const std::size_t row_bytes = n * sizeof(double) * na;
  const std::size_t w = std::max<std::size_t>(1, std::min(m, (std::size_t(4) << 30) / row_bytes));
  double* dv[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  cudaError_t err = cudaSuccess;
  for (int q = 0; q < na && err == cudaSuccess; ++q) err = cudaMalloc(&dv[q], n * w * sizeof(double));
  bandsolve_status st = BANDSOLVE_OK;
  for (std::size_t j0 = 0; j0 < m && err == cudaSuccess && st == BANDSOLVE_OK; j0 += w) {
    const std::size_t cw = std::min(w, m - j0);
    for (int q = 0; q < na && err == cudaSuccess; ++q)
      err = cudaMemcpy2D(dv[q], cw * sizeof(double), arr[q] + j0, m * sizeof(double), cw * sizeof(double), n,
                         cudaMemcpyHostToDevice);
    if (err != cudaSuccess) break;
    st = per_system_device(pent, dv, n, cw, cw, nullptr);
    // the reference overwrites every band but a; copy them back even on breakdown
    for (int q = 1; q < na && err == cudaSuccess; ++q)
      err = cudaMemcpy2D(arr[q] + j0, m * sizeof(double), dv[q], cw * sizeof(double), cw * sizeof(double), n,
                         cudaMemcpyDeviceToHost);
  }
  for (int q = 0; q < na; ++q)
    if (dv[q]) cudaFree(dv[q]);
  if (err != cudaSuccess) return cuda_fail(err, "per-system staging");
  return st;
}

}  // namespace bsb
