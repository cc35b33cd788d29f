// Partitioned (SPIKE-style) shared-LHS solve for few long systems, fast mode.
//
// With one thread per system, a batch of m systems keeps only m dependent
// chains in flight: for m below ~one warp per SM (configs[0]: 4096 systems;
// the ADI axes: 4096 systems of 4096 rows) the sweep is latency-bound far
// from the HBM roofline. Because the LHS is shared, the partition method's
// expensive parts are per-matrix, not per-system, and are computed once on
// the host:
//
//   A = diag(A_0 .. A_{K-1}) + couplings between adjacent blocks of L rows.
//   Per block k: y_k = A_k^-1 b_k (block factors: one record per row, the
//   same packed fast records as the full sweep), and spikes W_k / V_k =
//   A_k^-1 (coupling columns) (tri: 2, pent: 4 vectors of n).
//   x_k = y_k - W_k x_(left interface) - V_k x_(right interface), so the 2K
//   (tri) / 4K (pent) interface unknowns satisfy one dense R x R system whose
//   matrix is shared: its LU (partial pivoting) is precomputed.
//
// Device passes (4 HBM passes over the batch, like an off-chip sequential
// sweep): (A) K*m independent block forward sweeps (thread per block-system,
// deep register prefetch) that also emit the block's interface values of y =
// A_k^-1 b_k -- the bottom ones are forward values, the top ones dot products
// of the forward values with precomputed rows of the block's U^-1; (B) per
// system, the R x R interface solve (LU in smem, banded loops); (C) K*m block
// backward sweeps that start from the block's own solved bottom values and
// fold the left-neighbour coupling in as g_i - F_i x_left (F = the forward
// image of the coupling column). Arithmetic differs from the sequential sweep
// by rounding only (fast mode, 1e-12).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstring>
#include <vector>

#include "internal.hpp"
#include "sweep_kernels.cuh"

namespace bsb {

struct PartPlan {
  int K = 0, R = 0, L = 0;
  bool pent = false;
  std::vector<int> start;                  // K + 1 block starts (block K-1 absorbs n % K)
  std::vector<double> fwd, bwd;            // packed fast records, one per row (block-local factors)
  std::vector<double> fl;                  // forward images of the left coupling (tri: F, pent: F1 | F2)
  std::vector<double> pr;                  // rows of the block U^-1 (tri: P0, pent: P0 | P1)
  std::vector<double> lu;                  // R x R, row-major, L unit-lower + U
  std::vector<int> perm;                   // row permutation of the LU | row lo | row hi
  std::vector<std::pair<int, void*>> dev;  // device blobs
  ~PartPlan() {
    for (auto& d : dev) {
      int prev = -1;
      if (cudaGetDevice(&prev) == cudaSuccess && prev != d.first) cudaSetDevice(d.first);
      cudaFree(d.second);
      if (prev >= 0 && prev != d.first) cudaSetDevice(prev);
    }
    cudaGetLastError();
  }
};
void PartPlanDeleter::operator()(PartPlan* p) const { delete p; }

namespace {

constexpr int kPartMaxR = 64;  // reduced-system order cap: the LU (32 KB) lives in smem

// block factor forward / backward (any rounding: fast path), in place
void tri_block_fwd(const Factor& f, double* v) {
  v[0] *= f.inv_denom[0];
  for (std::size_t i = 1; i < f.n; ++i) v[i] = (v[i] - f.sub[i] * v[i - 1]) * f.inv_denom[i];
}
void tri_block_bwd(const Factor& f, double* v) {
  for (std::size_t i = f.n - 1; i-- > 0;) v[i] -= f.chat[i] * v[i + 1];
}
void pent_block_fwd(const Factor& f, double* v) {
  v[0] *= f.inv_alpha[0];
  v[1] = (v[1] - f.beta[1] * v[0]) * f.inv_alpha[1];
  for (std::size_t i = 2; i < f.n; ++i) v[i] = (v[i] - f.epsilon[i] * v[i - 2] - f.beta[i] * v[i - 1]) * f.inv_alpha[i];
}
void pent_block_bwd(const Factor& f, double* v) {
  const std::size_t n = f.n;
  v[n - 2] -= f.gamma[n - 2] * v[n - 1];
  for (std::size_t i = n - 2; i-- > 0;) v[i] -= f.gamma[i] * v[i + 1] + f.delta[i] * v[i + 2];
}

// dense LU with partial pivoting, in place; false when singular
bool lu_factor(std::vector<double>& a, std::vector<int>& perm, int r) {
  perm.resize(r);
  for (int i = 0; i < r; ++i) perm[i] = i;
  for (int k = 0; k < r; ++k) {
    int p = k;
    for (int i = k + 1; i < r; ++i)
      if (std::abs(a[i * r + k]) > std::abs(a[p * r + k])) p = i;
    if (!(std::abs(a[p * r + k]) > 1e-300)) return false;
    if (p != k) {
      for (int c = 0; c < r; ++c) std::swap(a[k * r + c], a[p * r + c]);
      std::swap(perm[k], perm[p]);
    }
    for (int i = k + 1; i < r; ++i) {
      a[i * r + k] /= a[k * r + k];
      for (int c = k + 1; c < r; ++c) a[i * r + c] -= a[i * r + k] * a[k * r + c];
    }
  }
  return true;
}

std::unique_ptr<PartPlan, PartPlanDeleter> build_plan(const Factor& f, int K) {
  const int n = static_cast<int>(f.n);
  const bool pent = f.kind != Kind::Tri;
  const int nb = pent ? 5 : 3;
  if (f.bands.size() != static_cast<std::size_t>(nb) * n) return nullptr;
  std::unique_ptr<PartPlan, PartPlanDeleter> p(new PartPlan);
  p->K = K;
  p->pent = pent;
  p->L = n / K;
  p->R = (pent ? 4 : 2) * K;
  p->start.resize(K + 1);
  for (int k = 0; k < K; ++k) p->start[k] = k * p->L;
  p->start[K] = n;
  const int rec_f = pent ? 4 : 2, rec_b = pent ? 2 : 1;
  p->fwd.assign(static_cast<std::size_t>(n) * rec_f, 0.0);
  p->bwd.assign(static_cast<std::size_t>(n) * rec_b, 0.0);
  const int nsp = pent ? 4 : 2;
  const int nl = pent ? 2 : 1;
  p->fl.assign(static_cast<std::size_t>(n) * nl, 0.0);
  p->pr.assign(static_cast<std::size_t>(n) * nl, 0.0);
  double worst = 0.0;
  const double* band[5];
  for (int q = 0; q < nb; ++q) band[q] = f.bands.data() + static_cast<std::size_t>(q) * n;
  // local interface rows of a block of length Lk
  auto iface = [&](int q, int Lk) { return pent ? (q < 2 ? q : Lk - 4 + q) : (q == 0 ? 0 : Lk - 1); };
  std::vector<double> R(static_cast<std::size_t>(p->R) * p->R, 0.0);
  for (int k = 0; k < K; ++k) {
    const int s = p->start[k], e = p->start[k + 1], Lk = e - s;
    std::vector<double> bb[5];
    for (int q = 0; q < nb; ++q) bb[q].assign(band[q] + s, band[q] + e);
    std::unique_ptr<Factor> fb;
    bandsolve_status st;
    if (!pent) {
      bb[0][0] = 0.0;
      bb[2][Lk - 1] = 0.0;
      st = make_tri_factor(bb[0].data(), bb[1].data(), bb[2].data(), Lk, fb);
    } else {
      bb[0][0] = bb[0][1] = bb[1][0] = 0.0;
      bb[3][Lk - 1] = bb[4][Lk - 1] = bb[4][Lk - 2] = 0.0;
      st = make_pent_factor(bb[0].data(), bb[1].data(), bb[2].data(), bb[3].data(), bb[4].data(), Lk, fb);
    }
    clear_error();
    if (st != BANDSOLVE_OK) return nullptr;
    // packed fast records (same layout as solve.cu pack_*: fwd {a m, m} /
    // {e ia, b ia, ia, 0}; bwd chat / {gamma, delta})
    for (int i = 0; i < Lk; ++i) {
      const std::size_t g = static_cast<std::size_t>(s + i);
      if (!pent) {
        const double a = i == 0 ? 0.0 : fb->sub[i], mm = fb->inv_denom[i];
        p->fwd[2 * g] = a * mm;
        p->fwd[2 * g + 1] = mm;
        p->bwd[g] = i + 1 < Lk ? fb->chat[i] : 0.0;
      } else {
        const double ia = fb->inv_alpha[i];
        const double ep = i < 2 ? 0.0 : fb->epsilon[i], be = i == 0 ? 0.0 : fb->beta[i];
        p->fwd[4 * g] = ep * ia;
        p->fwd[4 * g + 1] = be * ia;
        p->fwd[4 * g + 2] = ia;
        p->bwd[2 * g] = i + 1 < Lk ? fb->gamma[i] : 0.0;
        p->bwd[2 * g + 1] = i + 2 < Lk ? fb->delta[i] : 0.0;
      }
    }
    // spikes: A_k^-1 times the coupling columns of the neighbour unknowns
    std::vector<std::vector<double>> sp(nsp, std::vector<double>(Lk, 0.0));
    if (!pent) {
      if (k > 0) sp[0][0] = band[0][s];           // sub[s] x_{s-1}
      if (k + 1 < K) sp[1][Lk - 1] = band[2][e - 1];  // sup[e-1] x_e
    } else {
      if (k > 0) {
        sp[0][0] = band[0][s];          // a[s] x_{s-2}
        sp[1][0] = band[1][s];          // b[s] x_{s-1}
        sp[1][1] = band[0][s + 1];      // a[s+1] x_{s-1}
      }
      if (k + 1 < K) {
        sp[2][Lk - 2] = band[4][e - 2];  // e[e-2] x_e
        sp[2][Lk - 1] = band[3][e - 1];  // d[e-1] x_e
        sp[3][Lk - 1] = band[4][e - 1];  // e[e-1] x_{e+1}
      }
    }
    for (int q = 0; q < nsp; ++q) {
      if (pent) pent_block_fwd(*fb, sp[q].data());
      else tri_block_fwd(*fb, sp[q].data());
      if (q < nl)  // left spikes: keep the forward image for pass C
        for (int i = 0; i < Lk; ++i) {
          p->fl[static_cast<std::size_t>(q) * n + s + i] = sp[q][i];
          worst = std::max(worst, std::abs(sp[q][i]));
        }
      if (pent) pent_block_bwd(*fb, sp[q].data());
      else tri_block_bwd(*fb, sp[q].data());
    }
    // rows 0 (and 1) of the block's U^-1: U^T p = e_r, a forward recurrence
    for (int q = 0; q < nl; ++q) {
      double* pv = p->pr.data() + static_cast<std::size_t>(q) * n + s;
      for (int i = 0; i < Lk; ++i) {
        double v = i == q ? 1.0 : 0.0;
        if (!pent) {
          if (i >= 1) v -= fb->chat[i - 1] * pv[i - 1];
        } else {
          if (i >= 1) v -= fb->gamma[i - 1] * pv[i - 1];
          if (i >= 2) v -= fb->delta[i - 2] * pv[i - 2];
        }
        pv[i] = v;
        worst = std::max(worst, std::abs(v));
      }
    }
    // reduced-system rows of this block's interface unknowns
    const int nq = pent ? 4 : 2;
    for (int q = 0; q < nq; ++q) {
      const int row = nq * k + q, r = iface(q, Lk);
      R[static_cast<std::size_t>(row) * p->R + row] += 1.0;
      if (!pent) {
        if (k > 0) R[static_cast<std::size_t>(row) * p->R + 2 * (k - 1) + 1] += sp[0][r];
        if (k + 1 < K) R[static_cast<std::size_t>(row) * p->R + 2 * (k + 1)] += sp[1][r];
      } else {
        if (k > 0) {
          R[static_cast<std::size_t>(row) * p->R + 4 * (k - 1) + 2] += sp[0][r];
          R[static_cast<std::size_t>(row) * p->R + 4 * (k - 1) + 3] += sp[1][r];
        }
        if (k + 1 < K) {
          R[static_cast<std::size_t>(row) * p->R + 4 * (k + 1)] += sp[2][r];
          R[static_cast<std::size_t>(row) * p->R + 4 * (k + 1) + 1] += sp[3][r];
        }
      }
    }
  }
  if (!(worst < 1e100)) return nullptr;  // growth: leave it to the sequential sweep
  if (!lu_factor(R, p->perm, p->R)) return nullptr;
  // per-row extent of the (block-banded) factors: the solves skip exact zeros
  const int r = p->R;
  p->perm.resize(3 * r);
  for (int i = 0; i < r; ++i) {
    int lo = i, hi = i;
    for (int c = 0; c < i; ++c)
      if (R[static_cast<std::size_t>(i) * r + c] != 0.0) { lo = c; break; }
    for (int c = r - 1; c > i; --c)
      if (R[static_cast<std::size_t>(i) * r + c] != 0.0) { hi = c; break; }
    p->perm[r + i] = lo;
    p->perm[2 * r + i] = hi;
  }
  p->lu = std::move(R);
  return p;
}

// ---- kernels ------------------------------------------------------------------
constexpr int kPartU = 16;  // rows per register block (two in flight per thread)

template <bool PENT>
struct DotHook {  // accumulates the top interface values of y during the forward sweep
  const double* p0;
  const double* p1;
  double* a0;
  double* a1;
  __device__ __forceinline__ void operator()(int i, double v) const {
    *a0 = fma(p0[i], v, *a0);
    if constexpr (PENT) *a1 = fma(p1[i], v, *a1);
  }
};

template <bool PENT>
__global__ void __launch_bounds__(128) part_fwd_kernel(double* __restrict__ x, int n, long long m, long long ld,
                                                       int K, int L, const double* __restrict__ fwd,
                                                       const double* __restrict__ bwd,
                                                       const double* __restrict__ pr, double* __restrict__ yi) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(K) * m) return;
  const int k = static_cast<int>(t / m);
  const long long j = t - static_cast<long long>(k) * m;
  const int r0 = k * L;
  const int len = k + 1 < K ? L : n - r0;
  const dev::Rows<double, PENT, true> rows{fwd + static_cast<long long>(r0) * (PENT ? 4 : 2),
                                           bwd + static_cast<long long>(r0) * (PENT ? 2 : 1)};
  double s1 = 0.0, s2 = 0.0, a0 = 0.0, a1 = 0.0;
  const DotHook<PENT> hook{pr + r0, pr + n + r0, &a0, &a1};
  dev::column_forward<double, PENT, true, kPartU>(x + static_cast<long long>(r0) * ld + j, len, ld, rows, s1, s2,
                                                  hook);
  if constexpr (PENT) {
    const double g = static_cast<const double*>(rows.bwd)[2 * (len - 2)];  // gamma_{L-2}
    yi[static_cast<long long>(4 * k) * m + j] = a0;
    yi[static_cast<long long>(4 * k + 1) * m + j] = a1;
    yi[static_cast<long long>(4 * k + 2) * m + j] = fma(-g, s1, s2);
    yi[static_cast<long long>(4 * k + 3) * m + j] = s1;
  } else {
    yi[static_cast<long long>(2 * k) * m + j] = a0;
    yi[static_cast<long long>(2 * k + 1) * m + j] = s1;
  }
}

template <bool PENT>
__global__ void part_reduce_kernel(int K, long long m, const double* __restrict__ lu_g,
                                   const int* __restrict__ idx_g, double* __restrict__ z) {
  extern __shared__ double sm[];
  constexpr int NQ = PENT ? 4 : 2;
  const int R = NQ * K;
  double* lu = sm;
  int* idx = reinterpret_cast<int*>(sm + R * R);  // perm | lo | hi
  for (int t = threadIdx.x; t < R * R; t += blockDim.x) lu[t] = lu_g[t];
  for (int t = threadIdx.x; t < 3 * R; t += blockDim.x) idx[t] = idx_g[t];
  __syncthreads();
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  // interface values of y in pivot order, then P A = L U; z overwrites y in place
  double w[kPartMaxR];
  for (int i = 0; i < R; ++i) w[i] = z[static_cast<long long>(idx[i]) * m + j];
  const int* lo = idx + R;
  const int* hi = idx + 2 * R;
  for (int i = 0; i < R; ++i) {
    double v = w[i];
    for (int c = lo[i]; c < i; ++c) v = fma(-lu[i * R + c], w[c], v);
    w[i] = v;
  }
  for (int i = R - 1; i >= 0; --i) {
    double v = w[i];
    for (int c = i + 1; c <= hi[i]; ++c) v = fma(-lu[i * R + c], w[c], v);
    w[i] = v / lu[i * R + i];
  }
  for (int i = 0; i < R; ++i) z[static_cast<long long>(i) * m + j] = w[i];
}

template <bool PENT>
struct LeftHook {  // g_i - F_i x_left (the left-neighbour coupling's forward image)
  const double* f1;
  const double* f2;
  double xl1, xl2;
  __device__ __forceinline__ double operator()(int i, double g) const {
    if constexpr (PENT) return fma(-f1[i], xl2, fma(-f2[i], xl1, g));
    else return fma(-f1[i], xl1, g);
  }
};

template <bool PENT>
__global__ void __launch_bounds__(128) part_bwd_kernel(double* __restrict__ x, int n, long long m, long long ld,
                                                       int K, int L, const double* __restrict__ fwd,
                                                       const double* __restrict__ bwd,
                                                       const double* __restrict__ fl, const double* __restrict__ z) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(K) * m) return;
  const int k = static_cast<int>(t / m);
  const long long j = t - static_cast<long long>(k) * m;
  const int r0 = k * L;
  const int len = k + 1 < K ? L : n - r0;
  const dev::Rows<double, PENT, true> rows{fwd + static_cast<long long>(r0) * (PENT ? 4 : 2),
                                           bwd + static_cast<long long>(r0) * (PENT ? 2 : 1)};
  double* col = x + static_cast<long long>(r0) * ld + j;
  constexpr int NQ = PENT ? 4 : 2;
  LeftHook<PENT> hook{fl + r0, fl + n + r0, 0.0, 0.0};
  double s1, s2 = 0.0;
  if constexpr (PENT) {
    if (k > 0) {
      hook.xl2 = z[static_cast<long long>(NQ * k - 2) * m + j];  // x_{s-2}
      hook.xl1 = z[static_cast<long long>(NQ * k - 1) * m + j];  // x_{s-1}
    }
    s1 = z[static_cast<long long>(NQ * k + 2) * m + j];  // own rows L-2, L-1
    s2 = z[static_cast<long long>(NQ * k + 3) * m + j];
    col[static_cast<long long>(len - 2) * ld] = s1;
    col[static_cast<long long>(len - 1) * ld] = s2;
    dev::column_backward<double, PENT, true, kPartU>(col, len - 2, ld, rows, s1, s2, hook);
  } else {
    if (k > 0) hook.xl1 = z[static_cast<long long>(NQ * k - 1) * m + j];
    s1 = z[static_cast<long long>(NQ * k + 1) * m + j];  // own row L-1
    col[static_cast<long long>(len - 1) * ld] = s1;
    dev::column_backward<double, PENT, true, kPartU>(col, len - 1, ld, rows, s1, s2, hook);
  }
}

}  // namespace

int partition_blocks(std::size_t n, std::size_t m, int sms, bool pent) {
  const char* env = std::getenv("BANDSOLVE_PARTITION");
  if (env && std::strcmp(env, "0") == 0) return 0;
  if (std::getenv("BANDSOLVE_PLAN")) return 0;  // a forced sweep plan (tests / tuning)
  const bool forced = env && std::strcmp(env, "1") == 0;
  if (n > static_cast<std::size_t>(INT_MAX) || m == 0 || current_mode() != BANDSOLVE_MODE_FAST) return 0;
  // few systems only: below ~one warp of systems per SM the sweep is latency-bound
  // (short systems: three launches cost more than the latency they hide)
  if (!forced && (m > static_cast<std::size_t>(sms) * 64 || n < 1024)) return 0;
  const int kmax = kPartMaxR / (pent ? 4 : 2);
  const char* ke = std::getenv("BANDSOLVE_PART_K");  // tuning override (power of two)
  if (ke && std::atoi(ke) >= 2 && std::atoi(ke) <= kmax && static_cast<int>(n) / std::atoi(ke) >= 16)
    return std::atoi(ke);
  int K = 2;
  while (K < kmax && static_cast<std::size_t>(K) * m < static_cast<std::size_t>(sms) * 512 &&
         static_cast<int>(n) / (2 * K) >= 32)
    K *= 2;
  return static_cast<int>(n) / K < 16 ? 0 : K;
}

bandsolve_status partition_solve_device(const Factor& f, double* x, std::size_t n, std::size_t m, std::size_t ld,
                                        void* stream, int sms, bool* done) {
  *done = false;
  const bool pent = f.kind != Kind::Tri;
  const int K = partition_blocks(n, m, sms, pent);
  if (K == 0) return BANDSOLVE_OK;
  int device = 0;
  if (cudaGetDevice(&device) != cudaSuccess) {
    cudaGetLastError();
    return BANDSOLVE_OK;
  }
  // plan (host, once per factor and K) and its device blob (once per device)
  PartPlan* p = nullptr;
  void* blob = nullptr;
  {
    std::lock_guard<std::mutex> lock(f.mu);
    for (auto& q : f.parts)
      if (q && q->K == K) p = q.get();
    if (!p) {
      auto q = build_plan(f, K);
      if (!q) return BANDSOLVE_OK;  // a block pivot broke down: the sequential sweep handles it
      p = q.get();
      f.parts.push_back(std::move(q));
    }
    for (auto& d : p->dev)
      if (d.first == device) blob = d.second;
    if (!blob) {
      const std::size_t bytes = (p->fwd.size() + p->bwd.size() + p->fl.size() + p->pr.size() + p->lu.size()) * sizeof(double) +
                                p->perm.size() * sizeof(int);
      if (cudaMalloc(&blob, bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(BANDSOLVE_ERR_INTERNAL, "partition plan upload");
      }
      char* c = static_cast<char*>(blob);
      for (const auto* v : {&p->fwd, &p->bwd, &p->fl, &p->pr, &p->lu}) {
        cudaMemcpy(c, v->data(), v->size() * sizeof(double), cudaMemcpyHostToDevice);
        c += v->size() * sizeof(double);
      }
      cudaMemcpy(c, p->perm.data(), p->perm.size() * sizeof(int), cudaMemcpyHostToDevice);
      p->dev.emplace_back(device, blob);
    }
  }
  const double* fwd = static_cast<const double*>(blob);
  const double* bwd = fwd + p->fwd.size();
  const double* fl = bwd + p->bwd.size();
  const double* pr = fl + p->fl.size();
  const double* lu = pr + p->pr.size();
  const int* idx = reinterpret_cast<const int*>(lu + p->lu.size());
  auto s = static_cast<cudaStream_t>(stream);
  const int N = static_cast<int>(n);
  const long long M = static_cast<long long>(m), LD = static_cast<long long>(ld);
  double* z = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&z), static_cast<std::size_t>(p->R) * m * sizeof(double), s) !=
      cudaSuccess) {
    cudaGetLastError();
    return fail(BANDSOLVE_ERR_INTERNAL, "partition scratch");
  }
  const long long tot = static_cast<long long>(K) * M;
  const unsigned g1 = static_cast<unsigned>((tot + 127) / 128);
  const unsigned gj = static_cast<unsigned>((M + 127) / 128);
  const std::size_t red_smem = static_cast<std::size_t>(p->R) * p->R * sizeof(double) + 3 * p->R * sizeof(int);
  if (pent) {
    part_fwd_kernel<true><<<g1, 128, 0, s>>>(x, N, M, LD, K, p->L, fwd, bwd, pr, z);
    part_reduce_kernel<true><<<gj, 128, red_smem, s>>>(K, M, lu, idx, z);
    part_bwd_kernel<true><<<g1, 128, 0, s>>>(x, N, M, LD, K, p->L, fwd, bwd, fl, z);
  } else {
    part_fwd_kernel<false><<<g1, 128, 0, s>>>(x, N, M, LD, K, p->L, fwd, bwd, pr, z);
    part_reduce_kernel<false><<<gj, 128, red_smem, s>>>(K, M, lu, idx, z);
    part_bwd_kernel<false><<<g1, 128, 0, s>>>(x, N, M, LD, K, p->L, fwd, bwd, fl, z);
  }
  note_launches(3);
  cudaFreeAsync(z, s);
  if (cudaError_t e = cudaGetLastError(); e != cudaSuccess)
    return fail(BANDSOLVE_ERR_INTERNAL, std::string("partition launch: ") + cudaGetErrorString(e));
  *done = true;
  return BANDSOLVE_OK;
}

}  // namespace bsb
