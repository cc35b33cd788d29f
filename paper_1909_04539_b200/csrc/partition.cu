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
//   matrix is shared: its inverse is precomputed (LU with partial pivoting).
//
// Two launches, 4 HBM passes over the batch (like an off-chip sequential
// sweep): (A) K*m independent block forward sweeps (thread per block-system,
// deep register prefetch) that also emit the block's interface values of y =
// A_k^-1 b_k -- the bottom ones are forward values, the top ones dot products
// of the forward values with precomputed rows of the block's U^-1; (B) K*m
// block backward sweeps: each thread first forms the interface values it
// needs (its own bottom rows and its left neighbour's) as rows of R^-1 times
// the system's y interface vector (R independent FMAs, L2-resident), then
// sweeps up from its own bottom values, folding the left coupling in as
// g_i - F_i x_left (F = the forward image of the coupling column). A periodic
// (Woodbury) correction fuses into (B): its coefficients need only x_0, x_1,
// x_{n-2}, x_{n-1}, which are interface unknowns. Arithmetic differs from the
// sequential sweep by rounding only (fast mode, 1e-12).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "internal.hpp"
#include "sweep_spike.cuh"

namespace bsb {

cudaError_t upload_sync(void* dst, const void* src, std::size_t bytes);  // solve.cu
bool encode_tile_map(CUtensorMap* map, void* x, std::size_t elem, long long n, long long m, long long ld,
                     int box_w, int box_r);              // solve.cu
cudaError_t allow_max_smem(const void* kern);            // solve.cu
std::size_t max_smem_per_block();                        // solve.cu

struct PartPlan {
  int K = 0, R = 0, L = 0;
  bool pent = false;
  std::vector<int> start;                  // K + 1 block starts (block K-1 absorbs n % K)
  std::vector<double> fwd, bwd;            // packed fast records, one per row (block-local factors)
  std::vector<double> fl;                  // forward images of the left coupling (tri: F, pent: F1 | F2)
  std::vector<double> pr;                  // rows of the block U^-1 (tri: P0, pent: P0 | P1)
  std::vector<double> rinv;                // R x R inverse of the interface matrix, row-major
  bool ok = false;                         // false: the plan broke down (sequential sweep instead)
  std::vector<std::pair<int, void*>> dev;  // device blobs
  // device blobs of the one-pass kernel's records, keyed 2 device + (fp32 ? 1 : 0)
  std::vector<std::pair<int, void*>> spike_dev;
  int sp_dp = -1, sp_df = -1;  // spike decay cut-offs in chunks (spike_cutoffs), -1: not computed
  ~PartPlan() {
    auto release = [](int device, void* ptr) {
      int prev = -1;
      if (cudaGetDevice(&prev) == cudaSuccess && prev != device) cudaSetDevice(device);
      cudaFree(ptr);
      if (prev >= 0 && prev != device) cudaSetDevice(prev);
    };
    for (auto& d : dev) release(d.first, d.second);
    for (auto& d : spike_dev) release(d.first / 2, d.second);
    cudaGetLastError();
  }
};
void PartPlanDeleter::operator()(PartPlan* p) const { delete p; }

namespace {

constexpr int kPartMaxR = 64;  // interface-system order cap (R^-1 rows read per thread)
// Largest accepted growth of the block eliminations (pivot reciprocal x band
// scale, spike / U^-1 / interface-inverse entries). Diagonally dominant and
// the SPD stencil matrices stay below ~10; 1e6 keeps the rounding
// amplification of the partitioned path well inside the 1e-12 contract.
constexpr double kPartMaxGrowth = 1e6;

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
    if (st != BANDSOLVE_OK) return p;
    // A block k > 0 is not a leading principal submatrix: its unpivoted
    // elimination can meet a tiny pivot even when the sequential factor is
    // well conditioned (e.g. a near-zero diagonal entry at a block start).
    // Reject block pivots that grow the elimination beyond kPartMaxGrowth
    // relative to the band scale; the sequential sweep then runs instead.
    {
      double scale = 0.0, inv_max = 0.0;
      for (int q = 0; q < nb; ++q)
        for (int i = 0; i < Lk; ++i) scale = std::max(scale, std::abs(bb[q][i]));
      const std::vector<double>& inv = pent ? fb->inv_alpha : fb->inv_denom;
      for (int i = 0; i < Lk; ++i) inv_max = std::max(inv_max, std::abs(inv[i]));
      if (!(scale * inv_max < kPartMaxGrowth)) return p;
    }
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
  if (!(worst < kPartMaxGrowth)) return p;  // growth: leave it to the sequential sweep
  const int r = p->R;
  std::vector<int> perm;
  if (!lu_factor(R, perm, r)) return p;
  // R^-1 column by column: P A = L U  =>  A^-1 e_c = U^-1 L^-1 P e_c
  p->rinv.assign(static_cast<std::size_t>(r) * r, 0.0);
  std::vector<double> w(r);
  for (int c = 0; c < r; ++c) {
    for (int i = 0; i < r; ++i) {
      double v = perm[i] == c ? 1.0 : 0.0;
      for (int q = 0; q < i; ++q) v -= R[static_cast<std::size_t>(i) * r + q] * w[q];
      w[i] = v;
    }
    for (int i = r - 1; i >= 0; --i) {
      double v = w[i];
      for (int q = i + 1; q < r; ++q) v -= R[static_cast<std::size_t>(i) * r + q] * w[q];
      w[i] = v / R[static_cast<std::size_t>(i) * r + i];
    }
    for (int i = 0; i < r; ++i) {
      p->rinv[static_cast<std::size_t>(i) * r + c] = w[i];
      if (!(std::abs(w[i]) < kPartMaxGrowth)) return p;
    }
  }
  p->ok = true;
  return p;
}

// ---- kernels ------------------------------------------------------------------
constexpr int kPartU = 16;  // rows per register block (two in flight per thread)

// Per-row arrays of the block a CTA solves, staged once into shared memory
// when every thread of the CTA works on the same block (the ADI axes: m a
// multiple of 128): the rows' factor records, U^-1 rows, coupling images and
// periodic z are then shared loads instead of an L2 round trip per row on
// the dependency chain. Returns that block, or -1 (the global arrays are used).
__device__ __forceinline__ int cta_block(long long m, int K, int stage) {
  if (!stage) return -1;
  const long long t0 = static_cast<long long>(blockIdx.x) * blockDim.x, t1 = t0 + blockDim.x - 1;
  if (t1 >= static_cast<long long>(K) * m) return -1;
  return t0 / m == t1 / m ? static_cast<int>(t0 / m) : -1;
}
__device__ __forceinline__ void cta_copy(double* dst, const double* src, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = src[i];
}

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
                                                       const double* __restrict__ pr, double* __restrict__ yi,
                                                       int stage) {
  extern __shared__ __align__(128) double pst[];
  constexpr int FW = PENT ? 4 : 2;
  const int kc = cta_block(m, K, stage);
  if (kc >= 0) {  // [records FW x len | P0 | P1]
    const int r0c = kc * L, lenc = kc + 1 < K ? L : n - r0c;
    cta_copy(pst, fwd + static_cast<long long>(r0c) * FW, lenc * FW);
    cta_copy(pst + lenc * FW, pr + r0c, lenc);
    if constexpr (PENT) cta_copy(pst + lenc * (FW + 1), pr + n + r0c, lenc);
  }
  __syncthreads();
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(K) * m) return;
  const int k = static_cast<int>(t / m);
  const long long j = t - static_cast<long long>(k) * m;
  const int r0 = k * L;
  const int len = k + 1 < K ? L : n - r0;
  const bool sh = kc >= 0;
  const dev::Rows<double, PENT, true> rows{sh ? pst : fwd + static_cast<long long>(r0) * FW,
                                           bwd + static_cast<long long>(r0) * (PENT ? 2 : 1)};
  double s1 = 0.0, s2 = 0.0, a0 = 0.0, a1 = 0.0;
  const DotHook<PENT> hook{sh ? pst + len * FW : pr + r0, sh ? pst + len * (FW + 1) : pr + n + r0, &a0, &a1};
  dev::column_forward<double, PENT, true, kPartU, DotHook<PENT>, 2>(x + static_cast<long long>(r0) * ld + j, len, ld,
                                                                    rows, s1, s2, hook);
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

// Pass A with the ADI explicit half fused in (adi_step_device, fast mode):
// the RHS row i of system j is the periodic Crank-Nicolson stencil across
// systems of a source array laid out the other way round, src[j * lds + i]
// (the field before its transpose). Each thread reads its own source row
// contiguously (16-byte loads; the 8 rows of a register block are one 64-byte
// run), takes the stencil neighbours j +- 1 (+- 2) from adjacent lanes by
// shuffles (edge lanes load theirs), and writes the forward values to x in
// the interleaved layout: the stencil, the transpose and the forward sweep
// in one pass. Needs m % 32 == 0 (whole warps per block) and even L, lds.
constexpr int kStU = 8;

template <bool PENT>
__global__ void __launch_bounds__(128) part_fwd_stencil_kernel(
    double* __restrict__ x, int n, long long m, long long ld, int K, int L, const double* __restrict__ fwd,
    const double* __restrict__ bwd, const double* __restrict__ pr, double* __restrict__ yi,
    const double* __restrict__ src, long long lds, double cs, double cs4, double cmid, int stage) {
  using namespace dev;
  extern __shared__ __align__(128) double pst[];
  constexpr int FW = PENT ? 4 : 2;
  const int kc = cta_block(m, K, stage);
  if (kc >= 0) {  // [records FW x len | P0 | P1]
    const int r0c = kc * L, lenc = kc + 1 < K ? L : n - r0c;
    cta_copy(pst, fwd + static_cast<long long>(r0c) * FW, lenc * FW);
    cta_copy(pst + lenc * FW, pr + r0c, lenc);
    if constexpr (PENT) cta_copy(pst + lenc * (FW + 1), pr + n + r0c, lenc);
  }
  __syncthreads();
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(K) * m) return;  // whole warps (m % 32 == 0)
  const int lane = threadIdx.x & 31;
  const int k = static_cast<int>(t / m);
  const long long j = t - static_cast<long long>(k) * m;
  const int r0 = k * L;
  const int len = k + 1 < K ? L : n - r0;
  const bool sh = kc >= 0;
  const dev::Rows<double, PENT, true> rows{sh ? pst : fwd + static_cast<long long>(r0) * FW,
                                           bwd + static_cast<long long>(r0) * (PENT ? 2 : 1)};
  // rows outside the warp: A = the nearer neighbour (lanes 0 / 31), B = the
  // farther (pent: lanes 0, 1 / 30, 31); periodic across the m systems
  auto wrap = [&](long long q) { return q < 0 ? q + m : (q >= m ? q - m : q); };
  const double* own = src + j * lds + r0;
  const double* rowA = own;
  const double* rowB = own;
  if (lane == 0) rowA = src + wrap(j - 1) * lds + r0;
  if (lane == 31) rowA = src + wrap(j + 1) * lds + r0;
  if constexpr (PENT) {
    if (lane <= 1) rowB = src + wrap(j - 2) * lds + r0;
    if (lane >= 30) rowB = src + wrap(j + 2) * lds + r0;
  }
  const bool needA = lane == 0 || lane == 31;
  const bool needB = PENT && (lane <= 1 || lane >= 30);
  double* col = x + static_cast<long long>(r0) * ld + j;
  const double* p0 = sh ? pst + len * FW : pr + r0;
  const double* p1 = sh ? pst + len * (FW + 1) : pr + n + r0;
  double s1 = 0.0, s2 = 0.0, a0 = 0.0, a1 = 0.0;
  auto rhs_row = [&](double c, double d1, double u1, double d2, double u2) {
    if constexpr (PENT) {  // pde.cpp:108 order
      const double q = add_rn(mul_rn(-cs, add_rn(d2, u2)), mul_rn(cs4, add_rn(d1, u1)));
      return add_rn(q, mul_rn(cmid, c));
    } else {  // pde.cpp:85 order
      return add_rn(mul_rn(cs, add_rn(d1, u1)), mul_rn(cmid, c));
    }
  };
  auto load8 = [&](const double* p, int i0, double* v) {
#pragma unroll
    for (int u = 0; u < kStU; u += 2) {
      const double2 w = *reinterpret_cast<const double2*>(p + i0 + u);
      v[u] = w.x;
      v[u + 1] = w.y;
    }
  };
  const int full = len / kStU;
  double c[kStU], cA[kStU], cB[kStU], n0[kStU], nA[kStU], nB[kStU];
  if (full > 0) {
    load8(own, 0, c);
    if (needA) load8(rowA, 0, cA);
    if (needB) load8(rowB, 0, cB);
  }
  for (int b = 0; b < full; ++b) {
    const int i0 = b * kStU;
    if (b + 3 < full) {  // L2 prefetch two runs beyond the register double buffer
      prefetch_l2(own + i0 + 3 * kStU);
      if (needA) prefetch_l2(rowA + i0 + 3 * kStU);
      if (needB) prefetch_l2(rowB + i0 + 3 * kStU);
    }
    if (b + 1 < full) {
      load8(own, i0 + kStU, n0);
      if (needA) load8(rowA, i0 + kStU, nA);
      if (needB) load8(rowB, i0 + kStU, nB);
    }
#pragma unroll
    for (int u = 0; u < kStU; ++u) {
      double d1 = __shfl_up_sync(0xffffffffu, c[u], 1);
      double u1 = __shfl_down_sync(0xffffffffu, c[u], 1);
      if (lane == 0) d1 = cA[u];
      if (lane == 31) u1 = cA[u];
      double d2 = 0.0, u2 = 0.0;
      if constexpr (PENT) {
        d2 = __shfl_up_sync(0xffffffffu, c[u], 2);
        u2 = __shfl_down_sync(0xffffffffu, c[u], 2);
        if (lane <= 1) d2 = cB[u];
        if (lane >= 30) u2 = cB[u];
      }
      const double v = rows.forward(i0 + u, rhs_row(c[u], d1, u1, d2, u2), s1, s2);
      a0 = fma(p0[i0 + u], v, a0);
      if constexpr (PENT) a1 = fma(p1[i0 + u], v, a1);
      col[static_cast<long long>(i0 + u) * ld] = v;
    }
#pragma unroll
    for (int u = 0; u < kStU; ++u) {
      c[u] = n0[u];
      cA[u] = nA[u];
      cB[u] = nB[u];
    }
  }
  for (int i = full * kStU; i < len; ++i) {  // tail rows: scalar loads
    const double cc = own[i];
    const double ea = needA ? rowA[i] : 0.0, eb = needB ? rowB[i] : 0.0;
    double d1 = __shfl_up_sync(0xffffffffu, cc, 1);
    double u1 = __shfl_down_sync(0xffffffffu, cc, 1);
    if (lane == 0) d1 = ea;
    if (lane == 31) u1 = ea;
    double d2 = 0.0, u2 = 0.0;
    if constexpr (PENT) {
      d2 = __shfl_up_sync(0xffffffffu, cc, 2);
      u2 = __shfl_down_sync(0xffffffffu, cc, 2);
      if (lane <= 1) d2 = eb;
      if (lane >= 30) u2 = eb;
    }
    const double v = rows.forward(i, rhs_row(cc, d1, u1, d2, u2), s1, s2);
    a0 = fma(p0[i], v, a0);
    if constexpr (PENT) a1 = fma(p1[i], v, a1);
    col[static_cast<long long>(i) * ld] = v;
  }
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
struct CorrHook {  // stores x_i - (z1_i t1 + z2_i t2)
  const double* z1;
  const double* z2;
  double t1, t2;
  __device__ __forceinline__ double operator()(int i, double v) const {
    if constexpr (PENT) return fma(-z1[i], t1, fma(-z2[i], t2, v));
    else return fma(-z1[i], t1, v);
  }
};

// (tri: <= 128 registers, 4 CTAs per SM keep 16 blocks x 4096 systems in one
// wave; pent runs 8 blocks and keeps its registers)
template <bool PENT, bool PER>
__global__ void __launch_bounds__(128, PENT ? 1 : 4) part_bwd_kernel(double* __restrict__ x, int n, long long m, long long ld,
                                                       int K, int L, const double* __restrict__ fwd,
                                                       const double* __restrict__ bwd,
                                                       const double* __restrict__ fl,
                                                       const double* __restrict__ rinv,
                                                       const double* __restrict__ yi, PartPeriodic per,
                                                       int stage) {
  extern __shared__ __align__(128) double pst[];
  constexpr int BWN = PENT ? 2 : 1;  // doubles per bwd record; also F / z arrays per row
  const int kc = cta_block(m, K, stage);
  if (kc >= 0) {  // [bwd records | F1 (| F2) | (PER) z1 (| z2)]
    const int r0c = kc * L, lenc = kc + 1 < K ? L : n - r0c;
    cta_copy(pst, bwd + static_cast<long long>(r0c) * BWN, lenc * BWN);
    cta_copy(pst + lenc * BWN, fl + r0c, lenc);
    if constexpr (PENT) cta_copy(pst + lenc * (BWN + 1), fl + n + r0c, lenc);
    if constexpr (PER) {
      cta_copy(pst + lenc * 2 * BWN, per.z1 + r0c, lenc);
      if constexpr (PENT) cta_copy(pst + lenc * (2 * BWN + 1), per.z2 + r0c, lenc);
    }
  }
  __syncthreads();
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(K) * m) return;
  const int k = static_cast<int>(t / m);
  const long long j = t - static_cast<long long>(k) * m;
  const int r0 = k * L;
  const int len = k + 1 < K ? L : n - r0;
  constexpr int NQ = PENT ? 4 : 2;
  constexpr int NH = NQ / 2;  // bottom interface rows per block
  const int R = NQ * K;
  // interface values: [own bottom NH | left bottom NH | (PER) global first NH | global last NH]
  constexpr int NU = PER ? 4 * NH : 2 * NH;
  int rowsel[NU];
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    rowsel[h] = NQ * k + NH + h;
    rowsel[NH + h] = k > 0 ? NQ * k - NH + h : NQ * k + NH + h;  // (unused when k == 0)
    if constexpr (PER) {
      rowsel[2 * NH + h] = h;
      rowsel[3 * NH + h] = R - NH + h;
    }
  }
  double zu[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) zu[u] = 0.0;
  // batches of 16 independent L2 loads in flight (one L2 round trip per
  // batch instead of per interface value)
  constexpr int CB = 16;
  int c0 = 0;
  for (; c0 + CB <= R; c0 += CB) {
    double y[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) y[c] = yi[static_cast<long long>(c0 + c) * m + j];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const double* row = rinv + rowsel[u] * R + c0;
#pragma unroll
      for (int c = 0; c < CB; ++c) zu[u] = fma(__ldg(row + c), y[c], zu[u]);
    }
  }
  for (int c = c0; c < R; ++c) {
    const double y = yi[static_cast<long long>(c) * m + j];
#pragma unroll
    for (int u = 0; u < NU; ++u) zu[u] = fma(__ldg(rinv + rowsel[u] * R + c), y, zu[u]);
  }
  const bool sh = kc >= 0;
  const dev::Rows<double, PENT, true> rows{fwd + static_cast<long long>(r0) * (PENT ? 4 : 2),
                                           sh ? pst : bwd + static_cast<long long>(r0) * BWN};
  double* col = x + static_cast<long long>(r0) * ld + j;
  LeftHook<PENT> hook{sh ? pst + len * BWN : fl + r0, sh ? pst + len * (BWN + 1) : fl + n + r0, 0.0, 0.0};
  if (k > 0) {
    if constexpr (PENT) {
      hook.xl2 = zu[2];  // x_{s-2}
      hook.xl1 = zu[3];  // x_{s-1}
    } else {
      hook.xl1 = zu[1];  // x_{s-1}
    }
  }
  CorrHook<PENT> corr{sh ? pst + len * 2 * BWN : per.z1 + r0, sh ? pst + len * (2 * BWN + 1) : per.z2 + r0, 0.0,
                      0.0};
  if constexpr (PER) {
    if constexpr (PENT) {  // periodic.cpp:189-194 (fast-mode rounding)
      const double w1 = zu[4] - zu[7], w2 = zu[5] - zu[6];
      corr.t1 = fma(per.c[0], w1, per.c[1] * w2);
      corr.t2 = fma(per.c[2], w1, per.c[3] * w2);
    } else {  // periodic.cpp:80
      corr.t1 = fma(per.c[0], zu[3], zu[2]) * per.c[1];
    }
  }
  double s1, s2 = 0.0;
  if constexpr (PENT) {
    s1 = zu[0];  // own rows L-2, L-1
    s2 = zu[1];
    if constexpr (PER) {
      col[static_cast<long long>(len - 2) * ld] = corr(len - 2, s1);
      col[static_cast<long long>(len - 1) * ld] = corr(len - 1, s2);
      dev::column_backward<double, PENT, true, kPartU, LeftHook<PENT>, CorrHook<PENT>, 2>(col, len - 2, ld, rows, s1, s2, hook, corr);
    } else {
      col[static_cast<long long>(len - 2) * ld] = s1;
      col[static_cast<long long>(len - 1) * ld] = s2;
      dev::column_backward<double, PENT, true, kPartU, LeftHook<PENT>, dev::NoHook, 2>(col, len - 2, ld, rows, s1, s2, hook);
    }
  } else {
    s1 = zu[0];  // own row L-1
    if constexpr (PER) {
      col[static_cast<long long>(len - 1) * ld] = corr(len - 1, s1);
      dev::column_backward<double, PENT, true, kPartU, LeftHook<PENT>, CorrHook<PENT>, 2>(col, len - 1, ld, rows, s1, s2, hook, corr);
    } else {
      col[static_cast<long long>(len - 1) * ld] = s1;
      dev::column_backward<double, PENT, true, kPartU, LeftHook<PENT>, dev::NoHook, 2>(col, len - 1, ld, rows, s1, s2, hook);
    }
  }
}

}  // namespace

bool partition_stencil_ok(std::size_t n, std::size_t m, int K, std::size_t lds) {
  return K > 0 && m % 32 == 0 && (n / K) % 2 == 0 && lds % 2 == 0 && lds >= n;
}

int partition_blocks(std::size_t n, std::size_t m, int sms, bool pent) {
  const long long sel = tune_int("PARTITION", -1);  // 0: never, 1: whenever it applies
  if (sel == 0) return 0;
  if (tune_flag("PLAN")) return 0;  // a forced sweep plan (tests / tuning)
  const bool forced = sel == 1;
  if (n > static_cast<std::size_t>(INT_MAX) || m == 0 || current_mode() != BANDSOLVE_MODE_FAST) return 0;
  // few systems only: below ~one warp of systems per SM the sweep is latency-bound
  // (short systems: three launches cost more than the latency they hide)
  if (!forced && (m > static_cast<std::size_t>(sms) * 64 || n < 1024)) return 0;
  // each backward thread forms 4 (tri) / 8 (pent) interface values from
  // R^-1 rows, so a small interface system wins over more blocks (measured at
  // 4096 x 4096: tri K=16 1.12e11 vs K=32 1.0e11 rows/s; pent K=8 = K=16)
  const int kmax = pent ? 8 : 16;
  const int ke = static_cast<int>(tune_int("PART_K", 0));  // tuning override (power of two)
  if (ke >= 2 && ke <= kPartMaxR / (pent ? 4 : 2) && static_cast<int>(n) / ke >= 16) return ke;
  int K = 2;
  while (K < kmax && static_cast<std::size_t>(K) * m < static_cast<std::size_t>(sms) * 512 &&
         static_cast<int>(n) / (2 * K) >= 32)
    K *= 2;
  return static_cast<int>(n) / K < 16 ? 0 : K;
}

bandsolve_status partition_solve_device(const Factor& f, double* x, std::size_t n, std::size_t m, std::size_t ld,
                                        void* stream, int sms, bool* done, const PartPeriodic* per,
                                        const PartStencil* st) {
  *done = false;
  const bool pent = f.kind != Kind::Tri;
  const int K = partition_blocks(n, m, sms, pent);
  if (K == 0) return BANDSOLVE_OK;
  if (st && !partition_stencil_ok(n, m, K, st->lds)) return BANDSOLVE_OK;
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
      if (!q) return BANDSOLVE_OK;
      p = q.get();
      f.parts.push_back(std::move(q));
    }
    if (!p->ok) return BANDSOLVE_OK;  // a block pivot broke down or grew: the sequential sweep handles it
    for (auto& d : p->dev)
      if (d.first == device) blob = d.second;
    if (!blob) {
      const std::size_t bytes =
          (p->fwd.size() + p->bwd.size() + p->fl.size() + p->pr.size() + p->rinv.size()) * sizeof(double);
      if (cudaMalloc(&blob, bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(BANDSOLVE_ERR_INTERNAL, "partition plan upload");
      }
      char* c = static_cast<char*>(blob);
      for (const auto* v : {&p->fwd, &p->bwd, &p->fl, &p->pr, &p->rinv}) {
        if (upload_sync(c, v->data(), v->size() * sizeof(double)) != cudaSuccess) {
          cudaGetLastError();
          cudaFree(blob);
          return fail(BANDSOLVE_ERR_INTERNAL, "partition plan upload");
        }
        c += v->size() * sizeof(double);
      }
      p->dev.emplace_back(device, blob);
    }
  }
  const double* fwd = static_cast<const double*>(blob);
  const double* bwd = fwd + p->fwd.size();
  const double* fl = bwd + p->bwd.size();
  const double* pr = fl + p->fl.size();
  const double* rinv = pr + p->pr.size();
  auto s = static_cast<cudaStream_t>(stream);
  const int N = static_cast<int>(n);
  const long long M = static_cast<long long>(m), LD = static_cast<long long>(ld);
  double* yi = nullptr;  // interface values of y, [R][m]
  if (pool_malloc_async(reinterpret_cast<void**>(&yi), static_cast<std::size_t>(p->R) * m * sizeof(double), s) !=
      cudaSuccess) {
    cudaGetLastError();
    return fail(BANDSOLVE_ERR_INTERNAL, "partition scratch");
  }
  const long long tot = static_cast<long long>(K) * M;
  const unsigned g1 = static_cast<unsigned>((tot + 127) / 128);
  const PartPeriodic pa = per ? *per : PartPeriodic{};
  // shared-memory staging of the CTA's block rows (cta_block): the longest
  // block (the last absorbs n % K), within the default 48 KB
  const int lmax = N - (K - 1) * p->L;
  const std::size_t fb = static_cast<std::size_t>(lmax) * (pent ? 6 : 3) * sizeof(double);
  const std::size_t bb = static_cast<std::size_t>(lmax) * (pent ? 4 : 2) * (per ? 2 : 1) * sizeof(double);
  const bool stage_ok = fb <= 48 * 1024 && bb <= 48 * 1024 && !tune_flag("PART_NOSTAGE");
  const int sg = stage_ok ? 1 : 0;
  const std::size_t sf = stage_ok ? fb : 0, sb = stage_ok ? bb : 0;
  if (st) {
    if (pent)
      part_fwd_stencil_kernel<true><<<g1, 128, sf, s>>>(x, N, M, LD, K, p->L, fwd, bwd, pr, yi, st->src, st->lds,
                                                        st->s, st->s4, st->mid, sg);
    else
      part_fwd_stencil_kernel<false><<<g1, 128, sf, s>>>(x, N, M, LD, K, p->L, fwd, bwd, pr, yi, st->src, st->lds,
                                                         st->s, st->s4, st->mid, sg);
    if (per) {
      if (pent) part_bwd_kernel<true, true><<<g1, 128, sb, s>>>(x, N, M, LD, K, p->L, fwd, bwd, fl, rinv, yi, pa, sg);
      else part_bwd_kernel<false, true><<<g1, 128, sb, s>>>(x, N, M, LD, K, p->L, fwd, bwd, fl, rinv, yi, pa, sg);
    } else {
      if (pent) part_bwd_kernel<true, false><<<g1, 128, sb, s>>>(x, N, M, LD, K, p->L, fwd, bwd, fl, rinv, yi, pa, sg);
      else part_bwd_kernel<false, false><<<g1, 128, sb, s>>>(x, N, M, LD, K, p->L, fwd, bwd, fl, rinv, yi, pa, sg);
    }
  } else if (pent) {
    part_fwd_kernel<true><<<g1, 128, sf, s>>>(x, N, M, LD, K, p->L, fwd, bwd, pr, yi, sg);
    if (per) part_bwd_kernel<true, true><<<g1, 128, sb, s>>>(x, N, M, LD, K, p->L, fwd, bwd, fl, rinv, yi, pa, sg);
    else part_bwd_kernel<true, false><<<g1, 128, sb, s>>>(x, N, M, LD, K, p->L, fwd, bwd, fl, rinv, yi, pa, sg);
  } else {
    part_fwd_kernel<false><<<g1, 128, sf, s>>>(x, N, M, LD, K, p->L, fwd, bwd, pr, yi, sg);
    if (per) part_bwd_kernel<false, true><<<g1, 128, sb, s>>>(x, N, M, LD, K, p->L, fwd, bwd, fl, rinv, yi, pa, sg);
    else part_bwd_kernel<false, false><<<g1, 128, sb, s>>>(x, N, M, LD, K, p->L, fwd, bwd, fl, rinv, yi, pa, sg);
  }
  note_launches(2);
  cudaFreeAsync(yi, s);
  if (cudaError_t e = cudaGetLastError(); e != cudaSuccess)
    return fail(BANDSOLVE_ERR_INTERNAL, std::string("partition launch: ") + cudaGetErrorString(e));
  *done = true;
  return BANDSOLVE_OK;
}

// ---- one-pass partitioned sweep for many long systems (sweep_spike.cuh) ----------

namespace {

// Records of the one-pass kernel: [SpF<T> x n][SpB<T> x n] (the plan's block
// factors, U^-1 rows and left-coupling images, interleaved per row), then
// R^-1 (R x R, row-major), all in T.
template <typename T>
std::vector<unsigned char> spike_blob(const PartPlan& p, int n) {
  const std::size_t nf = static_cast<std::size_t>(n);
  const std::size_t sf = p.pent ? sizeof(dev::SpF<T, true>) : sizeof(dev::SpF<T, false>);
  const std::size_t sb = p.pent ? sizeof(dev::SpB<T, true>) : sizeof(dev::SpB<T, false>);
  // [F x n][B x n][pent: U^-1 row 1 x n][R^-1]
  const std::size_t sp = p.pent ? sizeof(T) : 0;
  std::vector<unsigned char> blob(nf * (sf + sb + sp) + p.rinv.size() * sizeof(T), 0);
  for (std::size_t u = 0; u < nf; ++u) {
    if (p.pent) {
      dev::SpF<T, true> f{};
      f.e = static_cast<T>(p.fwd[4 * u]);       // eps/alpha
      f.b = static_cast<T>(p.fwd[4 * u + 1]);   // beta/alpha
      f.ia = static_cast<T>(p.fwd[4 * u + 2]);  // 1/alpha
      f.p0 = static_cast<T>(p.pr[u]);           // U^-1 row 0
      const T p1 = static_cast<T>(p.pr[nf + u]);  // U^-1 row 1
      std::memcpy(blob.data() + nf * (sf + sb) + u * sp, &p1, sp);
      dev::SpB<T, true> b{};
      b.g = static_cast<T>(p.bwd[2 * u]);       // gamma
      b.d = static_cast<T>(p.bwd[2 * u + 1]);   // delta
      b.f1 = static_cast<T>(p.fl[u]);           // F (x_{s-2})
      b.f2 = static_cast<T>(p.fl[nf + u]);      // F (x_{s-1})
      std::memcpy(blob.data() + u * sf, &f, sf);
      std::memcpy(blob.data() + nf * sf + u * sb, &b, sb);
    } else {
      dev::SpF<T, false> f{};
      f.am = static_cast<T>(p.fwd[2 * u]);      // a/denom
      f.m = static_cast<T>(p.fwd[2 * u + 1]);   // 1/denom
      f.p0 = static_cast<T>(p.pr[u]);           // U^-1 row 0
      dev::SpB<T, false> b{};
      b.c = static_cast<T>(p.bwd[u]);           // chat
      b.f1 = static_cast<T>(p.fl[u]);           // F (x_{s-1})
      std::memcpy(blob.data() + u * sf, &f, sf);
      std::memcpy(blob.data() + nf * sf + u * sb, &b, sb);
    }
  }
  T* r = reinterpret_cast<T*>(blob.data() + nf * (sf + sb + sp));
  for (std::size_t i = 0; i < p.rinv.size(); ++i) r[i] = static_cast<T>(p.rinv[i]);
  return blob;
}

// the plan for K blocks (cached on the factor), or nullptr when it broke down
PartPlan* cached_plan(const Factor& f, int K) {
  for (auto& q : f.parts)
    if (q && q->K == K) return q->ok ? q.get() : nullptr;
  auto q = build_plan(f, K);
  if (!q) return nullptr;
  PartPlan* p = q.get();
  f.parts.push_back(std::move(q));
  return p->ok ? p : nullptr;
}

}  // namespace

// A per-device scratch word per lane: lanes past the batch edge store there
// (branch-free stores in the spike and pipe kernels). nullptr on failure.
double* dead_lane_sink(int device) {
  static double* sinks[64] = {};
  static std::mutex mu;
  if (device < 0 || device >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!sinks[device] && cudaMalloc(reinterpret_cast<void**>(&sinks[device]), 32 * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    sinks[device] = nullptr;
  }
  return sinks[device];
}

namespace {

// CTAs per cluster for K blocks (8 blocks per CTA beyond one CTA)
int spike_cluster(int K) { return K > dev::kSpWarps ? K / dev::kSpWarps : 1; }

int spike_ring_slots(int n, int K, bool pent, bool per, std::size_t elem, std::size_t rec = 0) {
  const std::size_t cap = max_smem_per_block();
  const int CS = spike_cluster(K);
  const int Kc = CS > 1 ? dev::kSpWarps : K;
  const int nl = n / K * Kc;
  const int R = (pent ? 4 : 2) * K;
  for (int kb = 6; kb >= 2; --kb)
    if (dev::SpikeLayout::make(nl, R, Kc, kb, pent, per, elem, rec).total <= cap) return kb;
  return 0;
}

// Clusters of CS CTAs that can be co-resident (GPC packing), 0 if none.
int spike_active_clusters(const void* kern, int CS, std::size_t smem, int sms) {
  if (CS == 1) return sms;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(kern, CS);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(CS * (sms / CS)), 1, 1);
  cfg.blockDim = dim3(32 * (dev::kSpWarps + 1), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(CS);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cache[key] = n;
  return n;
}

}  // namespace

int spike_blocks(std::size_t n, std::size_t m, std::size_t ld, const void* x, int sms, bool pent, std::size_t elem) {
  const long long sel = tune_int("SPIKE", -1);  // 0: never, 1: whenever it applies
  if (sel == 0 || tune_flag("PLAN")) return 0;
  // fp32 runs as pairs of adjacent systems per lane (8 bytes, like fp64)
  const bool fp32 = elem == 4;
  const std::size_t maxl = dev::spike_max_rows<double>();
  if (current_mode() != BANDSOLVE_MODE_FAST || n > static_cast<std::size_t>(dev::kSpMaxK) * maxl || m == 0) return 0;
  // TMA: 16-byte aligned base and pitch; the batch edge inside a 16-byte
  // granule (odd fp64 / non-multiple-of-4 fp32 batches would straddle one)
  const std::size_t gran = 16 / elem;
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0 || ld % gran != 0 || m > static_cast<std::size_t>(INT_MAX) / 2) return 0;
  if (m % gran != 0) return 0;
  if (fp32) m /= 2;
  // fp32 moves half the bytes per row through the same per-row work: the
  // kernel runs at ~0.5 of the fp32 roofline, above the sequential plans only
  // for long systems (tri 2^20 systems: N = 1024 / 4096 0.51 / 0.58 vs 0.43 /
  // 0.40; N = 512: 0.50 vs 0.78)
  if (fp32 && n < static_cast<std::size_t>(tune_int("SPIKE_F32_MIN_N", 0)) && sel != 1) return 0;
  const int kf = static_cast<int>(tune_int("SPIKE_K", 0));  // tuning override
  // K <= 8: one CTA holds every block; K = 16 / 32: a cluster of K / 8 CTAs
  int K = 0;
  for (int k = 2; k <= dev::kSpMaxK; k *= 2)
    if (n % k == 0 && (n / k) % dev::kSpR == 0 && n / k <= maxl &&
        n / k >= 2 * dev::kSpR && (kf == 0 || k == kf)) {
      K = k;
      break;
    }
  if (K == 0) return 0;
  // many systems: at least one full wave of groups (32 (8 / K) systems per
  // CTA; a cluster of K / 8 CTAs per 32 systems)
  const int CS = spike_cluster(K);
  const std::size_t per_wave = CS > 1 ? 32u * static_cast<std::size_t>(sms / CS)
                                      : 32u * static_cast<std::size_t>(dev::kSpWarps / K) * sms;
  if (sel != 1 && m < per_wave) {
    // Few systems: shorter blocks put more CTAs to work (configs[0], tri
    // N = 256 x 4096: K = 2 0.14, K = 8 0.33 of the HBM roofline, vs 0.21
    // for the sequential sweep). Long ones (n >= 1024) take the two-launch
    // partitioned path instead.
    if (n >= 1024 || kf != 0) return 0;
    while (K * 2 <= dev::kSpWarps && n % (2 * K) == 0 && (n / (2 * K)) % dev::kSpR == 0 &&
           n / (2 * K) >= 2 * dev::kSpR)
      K *= 2;
  }
  if (spike_ring_slots(static_cast<int>(n), K, pent, !fp32, 8, fp32 ? 4 : 8) == 0) return 0;
  return K;
}

namespace {

// First block-local chunk (of kSpR rows) past which every entry of the
// per-row vectors (arrays of n values, block length L) is below 1e-18 of the
// vector's largest magnitude, over all blocks: from there on their FMAs
// contribute nothing above fp64 rounding (fast mode).
int spike_cutoff(const std::vector<double>& v, std::size_t off, int n, int L) {
  double mx = 0.0;
  for (int u = 0; u < n; ++u) mx = std::max(mx, std::abs(v[off + u]));
  const double thr = 1e-18 * mx;
  int last = -1;  // last block-local row with a non-negligible entry
  for (int u = 0; u < n; ++u)
    if (!(std::abs(v[off + u]) < thr)) last = std::max(last, u % L);
  return last / dev::kSpR + 1;
}
void spike_cutoffs(PartPlan& p, int n) {
  if (p.sp_dp >= 0) return;
  const int L = n / p.K;
  const bool off = tune_int("SPIKE_CUT", 1) == 0;  // 0: never skip (A/B)
  p.sp_dp = off ? (1 << 30) : spike_cutoff(p.pr, 0, n, L);
  p.sp_df = off ? (1 << 30) : spike_cutoff(p.fl, 0, n, L);
  if (p.pent && !off) {
    p.sp_dp = std::max(p.sp_dp, spike_cutoff(p.pr, static_cast<std::size_t>(n), n, L));
    p.sp_df = std::max(p.sp_df, spike_cutoff(p.fl, static_cast<std::size_t>(n), n, L));
  }
}

template <typename T>
bandsolve_status spike_solve_t(const Factor& f, T* x, std::size_t n, std::size_t m, std::size_t ld, void* stream,
                               int sms, bool* done, const PartPeriodic* per, const SpikeCN* cn) {
  *done = false;
  const bool pent = f.kind != Kind::Tri;
  if (cn && (!per || reinterpret_cast<uintptr_t>(cn->u) % 16 != 0)) return BANDSOLVE_OK;
  // fp32: two adjacent systems per lane (T = float2), plain solves only
  constexpr bool kPair = std::is_same<T, float2>::value;
  using S = dev::Scalar<T>;
  if (kPair && (per || cn)) return BANDSOLVE_OK;
  const int K = spike_blocks(n, m, ld, x, sms, pent, kPair ? 4 : sizeof(T));
  if (kPair) {  // the kernel sees pairs
    m /= 2;
    ld /= 2;
  }
  if (K == 0) return BANDSOLVE_OK;
  int device = 0;
  if (cudaGetDevice(&device) != cudaSuccess) {
    cudaGetLastError();
    return BANDSOLVE_OK;
  }
  PartPlan* p = nullptr;
  void* blob = nullptr;
  {
    std::lock_guard<std::mutex> lock(f.mu);
    p = cached_plan(f, K);
    if (!p) return BANDSOLVE_OK;  // a block pivot broke down or grew: the sequential sweep handles it
    spike_cutoffs(*p, static_cast<int>(n));
    const int key = device * 2 + (sizeof(S) == 8 ? 0 : 1);  // one blob per device and precision
    for (auto& d : p->spike_dev)
      if (d.first == key) blob = d.second;
    if (!blob) {
      const std::vector<unsigned char> hb = spike_blob<S>(*p, static_cast<int>(n));
      if (cudaMalloc(&blob, hb.size()) != cudaSuccess) {
        cudaGetLastError();
        return fail(BANDSOLVE_ERR_INTERNAL, "spike plan upload");
      }
      if (upload_sync(blob, hb.data(), hb.size()) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(blob);
        return fail(BANDSOLVE_ERR_INTERNAL, "spike plan upload");
      }
      p->spike_dev.emplace_back(key, blob);
    }
  }
  const int N = static_cast<int>(n);
  const int CS = spike_cluster(K);
  const int Kc = CS > 1 ? dev::kSpWarps : K;
  const int R = p->R;
  const int KB = spike_ring_slots(N, K, pent, per != nullptr, sizeof(T), sizeof(S));
  const std::size_t rec_bytes =
      static_cast<std::size_t>(n) * (pent ? sizeof(dev::SpF<S, true>) + sizeof(dev::SpB<S, true>) + sizeof(S)
                                          : sizeof(dev::SpF<S, false>) + sizeof(dev::SpB<S, false>));
  const S* rinv = reinterpret_cast<const S*>(static_cast<const unsigned char*>(blob) + rec_bytes);
  CUtensorMap map;
  // the tensor map reads b (in place: x; Crank-Nicolson: the old field u)
  void* src = cn ? const_cast<double*>(cn->u) : static_cast<void*>(x);
  if (!encode_tile_map(&map, src, sizeof(T), N, static_cast<long long>(m), static_cast<long long>(ld), 32,
                       dev::kSpR))
    return BANDSOLVE_OK;  // no tensor map: the sweep plans take it
  const int Wg = CS > 1 ? 32 : 32 * (dev::kSpWarps / K);
  const long long groups = (static_cast<long long>(m) + Wg - 1) / Wg;
  const std::size_t smem =
      dev::SpikeLayout::make(N / K * Kc, R, Kc, KB, pent, per != nullptr, sizeof(T), sizeof(S)).total;
  const int PD = static_cast<int>(tune_int("SPD", 4));
  auto s = static_cast<cudaStream_t>(stream);
  using Kern = decltype(&dev::sweep_spike<T, true, false, false, 1>);
  static_assert(sizeof(T) == 8, "8-byte lane values (fp64, or fp32 pairs)");
  const int csi = CS == 4 ? 2 : CS == 2 ? 1 : 0;
  Kern kern;
  if constexpr (!kPair) {
    // [cluster size 1/2/4][cn][pent][per]
#define BSB_SPIKE_SET(CSZ)                                                                                        \
  {{{dev::sweep_spike<T, false, false, false, CSZ>, dev::sweep_spike<T, false, true, false, CSZ>},               \
    {dev::sweep_spike<T, true, false, false, CSZ>, dev::sweep_spike<T, true, true, false, CSZ>}},                \
   {{dev::sweep_spike<T, false, true, true, CSZ>, dev::sweep_spike<T, false, true, true, CSZ>},                  \
    {dev::sweep_spike<T, true, true, true, CSZ>, dev::sweep_spike<T, true, true, true, CSZ>}}}
    static const Kern kerns[3][2][2][2] = {BSB_SPIKE_SET(1), BSB_SPIKE_SET(2), BSB_SPIKE_SET(4)};
#undef BSB_SPIKE_SET
    kern = kerns[csi][cn != nullptr][pent][per != nullptr];
  } else {  // fp32: plain solves
    static const Kern kerns[3][2] = {{dev::sweep_spike<T, false, false, false, 1>, dev::sweep_spike<T, true, false, false, 1>},
                                     {dev::sweep_spike<T, false, false, false, 2>, dev::sweep_spike<T, true, false, false, 2>},
                                     {dev::sweep_spike<T, false, false, false, 4>, dev::sweep_spike<T, true, false, false, 4>}};
    kern = kerns[csi][pent];
  }
  const int ki = (kPair ? 24 : 0) + csi * 8 + (cn ? 4 : 0) + (pent ? 2 : 0) + (per ? 1 : 0);
  static std::atomic<uint64_t> configured[48];
  const uint64_t bit = device < 64 ? (1ull << device) : 0;
  std::atomic<uint64_t>& attr_set = configured[ki];
  dev::SpikePer sp;
  sp.dp = p->sp_dp;
  sp.df = p->sp_df;
  if (per) {
    sp.z1 = per->z1;
    sp.z2 = per->z2;
    for (int q = 0; q < 4; ++q) sp.c[q] = per->c[q];
  }
  if (cn) {
    sp.u = cn->u;
    for (int q = 0; q < 3; ++q) sp.cn[q] = cn->c[q];
  }
  if (!(bit && (attr_set.load(std::memory_order_relaxed) & bit))) {
    if (cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern)); e != cudaSuccess)
      return fail(BANDSOLVE_ERR_INTERNAL, std::string("spike attributes: ") + cudaGetErrorString(e));
    if (CS > 1)  // clusters of up to 4: portable size, no opt-in needed
      cudaFuncSetAttribute(reinterpret_cast<const void*>(kern), cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    if (bit) attr_set.fetch_or(bit, std::memory_order_relaxed);
  }
  // lanes past the batch edge write their values here (branch-free stores)
  T* sink = reinterpret_cast<T*>(dead_lane_sink(device));
  if (!sink) return fail(BANDSOLVE_ERR_INTERNAL, "spike scratch");
  const int active = spike_active_clusters(reinterpret_cast<const void*>(kern), CS, smem, sms);
  if (active <= 0) return BANDSOLVE_OK;  // the cluster does not fit: the sweep plans take it
  const unsigned grid = static_cast<unsigned>(CS * std::min<long long>(active, groups));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(32 * (dev::kSpWarps + 1), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (!tune_flag("NO_PDL")) {  // the prologue may overlap the previous kernel (griddepcontrol.wait inside)
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (CS > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = static_cast<unsigned>(CS);
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, map, x, N, static_cast<long long>(m), static_cast<long long>(ld), K,
                                     p->L, KB, PD, groups, static_cast<const void*>(blob), rinv, sink, sp);
  note_launches(1);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BANDSOLVE_ERR_INTERNAL, std::string("spike launch: ") + cudaGetErrorString(e));
  *done = true;
  return BANDSOLVE_OK;
}

}  // namespace

bandsolve_status spike_solve_device(const Factor& f, double* x, std::size_t n, std::size_t m, std::size_t ld,
                                    void* stream, int sms, bool* done, const PartPeriodic* per, const SpikeCN* cn) {
  return spike_solve_t<double>(f, x, n, m, ld, stream, sms, done, per, cn);
}

bandsolve_status spike_solve_device_f32(const Factor& f, float* x, std::size_t n, std::size_t m, std::size_t ld,
                                        void* stream, int sms, bool* done) {
  return spike_solve_t<float2>(f, reinterpret_cast<float2*>(x), n, m, ld, stream, sms, done, nullptr, nullptr);
}

}  // namespace bsb
