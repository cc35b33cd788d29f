// Device layer of libbandsolve_b200: factor upload, kernel plans, launches,
// the staged host-batch pipeline, residual and synthetic-RHS kernels.
#include <cudaTypedefs.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.hpp"
#include "sweep_kernels.cuh"
#include "sweep_persist.cuh"
#include "sweep_stream.cuh"

namespace bsb {

namespace {

std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_mode{-1};

int mode_from_env() {
  const char* e = std::getenv("BANDSOLVE_MODE");
  if (e && (std::strcmp(e, "fast") == 0 || std::strcmp(e, "FAST") == 0 || std::strcmp(e, "1") == 0))
    return BANDSOLVE_MODE_FAST;
  return BANDSOLVE_MODE_EXACT;
}

}  // namespace

bandsolve_status cuda_fail(cudaError_t err, const char* what) {
  return fail(BANDSOLVE_ERR_INTERNAL,
              std::string(what) + ": " + cudaGetErrorName(err) + " (" + cudaGetErrorString(err) + ")");
}

#define BSB_CUDA(call)                                  \
  do {                                                  \
    cudaError_t err_ = (call);                          \
    if (err_ != cudaSuccess) return cuda_fail(err_, #call); \
  } while (0)

// Upload of a per-device constant (factor records, correction vectors,
// partition plans) that later solves read from ANY stream. A pageable
// cudaMemcpy may return before its DMA lands, and kernels on non-blocking
// streams are not ordered after the legacy stream, so the copy goes through a
// private stream that is synchronised before the pointer is published.
cudaError_t upload_sync(void* dst, const void* src, std::size_t bytes) {
  cudaStream_t s = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return e != cudaSuccess ? e : e2;
}

int device_count_cached() {
  static int count = [] {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return c;
  }();
  return count;
}

namespace {

// ---- packed factor records --------------------------------------------------
// The signed zeros below make the generic row formulas of sweep_kernels.cuh
// reproduce the reference's peeled boundary rows exactly:
//   tri fwd row 0   (tri_solver.cpp:27)  : a_0 = +0        -> (d - (+0)) * m0 = d * m0
//   tri bwd row n-1 (tri_solver.cpp:39)  : chat_{n-1} = +0 -> dhat - (+0) = dhat
//   pent fwd rows 0,1 (pent_solver.cpp:19-31): eps_0 = eps_1 = beta_0 = +0
//   pent bwd row n-1: gamma = delta = +0; row n-2 (pent_solver.cpp:44-50):
//     exact mode delta_{n-2} = -0 so gamma*x1 + (-0) == gamma*x1 bit for bit.
template <typename T>
void pack_tri(const Factor& f, bool fast, std::vector<unsigned char>& fwd, std::vector<unsigned char>& bwd) {
  const std::size_t n = f.n;
  fwd.assign(n * sizeof(dev::TriFwd<T>), 0);
  bwd.assign(n * sizeof(T), 0);
  auto* rf = reinterpret_cast<dev::TriFwd<T>*>(fwd.data());
  auto* rb = reinterpret_cast<T*>(bwd.data());
  for (std::size_t i = 0; i < n; ++i) {
    const double a = (i == 0) ? 0.0 : f.sub[i];
    const double m = f.inv_denom[i];
    rf[i].a = static_cast<T>(fast ? a * m : a);
    rf[i].m = static_cast<T>(m);
    rb[i] = static_cast<T>(i + 1 < n ? f.chat[i] : 0.0);
  }
}

template <typename T>
void pack_pent(const Factor& f, bool fast, std::vector<unsigned char>& fwd, std::vector<unsigned char>& bwd) {
  const std::size_t n = f.n;
  fwd.assign(n * sizeof(dev::PentFwd<T>), 0);
  bwd.assign(n * sizeof(dev::PentBwd<T>), 0);
  auto* rf = reinterpret_cast<dev::PentFwd<T>*>(fwd.data());
  auto* rb = reinterpret_cast<dev::PentBwd<T>*>(bwd.data());
  const bool uniform = f.kind == Kind::Uniform;
  for (std::size_t i = 0; i < n; ++i) {
    const double ia = f.inv_alpha[i];
    // pent_solver.cpp:33: eps_i is read only for i >= 2 (scalar for uniform, :115)
    const double e = (i < 2) ? 0.0 : (uniform ? f.eps_scalar : f.epsilon[i]);
    const double b = (i == 0) ? 0.0 : f.beta[i];
    rf[i].e = static_cast<T>(fast ? e * ia : e);
    rf[i].b = static_cast<T>(fast ? b * ia : b);
    rf[i].ia = static_cast<T>(ia);
    rf[i].pad = T(0);
    const double g = (i + 1 < n) ? f.gamma[i] : 0.0;
    double d;
    if (i + 2 < n) d = f.delta[i];
    else if (i + 2 == n) d = fast ? 0.0 : -0.0;
    else d = 0.0;
    rb[i].g = static_cast<T>(g);
    rb[i].d = static_cast<T>(d);
  }
}

bandsolve_status ensure_device_factor(const Factor& f, int device, const DeviceFactor** out) {
  std::lock_guard<std::mutex> lock(f.mu);
  for (const DeviceFactor& d : f.devices) {
    if (d.device == device) {
      *out = &d;
      return BANDSOLVE_OK;
    }
  }
  // four variants {f64, f32} x {exact, fast}, each a fwd and a bwd array
  std::vector<unsigned char> fw[2][2], bw[2][2];
  for (int fast = 0; fast < 2; ++fast) {
    if (f.kind == Kind::Tri) {
      pack_tri<double>(f, fast, fw[0][fast], bw[0][fast]);
      pack_tri<float>(f, fast, fw[1][fast], bw[1][fast]);
    } else {
      pack_pent<double>(f, fast, fw[0][fast], bw[0][fast]);
      pack_pent<float>(f, fast, fw[1][fast], bw[1][fast]);
    }
  }
  std::size_t total = 0;
  std::size_t off_f[2][2], off_b[2][2];
  auto align256 = [](std::size_t v) { return (v + 255) & ~std::size_t(255); };
  for (int p = 0; p < 2; ++p)
    for (int q = 0; q < 2; ++q) {
      off_f[p][q] = total;
      total = align256(total + fw[p][q].size());
      off_b[p][q] = total;
      total = align256(total + bw[p][q].size());
    }
  std::vector<unsigned char> blob(total, 0);
  for (int p = 0; p < 2; ++p)
    for (int q = 0; q < 2; ++q) {
      std::memcpy(blob.data() + off_f[p][q], fw[p][q].data(), fw[p][q].size());
      std::memcpy(blob.data() + off_b[p][q], bw[p][q].data(), bw[p][q].size());
    }
  DeviceFactor d;
  d.device = device;
  BSB_CUDA(cudaMalloc(&d.base, total));
  cudaError_t err = upload_sync(d.base, blob.data(), total);
  if (err != cudaSuccess) {
    cudaFree(d.base);
    return cuda_fail(err, "factor upload");
  }
  auto* base = static_cast<unsigned char*>(d.base);
  for (int p = 0; p < 2; ++p)
    for (int q = 0; q < 2; ++q) {
      d.fwd[p][q] = base + off_f[p][q];
      d.bwd[p][q] = base + off_b[p][q];
    }
  f.devices.push_back(d);  // a deque: earlier entries never move
  *out = &f.devices.back();
  return BANDSOLVE_OK;
}

// ---- tensor maps --------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// ---- plans ----------------------------------------------------------------------
constexpr int kChunkRows = 32;
constexpr std::size_t kSmemPerSm = 233472;        // 228 KB per SM on sm_100 (cudaGetDeviceProperties)
constexpr std::size_t kSmemPerBlockMax = 232448;  // 227 KB opt-in per CTA
constexpr std::size_t kSmemReservedPerCta = 1024;
constexpr double kSpillBudget = 64.0 * (1 << 20);  // bytes of spilled d-hat kept L2-resident (of 126 MB)

enum class PlanKind { Global, Smem, Persist, Stream };

struct Plan {
  PlanKind kind = PlanKind::Global;
  int W = 0;                 // smem: systems per CTA
  int ctas_per_sm = 0;       // smem
  int warps = 0;             // persist: warps per CTA (32 systems each)
  int H = 0, TC = 0;         // persist/stream: spilled head rows, tail chunks
  int Wg = 0, KB = 0, KR = 0, PD = 0;  // stream: systems per group, b / reload ring slots, L2 prefetch distance
  int stagger_ns = 0;                  // stream: start delay of odd CTAs
  int V = 1;                           // stream: systems per lane
  int tmem_chunks = 0;                 // stream: head chunks kept in Tensor Memory
  int rc_chunks = 0;                   // stream: head chunks recomputed from checkpoints (not stored)
  int seg_chunks = 0;                  // stream: chunks per recomputed segment
  double model_us = 0;       // stream: modelled time
  std::size_t smem_bytes = 0;
  std::string why;
};

int num_sms(int device) {
  static std::atomic<int> cached[64];
  if (device < 0 || device >= 64) return 148;
  int v = cached[device].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) {
      cudaGetLastError();
      v = 148;
    }
    cached[device].store(v, std::memory_order_relaxed);
  }
  return v;
}

// Stream-ordered allocations (spill scratch, residual buffers, ADI work)
// come from a pool the library owns, one per device, that keeps freed blocks
// mapped so steady-state solves never go back to the driver. The
// application's default pool and its release threshold are left alone.
cudaMemPool_t library_pool(int device) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  if (device < 0 || device >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[device]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
      uint64_t threshold = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
      pools[device] = pool;
    }
    cudaGetLastError();
  }
  return pools[device];
}

}  // namespace

cudaError_t pool_malloc_async_raw(void** p, std::size_t bytes, cudaStream_t s) {
  int device = 0;
  if (cudaError_t e = cudaGetDevice(&device); e != cudaSuccess) return e;
  cudaMemPool_t pool = library_pool(device);
  if (!pool) return cudaMallocAsync(p, bytes, s);
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

namespace {

// The spill scratch is written and re-read within one tile; its evict_last
// lines are only protected from the evict-first b/x streams inside the L2
// persisting set-aside, which is 0 by default. Opt-in (tuning key
// L2_SETASIDE=1, since the limit is process-wide device state): grow the
// set-aside (never shrink it) to cover the scratch, up to the device maximum.
// Off, the solve is the same; only spilled rows may round-trip through HBM.
void ensure_l2_setaside(int device, std::size_t bytes) {
  if (tune_int("L2_SETASIDE", 0) == 0) return;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int max_persist = 0;
  if (cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device) != cudaSuccess ||
      max_persist <= 0) {
    cudaGetLastError();
    return;
  }
  const std::size_t want = std::min<std::size_t>(bytes + bytes / 8, static_cast<std::size_t>(max_persist));
  std::size_t cur = 0;
  if (cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) == cudaSuccess && cur < want)
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
  cudaGetLastError();
}

std::size_t smem_bytes_for(std::size_t n, int W, std::size_t elem) {
  const std::size_t chunks = (n + kChunkRows - 1) / kChunkRows;
  return chunks * kChunkRows * W * elem + chunks * sizeof(uint64_t);
}

std::size_t fwd_rec_bytes(bool pent, std::size_t elem) { return (pent ? 4 : 2) * elem; }
std::size_t bwd_rec_bytes(bool pent, std::size_t elem) { return (pent ? 2 : 1) * elem; }

// Dependent-latency cycles per row (forward + backward) on B200: fp64
// DADD/DMUL/DFMA 8 cycles, fp32 4 (tools/microbench/dplat.cu).
int chain_cycles(bool pent, bool fast, std::size_t elem) {
  const int lat = elem == 8 ? 8 : 4;
  if (fast) return 2 * lat;
  return (pent ? 6 : 5) * lat;
}

// Persistent plan: as many systems per SM as the chain needs (2x margin over
// 1.125 rows/cycle/SM), all rows in smem when they fit, otherwise the head
// rows spill to L2 within kSpillBudget.
bool plan_persist(std::size_t n, std::size_t elem, bool pent, bool fast, int sms, Plan& p) {
  const std::size_t fr = fwd_rec_bytes(pent, elem), br = bwd_rec_bytes(pent, elem);
  const std::size_t fac = dev::align128(n * fr) + dev::align128(n * br);
  if (fac > kSmemPerBlockMax / 2) return false;
  const int tail_full_chunks = static_cast<int>((n + dev::kRT - 1) / dev::kRT);
  const int need_sys = static_cast<int>(2.0 * 1.125 * chain_cycles(pent, fast, elem));
  int target = std::max(2, std::min(dev::kMaxWarps, (need_sys + dev::kPW - 1) / dev::kPW));
  const bool forced_warps = tune_flag("PWARPS");
  if (forced_warps) target = std::max(1, std::min(dev::kMaxWarps, static_cast<int>(tune_int("PWARPS", 1))));
  const int forced_tail = static_cast<int>(tune_int("PTAIL", -1));

  auto fit = [&](int warps, int H, int TC) {
    return dev::PersistLayout::make(static_cast<int>(n), H, TC, warps, elem, fr, br).total <= kSmemPerBlockMax;
  };
  // 1) everything resident: the most warps that fit (at least `target`)
  if (forced_tail < 0) {
    int w = 0;
    for (int k = dev::kMaxWarps; k >= 1; --k)
      if (fit(k, 0, tail_full_chunks)) {
        w = k;
        break;
      }
    if (w >= target) {
      p.kind = PlanKind::Persist;
      p.warps = w;
      p.H = 0;
      p.TC = tail_full_chunks;
      p.smem_bytes = dev::PersistLayout::make(static_cast<int>(n), 0, p.TC, w, elem, fr, br).total;
      return true;
    }
  }
  // 2) spill the head: the largest tail that fits for `warps`, head in L2
  for (int warps = target; warps >= 1; --warps) {
    int best_tc = -1;
    for (int tc = tail_full_chunks; tc >= 0; --tc) {
      int tail_rows = std::min<int>(static_cast<int>(n), tc * dev::kRT);
      if (forced_tail >= 0) tail_rows = std::min<int>(static_cast<int>(n), forced_tail);
      int H = static_cast<int>(n) - tail_rows;
      H = (H + dev::kHAlign - 1) / dev::kHAlign * dev::kHAlign;  // head rows: whole ring chunks / reload blocks
      if (H > static_cast<int>(n)) H = static_cast<int>(n) / dev::kHAlign * dev::kHAlign;
      const int TC = (static_cast<int>(n) - H + dev::kRT - 1) / dev::kRT;
      if (H + TC * dev::kRT < static_cast<int>(n)) continue;
      if (fit(warps, H, TC)) {
        best_tc = TC;
        p.H = H;
        break;
      }
      if (forced_tail >= 0) break;
    }
    if (best_tc < 0) continue;
    const double spill = static_cast<double>(warps) * dev::kPW * sms * p.H * elem;
    if (spill <= kSpillBudget || warps == 1 || forced_tail >= 0 || forced_warps) {
      p.kind = PlanKind::Persist;
      p.warps = warps;
      p.TC = best_tc;
      p.smem_bytes = dev::PersistLayout::make(static_cast<int>(n), p.H, p.TC, warps, elem, fr, br).total;
      return true;
    }
  }
  return false;
}


// Measured fraction of HBM bandwidth the streaming kernel reaches with S
// systems per SM and no spill (B200, n = 256, 2^21 systems, V = 1, KR = 4;
// tools/gpu_calib.sh). Below S = 64 a warp's recurrence latency, not HBM,
// bounds the SM, so the fraction scales with S.
double stream_compute_frac(int S, bool pent, bool fast) {
  const double f64 = pent ? (fast ? 0.80 : 0.60) : (fast ? 0.93 : 0.72);
  const double f96 = pent ? (fast ? 0.82 : 0.87) : (fast ? 0.82 : 0.84);
  if (S <= 64) return f64 * S / 64.0;
  if (S <= 96) return f64 + (f96 - f64) * (S - 64) / 32.0;
  return f96 * (1.0 - 0.04 * (S - 96) / 32.0);
}

// Measured slowdown from the d-hat spill (total MB over all SMs): any spill
// costs ~20% (ring waits on L2 round trips); beyond ~45 MB the spill no
// longer stays L2-resident alongside the b/x streams and it falls off
// quickly (n = 512 / 1024 sweeps, tools/gpu_calib.sh).
double stream_spill_factor(double spill_mb) {
  static const double pts[][2] = {{0, 1.0}, {1, 0.82}, {45, 0.80}, {57, 0.74}, {65, 0.56}, {98, 0.40}, {200, 0.25}};
  const int np = sizeof(pts) / sizeof(pts[0]);
  if (spill_mb >= pts[np - 1][0]) return pts[np - 1][1];
  for (int k = 1; k < np; ++k)
    if (spill_mb <= pts[k][0]) {
      const double t = (spill_mb - pts[k - 1][0]) / (pts[k][0] - pts[k - 1][0]);
      return pts[k - 1][1] + t * (pts[k][1] - pts[k - 1][1]);
    }
  return pts[np - 1][1];
}

int env_int(const char* key, int dflt) { return static_cast<int>(tune_int(key, dflt)); }

// Streaming plan (sweep_stream.cuh): pick the systems per lane V, the group
// width Wg (systems per SM in flight), the head/tail split and the ring
// depths that maximise the calibrated throughput estimate
//   frac = compute(S) x spill_factor(spill) x (round utilisation),
// preferring the smaller spill on ties.
bool plan_stream(std::size_t n, std::size_t m, std::size_t elem, bool pent, bool fast, int sms, Plan& p,
                 int per_arrays = 0, bool allow_tmem = true, int only_wg = 0, bool allow_rc = false) {
  const std::size_t fr = fwd_rec_bytes(pent, elem), br = bwd_rec_bytes(pent, elem);
  const std::size_t fac = dev::align128(n * fr) + dev::align128(n * br);
  if (fac > kSmemPerBlockMax / 2 || n < 2) return false;
  const int forced_wg = only_wg ? only_wg : env_int("SWG", 0);
  const int forced_tail = env_int("STAIL", -1);
  // KR = 0: one FIFO ring of KB slots carries both the b chunks and the
  // spill reloads (every slot serves whichever head phase is running)
  const int KB = std::max(1, env_int("SKB", 4));
  const int KR = std::max(0, env_int("SKR", 4));
  const int PD = std::max(0, env_int("SPD", 4));
  // recompute tier (plain solves only): rows forced by BANDSOLVE_SRC (-1: none)
  const int forced_rc = allow_rc ? env_int("SRC", -1) : -1;
  const int forced_seg = env_int("SSEG", 0);
  const bool tm8 = allow_rc && env_int("TM8", 0) != 0;  // TMEM tier with 5..8 compute warps
  const int N = static_cast<int>(n);
  bool found = false;
  double best_t = 1e300;
  double best_spill = 1e300;
  int tmem_pick = 0;
  const int forced_v = env_int("SV", 0);
  for (int cand = 0; cand < 16; ++cand) {
    const int V = cand < 8 ? 1 : 2;
    const int P = cand < 8 ? cand + 1 : cand - 7;
    if (P > dev::stream_max_warps(V)) continue;
    if (forced_v && V != forced_v) continue;
    const int Wg = 32 * V * P;
    if (forced_wg && Wg != forced_wg) continue;
    const long long groups = (static_cast<long long>(m) + Wg - 1) / Wg;
    const long long grid = std::min<long long>(sms, groups);
    const bool tm_ok = allow_tmem && V == 1 && (P <= 4 || tm8) && env_int("TMEM", 1) != 0;
    const int tcap = tm_ok ? dev::stream_tmem_cap_chunks(P, elem) : 0;
    // recompute chunks / segment chunks for a head of h rows
    auto rc_for = [&](int h) {
      if (forced_rc < 0 || tcap == 0) return 0;
      return std::max(0, std::min(forced_rc / dev::kSR, h / dev::kSR - std::min(h / dev::kSR, tcap)));
    };
    const int seg = std::max(1, std::min(tcap, forced_seg > 0 ? forced_seg : tcap));
    auto ckpts_for = [&](int rc) { return rc > 0 ? (rc + seg - 1) / seg - 1 : 0; };
    auto fits = [&](int H, int TC) {
      return dev::StreamLayout::make(N, H, TC, Wg, KB, KR, elem, fr, br, per_arrays, ckpts_for(rc_for(H))).total <=
             kSmemPerBlockMax;
    };
    int H = -1;
    const int all_tc = (N + dev::kSR - 1) / dev::kSR;
    if (forced_tail >= 0) {
      const int t = std::min(N, forced_tail);
      H = (N - t + dev::kSR - 1) / dev::kSR * dev::kSR;
      if (H > N) H = N / dev::kSR * dev::kSR;
      if (!fits(H, (N - H + dev::kSR - 1) / dev::kSR)) continue;
    } else if (fits(0, all_tc)) {
      H = 0;
    } else {
      for (int tc = all_tc; tc >= 0; --tc) {
        int h = (N - tc * dev::kSR + dev::kSR - 1) / dev::kSR * dev::kSR;
        if (h < 0) h = 0;
        if (h > N) h = N / dev::kSR * dev::kSR;
        const int TC = (N - h + dev::kSR - 1) / dev::kSR;
        if (fits(h, TC)) {
          H = h;
          break;
        }
      }
    }
    if (H < 0) continue;
    const int TC = (N - H + dev::kSR - 1) / dev::kSR;
    // TMEM tier (V = 1, one warp per TMEM lane quadrant): up to 2 KB per system
    const int rc = rc_for(H);
    const int rtc = std::min(H / dev::kSR - rc, tcap);
    const double spill = static_cast<double>(grid) * Wg * (H - (rtc + rc) * dev::kSR) * elem;
    const double rounds = static_cast<double>(m) / (static_cast<double>(Wg) * sms);
    const double util = rounds / std::ceil(rounds);
    // fp32 fast mode: the fp64 fast calibration underrates wider groups
    // (measured tri N = 512, 2^20: Wg = 64 0.53, Wg = 96 0.78); the exact
    // curve ranks fp32 groups correctly
    const double frac = stream_compute_frac(Wg, pent, fast && elem == 8) * (V == 2 ? 0.95 : 1.0) *
                        stream_spill_factor(spill / (1 << 20)) * util *
                        (16.0 / (16.0 + 8.0 * rc * dev::kSR / N));  // the recomputed rows read b twice
    const double t = static_cast<double>(n) * m * 2.0 * elem / (frac * 6.5e12);
    // TMEM-tier rule (measured at N = 384..512, tools/gpu_calib.sh): with the
    // forward intermediates split over TMEM + smem, the largest group whose
    // residual L2 spill stays <= 30 MB wins (capped at 96 systems in fast
    // mode); the calibrated model below decides everything else.
    if (rtc > 0 && rc == 0 && elem == 8 && N >= 384 && Wg >= 96 && spill <= 30.0 * (1 << 20) &&
        Wg <= (fast ? 96 : 128) && !forced_wg) {
      tmem_pick = Wg;
    }
    if (!found || t < best_t * 0.995 || (t <= best_t * 1.005 && spill < best_spill)) {
      found = true;
      best_t = t;
      best_spill = spill;
      p.kind = PlanKind::Stream;
      p.Wg = Wg;
      p.H = H;
      p.TC = TC;
      p.KB = KB;
      p.KR = KR;
      p.PD = PD;
      p.stagger_ns = env_int("SSTAG", 0);
      p.warps = P;
      p.model_us = t * 1e6;
      p.smem_bytes = dev::StreamLayout::make(N, H, TC, Wg, KB, KR, elem, fr, br, per_arrays, ckpts_for(rc)).total;
      p.V = V;
      p.tmem_chunks = rtc;
      p.rc_chunks = rc;
      p.seg_chunks = rc > 0 ? seg : 0;
    }
  }
  if (found && tmem_pick && tmem_pick != p.Wg && forced_rc < 0) {
    // re-plan with the TMEM rule's group width (same layout rules)
    Plan q;
    if (plan_stream(n, m, elem, pent, fast, sms, q, per_arrays, allow_tmem, tmem_pick, allow_rc)) p = q;
  }
  return found;
}


Plan choose_plan(std::size_t n, std::size_t m, std::size_t ld, std::size_t elem, const void* x, bool pent,
                 bool fast, int sms) {
  Plan p;
  // BANDSOLVE_PLAN = stream | global | persist | smem | smemW8 | smemW16 | smemW32 (tuning / tests)
  const std::optional<std::string> force_s = tune_str("PLAN");
  const char* force = force_s ? force_s->c_str() : nullptr;
  int forced_w = 0;
  bool force_smem = false;
  bool force_persist = false;
  if (force) {
    force_persist = std::strcmp(force, "persist") == 0;
    if (std::strcmp(force, "global") == 0) {
      p.why = "forced global";
      return p;
    }
    if (std::strncmp(force, "smem", 4) == 0) {
      force_smem = true;
      if (std::strncmp(force, "smemW", 5) == 0) forced_w = std::atoi(force + 5);
    }
  }
  const bool aligned = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && ((ld * elem) % 16 == 0);
  if (!aligned) {
    p.why = "row pitch or base not 16-byte aligned (TMA rule)";
    return p;
  }
  if (n > static_cast<std::size_t>(INT_MAX) || m > static_cast<std::size_t>(INT_MAX) / 2) {
    p.why = "shape beyond 32-bit TMA coordinates";
    return p;
  }
  // Many long systems: once the forward intermediates mostly spill past L2,
  // the on-chip plans fall below two plain streaming passes (thread per
  // system in global memory: fwd read+write, bwd read+write at ~0.95 of HBM
  // each = 0.48 of the 16 B/row roofline). Measured with 2^20 systems:
  // tri/pent N=1536..4096 fp64 0.47-0.48 vs stream 0.24-0.41; fp32 N>=2048
  // 0.40 vs 0.15-0.31; at 65536 systems of 2048, 0.42 vs 0.27.
  if (!force && m >= static_cast<std::size_t>(sms) * 384 && n >= (elem == 8 ? 1536u : 2048u)) {
    p.why = "many long systems: two streaming passes beat the spilling on-chip plans";
    return p;
  }
  // Few long systems (< ~1 warp per SM) take the same order: with the TMEM
  // tier a streaming plan that fits beats the thread-per-system global sweep
  // (ADI axis 4096 x 4096 tri: 1.46x; 4096 x 1024: 1.39x; fp32 1024 x 4096:
  // 3.4x, measured); shapes no on-chip plan fits fall through to global.
  // (Fast mode first tries the partitioned path, partition.cu.)
  if (!force_smem && !force_persist && plan_stream(n, m, elem, pent, fast, sms, p, 0, true, 0, true)) return p;
  if (!force_smem && plan_persist(n, elem, pent, fast, sms, p)) return p;
  int best_sys = 0;
  for (int W : {8, 16, 32}) {
    if (forced_w && W != forced_w) continue;
    const std::size_t bytes = smem_bytes_for(n, W, elem);
    if (bytes > kSmemPerBlockMax) continue;
    int k = static_cast<int>(kSmemPerSm / (bytes + kSmemReservedPerCta));
    k = std::min(k, 32);
    const int sys = k * W;
    // prefer more systems in flight; on ties the wider (more coalesced) box
    if (sys > best_sys || (sys == best_sys && W > p.W)) {
      best_sys = sys;
      p.kind = PlanKind::Smem;
      p.W = W;
      p.smem_bytes = bytes;
      p.ctas_per_sm = k;
    }
  }
  if (p.kind != PlanKind::Smem) p.why = "tile does not fit shared memory";
  return p;
}

bool encode_map(CUtensorMap* map, void* x, std::size_t elem, long long n, long long m, long long ld, int box_w,
                int box_r) {
  auto encode = tensor_map_encoder();
  if (!encode) return false;
  const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(n)};
  const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(ld) * elem};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_r)};
  const cuuint32_t estride[2] = {1, 1};
  CUresult r = encode(map, elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x,
                      gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <typename K>
cudaError_t allow_big_smem(K kern);
// Set the large-smem attributes of `kern` once per device.
template <typename K>
cudaError_t allow_big_smem_once(K kern, std::atomic<uint64_t>& done) {
  int device = 0;
  if (cudaError_t e = cudaGetDevice(&device); e != cudaSuccess) return e;
  const uint64_t bit = device < 64 ? (1ull << device) : 0;
  if (bit && (done.load(std::memory_order_relaxed) & bit)) return cudaSuccess;
  cudaError_t e = allow_big_smem(kern);
  if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_relaxed);
  return e;
}

template <typename K>
cudaError_t allow_big_smem(K kern) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kSmemPerBlockMax));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}

template <typename T, int W, bool PENT, bool FAST>
cudaError_t launch_smem(const Plan& plan, T* x, int n, long long m, long long ld, const void* fwd,
                        const void* bwd, cudaStream_t s) {
  auto kern = dev::sweep_smem<T, W, kChunkRows, PENT, FAST>;
  static std::atomic<uint64_t> configured{0};  // one bit per device: attributes are per context
  if (cudaError_t e = allow_big_smem_once(kern, configured); e != cudaSuccess) return e;
  CUtensorMap map;
  if (!encode_map(&map, x, sizeof(T), n, m, ld, W, kChunkRows)) return cudaErrorInvalidValue;
  const long long grid = (m + W - 1) / W;
  kern<<<static_cast<unsigned>(grid), W, plan.smem_bytes, s>>>(map, x, n, m, ld, fwd, bwd);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <typename T, bool PENT, bool FAST>
cudaError_t launch_persist(const Plan& plan, T* x, int n, long long m, long long ld, const void* fwd,
                           const void* bwd, cudaStream_t s, int sms) {
  auto kern = dev::sweep_persist<T, PENT, FAST>;
  static std::atomic<uint64_t> configured{0};  // one bit per device: attributes are per context
  if (cudaError_t e = allow_big_smem_once(kern, configured); e != cudaSuccess) return e;
  CUtensorMap map_ring, map_tail;
  if (!encode_map(&map_ring, x, sizeof(T), n, m, ld, dev::kPW, dev::kRH) ||
      !encode_map(&map_tail, x, sizeof(T), n, m, ld, dev::kPW, dev::kRT))
    return cudaErrorInvalidValue;
  const long long tiles = (m + dev::kPW - 1) / dev::kPW;
  // spread small batches over all SMs before stacking warps per CTA
  int warps = plan.warps;
  if (tiles < static_cast<long long>(sms) * warps)
    warps = static_cast<int>(std::max<long long>(1, (tiles + sms - 1) / sms));
  const long long grid = std::min<long long>(sms, (tiles + warps - 1) / warps);
  const std::size_t smem = dev::PersistLayout::make(n, plan.H, plan.TC, warps, sizeof(T),
                                                    sizeof(typename dev::Recs<T, PENT>::Fwd),
                                                    sizeof(typename dev::Recs<T, PENT>::Bwd)).total;
  // head-row spill scratch, one H x 32 block per warp, stream-ordered so
  // concurrent launches on other streams never share it
  T* scratch = nullptr;
  if (plan.H > 0) {
    const std::size_t bytes = static_cast<std::size_t>(grid) * warps * plan.H * dev::kPW * sizeof(T);
    int device = 0;
    if (cudaGetDevice(&device) == cudaSuccess) ensure_l2_setaside(device, bytes);
    cudaError_t e = pool_malloc_async(reinterpret_cast<void**>(&scratch), bytes, s);
    if (e != cudaSuccess) return e;
  }
  kern<<<static_cast<unsigned>(grid), warps * 32, smem, s>>>(map_ring, map_tail, x, n, m, ld, plan.H, plan.TC,
                                                            tiles, fwd, bwd, scratch);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (scratch) {
    cudaError_t f = cudaFreeAsync(scratch, s);
    if (e == cudaSuccess) e = f;
  }
  return e;
}


template <typename T, int V, bool PENT, bool FAST, int PER = 0, bool CN = false, int TM = 0>
cudaError_t launch_stream_v(const Plan& plan, T* x, int n, long long m, long long ld, const void* fwd,
                            const void* bwd, cudaStream_t s, int sms, const dev::PerArgs& per_in = dev::PerArgs{}) {
  auto kern = dev::sweep_stream<T, V, PENT, FAST, PER, CN, TM>;
  dev::PerArgs per = per_in;
  per.tmem_chunks = TM ? plan.tmem_chunks : 0;
  per.rc_chunks = (TM >= 2 && !CN) ? plan.rc_chunks : 0;
  per.seg_chunks = per.rc_chunks > 0 ? plan.seg_chunks : 0;
  if (plan.warps > dev::stream_tm_warps(TM) && TM) return cudaErrorInvalidConfiguration;
  static std::atomic<uint64_t> configured{0};  // one bit per device: attributes are per context
  if (cudaError_t e = allow_big_smem_once(kern, configured); e != cudaSuccess) return e;
  CUtensorMap map;
  if (!encode_map(&map, x, sizeof(T), n, m, ld, 32 * V, dev::kSR)) return cudaErrorInvalidValue;
  const long long groups = (m + plan.Wg - 1) / plan.Wg;
  const long long grid = std::min<long long>(sms, groups);
  const int P = plan.Wg / (32 * V);
  T* scratch = nullptr;
  const int spilled_rows = plan.H - (per.tmem_chunks + per.rc_chunks) * dev::kSR;
  if (spilled_rows > 0) {
    const std::size_t bytes = static_cast<std::size_t>(grid) * plan.Wg * spilled_rows * sizeof(T);
    int device = 0;
    if (cudaGetDevice(&device) == cudaSuccess) ensure_l2_setaside(device, bytes);
    cudaError_t e = pool_malloc_async(reinterpret_cast<void**>(&scratch), bytes, s);
    if (e != cudaSuccess) return e;
  }
  // the scratch as rows of 32 V elements for the reload TMA (box: one chunk of all warps)
  CUtensorMap map_s = map;
  if (scratch) {
    const long long rows = grid * static_cast<long long>(P) * (spilled_rows / dev::kSR) * dev::kSR;
    if (!encode_map(&map_s, scratch, sizeof(T), rows, 32 * V, 32 * V, 32 * V, dev::kSR * P)) {
      cudaFreeAsync(scratch, s);
      return cudaErrorInvalidValue;
    }
  }
  kern<<<static_cast<unsigned>(grid), (P + 2) * 32, plan.smem_bytes, s>>>(map, x, n, m, ld, plan.H, plan.TC, plan.KB,
                                                                         plan.KR, plan.PD, plan.stagger_ns, groups, fwd, bwd,
                                                                         scratch, per, map_s);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (scratch) {
    cudaError_t f = cudaFreeAsync(scratch, s);
    if (e == cudaSuccess) e = f;
  }
  return e;
}

template <typename T, bool PENT, bool FAST>
cudaError_t launch_stream(const Plan& plan, T* x, int n, long long m, long long ld, const void* fwd,
                          const void* bwd, cudaStream_t s, int sms) {
  if (plan.V == 1 && plan.warps > 4 && (plan.tmem_chunks > 0 || plan.rc_chunks > 0))
    return launch_stream_v<T, 1, PENT, FAST, 0, false, 3>(plan, x, n, m, ld, fwd, bwd, s, sms);
  if (plan.V == 1 && plan.rc_chunks > 0)
    return launch_stream_v<T, 1, PENT, FAST, 0, false, 2>(plan, x, n, m, ld, fwd, bwd, s, sms);
  if (plan.V == 1 && plan.tmem_chunks > 0)
    return launch_stream_v<T, 1, PENT, FAST, 0, false, 1>(plan, x, n, m, ld, fwd, bwd, s, sms);
  if (plan.V == 2) return launch_stream_v<T, 2, PENT, FAST>(plan, x, n, m, ld, fwd, bwd, s, sms);
  return launch_stream_v<T, 1, PENT, FAST>(plan, x, n, m, ld, fwd, bwd, s, sms);
}


template <typename T, bool PENT, bool FAST>
cudaError_t launch_global(T* x, int n, long long m, long long ld, const void* fwd, const void* bwd,
                          cudaStream_t s, int sms = 148) {
  // thread per system: spread few systems over every SM (latency-bound regime)
  int threads = 128;
  while (threads > 32 && (m + threads - 1) / threads < sms) threads >>= 1;
  const long long grid = (m + threads - 1) / threads;
  const bool deep = m <= static_cast<long long>(sms) * 64 && n >= 256;  // few long systems
  // records in shared memory (16-byte rounded; the packed arrays are 256-byte padded)
  const int rec_f = (n * static_cast<int>(PENT ? sizeof(dev::PentFwd<T>) : sizeof(dev::TriFwd<T>)) + 15) / 16 * 16;
  const int rec_b = (n * static_cast<int>(PENT ? sizeof(dev::PentBwd<T>) : sizeof(T)) + 15) / 16 * 16;
  if (deep && static_cast<std::size_t>(rec_f + rec_b) <= kSmemPerBlockMax && !tune_flag("GLOBAL_NOREC")) {
    auto kern = dev::sweep_global_rec<T, PENT, FAST, 32>;  // 16-row blocks / L2 prefetch measured slower
    static std::atomic<uint64_t> configured{0};
    if (cudaError_t e = allow_big_smem_once(kern, configured); e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(grid), threads, rec_f + rec_b, s>>>(x, n, m, ld, fwd, bwd, rec_f, rec_b);
  } else if (deep)
    dev::sweep_global<T, PENT, FAST, 32><<<static_cast<unsigned>(grid), threads, 0, s>>>(x, n, m, ld, fwd, bwd);
  else
    dev::sweep_global<T, PENT, FAST><<<static_cast<unsigned>(grid), threads, 0, s>>>(x, n, m, ld, fwd, bwd);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <typename T, bool PENT, bool FAST>
cudaError_t dispatch(const Plan& plan, T* x, int n, long long m, long long ld, const void* fwd,
                     const void* bwd, cudaStream_t s, int sms) {
  if (plan.kind == PlanKind::Stream) return launch_stream<T, PENT, FAST>(plan, x, n, m, ld, fwd, bwd, s, sms);
  if (plan.kind == PlanKind::Persist) return launch_persist<T, PENT, FAST>(plan, x, n, m, ld, fwd, bwd, s, sms);
  if (plan.kind == PlanKind::Smem) {
    switch (plan.W) {
      case 8: return launch_smem<T, 8, PENT, FAST>(plan, x, n, m, ld, fwd, bwd, s);
      case 16: return launch_smem<T, 16, PENT, FAST>(plan, x, n, m, ld, fwd, bwd, s);
      case 32: return launch_smem<T, 32, PENT, FAST>(plan, x, n, m, ld, fwd, bwd, s);
      default: return cudaErrorInvalidValue;
    }
  }
  return launch_global<T, PENT, FAST>(x, n, m, ld, fwd, bwd, s, sms);
}

template <typename T>
cudaError_t dispatch_kind(const Plan& plan, bool pent, bool fast, T* x, int n, long long m, long long ld,
                          const void* fwd, const void* bwd, cudaStream_t s, int sms) {
  if (pent)
    return fast ? dispatch<T, true, true>(plan, x, n, m, ld, fwd, bwd, s, sms)
                : dispatch<T, true, false>(plan, x, n, m, ld, fwd, bwd, s, sms);
  return fast ? dispatch<T, false, true>(plan, x, n, m, ld, fwd, bwd, s, sms)
              : dispatch<T, false, false>(plan, x, n, m, ld, fwd, bwd, s, sms);
}

// ---- residual ---------------------------------------------------------------
// One thread per system, the reference's accumulation order
// (tri_solver.cpp:116-136, pent_solver.cpp:223-251) with separately rounded
// operations, then a max over systems. The per-system value is >= 0 and
// NaN-free (std::max drops NaNs), so the max can be taken on the bit pattern.
__device__ __forceinline__ double ref_max(double a, double b) { return (a < b) ? b : a; }

__global__ void residual_tri_kernel(const double* __restrict__ x, const double* __restrict__ rhs, int n,
                                    long long m, long long ld, const double* __restrict__ sub,
                                    const double* __restrict__ diag, const double* __restrict__ sup,
                                    double corner_tr, double corner_bl, unsigned long long* out) {
  using namespace dev;
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  double w = 0.0;
  if (j < m) {
    auto X = [&](int i) { return x[static_cast<long long>(i) * ld + j]; };
    double rmax = 0.0, dmax = 0.0;
    for (int i = 0; i < n; ++i) {
      double acc = mul_rn(diag[i], X(i));
      if (i > 0) acc = add_rn(acc, mul_rn(sub[i], X(i - 1)));
      if (i + 1 < n) acc = add_rn(acc, mul_rn(sup[i], X(i + 1)));
      if (i == 0) acc = add_rn(acc, mul_rn(corner_tr, X(n - 1)));
      if (i == n - 1) acc = add_rn(acc, mul_rn(corner_bl, X(0)));
      const double b = rhs[static_cast<long long>(i) * ld + j];
      rmax = ref_max(rmax, fabs(sub_rn(acc, b)));
      dmax = ref_max(dmax, fabs(b));
    }
    w = dmax > 0.0 ? __ddiv_rn(rmax, dmax) : rmax;
  }
  for (int o = 16; o > 0; o >>= 1) w = ref_max(w, __shfl_xor_sync(0xffffffffu, w, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(w)));
}

__global__ void residual_pent_kernel(const double* __restrict__ x, const double* __restrict__ rhs, int n,
                                     long long m, long long ld, const double* __restrict__ bands, int cyclic,
                                     double ca, double cb, double cd, double ce, unsigned long long* out) {
  using namespace dev;
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const double* a = bands;
  const double* b = bands + n;
  const double* c = bands + 2 * n;
  const double* d = bands + 3 * n;
  const double* e = bands + 4 * n;
  double w = 0.0;
  if (j < m) {
    auto X = [&](int i) { return x[static_cast<long long>(i) * ld + j]; };
    double rmax = 0.0, dmax = 0.0;
    for (int i = 0; i < n; ++i) {
      double acc = mul_rn(c[i], X(i));
      if (i >= 2) acc = add_rn(acc, mul_rn(a[i], X(i - 2)));
      if (i >= 1) acc = add_rn(acc, mul_rn(b[i], X(i - 1)));
      if (i + 1 < n) acc = add_rn(acc, mul_rn(d[i], X(i + 1)));
      if (i + 2 < n) acc = add_rn(acc, mul_rn(e[i], X(i + 2)));
      if (cyclic) {
        if (i == 0) acc = add_rn(acc, add_rn(mul_rn(ca, X(n - 2)), mul_rn(cb, X(n - 1))));
        if (i == 1) acc = add_rn(acc, mul_rn(ca, X(n - 1)));
        if (i == n - 2) acc = add_rn(acc, mul_rn(ce, X(0)));
        if (i == n - 1) acc = add_rn(acc, add_rn(mul_rn(cd, X(0)), mul_rn(ce, X(1))));
      }
      const double r = rhs[static_cast<long long>(i) * ld + j];
      rmax = ref_max(rmax, fabs(sub_rn(acc, r)));
      dmax = ref_max(dmax, fabs(r));
    }
    w = dmax > 0.0 ? __ddiv_rn(rmax, dmax) : rmax;
  }
  for (int o = 16; o > 0; o >>= 1) w = ref_max(w, __shfl_xor_sync(0xffffffffu, w, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(w)));
}

// ---- synthetic RHS (bit-identical to oracle_rhs_value) ------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void fill_rhs_kernel(T* __restrict__ x, int n, long long m, long long ld, uint64_t seed_hash,
                                uint64_t j_offset) {
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  for (int i = blockIdx.y; i < n; i += gridDim.y) {
    uint64_t h = splitmix64(seed_hash ^ static_cast<uint64_t>(i));
    h = splitmix64(h ^ (j_offset + static_cast<uint64_t>(j)));
    const double v = __dsub_rn(__dmul_rn(static_cast<double>(h >> 11), 0x1.0p-52), 1.0);
    x[static_cast<long long>(i) * ld + j] = static_cast<T>(v);
  }
}

// ---- periodic wrap correction (reference periodic.cpp:57-89, :172-208) -----
// Two phases so rows can be corrected in parallel without racing on the
// rows the coefficients read: (1) one thread per system forms its
// coefficient(s) from y_0 (y_1) and y_{n-1} (y_{n-2}) into coef[]; (2) a 2D
// grid applies x_i = y_i - w z_i (pent: - (z1_i t1 + z2_i t2)) to every row,
// the reference's operation order with separately rounded operations.
__global__ void periodic_coef_kernel(const double* __restrict__ x, int n, long long m, long long ld, bool pent,
                                     double c0, double c1, double c2, double c3, double* __restrict__ coef) {
  using namespace dev;
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  auto Y = [&](int i) { return x[static_cast<long long>(i) * ld + j]; };
  if (!pent) {
    // w = (y_0 + v_last * y_{n-1}) * scale                          periodic.cpp:80
    coef[j] = mul_rn(add_rn(Y(0), mul_rn(c0, Y(n - 1))), c1);
  } else {
    // periodic.cpp:189-194
    const double w1 = sub_rn(Y(0), Y(n - 1));
    const double w2 = sub_rn(Y(1), Y(n - 2));
    coef[j] = add_rn(mul_rn(c0, w1), mul_rn(c1, w2));
    coef[m + j] = add_rn(mul_rn(c2, w1), mul_rn(c3, w2));
  }
}

constexpr int kCorrRows = 16;  // rows per thread of the apply kernel

template <bool PENT>
__global__ void periodic_apply_kernel(double* __restrict__ x, int n, long long m, long long ld,
                                      const double* __restrict__ z1, const double* __restrict__ z2,
                                      const double* __restrict__ coef) {
  using namespace dev;
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int i0 = blockIdx.y * kCorrRows;
  const int i1 = min(n, i0 + kCorrRows);
  double* col = x + j;
  if constexpr (!PENT) {
    const double w = coef[j];
    for (int i = i0; i < i1; ++i)  // periodic.cpp:85: row -= w * z_i
      col[static_cast<long long>(i) * ld] = sub_rn(col[static_cast<long long>(i) * ld], mul_rn(w, __ldg(z1 + i)));
  } else {
    const double t1 = coef[j], t2 = coef[m + j];
    for (int i = i0; i < i1; ++i)  // periodic.cpp:203: row -= z1_i t1 + z2_i t2
      col[static_cast<long long>(i) * ld] = sub_rn(
          col[static_cast<long long>(i) * ld], add_rn(mul_rn(__ldg(z1 + i), t1), mul_rn(__ldg(z2 + i), t2)));
  }
}

// ---- Crank-Nicolson explicit half, periodic stencil (reference pde.cpp:73-114) --
// One thread per system walks its column with a register window of the
// stencil's neighbours (wrap-around rows preloaded), so each row of u is
// read once and each row of out written once; the reference's operation
// order with separately rounded operations:
//   diffusion  o = s*(u[i-1] + u[i+1]) + mid*u[i]                    (:85)
//   hyper      o = -s*(u[i-2] + u[i+2]) + s4*(u[i-1] + u[i+1]) + mid*u[i]   (:108)
constexpr int kStencilRows = 16;  // rows per thread of the stencil kernel

template <bool PENT>
__global__ void cn_rhs_kernel(const double* __restrict__ u, double* __restrict__ out, int n, long long m,
                              long long ld, double s, double s4, double mid) {
  using namespace dev;
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int i0 = blockIdx.y * kStencilRows;
  const int i1 = min(n, i0 + kStencilRows);
  auto U = [&](int i) {  // periodic row index (|offset| <= 2 < n)
    i = i < 0 ? i + n : (i >= n ? i - n : i);
    return u[static_cast<long long>(i) * ld + j];
  };
  double* o = out + j;
  if constexpr (!PENT) {
    double um = U(i0 - 1), ui = U(i0);
    for (int i = i0; i < i1; ++i) {
      const double up = U(i + 1);
      o[static_cast<long long>(i) * ld] = add_rn(mul_rn(s, add_rn(um, up)), mul_rn(mid, ui));
      um = ui;
      ui = up;
    }
  } else {
    double a2 = U(i0 - 2), a1 = U(i0 - 1), c = U(i0), b1 = U(i0 + 1);  // u[i-2], u[i-1], u[i], u[i+1]
    for (int i = i0; i < i1; ++i) {
      const double b2 = U(i + 2);
      const double t = add_rn(mul_rn(-s, add_rn(a2, b2)), mul_rn(s4, add_rn(a1, b1)));
      o[static_cast<long long>(i) * ld] = add_rn(t, mul_rn(mid, c));
      a2 = a1;
      a1 = c;
      c = b1;
      b1 = b2;
    }
  }
}

// band -> n x m replicated copy (the per-system engine's fill_replicated,
// pde.cpp:178-180)
__global__ void replicate_band_kernel(const double* __restrict__ band, double* __restrict__ out, long long n,
                                      long long m, long long ld) {
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  for (long long i = blockIdx.y; i < n; i += gridDim.y) out[i * ld + j] = band[i];
}

// ---- fused stencil + transpose for the ADI half steps ---------------------------
// out[c * ldo + r] = stencil_r(u)[r][c]: the periodic Crank-Nicolson explicit
// half along rows (same operation order as cn_rhs_kernel) written transposed,
// so the next implicit half sweeps the other axis with its systems
// interleaved. One read of u (32 x 32 tile + 2-row halos through smem) and one
// write of out per element instead of stencil and transpose as two passes.
template <bool PENT>
__global__ void cn_rhs_transpose_kernel(const double* __restrict__ u, double* __restrict__ out, int rows, int cols,
                                        long long ldi, long long ldo, double s, double s4, double mid) {
  using namespace dev;
  constexpr int H = PENT ? 2 : 1;
  __shared__ double tile[32 + 2 * H][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32 + 2 * H; k += blockDim.y) {
    int r = r0 + k - H;
    r = r < 0 ? r + rows : (r >= rows ? r - rows : r);  // periodic rows (|offset| <= 2 < rows)
    const int c = c0 + threadIdx.x;
    if (r0 + k - H < rows + H && c < cols) tile[k][threadIdx.x] = u[static_cast<long long>(r) * ldi + c];
  }
  __syncthreads();
  const int x = threadIdx.x;  // tile row r0 + x
  const int r = r0 + x;
  if (r >= rows) return;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k;
    if (c >= cols) break;
    const double* t = &tile[x + H][k];
    double o;
    if constexpr (!PENT) {
      o = add_rn(mul_rn(s, add_rn(t[-33], t[33])), mul_rn(mid, t[0]));
    } else {
      const double q = add_rn(mul_rn(-s, add_rn(t[-66], t[66])), mul_rn(s4, add_rn(t[-33], t[33])));
      o = add_rn(q, mul_rn(mid, t[0]));
    }
    out[static_cast<long long>(c) * ldo + r] = o;
  }
}

uint64_t host_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ---- per-thread staging context for host batches --------------------------------
constexpr int kStages = 4;
struct StageContext {
  int device = -1;
  int slot = 0;  // position in the device list (a device may be listed more than once)
  cudaStream_t streams[kStages] = {};
  void* buf[kStages] = {};
  std::size_t cap[kStages] = {};
};
// Freed when the thread exits (its streams and staging buffers). CUDA calls
// made after the runtime has been unloaded at process exit just return
// cudaErrorCudartUnloading, so the release is safe at any point.
struct StageContexts {
  std::vector<StageContext*> list;
  ~StageContexts() {
    for (StageContext* c : list) {
      int prev = -1;
      if (cudaGetDevice(&prev) == cudaSuccess && prev != c->device) cudaSetDevice(c->device);
      for (int s = 0; s < kStages; ++s) {
        if (c->streams[s]) cudaStreamSynchronize(c->streams[s]);
        if (c->buf[s]) cudaFree(c->buf[s]);
        if (c->streams[s]) cudaStreamDestroy(c->streams[s]);
      }
      if (prev >= 0 && prev != c->device) cudaSetDevice(prev);
      delete c;
    }
    cudaGetLastError();
  }
};
thread_local StageContexts t_contexts;

bandsolve_status stage_context(int device, int slot, StageContext** out) {
  for (StageContext* c : t_contexts.list)
    if (c->device == device && c->slot == slot) {
      *out = c;
      return BANDSOLVE_OK;
    }
  auto* c = new StageContext;
  c->device = device;
  c->slot = slot;
  t_contexts.list.push_back(c);  // owned from here on, even if a stream fails below
  for (int s = 0; s < kStages; ++s) BSB_CUDA(cudaStreamCreateWithFlags(&c->streams[s], cudaStreamNonBlocking));
  *out = c;
  return BANDSOLVE_OK;
}

}  // namespace

// ---------------------------------------------------------------------------------
int current_mode() {
  int m = g_mode.load(std::memory_order_relaxed);
  if (m < 0) {
    m = mode_from_env();
    g_mode.store(m, std::memory_order_relaxed);
  }
  return m;
}
void set_mode(int mode) { g_mode.store(mode, std::memory_order_relaxed); }
uint64_t kernel_launches() { return g_launches.load(std::memory_order_relaxed); }
void note_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

void release_device_factor(DeviceFactor& d) {
  if (!d.base) return;
  int prev = -1;
  if (cudaGetDevice(&prev) == cudaSuccess && prev != d.device) cudaSetDevice(d.device);
  cudaFree(d.base);
  if (prev >= 0 && prev != d.device) cudaSetDevice(prev);
  cudaGetLastError();
  d.base = nullptr;
}

Factor::~Factor() {
  for (DeviceFactor& d : devices) release_device_factor(d);
}

double* host_alloc_zeroed(std::size_t count, bool* pinned) {
  *pinned = false;
  const std::size_t bytes = count * sizeof(double);
  if (device_count_cached() > 0) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) == cudaSuccess) {
      std::memset(p, 0, bytes);
      *pinned = true;
      return static_cast<double*>(p);
    }
    cudaGetLastError();
  }
  return static_cast<double*>(std::calloc(count, sizeof(double)));
}

void host_free(double* p, bool pinned) {
  if (!p) return;
  if (pinned) cudaFreeHost(p);
  else std::free(p);
}

bool encode_tile_map(CUtensorMap* map, void* x, std::size_t elem, long long n, long long m, long long ld, int box_w,
                     int box_r) {
  return encode_map(map, x, elem, n, m, ld, box_w, box_r);
}
cudaError_t allow_max_smem(const void* kern) { return allow_big_smem(kern); }
std::size_t max_smem_per_block() { return kSmemPerBlockMax; }

bandsolve_status describe_plan(Kind kind, std::size_t n, std::size_t m, std::size_t ld, bool f32,
                               std::string& out) {
  alignas(16) static const double kProbe[2] = {0.0, 0.0};  // 16-byte aligned stand-in base
  int device = 0;
  int sms = 148;
  if (device_count_cached() > 0 && cudaGetDevice(&device) == cudaSuccess) sms = num_sms(device);
  cudaGetLastError();
  const bool pent = kind != Kind::Tri;
  const bool fast = current_mode() == BANDSOLVE_MODE_FAST;
  const Plan p = choose_plan(n, m, ld, f32 ? 4 : 8, kProbe, pent, fast, sms);
  char buf[256];
  const int KS = spike_blocks(n, m, ld, kProbe, sms, pent, f32 ? 4 : 8);
  const int K = f32 ? 0 : partition_blocks(n, m, sms, pent);
  int pkb = 0, prt = 0, pst = 0;
  const int PP = (KS > 0 || K > 0 || (f32 && (m % 4 != 0 || ld % 4 != 0)))
                     ? 0
                     : pipe_warps(n, f32 ? m / 2 : m, f32 ? ld / 2 : ld, kProbe, pent, sms, &pkb, &prt, &pst);
  if (PP > 0) {
    const std::size_t tm = std::min<std::size_t>(n, 256), rg = static_cast<std::size_t>(prt) * 16,
                      sm = static_cast<std::size_t>(pst) * 16;
    std::snprintf(buf, sizeof buf,
                  "pipe Wg=%d warps=%d+1 tmem=%zu reg-rows=%zu smem-rows=%zu l2-rows=%zu ring=%d%s (1 launch)",
                  (f32 ? 64 : 32) * PP, PP, tm, rg, sm, n - tm - rg - sm, pkb, f32 ? " fp32 pairs" : "");
  }
  else if (KS > 0)
    std::snprintf(buf, sizeof buf, "spike K=%d blocks of %zu rows, interface system %d, 1 launch (TMEM-resident blocks%s)",
                  KS, n / KS, (pent ? 4 : 2) * KS, KS > 8 ? (KS == 16 ? ", clusters of 2 CTAs" : ", clusters of 4 CTAs") : "");
  else if (K > 0)
    std::snprintf(buf, sizeof buf, "partition K=%d blocks of %zu rows, interface system %d (dense LU), 2 launches", K,
                  n / K, (pent ? 4 : 2) * K);
  else if (p.kind == PlanKind::Stream)
    std::snprintf(buf, sizeof buf, "stream Wg=%d V=%d warps=%d+2 recompute=%d(seg %d) tmem=%d head(L2)=%d tail(smem)=%d rings=%d/%d pd=%d smem=%zu B model=%.1f us",
                  p.Wg, p.V, p.warps, p.rc_chunks * dev::kSR, p.seg_chunks * dev::kSR, p.tmem_chunks * dev::kSR,
                  p.H - (p.tmem_chunks + p.rc_chunks) * dev::kSR, static_cast<int>(n) - p.H,
                  p.KB, p.KR, p.PD, p.smem_bytes, p.model_us);
  else if (p.kind == PlanKind::Persist)
    std::snprintf(buf, sizeof buf, "persist warps=%d systems/sm=%d head(L2)=%d tail(smem)=%d smem=%zu B", p.warps,
                  p.warps * dev::kPW, p.H, static_cast<int>(n) - p.H, p.smem_bytes);
  else if (p.kind == PlanKind::Smem)
    std::snprintf(buf, sizeof buf, "smem-tma W=%d R=%d smem=%zu B ctas/sm=%d systems/sm=%d", p.W, kChunkRows,
                  p.smem_bytes, p.ctas_per_sm, p.ctas_per_sm * p.W);
  else
    std::snprintf(buf, sizeof buf, "global-inplace (%s)", p.why.c_str());
  out = buf;
  return BANDSOLVE_OK;
}

bandsolve_status solve_device(const Factor& f, void* x, bool f32, std::size_t n, std::size_t m,
                              std::size_t ld, void* stream) {
  if (!x) return fail(BANDSOLVE_ERR_BAD_ARG, "null device pointer");
  if (n != f.n) return fail(BANDSOLVE_ERR_SHAPE_MISMATCH, "factor order != batch rows");
  if (ld < m) return fail(BANDSOLVE_ERR_BAD_ARG, "row pitch ld < m");
  if (m == 0) return BANDSOLVE_OK;
  if (n > static_cast<std::size_t>(INT_MAX)) return fail(BANDSOLVE_ERR_BAD_ARG, "n too large");
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  int device = 0;
  BSB_CUDA(cudaGetDevice(&device));
  const DeviceFactor* df = nullptr;
  bandsolve_status st = ensure_device_factor(f, device, &df);
  if (st != BANDSOLVE_OK) return st;
  const bool fast = current_mode() == BANDSOLVE_MODE_FAST;
  const bool pent = f.kind != Kind::Tri;
  const int p = f32 ? 1 : 0;
  const int q = fast ? 1 : 0;
  auto s = static_cast<cudaStream_t>(stream);
  const int sms = num_sms(device);
  if (fast && f32) {  // fp32: the one-pass partitioned kernel in float (1e-5 contract)
    bool done = false;
    st = spike_solve_device_f32(f, static_cast<float*>(x), n, m, ld, stream, sms, &done);
    if (st != BANDSOLVE_OK || done) return st;
  }
  if (fast && !f32) {
    bool done = false;
    st = spike_solve_device(f, static_cast<double*>(x), n, m, ld, stream, sms, &done);
    if (st != BANDSOLVE_OK || done) return st;
    st = partition_solve_device(f, static_cast<double*>(x), n, m, ld, stream, sms, &done);
    if (st != BANDSOLVE_OK || done) return st;
  }
  {  // every forward intermediate on chip, pipelined across groups (fp32: system pairs per lane)
    bool done = false;
    st = pipe_solve_device(pent, fast, df->fwd[p][q], df->bwd[p][q], static_cast<double*>(x), n, m, ld, stream, sms,
                           &done, nullptr, nullptr, f32);
    if (st != BANDSOLVE_OK || done) return st;
  }
  const Plan plan = choose_plan(n, m, ld, f32 ? 4 : 8, x, pent, fast, sms);
  cudaError_t err;
  if (f32)
    err = dispatch_kind<float>(plan, pent, fast, static_cast<float*>(x), static_cast<int>(n),
                               static_cast<long long>(m), static_cast<long long>(ld), df->fwd[p][q],
                               df->bwd[p][q], s, sms);
  else
    err = dispatch_kind<double>(plan, pent, fast, static_cast<double*>(x), static_cast<int>(n),
                                static_cast<long long>(m), static_cast<long long>(ld), df->fwd[p][q],
                                df->bwd[p][q], s, sms);
  if (err != cudaSuccess) return cuda_fail(err, "sweep launch");
  return BANDSOLVE_OK;
}

Periodic::~Periodic() {
  for (auto& d : devices) {
    int prev = -1;
    if (cudaGetDevice(&prev) == cudaSuccess && prev != d.first) cudaSetDevice(d.first);
    cudaFree(d.second);
    if (prev >= 0 && prev != d.first) cudaSetDevice(prev);
  }
  cudaGetLastError();
}

namespace {
bandsolve_status periodic_device_z(const Periodic& p, int device, const double** out) {
  std::lock_guard<std::mutex> lock(p.mu);
  for (const auto& d : p.devices)
    if (d.first == device) {
      *out = d.second;
      return BANDSOLVE_OK;
    }
  const std::size_t n = p.n;
  // z1 | z2 (correction kernel) followed by the fused-sweep arrays
  std::vector<double> host(2 * n + p.fused.size(), 0.0);
  std::memcpy(host.data(), p.z1.data(), n * sizeof(double));
  if (!p.z2.empty()) std::memcpy(host.data() + n, p.z2.data(), n * sizeof(double));
  std::memcpy(host.data() + 2 * n, p.fused.data(), p.fused.size() * sizeof(double));
  double* d = nullptr;
  BSB_CUDA(cudaMalloc(&d, host.size() * sizeof(double)));
  cudaError_t err = upload_sync(d, host.data(), host.size() * sizeof(double));
  if (err != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(err, "periodic z upload");
  }
  p.devices.emplace_back(device, d);
  *out = d;
  return BANDSOLVE_OK;
}

bandsolve_status launch_periodic_correct(const Periodic& p, double* x, std::size_t n, std::size_t m,
                                         std::size_t ld, cudaStream_t s) {
  int device = 0;
  BSB_CUDA(cudaGetDevice(&device));
  const double* z = nullptr;
  bandsolve_status st = periodic_device_z(p, device, &z);
  if (st != BANDSOLVE_OK) return st;
  const bool pent = p.kind != Kind::Tri;
  double* coef = nullptr;
  BSB_CUDA(pool_malloc_async(reinterpret_cast<void**>(&coef), (pent ? 2 : 1) * m * sizeof(double), s));
  const int threads = 128;
  const unsigned gx = static_cast<unsigned>((m + threads - 1) / threads);
  if (pent)
    periodic_coef_kernel<<<gx, threads, 0, s>>>(x, static_cast<int>(n), static_cast<long long>(m),
                                                static_cast<long long>(ld), true, p.cap_inv[0], p.cap_inv[1],
                                                p.cap_inv[2], p.cap_inv[3], coef);
  else
    periodic_coef_kernel<<<gx, threads, 0, s>>>(x, static_cast<int>(n), static_cast<long long>(m),
                                                static_cast<long long>(ld), false, p.v_last, p.scale, 0.0, 0.0, coef);
  const dim3 grid(gx, static_cast<unsigned>((n + kCorrRows - 1) / kCorrRows));
  if (pent)
    periodic_apply_kernel<true><<<grid, threads, 0, s>>>(x, static_cast<int>(n), static_cast<long long>(m),
                                                         static_cast<long long>(ld), z, z + n, coef);
  else
    periodic_apply_kernel<false><<<grid, threads, 0, s>>>(x, static_cast<int>(n), static_cast<long long>(m),
                                                          static_cast<long long>(ld), z, nullptr, coef);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  cudaFreeAsync(coef, s);
  BSB_CUDA(cudaGetLastError());
  return BANDSOLVE_OK;
}
}  // namespace

// One Crank-Nicolson step out = A^-1 (B u) in one streaming pass: the
// stencil is fused into the forward sweep (sweep_stream CN), and in fast
// mode the periodic correction as well (PER); exact mode follows with the
// bitwise correction kernel on `out`. Falls back to stencil kernel + solve
// when no streaming plan fits.
bandsolve_status cn_step_device(const Periodic& p, double sigma_x, const double* u, double* out, std::size_t n,
                                std::size_t m, std::size_t ld, void* stream) {
  if (!u || !out) return fail(BANDSOLVE_ERR_BAD_ARG, "null device pointer");
  if (u == out) return fail(BANDSOLVE_ERR_BAD_ARG, "the stencil needs distinct input and output arrays");
  if (n != p.n) return fail(BANDSOLVE_ERR_SHAPE_MISMATCH, "correction order != batch rows");
  if (ld < m) return fail(BANDSOLVE_ERR_BAD_ARG, "row pitch ld < m");
  if (m == 0) return BANDSOLVE_OK;
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  auto s = static_cast<cudaStream_t>(stream);
  const bool pent = p.kind != Kind::Tri;
  const bool fast = current_mode() == BANDSOLVE_MODE_FAST;
  int device = 0;
  BSB_CUDA(cudaGetDevice(&device));
  const int sms = num_sms(device);
  const bool aligned = (reinterpret_cast<uintptr_t>(u) % 16 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0) &&
                       ((ld * sizeof(double)) % 16 == 0);
  if (fast && aligned && !tune_flag("CN_UNFUSED") && spike_blocks(n, m, ld, out, sms, pent) > 0) {
    // many long systems: stencil + one-pass partitioned sweep + Woodbury
    // correction in one launch (sweep_spike.cuh, template CN)
    const double* blob = nullptr;
    bandsolve_status st = periodic_device_z(p, device, &blob);
    if (st != BANDSOLVE_OK) return st;
    PartPeriodic pa{blob, blob + n, {0.0, 0.0, 0.0, 0.0}};
    if (pent) {
      for (int k = 0; k < 4; ++k) pa.c[k] = p.cap_inv[k];
    } else {
      pa.c[0] = p.v_last;
      pa.c[1] = p.scale;
    }
    // pde.cpp:80-81 / :101-103
    const SpikeCN cn{u, {sigma_x, pent ? 4.0 * sigma_x : 0.0, pent ? 1.0 - 6.0 * sigma_x : 1.0 - 2.0 * sigma_x}};
    bool done = false;
    st = spike_solve_device(*p.factor, out, n, m, ld, stream, sms, &done, &pa, &cn);
    if (st != BANDSOLVE_OK || done) return st;
  }
  if (aligned && !tune_flag("CN_UNFUSED") && tune_flag("PIPE_CN")) {
    // stencil + pipelined on-chip sweep + correction (bitwise in exact mode),
    // one launch. Opt-in: the register pressure of the stencil + two backward
    // passes measured below the streaming CN kernel (pent N = 512 exact:
    // 0.24 with the register tier / 0.34 without, vs 0.37)
    const DeviceFactor* df = nullptr;
    bandsolve_status st = ensure_device_factor(*p.factor, device, &df);
    if (st != BANDSOLVE_OK) return st;
    const double* blob = nullptr;
    st = periodic_device_z(p, device, &blob);
    if (st != BANDSOLVE_OK) return st;
    PartPeriodic pa{blob, blob + n, {0.0, 0.0, 0.0, 0.0}};
    if (pent) {
      for (int k = 0; k < 4; ++k) pa.c[k] = p.cap_inv[k];
    } else {
      pa.c[0] = p.v_last;
      pa.c[1] = p.scale;
    }
    const SpikeCN cn{u, {sigma_x, pent ? 4.0 * sigma_x : 0.0, pent ? 1.0 - 6.0 * sigma_x : 1.0 - 2.0 * sigma_x}};
    bool done = false;
    st = pipe_solve_device(pent, fast, df->fwd[0][fast ? 1 : 0], df->bwd[0][fast ? 1 : 0], out, n, m, ld, stream, sms,
                           &done, &pa, &cn);
    if (st != BANDSOLVE_OK || done) return st;
  }
  Plan plan;
  if (!tune_flag("CN_UNFUSED") && aligned && n <= static_cast<std::size_t>(INT_MAX) &&
      m <= static_cast<std::size_t>(INT_MAX) / 2 &&
      plan_stream(n, m, sizeof(double), pent, fast, sms, plan, fast ? (pent ? 4 : 2) : 0)) {
    const DeviceFactor* df = nullptr;
    bandsolve_status st = ensure_device_factor(*p.factor, device, &df);
    if (st != BANDSOLVE_OK) return st;
    const double* blob = nullptr;
    st = periodic_device_z(p, device, &blob);
    if (st != BANDSOLVE_OK) return st;
    dev::PerArgs per;
    per.arrays = blob + 2 * n;
    if (pent) {
      for (int k = 0; k < 4; ++k) per.pc[k] = p.cap_inv[k];
    } else {
      per.pc[0] = p.v_last;
      per.pc[1] = p.scale;
    }
    per.out = out;
    // pde.cpp:80-81 / :101-103
    per.cn[0] = sigma_x;
    per.cn[1] = pent ? 4.0 * sigma_x : 0.0;
    per.cn[2] = pent ? 1.0 - 6.0 * sigma_x : 1.0 - 2.0 * sigma_x;
    const int N = static_cast<int>(n);
    const long long M = static_cast<long long>(m), LD = static_cast<long long>(ld);
    double* x = const_cast<double*>(u);  // read only (tensor map source); results go to per.out
    const int q = fast ? 1 : 0;
    const void* fw = df->fwd[0][q];
    const void* bw = df->bwd[0][q];
    cudaError_t err;
    const bool tm = plan.V == 1 && plan.tmem_chunks > 0;
    if (fast) {
      if (pent)
        err = tm ? launch_stream_v<double, 1, true, true, 2, true, true>(plan, x, N, M, LD, fw, bw, s, sms, per)
              : plan.V == 2 ? launch_stream_v<double, 2, true, true, 2, true>(plan, x, N, M, LD, fw, bw, s, sms, per)
                            : launch_stream_v<double, 1, true, true, 2, true>(plan, x, N, M, LD, fw, bw, s, sms, per);
      else
        err = tm ? launch_stream_v<double, 1, false, true, 1, true, true>(plan, x, N, M, LD, fw, bw, s, sms, per)
              : plan.V == 2 ? launch_stream_v<double, 2, false, true, 1, true>(plan, x, N, M, LD, fw, bw, s, sms, per)
                            : launch_stream_v<double, 1, false, true, 1, true>(plan, x, N, M, LD, fw, bw, s, sms, per);
    } else {
      if (pent)
        err = tm ? launch_stream_v<double, 1, true, false, 0, true, true>(plan, x, N, M, LD, fw, bw, s, sms, per)
              : plan.V == 2 ? launch_stream_v<double, 2, true, false, 0, true>(plan, x, N, M, LD, fw, bw, s, sms, per)
                            : launch_stream_v<double, 1, true, false, 0, true>(plan, x, N, M, LD, fw, bw, s, sms, per);
      else
        err = tm ? launch_stream_v<double, 1, false, false, 0, true, true>(plan, x, N, M, LD, fw, bw, s, sms, per)
              : plan.V == 2 ? launch_stream_v<double, 2, false, false, 0, true>(plan, x, N, M, LD, fw, bw, s, sms, per)
                            : launch_stream_v<double, 1, false, false, 0, true>(plan, x, N, M, LD, fw, bw, s, sms, per);
    }
    if (err != cudaSuccess) return cuda_fail(err, "fused Crank-Nicolson sweep launch");
    if (fast) return BANDSOLVE_OK;
    return launch_periodic_correct(p, out, n, m, ld, s);
  }
  bandsolve_status st = cn_rhs_device(pent, sigma_x, u, out, n, m, ld, stream);
  if (st != BANDSOLVE_OK) return st;
  return periodic_device(p, out, n, m, ld, stream, false);
}

bandsolve_status periodic_device(const Periodic& p, double* x, std::size_t n, std::size_t m, std::size_t ld,
                                 void* stream, bool correct_only) {
  if (!x) return fail(BANDSOLVE_ERR_BAD_ARG, "null device pointer");
  if (n != p.n) return fail(BANDSOLVE_ERR_SHAPE_MISMATCH, "correction order != batch rows");
  if (ld < m) return fail(BANDSOLVE_ERR_BAD_ARG, "row pitch ld < m");
  if (m == 0) return BANDSOLVE_OK;
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  auto s = static_cast<cudaStream_t>(stream);
  int device = 0;
  BSB_CUDA(cudaGetDevice(&device));
  const int sms = num_sms(device);
  const bool pent = p.kind != Kind::Tri;
  const bool fuse = !correct_only && current_mode() == BANDSOLVE_MODE_FAST &&
                    !tune_flag("PERIODIC_UNFUSED");
  if (fuse && (spike_blocks(n, m, ld, x, sms, pent) > 0 || partition_blocks(n, m, sms, pent) > 0)) {
    // many long systems: the one-pass partitioned sweep; few long systems:
    // the two-launch partitioned sweep; the correction fused into both
    const double* blob = nullptr;
    bandsolve_status st = periodic_device_z(p, device, &blob);
    if (st != BANDSOLVE_OK) return st;
    PartPeriodic pa{blob, blob + n, {0.0, 0.0, 0.0, 0.0}};
    if (pent) {
      for (int k = 0; k < 4; ++k) pa.c[k] = p.cap_inv[k];
    } else {
      pa.c[0] = p.v_last;
      pa.c[1] = p.scale;
    }
    bool done = false;
    st = spike_solve_device(*p.factor, x, n, m, ld, stream, sms, &done, &pa);
    if (st != BANDSOLVE_OK || done) return st;
    st = partition_solve_device(*p.factor, x, n, m, ld, stream, sms, &done, &pa);
    if (st != BANDSOLVE_OK || done) return st;
  }
  if (fuse && partition_blocks(n, m, sms, pent) == 0) {
    // fast mode: one fused pass (sweep_stream PER), when a streaming plan fits
    // (few long systems take the partitioned sweep + correction instead)
    const bool aligned = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && ((ld * sizeof(double)) % 16 == 0);
    Plan plan;
    if (aligned && n <= static_cast<std::size_t>(INT_MAX) && m <= static_cast<std::size_t>(INT_MAX) / 2 &&
        plan_stream(n, m, sizeof(double), pent, true, sms, plan, pent ? 4 : 2)) {
      const DeviceFactor* df = nullptr;
      bandsolve_status st = ensure_device_factor(*p.factor, device, &df);
      if (st != BANDSOLVE_OK) return st;
      const double* blob = nullptr;
      st = periodic_device_z(p, device, &blob);
      if (st != BANDSOLVE_OK) return st;
      dev::PerArgs per;
      per.arrays = blob + 2 * n;
      if (pent) {
        for (int k = 0; k < 4; ++k) per.pc[k] = p.cap_inv[k];
      } else {
        per.pc[0] = p.v_last;
        per.pc[1] = p.scale;
      }
      const int N = static_cast<int>(n);
      const long long M = static_cast<long long>(m), LD = static_cast<long long>(ld);
      cudaError_t err;
      const void* fw = df->fwd[0][1];
      const void* bw = df->bwd[0][1];
      const bool tm = plan.V == 1 && plan.tmem_chunks > 0;
      if (pent)
        err = tm ? launch_stream_v<double, 1, true, true, 2, false, true>(plan, x, N, M, LD, fw, bw, s, sms, per)
              : plan.V == 2 ? launch_stream_v<double, 2, true, true, 2>(plan, x, N, M, LD, fw, bw, s, sms, per)
                            : launch_stream_v<double, 1, true, true, 2>(plan, x, N, M, LD, fw, bw, s, sms, per);
      else
        err = tm ? launch_stream_v<double, 1, false, true, 1, false, true>(plan, x, N, M, LD, fw, bw, s, sms, per)
              : plan.V == 2 ? launch_stream_v<double, 2, false, true, 1>(plan, x, N, M, LD, fw, bw, s, sms, per)
                            : launch_stream_v<double, 1, false, true, 1>(plan, x, N, M, LD, fw, bw, s, sms, per);
      if (err != cudaSuccess) return cuda_fail(err, "fused periodic sweep launch");
      return BANDSOLVE_OK;
    }
  }
  if (!correct_only && !tune_flag("PERIODIC_UNFUSED")) {
    // exact mode (or fast without a fused plan): the pipelined on-chip sweep
    // with the bitwise correction fused (a first backward pass finds y_0..)
    const DeviceFactor* df = nullptr;
    bandsolve_status st = ensure_device_factor(*p.factor, device, &df);
    if (st != BANDSOLVE_OK) return st;
    const double* blob = nullptr;
    st = periodic_device_z(p, device, &blob);
    if (st != BANDSOLVE_OK) return st;
    PartPeriodic pa{blob, blob + n, {0.0, 0.0, 0.0, 0.0}};
    if (pent) {
      for (int k = 0; k < 4; ++k) pa.c[k] = p.cap_inv[k];
    } else {
      pa.c[0] = p.v_last;
      pa.c[1] = p.scale;
    }
    const bool fast = current_mode() == BANDSOLVE_MODE_FAST;
    bool done = false;
    st = pipe_solve_device(pent, fast, df->fwd[0][fast ? 1 : 0], df->bwd[0][fast ? 1 : 0], x, n, m, ld, stream, sms,
                           &done, &pa);
    if (st != BANDSOLVE_OK || done) return st;
  }
  if (!correct_only) {
    bandsolve_status st = solve_device(*p.factor, x, false, n, m, ld, stream);
    if (st != BANDSOLVE_OK) return st;
  }
  return launch_periodic_correct(p, x, n, m, ld, s);
}

// Fast-mode ADI half step in two launches: the explicit stencil across the
// systems of `src` (laid out src[j * lds + i]) fused into the partitioned
// forward pass, the periodic correction into the backward pass; *done =
// false when the shape does not qualify (caller runs stencil+transpose and
// periodic_device instead).
bandsolve_status periodic_stencil_partition(const Periodic& p, const double* src, std::size_t lds, double cs,
                                            double cs4, double cmid, double* x, std::size_t n, std::size_t m,
                                            std::size_t ld, void* stream, bool* done) {
  *done = false;
  if (current_mode() != BANDSOLVE_MODE_FAST || tune_flag("PERIODIC_UNFUSED") || tune_flag("ADI_UNFUSED"))
    return BANDSOLVE_OK;
  if (reinterpret_cast<uintptr_t>(src) % 16 != 0) return BANDSOLVE_OK;
  int device = 0;
  BSB_CUDA(cudaGetDevice(&device));
  const int sms = num_sms(device);
  const bool pent = p.kind != Kind::Tri;
  // tridiagonal only: the pentadiagonal variant (two neighbour rows per side
  // in registers) measured slower than stencil+transpose and the plain pass
  // (5.6e10 vs 6.7e10 rows/s at 4096^2); tri gains 1.11e11 -> 1.33e11
  if (pent && !tune_flag("ADI_FUSE_PENT")) return BANDSOLVE_OK;
  if (partition_blocks(n, m, sms, pent) == 0) return BANDSOLVE_OK;
  const double* blob = nullptr;
  bandsolve_status st = periodic_device_z(p, device, &blob);
  if (st != BANDSOLVE_OK) return st;
  PartPeriodic pa{blob, blob + n, {0.0, 0.0, 0.0, 0.0}};
  if (pent) {
    for (int k = 0; k < 4; ++k) pa.c[k] = p.cap_inv[k];
  } else {
    pa.c[0] = p.v_last;
    pa.c[1] = p.scale;
  }
  const PartStencil ps{src, lds, cs, cs4, cmid};
  return partition_solve_device(*p.factor, x, n, m, ld, stream, sms, done, &pa, &ps);
}

// ---- device list of the host-batch solves (bandsolve_set_devices) ------------------
namespace {
std::mutex g_dev_mu;
std::vector<int> g_devices;  // empty: the calling thread's current device
}  // namespace

bandsolve_status set_devices(const int* ids, int count) {
  if (count < 0 || (count > 0 && !ids)) return fail(BANDSOLVE_ERR_BAD_ARG, "bad device list");
  for (int k = 0; k < count; ++k)
    if (ids[k] < 0) return fail(BANDSOLVE_ERR_BAD_ARG, "negative device id");
  std::lock_guard<std::mutex> lock(g_dev_mu);
  g_devices.assign(ids, ids + count);
  return BANDSOLVE_OK;
}

int get_devices(int* ids, int capacity) {
  std::lock_guard<std::mutex> lock(g_dev_mu);
  const int count = static_cast<int>(g_devices.size());
  for (int k = 0; ids && k < std::min(count, capacity); ++k) ids[k] = g_devices[k];
  return count;
}

// Host-batch solve: the m columns are split over the device list exactly as
// the reference splits them over its workers (parallel.cpp:53-54, j0 =
// m*g/G); each shard streams ~64 MiB column chunks through its own device's
// staging pipeline (kStages streams: chunk k's H2D overlaps chunk k-1's sweep
// and chunk k-2's D2H), so each GPU's copies use that GPU's own PCIe link.
// One host thread issues everything asynchronously, round-robin over the
// shards, then waits for all of them. Columns are independent, so the result
// is bitwise the same for any device list.
bandsolve_status solve_host(const Factor& f, double* x, std::size_t n, std::size_t m, const Periodic* per,
                            bool correct_only) {
  if (n != f.n) return fail(BANDSOLVE_ERR_SHAPE_MISMATCH, "factor order != batch rows");
  if (m == 0) return BANDSOLVE_OK;
  const int ndev = device_count_cached();
  if (ndev == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  int caller = 0;
  BSB_CUDA(cudaGetDevice(&caller));
  std::vector<int> devs;
  {
    std::lock_guard<std::mutex> lock(g_dev_mu);
    devs = g_devices;
  }
  if (devs.empty()) devs.push_back(caller);
  for (int d : devs)
    if (d >= ndev) return fail(BANDSOLVE_ERR_BAD_ARG, "device list names a device that does not exist");

  struct Shard {
    int device;
    StageContext* ctx;
    std::size_t j0, j1, w, chunks;
    int stages;
  };
  const std::size_t G = devs.size();
  const std::size_t row_bytes = n * sizeof(double);
  const std::size_t chunk_mib = static_cast<std::size_t>(std::max(1, env_int("HOST_CHUNK_MIB", 64)));
  std::vector<Shard> shards;
  bandsolve_status st = BANDSOLVE_OK;
  for (std::size_t g = 0; g < G && st == BANDSOLVE_OK; ++g) {
    Shard sh{devs[g], nullptr, m * g / G, m * (g + 1) / G, 0, 0, 0};
    if (sh.j1 == sh.j0) continue;
    const std::size_t mg = sh.j1 - sh.j0;
    std::size_t w = (chunk_mib << 20) / row_bytes;
    w = std::max<std::size_t>(32, (w / 32) * 32);
    sh.w = std::min(w, mg);
    sh.chunks = (mg + sh.w - 1) / sh.w;
    sh.stages = static_cast<int>(std::min<std::size_t>(kStages, sh.chunks));
    if (cudaError_t e = cudaSetDevice(sh.device); e != cudaSuccess) {
      st = cuda_fail(e, "cudaSetDevice");
      break;
    }
    st = stage_context(sh.device, static_cast<int>(g), &sh.ctx);
    const std::size_t need = n * ((sh.w + 1) & ~std::size_t(1)) * sizeof(double);
    for (int q = 0; q < sh.stages && st == BANDSOLVE_OK; ++q) {
      StageContext* c = sh.ctx;
      if (c->cap[q] >= need) continue;
      cudaError_t e = cudaSuccess;
      if (c->buf[q]) {
        e = cudaStreamSynchronize(c->streams[q]);
        if (e == cudaSuccess) e = cudaFree(c->buf[q]);
        c->buf[q] = nullptr;
        c->cap[q] = 0;
      }
      if (e == cudaSuccess) e = cudaMalloc(&c->buf[q], need);
      if (e != cudaSuccess) st = cuda_fail(e, "staging buffer");
      else c->cap[q] = need;
    }
    shards.push_back(sh);
  }
  std::size_t max_chunks = 0;
  for (const Shard& sh : shards) max_chunks = std::max(max_chunks, sh.chunks);
  for (std::size_t k = 0; k < max_chunks && st == BANDSOLVE_OK; ++k) {
    for (const Shard& sh : shards) {
      if (k >= sh.chunks) continue;
      cudaError_t e = cudaSetDevice(sh.device);
      const int q = static_cast<int>(k % sh.stages);
      cudaStream_t strm = sh.ctx->streams[q];
      const std::size_t j0 = sh.j0 + k * sh.w;
      const std::size_t wk = std::min(sh.w, sh.j1 - j0);
      const std::size_t ldk = (wk + 1) & ~std::size_t(1);  // even pitch keeps the TMA path
      double* d = static_cast<double*>(sh.ctx->buf[q]);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(d, ldk * sizeof(double), x + j0, m * sizeof(double), wk * sizeof(double), n,
                              cudaMemcpyHostToDevice, strm);
      if (e != cudaSuccess) {
        st = cuda_fail(e, "host-to-device copy");
        break;
      }
      st = per ? periodic_device(*per, d, n, wk, ldk, strm, correct_only) : solve_device(f, d, false, n, wk, ldk, strm);
      if (st != BANDSOLVE_OK) break;
      e = cudaMemcpy2DAsync(x + j0, m * sizeof(double), d, ldk * sizeof(double), wk * sizeof(double), n,
                            cudaMemcpyDeviceToHost, strm);
      if (e != cudaSuccess) {
        st = cuda_fail(e, "device-to-host copy");
        break;
      }
    }
  }
  // drain every shard (also on failure: no copy may still target x after we return)
  for (const Shard& sh : shards) {
    cudaSetDevice(sh.device);
    for (int q = 0; q < sh.stages; ++q) {
      cudaError_t e = cudaStreamSynchronize(sh.ctx->streams[q]);
      if (e != cudaSuccess && st == BANDSOLVE_OK) st = cuda_fail(e, "staging stream");
    }
  }
  cudaSetDevice(caller);
  return st;
}

bandsolve_status cn_rhs_device(bool pent, double sigma_x, const double* u, double* out, std::size_t n,
                               std::size_t m, std::size_t ld, void* stream) {
  if (!u || !out) return fail(BANDSOLVE_ERR_BAD_ARG, "null device pointer");
  if (u == out) return fail(BANDSOLVE_ERR_BAD_ARG, "the stencil needs distinct input and output arrays");
  if (ld < m) return fail(BANDSOLVE_ERR_BAD_ARG, "row pitch ld < m");
  if (n < (pent ? 6u : 3u)) return fail(BANDSOLVE_ERR_BAD_ARG, "periodic stencil needs n >= 3 (tri) / 6 (pent)");
  if (n > static_cast<std::size_t>(INT_MAX)) return fail(BANDSOLVE_ERR_BAD_ARG, "n too large");
  if (m == 0) return BANDSOLVE_OK;
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  auto s = static_cast<cudaStream_t>(stream);
  const int threads = 128;
  const dim3 grid(static_cast<unsigned>((m + threads - 1) / threads),
                  static_cast<unsigned>((n + kStencilRows - 1) / kStencilRows));
  // pde.cpp:80-81 / :101-103: the coefficients are formed once on the host
  if (pent)
    cn_rhs_kernel<true><<<grid, threads, 0, s>>>(u, out, static_cast<int>(n), static_cast<long long>(m),
                                                 static_cast<long long>(ld), sigma_x, 4.0 * sigma_x,
                                                 1.0 - 6.0 * sigma_x);
  else
    cn_rhs_kernel<false><<<grid, threads, 0, s>>>(u, out, static_cast<int>(n), static_cast<long long>(m),
                                                  static_cast<long long>(ld), sigma_x, 0.0, 1.0 - 2.0 * sigma_x);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  BSB_CUDA(cudaGetLastError());
  return BANDSOLVE_OK;
}

bandsolve_status residual_device(Kind kind, const double* const* bands, std::size_t n, int cyclic,
                                 const double* x, const double* rhs, std::size_t m, std::size_t ld,
                                 void* stream, double* out) {
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  if (ld < m) return fail(BANDSOLVE_ERR_BAD_ARG, "row pitch ld < m");
  if (n > static_cast<std::size_t>(INT_MAX)) return fail(BANDSOLVE_ERR_BAD_ARG, "n too large");
  auto s = static_cast<cudaStream_t>(stream);
  const bool pent = kind != Kind::Tri;
  const int nb = pent ? 5 : 3;
  // bands as the residual reads them: constant bands + corners when cyclic
  // (tri_solver.cpp:149-156 via constant_tri_lhs; pent_solver.cpp:265-273)
  std::vector<double> host(nb * n + 1, 0.0);
  double corners[4] = {0, 0, 0, 0};
  if (cyclic) {
    if (!pent) {
      const double a = bands[0][1], b = bands[1][0], c = bands[2][0];
      for (std::size_t i = 0; i < n; ++i) {
        host[i] = a;
        host[n + i] = b;
        host[2 * n + i] = c;
      }
      host[0] = 0.0;
      host[2 * n + n - 1] = 0.0;
      corners[0] = a;
      corners[1] = c;
    } else {
      const double v[5] = {bands[0][2], bands[1][1], bands[2][0], bands[3][0], bands[4][0]};
      for (int k = 0; k < 5; ++k)
        for (std::size_t i = 0; i < n; ++i) host[k * n + i] = v[k];
      host[0] = host[1] = host[n] = 0.0;
      host[3 * n + n - 1] = host[4 * n + n - 1] = host[4 * n + n - 2] = 0.0;
      corners[0] = v[0];
      corners[1] = v[1];
      corners[2] = v[3];
      corners[3] = v[4];
    }
  } else {
    for (int k = 0; k < nb; ++k) std::memcpy(host.data() + k * n, bands[k], n * sizeof(double));
  }
  double* dbands = nullptr;
  unsigned long long* dout = nullptr;
  BSB_CUDA(pool_malloc_async(&dbands, host.size() * sizeof(double), s));
  BSB_CUDA(pool_malloc_async(&dout, sizeof(unsigned long long), s));
  BSB_CUDA(cudaMemcpyAsync(dbands, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  BSB_CUDA(cudaMemsetAsync(dout, 0, sizeof(unsigned long long), s));
  const int threads = 128;
  const unsigned grid = static_cast<unsigned>((m + threads - 1) / threads);
  if (grid > 0) {
    if (pent)
      residual_pent_kernel<<<grid, threads, 0, s>>>(x, rhs, static_cast<int>(n), static_cast<long long>(m),
                                                    static_cast<long long>(ld), dbands, cyclic, corners[0],
                                                    corners[1], corners[2], corners[3], dout);
    else
      residual_tri_kernel<<<grid, threads, 0, s>>>(x, rhs, static_cast<int>(n), static_cast<long long>(m),
                                                   static_cast<long long>(ld), dbands, dbands + n, dbands + 2 * n,
                                                   corners[0], corners[1], dout);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    BSB_CUDA(cudaGetLastError());
  }
  unsigned long long bits = 0;
  BSB_CUDA(cudaMemcpyAsync(&bits, dout, sizeof bits, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(dbands, s));
  BSB_CUDA(cudaFreeAsync(dout, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  double w;
  std::memcpy(&w, &bits, sizeof w);
  *out = w;
  return BANDSOLVE_OK;
}

// ---- 2D ADI step (configs[3]) -------------------------
// Peaceman-Rachford on a periodic ny x nx field C[y*ld + x]:
//   (I - s Lx) u* = (I + s Ly) u,   (I - s Ly) u' = (I + s Lx) u*
// with L the periodic second-difference (diffusion) or minus the fourth
// difference (hyperdiffusion) and the CN bands of pde.cpp:59-71. y-sweeps
// run on the field's own interleaved layout (rows = y, systems = x); the
// x-sweeps on its transpose (rows = x, systems = y).
bandsolve_status adi_step_device(const Periodic& px, const Periodic& py, double sigma, double* field, double* work,
                                 std::size_t nx, std::size_t ny, std::size_t ld, void* stream) {
  if (!field || !work) return fail(BANDSOLVE_ERR_BAD_ARG, "null device pointer");
  if (field == work) return fail(BANDSOLVE_ERR_BAD_ARG, "field and work must not alias");
  if (px.n != nx || py.n != ny) return fail(BANDSOLVE_ERR_SHAPE_MISMATCH, "ADI handle order != field shape");
  if (ld < nx) return fail(BANDSOLVE_ERR_BAD_ARG, "row pitch ld < nx");
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  auto s = static_cast<cudaStream_t>(stream);
  const bool pent = px.kind != Kind::Tri;
  const std::size_t ldt = (ny + 1) & ~std::size_t(1);  // transposed pitch (even: TMA plans)
  {
    int device = 0;
    BSB_CUDA(cudaGetDevice(&device));
  }
  // the transposed field lives in the caller's work array when it is large
  // enough (ny x ld doubles >= nx x ldt, 16-byte aligned: TMA), else in a
  // pool block for this step
  const bool own_t1 = !(reinterpret_cast<uintptr_t>(work) % 16 == 0 && ny * ld >= nx * ldt);
  double* t1 = own_t1 ? nullptr : work;
  if (own_t1) BSB_CUDA(pool_malloc_async(reinterpret_cast<void**>(&t1), nx * ldt * sizeof(double), s));
  // pde.cpp:80-81 / :101-103: the coefficients are formed once on the host
  const double cs = sigma, cs4 = pent ? 4.0 * sigma : 0.0, cmid = pent ? 1.0 - 6.0 * sigma : 1.0 - 2.0 * sigma;
  auto rhs_t = [&](const double* in, double* out, std::size_t rows, std::size_t cols, std::size_t ldi,
                   std::size_t ldo) {
    dim3 block(32, 8), grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
    if (pent)
      cn_rhs_transpose_kernel<true><<<grid, block, 0, s>>>(in, out, static_cast<int>(rows), static_cast<int>(cols),
                                                           static_cast<long long>(ldi), static_cast<long long>(ldo),
                                                           cs, cs4, cmid);
    else
      cn_rhs_transpose_kernel<false><<<grid, block, 0, s>>>(in, out, static_cast<int>(rows), static_cast<int>(cols),
                                                            static_cast<long long>(ldi), static_cast<long long>(ldo),
                                                            cs, cs4, cmid);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
  };
  bandsolve_status st = BANDSOLVE_OK;
  cudaError_t err;
  do {
    if (nx < (pent ? 6u : 3u) || ny < (pent ? 6u : 3u)) {
      st = fail(BANDSOLVE_ERR_BAD_ARG, "periodic stencil needs n >= 3 (tri) / 6 (pent)");
      break;
    }
    // half step 1: explicit along y, implicit along x (systems along x, interleaved after the transpose)
    bool done = false;
    if ((st = periodic_stencil_partition(px, field, ld, cs, cs4, cmid, t1, nx, ny, ldt, stream, &done)) !=
        BANDSOLVE_OK)
      break;
    if (!done) {
      if ((err = rhs_t(field, t1, ny, nx, ld, ldt)) != cudaSuccess) { st = cuda_fail(err, "ADI stencil"); break; }
      if ((st = periodic_device(px, t1, nx, ny, ldt, stream, false)) != BANDSOLVE_OK) break;
    }
    // half step 2: explicit along x, implicit along y
    if ((st = periodic_stencil_partition(py, t1, ldt, cs, cs4, cmid, field, ny, nx, ld, stream, &done)) !=
        BANDSOLVE_OK)
      break;
    if (!done) {
      if ((err = rhs_t(t1, field, nx, ny, ldt, ld)) != cudaSuccess) { st = cuda_fail(err, "ADI stencil"); break; }
      st = periodic_device(py, field, ny, nx, ld, stream, false);
    }
  } while (false);
  if (own_t1) cudaFreeAsync(t1, s);
  cudaGetLastError();
  return st;
}

// ---- Crank-Nicolson driver: bandsolve_bench_run (reference capi.cpp:369-411,
// pde.cpp run_benchmark :258-371) with the stepping loop on the GPU.
bandsolve_status bench_run_device(const bandsolve_bench_params& prm, bandsolve_bench_result* res,
                                  int threads_report) {
  // capi.cpp:374-401 and pde.cpp:258-277: the reference's checks, in order
  const bool diffusion = prm.problem == BANDSOLVE_PROBLEM_DIFFUSION;
  if (prm.problem != BANDSOLVE_PROBLEM_DIFFUSION && prm.problem != BANDSOLVE_PROBLEM_HYPERDIFFUSION)
    return fail(BANDSOLVE_ERR_BAD_ARG, "unknown problem");
  if (prm.variant != BANDSOLVE_VARIANT_SHARED && prm.variant != BANDSOLVE_VARIANT_PER_SYSTEM &&
      prm.variant != BANDSOLVE_VARIANT_UNIFORM && prm.variant != BANDSOLVE_VARIANT_CUSPARSE)
    return fail(BANDSOLVE_ERR_BAD_ARG, "unknown variant");
  const std::string prefix = prm.dump_prefix ? prm.dump_prefix : "";
  if (prm.dump_every > 0 && prefix.empty()) return fail(BANDSOLVE_ERR_BAD_ARG, "dump_every needs dump_prefix");
  const std::size_t n = prm.n, m = prm.m;
  if (n < 2 || m < 1) return fail(BANDSOLVE_ERR_BAD_ARG, "field shape must be at least 2 x 1");
  if (prm.steps < 1) return fail(BANDSOLVE_ERR_BAD_ARG, "steps must be >= 1");
  if (diffusion) {
    if (n < 3) return fail(BANDSOLVE_ERR_BAD_ARG, "diffusion benchmark needs n >= 3");
    if (prm.variant == BANDSOLVE_VARIANT_UNIFORM)
      return fail(BANDSOLVE_ERR_BAD_ARG, "uniform variant applies to hyperdiffusion only");
  } else if (n < 6) {
    return fail(BANDSOLVE_ERR_BAD_ARG, "hyperdiffusion benchmark needs n >= 6");
  }
  // pde.cpp:29-46: sigma_x = dt / (2 dx^p), default dt gives sigma_x = 1
  const double dx = 1.0 / static_cast<double>(n);
  const double pow_dx = diffusion ? dx * dx : dx * dx * dx * dx;
  const double dt = prm.dt > 0.0 ? prm.dt : 1.0 * 2.0 * pow_dx;
  const double sigma = dt / (2.0 * pow_dx);
  if (!(sigma > 0.0)) return fail(BANDSOLVE_ERR_BAD_ARG, "sigma_x must be positive");
  // preparation (outside the timed loop): periodic LHS of pde.cpp:59-71;
  // the uniform variant is bitwise the shared one (pent_solver.cpp:83-97)
  std::unique_ptr<Periodic> per;
  bandsolve_status st = diffusion ? make_periodic_tri(-sigma, 1.0 + 2.0 * sigma, -sigma, n, per)
                                  : make_periodic_pent(sigma, -4.0 * sigma, 1.0 + 6.0 * sigma, -4.0 * sigma,
                                                       sigma, n, per);
  if (st != BANDSOLVE_OK) return st;
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  // default_mode_initial, pde.cpp:48-58
  std::vector<double> field(n * m);
  const std::size_t mode_span = n / 4 > 0 ? n / 4 : 1;
  for (std::size_t j = 0; j < m; ++j) {
    const double k = static_cast<double>(1 + (j % mode_span));
    for (std::size_t i = 0; i < n; ++i) {
      const double xv = static_cast<double>(i + 1) / static_cast<double>(n);
      field[i * m + j] = std::sin(2.0 * 3.141592653589793238462643383279502884 * k * xv);  // std::numbers::pi
    }
  }
  // even pitch keeps the TMA plans; cuSPARSE's interleaved solvers take no pitch
  const bool cusp = prm.variant == BANDSOLVE_VARIANT_CUSPARSE;
  if (cusp && !cusparse_available()) return fail(BANDSOLVE_ERR_INTERNAL, "cuSPARSE comparator unavailable");
  const std::size_t ld = cusp ? m : (m + 1) & ~std::size_t(1);
  const std::size_t bytes = n * ld * sizeof(double);
  double *du = nullptr, *ds = nullptr;
  double* dbands = nullptr;  // per-system variant: A' bands (n each) | replicated copies (n x ld each)
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  auto cleanup = [&]() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (du) cudaFree(du);
    if (ds) cudaFree(ds);
    if (dbands) cudaFree(dbands);
    if (s) cudaStreamDestroy(s);
    cudaGetLastError();
  };
  // per-system variant (pde.cpp:168-185, :199-221): every step rewrites
  // replicated band copies of A', solves per system, then corrects. The
  // cuSPARSE variant (extension) is the same step with gtsv/gpsvInterleavedBatch
  // as the per-system solver (the paper's cuThomasBatch protocol).
  const bool per_sys = prm.variant == BANDSOLVE_VARIANT_PER_SYSTEM || cusp;
  const int nb = diffusion ? 3 : 5;
  auto step = [&](const double* from, double* to) -> bandsolve_status {
    if (!per_sys) return cn_step_device(*per, sigma, from, to, n, m, ld, s);
    bandsolve_status q = cn_rhs_device(!diffusion, sigma, from, to, n, m, ld, s);
    if (q != BANDSOLVE_OK) return q;
    double* arr[6];
    const dim3 grid(static_cast<unsigned>((m + 127) / 128), static_cast<unsigned>(std::min<std::size_t>(n, 4096)));
    for (int b = 0; b < nb; ++b) {
      arr[b] = dbands + nb * n + static_cast<std::size_t>(b) * n * ld;
      replicate_band_kernel<<<grid, 128, 0, s>>>(dbands + b * n, arr[b], static_cast<long long>(n),
                                                 static_cast<long long>(m), static_cast<long long>(ld));
    }
    g_launches.fetch_add(nb, std::memory_order_relaxed);
    arr[nb] = to;
    q = cusp ? cusparse_solve_device(!diffusion, arr, to, n, m, 0, s) : per_system_device(!diffusion, arr, n, m, ld, s);
    if (q != BANDSOLVE_OK) return q;
    return launch_periodic_correct(*per, to, n, m, ld, s);
  };
  cudaError_t err = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (err == cudaSuccess && per_sys) {
    err = cudaMalloc(&dbands, (nb * n + static_cast<std::size_t>(nb) * n * ld) * sizeof(double));
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(dbands, per->factor->bands.data(), nb * n * sizeof(double), cudaMemcpyHostToDevice, s);
  }
  if (err == cudaSuccess) err = cudaMalloc(&du, bytes);
  if (err == cudaSuccess) err = cudaMalloc(&ds, bytes);
  if (err == cudaSuccess) err = cudaEventCreate(&e0);
  if (err == cudaSuccess) err = cudaEventCreate(&e1);
  if (err == cudaSuccess)
    err = cudaMemcpy2DAsync(du, ld * sizeof(double), field.data(), m * sizeof(double), m * sizeof(double), n,
                            cudaMemcpyHostToDevice, s);
  if (err != cudaSuccess) {
    cleanup();
    return cuda_fail(err, "bench setup");
  }
  // one untimed warm-up step into the scratch buffer; the field is untouched
  st = step(du, ds);
  std::vector<double> per_step;
  per_step.reserve(static_cast<std::size_t>(prm.steps));
  for (long k = 0; st == BANDSOLVE_OK && k < prm.steps; ++k) {
    cudaEventRecord(e0, s);
    st = step(du, ds);
    cudaEventRecord(e1, s);
    if (st != BANDSOLVE_OK) break;
    err = cudaEventSynchronize(e1);
    if (err != cudaSuccess) {
      st = cuda_fail(err, "bench step");
      break;
    }
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    per_step.push_back(static_cast<double>(ms) * 1e-3);
    std::swap(du, ds);
    if (prm.dump_every > 0 && (k + 1) % prm.dump_every == 0) {
      err = cudaMemcpy2D(field.data(), m * sizeof(double), du, ld * sizeof(double), m * sizeof(double), n,
                         cudaMemcpyDeviceToHost);
      if (err != cudaSuccess) {
        st = cuda_fail(err, "bench dump");
        break;
      }
      st = ibat_write((prefix + "_step" + std::to_string(k + 1) + ".ibat").c_str(), field.data(), n, m);
    }
  }
  cleanup();
  if (st != BANDSOLVE_OK) return st;
  // pde.cpp:351-370 timing report; batch.cpp:72-111 storage footprint
  double total = 0.0;
  for (double t : per_step) total += t;
  const double mean = total / static_cast<double>(per_step.size());
  double var = 0.0;
  for (double t : per_step) var += (t - mean) * (t - mean);
  res->wall_s = total;
  res->per_step_mean_s = mean;
  res->per_step_std_s = per_step.size() > 1 ? std::sqrt(var / static_cast<double>(per_step.size() - 1)) : 0.0;
  const uint64_t un = n, um = m;
  res->elements = per_sys ? (diffusion ? 4 : 6) * un * um
                 : diffusion ? 3 * un + un * um
                             : (prm.variant == BANDSOLVE_VARIANT_UNIFORM ? 4 * un + un * um : 5 * un + un * um);
  res->threads = threads_report;
  res->steps = prm.steps;
  return BANDSOLVE_OK;
}

bandsolve_status residual_host(Kind kind, const double* const* bands, std::size_t n, int cyclic, const double* x,
                               const double* rhs, std::size_t m, double* out) {
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  int device = 0;
  BSB_CUDA(cudaGetDevice(&device));
  StageContext* ctx = nullptr;
  bandsolve_status st = stage_context(device, 0, &ctx);
  if (st != BANDSOLVE_OK) return st;
  cudaStream_t s = ctx->streams[0];
  const std::size_t bytes = n * m * sizeof(double);
  double *dx = nullptr, *dr = nullptr;
  BSB_CUDA(pool_malloc_async(&dx, bytes, s));
  BSB_CUDA(pool_malloc_async(&dr, bytes, s));
  BSB_CUDA(cudaMemcpyAsync(dx, x, bytes, cudaMemcpyHostToDevice, s));
  BSB_CUDA(cudaMemcpyAsync(dr, rhs, bytes, cudaMemcpyHostToDevice, s));
  st = residual_device(kind, bands, n, cyclic, dx, dr, m, m, s, out);
  cudaFreeAsync(dx, s);
  cudaFreeAsync(dr, s);
  cudaStreamSynchronize(s);
  return st;
}

bandsolve_status fill_rhs_device(void* x, bool f32, std::size_t n, std::size_t m, std::size_t ld, uint64_t seed,
                                 uint64_t j_offset, void* stream) {
  if (!x) return fail(BANDSOLVE_ERR_BAD_ARG, "null device pointer");
  if (ld < m) return fail(BANDSOLVE_ERR_BAD_ARG, "row pitch ld < m");
  if (n == 0 || m == 0) return BANDSOLVE_OK;
  if (device_count_cached() == 0) return fail(BANDSOLVE_ERR_INTERNAL, "no CUDA device available (no CPU fallback)");
  auto s = static_cast<cudaStream_t>(stream);
  const int threads = 256;
  dim3 grid(static_cast<unsigned>((m + threads - 1) / threads), static_cast<unsigned>(std::min<std::size_t>(n, 64)));
  const uint64_t sh = host_splitmix64(seed);
  if (f32)
    fill_rhs_kernel<float><<<grid, threads, 0, s>>>(static_cast<float*>(x), static_cast<int>(n),
                                                    static_cast<long long>(m), static_cast<long long>(ld), sh, j_offset);
  else
    fill_rhs_kernel<double><<<grid, threads, 0, s>>>(static_cast<double*>(x), static_cast<int>(n),
                                                     static_cast<long long>(m), static_cast<long long>(ld), sh, j_offset);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  BSB_CUDA(cudaGetLastError());
  return BANDSOLVE_OK;
}

}  // namespace bsb
