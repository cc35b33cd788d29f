// One-pass partitioned ("spike") shared-LHS sweep for MANY long systems,
// fast mode, fp64 (sm_100a).
//
// Why: a sequential sweep needs every forward intermediate of a system on
// chip until its backward sweep, and an SM must keep ~100 dependency chains
// in flight to pull HBM bandwidth. At N = 1024 that is ~800 KB per SM, more
// than TMEM + shared memory + registers; the spill to L2 caps the
// sequential plans near 0.5 of the HBM roofline (configs[4]).
//
// Because the LHS is shared, the partition method moves the per-system
// storage to per-BLOCK storage at no extra HBM traffic: each system of
// n = K L rows is split into K blocks (partition.cu build_plan: block
// factors, the forward images F of the left coupling columns, rows 0/1 of
// each block's U^-1, and the inverse of the R x R interface matrix, all per
// matrix, computed once on the host). One compute warp owns block k of 32
// systems, so a lane holds only L <= 128 forward values — half of its TMEM
// lane (warps w and w + 4 share lane quadrant w % 4) — and an SM runs
// 8 warps x 32 = 256 independent chains, two warps per scheduler:
//
//   forward   b streams in through a TMA ring (one {32 x 16} box per warp
//             and chunk); the lane runs the block-local forward recurrence,
//             gathers 16 rows and writes them to its TMEM lane with one
//             tcgen05.st.32x32b.x32, and accumulates the two (one)
//             interface dot products with the U^-1 rows;
//   interface each warp publishes its block's interface values of y =
//             A_k^-1 b_k in shared memory; after a barrier every lane forms
//             the x interface unknowns it needs (own bottom rows, the left
//             neighbour's bottom rows) as rows of R^-1 times the system's y
//             interface vector;
//   backward  from its own bottom x values the lane sweeps up over the TMEM
//             values (one tcgen05.ld per 16 rows, one chunk ahead), folding
//             the left coupling in as g_i - F_i x_left, and streams x to HBM.
//
// Systems longer than 8 blocks (N = 2048, 4096: K = 16, 32) span a thread-
// block CLUSTER of K / 8 CTAs, one per SM: each CTA holds 8 blocks of the
// same 32 systems in its TMEM, the interface values travel through
// distributed shared memory (ld.shared::cluster) after the hardware cluster
// barrier, and each CTA keeps only the R^-1 rows its blocks need.
//
// Software pipeline across groups: after the interface solve of group g a
// warp interleaves, chunk by chunk, the backward sweep of g with the forward
// sweep of g + 1 (two independent dependency chains per warp; b is read
// while x is written, so the SM's HBM traffic never comes in read-only /
// write-only bursts). Forward chunk k of a group with parity p lives in TMEM
// slot p ? CL-1-k : k, so in step k both use the slot the backward frees.
// Each 16-row chunk is computed in two stages so the dependency chain holds
// ONE fp64 FMA per row: first everything that does not depend on the
// recurrence (b * (1/alpha), the left-coupling update), for all 16 rows,
// then the chain itself.
//
// HBM traffic: read b once, write x once (16 B/row). Arithmetic differs
// from the sequential sweep by rounding only (fast mode, 1e-12 contract),
// exactly as the two-launch partitioned path of partition.cu.
#pragma once

#include "sweep_stream.cuh"

namespace bsb {
namespace dev {

constexpr int kSpR = 16;       // rows per chunk: one TMA box {32 systems, 16 rows} per warp
constexpr int kSpWarps = 8;    // compute warps: two per TMEM lane quadrant, 256 columns each
constexpr int kSpMaxL = 128;   // rows per block: 1 KB of TMEM lane per fp64 value
constexpr int kSpMaxK = 32;    // blocks per system (a cluster of up to 4 CTAs)
constexpr int kSpMaxCS = 4;    // CTAs per cluster

// per-row records in shared memory, split by phase (fp64 or fp32: the
// fp32 kernel runs the same plan rounded to float)
template <typename T, bool PENT>
struct SpF;  // forward: fast records + U^-1 row entries
template <typename T>
struct alignas(16) SpF<T, true> {
  T e, b, ia, p0;  // e = eps/alpha, b = beta/alpha, ia = 1/alpha (block-local); U^-1 row 1 in its own array
};
template <typename T>
struct alignas(16) SpF<T, false> {
  T am, m, p0, pad;  // am = a/denom, m = 1/denom
};
template <typename T, bool PENT>
struct SpB;  // backward: U entries + forward images of the left coupling
template <typename T>
struct alignas(16) SpB<T, true> {
  T g, d, f1, f2;  // gamma, delta, F (x_{s-2}), F (x_{s-1})
};
template <typename T>
struct alignas(16) SpB<T, false> {
  T c, f1;  // chat, F (x_{s-1})
};
// rows per block: one lane's TMEM share (256 columns) holds 128 fp64 / 256 fp32 values
template <typename T>
__host__ __device__ constexpr int spike_max_rows() { return 256 * 4 / static_cast<int>(sizeof(T)); }

// periodic (Woodbury) correction fused into the backward sweep: x_i -=
// z1_i t1 + z2_i t2, the coefficients from x_0, x_1, x_{n-2}, x_{n-1}, which
// are interface unknowns (periodic.cpp:57-89, :172-208; fast-mode rounding)
struct SpikePer {
  const double* z1 = nullptr;
  const double* z2 = nullptr;
  double c[4] = {0.0, 0.0, 0.0, 0.0};  // tri: v_last, scale; pent: cap_inv
  // Crank-Nicolson step (template CN): the right-hand side is the explicit
  // periodic stencil of the old field u (the tensor map's source, read
  // only), pde.cpp:73-114; x receives u_new. cn = s, 4s (pent), 1-2s / 1-6s
  const double* u = nullptr;
  double cn[3] = {0.0, 0.0, 0.0};
  // Decay cut-offs (block-local chunks): the U^-1 rows feeding the interface
  // dot products and the forward images of the left coupling decay away from
  // the block top; past chunk dp / df every entry is below 1e-18 of the
  // vector's largest, so those FMAs are skipped (fast mode only; far below
  // its rounding; plain pentadiagonal kernels). Defaults: never skip.
  int dp = 1 << 30;
  int df = 1 << 30;
};

// Rows of R^-1 a CTA keeps (its blocks kb0 .. kb0+Kc-1): the bottom NH
// unknowns of blocks kb0-1 .. kb0+Kc-1, then (periodic) the system's first
// and last NH unknowns.
__host__ __device__ constexpr int spike_rinv_rows(int Kc, int nh) { return (Kc + 3) * nh; }

struct SpikeLayout {
  size_t fwd_off, p1_off, bwd_off, z_off, rinv_off, xch_off, ring_off, bar_off, total;
  // nl: rows whose records this CTA holds; R: interface unknowns; Kc: blocks
  // per CTA; elem: 8 (fp64) / 4 (fp32)
  // rec: record / R^-1 element size (0: elem; 4 for the paired fp32 kernel)
  __host__ __device__ static SpikeLayout make(int nl, int R, int Kc, int KB, bool pent, bool per = false,
                                              size_t elem = 8, size_t rec = 0) {
    SpikeLayout L{};
    if (rec == 0) rec = elem;
    const size_t sf = rec == 8 ? (pent ? sizeof(SpF<double, true>) : sizeof(SpF<double, false>))
                               : (pent ? sizeof(SpF<float, true>) : sizeof(SpF<float, false>));
    const size_t sb = rec == 8 ? (pent ? sizeof(SpB<double, true>) : sizeof(SpB<double, false>))
                               : (pent ? sizeof(SpB<float, true>) : sizeof(SpB<float, false>));
    L.fwd_off = 0;
    // pent: U^-1 row 1 as a plain array (a 16-byte aligned 5-value record
    // would carry a pad word: 8 KB at N = 1024, the room of a fourth ring slot)
    L.p1_off = align128(static_cast<size_t>(nl) * sf);
    L.bwd_off = L.p1_off + (pent ? align128(static_cast<size_t>(nl) * rec) : 0);
    L.z_off = L.bwd_off + align128(static_cast<size_t>(nl) * sb);
    // z of the periodic correction: [nl] pairs (pent) / values (tri)
    L.rinv_off = L.z_off + (per ? align128(static_cast<size_t>(nl) * (pent ? 2 : 1) * sizeof(double)) : 0);
    L.xch_off = L.rinv_off + align128(static_cast<size_t>(spike_rinv_rows(Kc, pent ? 2 : 1)) * R * rec);
    // interface exchange, double-buffered: [2][warp][q][32 lanes]
    L.ring_off = L.xch_off + align128(2ull * kSpWarps * (pent ? 4 : 2) * 32 * elem);
    L.bar_off = L.ring_off + static_cast<size_t>(KB) * kSpWarps * kSpR * 32 * elem;
    // ring barriers, the TMEM base word
    L.total = L.bar_off + static_cast<size_t>(2 * KB + 1) * sizeof(uint64_t);
    return L;
  }
};

// ---- cluster primitives ----------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {  // own smem -> CTA rank's
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ double ld_cluster_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ float ld_cluster_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ float2 ld_cluster_f32x2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}
template <typename T>
__device__ __forceinline__ T ld_cluster(uint32_t addr) {
  if constexpr (std::is_same<T, float2>::value) return ld_cluster_f32x2(addr);
  else if constexpr (sizeof(T) == 8) return ld_cluster_f64(addr);
  else return ld_cluster_f32(addr);
}

// A lane's value type T: double (fp64), float (fp32), or float2 — two fp32
// systems per lane, packed FFMA2 arithmetic, moved and stored exactly like
// one fp64 value (8 bytes per lane and row). Records stay scalar (Scalar<T>).
template <typename T>
struct ScalarOf {
  using type = T;
};
template <>
struct ScalarOf<float2> {
  using type = float;
};
template <typename T>
using Scalar = typename ScalarOf<T>::type;
__device__ __forceinline__ double vfma(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float vfma(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ float2 vfma(float a, float2 b, float2 c) { return __ffma2_rn(make_float2(a, a), b, c); }
__device__ __forceinline__ double vmul(double b, double a) { return b * a; }
__device__ __forceinline__ float vmul(float b, float a) { return b * a; }
__device__ __forceinline__ float2 vmul(float2 b, float a) { return __fmul2_rn(b, make_float2(a, a)); }
// TMEM words: a float2 rides in the 64-bit slot of a double
template <typename T>
using TPieceOf = TPiece<std::conditional_t<sizeof(T) == 4, float, double>>;
template <typename T>
__device__ __forceinline__ auto to_word(T v) {
  if constexpr (std::is_same<T, float2>::value)
    return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(__float_as_uint(v.y)) << 32) |
                                                       __float_as_uint(v.x)));
  else return v;
}
template <typename T, typename W>
__device__ __forceinline__ T from_word(W w) {
  if constexpr (std::is_same<T, float2>::value) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(w));
    return make_float2(__uint_as_float(static_cast<unsigned>(u)), __uint_as_float(static_cast<unsigned>(u >> 32)));
  } else {
    return w;
  }
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// CS: CTAs per cluster (1; 2 / 4 for K = 16 / 32), a compile-time constant:
// with a runtime CS the single-CTA kernel measured 30% slower (tri N = 512:
// 0.68 vs 0.96 of the HBM roofline)
template <typename T, bool PENT, bool PER, bool CN = false, int CS = 1>
__global__ void __launch_bounds__(32 * (kSpWarps + 1), 1)
    sweep_spike(const __grid_constant__ CUtensorMap map_b, T* __restrict__ x, int n, long long m, long long ld,
                int K, int L, int KB, int PD, long long groups, const void* __restrict__ recs,
                const Scalar<T>* __restrict__ rinv_g, T* __restrict__ sink, SpikePer per) {
  static_assert(std::is_same<T, double>::value || (!PER && !CN), "fp32: plain solves only");
  using S = Scalar<T>;  // record / R^-1 type
  using F = SpF<S, PENT>;
  using B = SpB<S, PENT>;
  using TP = TPieceOf<T>;
  constexpr int NQ = PENT ? 4 : 2;  // interface rows per block (top NH, bottom NH)
  // decay cut-offs (SpikePer::dp / df): compiled into the plain pentadiagonal
  // kernels only, where they measured faster (configs[4] 0.78 -> 0.81; the
  // tri and Crank-Nicolson instances measured slower with the extra branch)
  constexpr bool kCut = PENT && !CN;
  constexpr int NH = NQ / 2;
  extern __shared__ __align__(128) unsigned char smem[];
  const int R = NQ * K;
  // CS == 1: the CTA holds all K blocks of G = 8/K groups of 32 systems;
  // CS > 1: it holds blocks [kb0, kb0 + 8) of one group (G = 1)
  const int rank = CS > 1 ? static_cast<int>(cluster_rank()) : 0;
  const int Kc = CS > 1 ? kSpWarps : K;
  const int kb0 = rank * Kc;
  const int G = CS > 1 ? 1 : kSpWarps / K;
  const int Wg = 32 * G;
  const int nl = Kc * L;      // rows whose records this CTA holds
  const int row0 = kb0 * L;   // first of them
  const long long cid = blockIdx.x / CS;  // cluster (group walker) index
  const long long ncl = gridDim.x / CS;
  const SpikeLayout Ly = SpikeLayout::make(nl, R, Kc, KB, PENT, PER, sizeof(T), sizeof(S));
  F* sf = reinterpret_cast<F*>(smem + Ly.fwd_off);
  S* sp1 = reinterpret_cast<S*>(smem + Ly.p1_off);
  B* sb = reinterpret_cast<B*>(smem + Ly.bwd_off);
  S* srinv = reinterpret_cast<S*>(smem + Ly.rinv_off);
  T* xch = reinterpret_cast<T*>(smem + Ly.xch_off);
  T* ring = reinterpret_cast<T*>(smem + Ly.ring_off);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Ly.bar_off);
  uint64_t* empty = full + KB;
  uint32_t& tmem_base_s = *reinterpret_cast<uint32_t*>(empty + KB);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int kBox = kSpR * 32;          // elements of one warp's box
  constexpr int kChunk = kSpWarps * kBox;  // elements of one ring slot
  const int CL = L / kSpR;                 // chunks per block

  {  // this CTA's records, its R^-1 rows and z -> smem
    const uint4* srcf = static_cast<const uint4*>(recs);
    const uint4* srcb = reinterpret_cast<const uint4*>(static_cast<const F*>(recs) + n);
    uint4* dstf = reinterpret_cast<uint4*>(smem + Ly.fwd_off);
    uint4* dstb = reinterpret_cast<uint4*>(smem + Ly.bwd_off);
    constexpr int wf = sizeof(F) / 16, wb = sizeof(B) / 16;
    for (int i = threadIdx.x; i < nl * wf; i += blockDim.x) dstf[i] = srcf[static_cast<size_t>(row0) * wf + i];
    for (int i = threadIdx.x; i < nl * wb; i += blockDim.x) dstb[i] = srcb[static_cast<size_t>(row0) * wb + i];
    if constexpr (PENT) {  // blob: [F x n][B x n][p1 x n][R^-1]
      const S* srcp = reinterpret_cast<const S*>(static_cast<const B*>(static_cast<const void*>(srcb)) + n);
      for (int i = threadIdx.x; i < nl; i += blockDim.x) sp1[i] = srcp[row0 + i];
    }
    const int nr = spike_rinv_rows(Kc, NH);
    for (int i = threadIdx.x; i < nr * R; i += blockDim.x) {
      const int t = i / R, c = i - t * R;
      int row;  // global row of R^-1 kept at local row t
      if (t < (Kc + 1) * NH) {
        const int kk = kb0 - 1 + t / NH;  // block whose bottom unknowns these are
        row = kk < 0 ? 0 : NQ * kk + NH + t % NH;
      } else if (t < (Kc + 2) * NH) {
        row = t - (Kc + 1) * NH;  // the system's first NH unknowns (block 0 top)
      } else {
        row = R - NH + (t - (Kc + 2) * NH);  // its last NH unknowns
      }
      srinv[i] = rinv_g[static_cast<size_t>(row) * R + c];
    }
    if constexpr (PER) {
      double* z = reinterpret_cast<double*>(smem + Ly.z_off);
      for (int i = threadIdx.x; i < nl; i += blockDim.x) {
        if constexpr (PENT) {
          z[2 * i] = per.z1[row0 + i];
          z[2 * i + 1] = per.z2[row0 + i];
        } else {
          z[i] = per.z1[row0 + i];
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < KB; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSpWarps);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_512(&tmem_base_s);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (CS > 1) cluster_sync_all();  // every CTA's barriers are initialised before remote arrivals
  // Programmatic dependent launch: the prologue above (records, barriers,
  // TMEM) overlaps the previous kernel's tail; the batch itself is touched
  // only after the previous grid has completed and flushed. The next launch
  // may be scheduled as soon as SMs free up.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // block / group slot of warp w, and the global first row of its block
  auto blk_of = [&](int w) { return CS > 1 ? kb0 + w : w % K; };
  auto gs_of = [&](int w) { return CS > 1 ? 0 : w / K; };

  if (warp == kSpWarps) {  // ---- producer: b chunks through the ring
    // (clusters: the other lanes exit, which takes them out of the cluster
    // barrier; lane 0 arrives once per group, see below)
    if (CS > 1 && lane != 0) return;
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const long long my_groups = (groups - cid + ncl - 1) / ncl;
      const long long total = my_groups * CL;
      long long pf = 0;
      auto chunk_at = [&](long long t, int& c0, int& c) {
        const long long gi = t / CL;
        c = static_cast<int>(t - gi * CL);
        c0 = static_cast<int>((cid + gi * ncl) * Wg);
      };
      int slot = 0;
      uint32_t phase = 0;
      for (long long t = 0; t < total; ++t) {
        for (; pf < total && pf < t + PD; ++pf) {  // keep PD chunks ahead in L2
          int c0, c;
          chunk_at(pf, c0, c);
          for (int w = 0; w < kSpWarps; ++w) tma_prefetch_2d(&map_b, c0 + gs_of(w) * 32, blk_of(w) * L + c * kSpR);
        }
        if (t >= KB) mbar_wait(&empty[slot], phase ^ 1u);
        int c0, c;
        chunk_at(t, c0, c);
        mbar_expect_tx(&full[slot], kChunk * sizeof(T));
        for (int w = 0; w < kSpWarps; ++w)
          tma_load_2d(ring + slot * kChunk + w * kBox, &map_b, c0 + gs_of(w) * 32, blk_of(w) * L + c * kSpR,
                      &full[slot], pol);
        if (++slot == KB) {
          slot = 0;
          phase ^= 1u;
        }
        if constexpr (CS > 1) {
          // one arrival per group's interface barrier (split phase: the wait
          // for the previous group's comes just before the next arrival, so
          // the ring keeps filling across the barrier)
          if (c == CL - 1) {
            if (t >= CL) asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
            asm volatile("barrier.cluster.arrive.release;" ::: "memory");
          }
        }
      }
      if constexpr (CS > 1) {
        if (total > 0) asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
        // the final cluster barrier (below) for this lane
        asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
        return;
      }
    }
  } else {
    // ---- compute warps: block k of the 32 systems of group slot gs
    const int k = blk_of(warp);
    const int gs = gs_of(warp);
    const int r0 = k * L;           // global first row of the block
    const int rl = r0 - row0;       // its first row in this CTA's records
    const uint32_t tlane = tmem_base_s + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                           static_cast<uint32_t>((warp >> 2) * 256);
    auto tslot = [&](uint32_t p, int c) {
      return tlane + static_cast<uint32_t>((p ? CL - 1 - c : c) * TP::kWords);
    };
    int slot = 0;
    uint32_t phase = 0;
    const F* fk = sf + rl;
    const S* p1k = sp1 + rl;
    const B* bk = sb + rl;
    const double* zk = reinterpret_cast<const double*>(smem + Ly.z_off) + (PENT ? 2 : 1) * rl;

    // forward state of the group being read, backward state of the one being written
    T fs1{}, fs2{}, a0{}, a1{};
    T bs1{}, bs2{}, xl1{}, xl2{}, t1{}, t2{};
    long long step = 0;
    T* out = sink + lane;
    TP cur;

    // CN: the stencil's halo rows. h1/h2 = u at the two rows above the chunk
    // (carried from the previous chunk; block starts load them), la0/la1 = the
    // two rows below it (plain loads issued one chunk ahead; the next block's
    // first rows at the block end), all with the periodic wrap.
    double h1 = 0.0, h2 = 0.0, la0 = 0.0, la1 = 0.0, nh1 = 0.0, nh2 = 0.0, nla0 = 0.0, nla1 = 0.0;
    auto u_at = [&](long long g, int row) -> double {  // u[row mod n] of this lane's system in group g
      if constexpr (CN) {
        row = row < 0 ? row + n : (row >= n ? row - n : row);
        long long j = g * Wg + gs * 32 + lane;
        j = j < m ? j : m - 1;
        return __ldg(per.u + static_cast<long long>(row) * ld + j);
      } else {
        return 0.0;
      }
    };
    auto halo_prefetch = [&](long long g) {  // chunk 0's halo of group g
      if constexpr (CN) {
        nh2 = u_at(g, r0 - 2);
        nh1 = u_at(g, r0 - 1);
        nla0 = u_at(g, r0 + kSpR);
        nla1 = u_at(g, r0 + kSpR + 1);
      }
    };

    auto fwd_chunk = [&](int c, uint32_t p, long long g) {
      mbar_wait(&full[slot], phase);
      const T* blk = ring + slot * kChunk + warp * kBox + lane;
      const F* fc = fk + c * kSpR;
      const S* p1c = p1k + c * kSpR;
      TP buf;
      T dv[kSpR];  // stage 1: b / pivot for the whole chunk (off the chain)
      if constexpr (CN) {
        if (c == 0) {
          h2 = nh2;
          h1 = nh1;
          la0 = nla0;
          la1 = nla1;
        }
        // the next chunk's look-ahead rows (the next block's first rows at the end)
        const int nb = (c + 2) * kSpR;
        const double n0 = c + 1 < CL ? u_at(g, r0 + nb) : 0.0;
        const double n1 = c + 1 < CL ? u_at(g, r0 + nb + 1) : 0.0;
        double e[kSpR + 4];  // u rows -2 .. kSpR + 1 of the chunk
        e[0] = h2;
        e[1] = h1;
#pragma unroll
        for (int r = 0; r < kSpR; ++r) e[r + 2] = blk[r * 32];
        e[kSpR + 2] = la0;
        e[kSpR + 3] = la1;
        const double cs = per.cn[0], cs4 = per.cn[1], cmid = per.cn[2];
#pragma unroll
        for (int r = 0; r < kSpR; ++r) {
          double f;
          if constexpr (PENT)  // pde.cpp:108  o = -s*(u2 + d2) + s4*(u1 + d1) + mid*mi
            f = (-cs * (e[r] + e[r + 4]) + cs4 * (e[r + 1] + e[r + 3])) + cmid * e[r + 2];
          else  // pde.cpp:85  o = s*(up + dn) + mid*mi
            f = cs * (e[r + 1] + e[r + 3]) + cmid * e[r + 2];
          if constexpr (PENT) dv[r] = f * fc[r].ia;
          else dv[r] = f * fc[r].m;
        }
        h2 = e[kSpR];
        h1 = e[kSpR + 1];
        la0 = n0;
        la1 = n1;
      } else {
#pragma unroll
        for (int r = 0; r < kSpR; ++r) {
          if constexpr (PENT) dv[r] = vmul(blk[r * 32], fc[r].ia);
          else dv[r] = vmul(blk[r * 32], fc[r].m);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == KB) {
        slot = 0;
        phase ^= 1u;
      }
      if (!kCut || c < per.dp) {
#pragma unroll
        for (int r = 0; r < kSpR; ++r) {  // stage 2: one FMA per row on the chain
          const F f = fc[r];
          T v;
          if constexpr (PENT) {
            v = vfma(-f.b, fs1, vfma(-f.e, fs2, dv[r]));
            a1 = vfma(p1c[r], v, a1);
          } else {
            v = vfma(-f.am, fs1, dv[r]);
          }
          a0 = vfma(f.p0, v, a0);
          fs2 = fs1;
          fs1 = v;
          buf.put(r, to_word(v));
        }
      } else {  // U^-1 rows 0/1 have decayed: no interface accumulation
#pragma unroll
        for (int r = 0; r < kSpR; ++r) {
          const F f = fc[r];
          T v;
          if constexpr (PENT) v = vfma(-f.b, fs1, vfma(-f.e, fs2, dv[r]));
          else v = vfma(-f.am, fs1, dv[r]);
          fs2 = fs1;
          fs1 = v;
          buf.put(r, to_word(v));
        }
      }
      buf.store(tslot(p, c));
    };

    auto corr = [&](int i, T v) {  // stored value of local row i (periodic correction)
      if constexpr (!PER) return v;
      else if constexpr (PENT) return fma(-zk[2 * i], t1, fma(-zk[2 * i + 1], t2, v));
      else return fma(-zk[i], t1, v);
    };

    // interface of the group just read (xch parity p): its backward state
    auto interface = [&](long long g, uint32_t p) {
      T* xw = xch + (static_cast<size_t>(p) * kSpWarps + warp) * NQ * 32 + lane;
      xw[0] = a0;
      if constexpr (PENT) {
        xw[32] = a1;
        xw[64] = vfma(-bk[L - 2].g, fs1, fs2);  // y_{L-2} = g_{L-2} - gamma_{L-2} g_{L-1}
        xw[96] = fs1;                          // y_{L-1} = g_{L-1}
      } else {
        xw[32] = fs1;
      }
      fs1 = fs2 = a0 = a1 = T{};
      if (CS == 1) {
        asm volatile("bar.sync 1, %0;" ::"r"(kSpWarps * 32) : "memory");
      } else {  // every warp of every CTA of the cluster has published its values
        // the hardware cluster barrier (every compute thread of every CTA,
        // plus each producer's one arrival per group)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                         "memory");
      }
      // x interface unknowns needed here, streamed over the R y values:
      // [own bottom NH | left bottom NH | (PER) first NH | last NH]
      constexpr int NU = PER ? 4 * NH : 2 * NH;
      int rows[NU];
#pragma unroll
      for (int h = 0; h < NU; ++h)
        rows[h] = h < NH       ? (k - kb0 + 1) * NH + h
                  : h < 2 * NH ? (k - kb0) * NH + (h - NH)
                               : (Kc + 1) * NH + (h - 2 * NH);
      T zu[NU];
#pragma unroll
      for (int h = 0; h < NU; ++h) zu[h] = T{};
      const uint32_t xbase = smem_u32(xch + static_cast<size_t>(p) * kSpWarps * NQ * 32 + lane);
      if constexpr (CS == 1) {
        for (int kk = 0; kk < K; ++kk) {
          T yv[NQ];
          const T* src = xch + ((static_cast<size_t>(p) * kSpWarps + gs * K + kk) * NQ) * 32 + lane;
#pragma unroll
          for (int q = 0; q < NQ; ++q) yv[q] = src[q * 32];
#pragma unroll
          for (int h = 0; h < NU; ++h) {
            const S* rr = srinv + static_cast<size_t>(rows[h]) * R + kk * NQ;
#pragma unroll
            for (int q = 0; q < NQ; ++q) zu[h] = vfma(rr[q], yv[q], zu[h]);
          }
        }
      } else {
        // K = 8 CS blocks, their y values in the CTAs of the cluster: the
        // remote (DSMEM) loads of KU blocks are issued back to back before
        // their FMAs, so the ~cluster-latency is paid K / KU times, not K
        constexpr int KU = PENT ? 4 : 8;
#pragma unroll 1
        for (int k0 = 0; k0 < 8 * CS; k0 += KU) {
          T yv[KU][NQ];
#pragma unroll
          for (int u = 0; u < KU; ++u) {
            const int kk = k0 + u;
            const uint32_t a = map_rank(xbase + static_cast<uint32_t>(((kk % kSpWarps) * NQ) * 32 * sizeof(T)),
                                        static_cast<uint32_t>(kk / kSpWarps));
#pragma unroll
            for (int q = 0; q < NQ; ++q) yv[u][q] = ld_cluster<T>(a + static_cast<uint32_t>(q * 32 * sizeof(T)));
          }
#pragma unroll
          for (int u = 0; u < KU; ++u) {
#pragma unroll
            for (int h = 0; h < NU; ++h) {
              const S* rr = srinv + static_cast<size_t>(rows[h]) * R + (k0 + u) * NQ;
#pragma unroll
              for (int q = 0; q < NQ; ++q) zu[h] = vfma(rr[q], yv[u][q], zu[h]);
            }
          }
        }
      }
      if (k == 0) {  // no left neighbour
#pragma unroll
        for (int h = NH; h < 2 * NH; ++h) zu[h] = T{};
      }
      if constexpr (PENT) {
        bs1 = zu[0];  // x_{L-2}
        bs2 = zu[1];  // x_{L-1}
        xl2 = zu[2];  // x_{s-2}
        xl1 = zu[3];  // x_{s-1}
      } else {
        bs1 = zu[0];  // x_{L-1}
        xl1 = zu[1];  // x_{s-1}
      }
      if constexpr (PER) {
        if constexpr (PENT) {  // periodic.cpp:189-194 (fast-mode rounding)
          const double w1 = zu[4] - zu[7], w2 = zu[5] - zu[6];
          t1 = fma(per.c[0], w1, per.c[1] * w2);
          t2 = fma(per.c[2], w1, per.c[3] * w2);
        } else {  // periodic.cpp:80
          t1 = fma(per.c[0], zu[3], zu[2]) * per.c[1];
        }
      }
      // x streamed to HBM (lanes past m write a scratch word: no branch)
      const long long j = g * Wg + gs * 32 + lane;
      const bool live = j < m;
      step = live ? ld : 0;
      out = live ? x + static_cast<long long>(r0 + L - 1) * ld + j : sink + lane;
      if constexpr (PENT) {
        __stcs(out - step, corr(L - 2, bs1));
        __stcs(out, corr(L - 1, bs2));
      } else {
        __stcs(out, corr(L - 1, bs1));
      }
      out -= NH * step;
      cur.load(tslot(p, CL - 1));  // the first backward chunk, loaded ahead
    };

    auto bwd_chunk = [&](int c, auto first) {
      constexpr int kTop = decltype(first)::value ? kSpR - 1 - NH : kSpR - 1;  // skip the interface rows
      cur.wait();
      const B* bc = bk + c * kSpR;
      T gv[kSpR];  // stage 1: left-coupling update (off the chain)
      if (!kCut || c < per.df) {
#pragma unroll
        for (int r = 0; r <= kTop; ++r) {
          const T g = from_word<T>(cur.get(r));
          if constexpr (PENT) gv[r] = vfma(-bc[r].f1, xl2, vfma(-bc[r].f2, xl1, g));
          else gv[r] = vfma(-bc[r].f1, xl1, g);
        }
      } else {  // the coupling's forward images have decayed
#pragma unroll
        for (int r = 0; r <= kTop; ++r) gv[r] = from_word<T>(cur.get(r));
      }
#pragma unroll
      for (int r = kTop; r >= 0; --r) {  // stage 2: one FMA per row on the chain
        T v;
        if constexpr (PENT) v = vfma(-bc[r].g, bs1, vfma(-bc[r].d, bs2, gv[r]));
        else v = vfma(-bc[r].c, bs1, gv[r]);
        bs2 = bs1;
        bs1 = v;
        __stcs(out, corr(c * kSpR + r, v));
        out -= step;
      }
    };

    const long long my = (groups - cid + ncl - 1) / ncl;
    if (my > 0) halo_prefetch(cid);
    uint32_t p = 0;  // parity of the group being read
    for (long long i = 0; i <= my; ++i, p ^= 1u) {
      const long long g = cid + i * ncl;  // group read in this round (i < my)
      // step kk: backward chunk CL-1-kk of the previous group, then forward
      // chunk kk of g (same TMEM slot)
      for (int kk = 0; kk < CL; ++kk) {
        if (i > 0) {
          const int c = CL - 1 - kk;
          if (kk == 0) bwd_chunk(c, std::true_type{});
          else bwd_chunk(c, std::false_type{});
          if (c > 0) cur.load(tslot(p ^ 1u, c - 1));
        }
        if (i < my) {
          fwd_chunk(kk, p, g);
          if (CN && kk == 0 && i + 1 < my) halo_prefetch(g + ncl);  // this group's halo is consumed
        }
      }
      if (i < my) interface(g, p);
    }
    tmem_fence_before();
    asm volatile("bar.sync 1, %0;" ::"r"(kSpWarps * 32) : "memory");
    if (warp == 0) {
      tmem_fence_after();
      tmem_dealloc_512(tmem_base_s);
    }
  }
  // a CTA's shared memory must outlive the cluster's remote reads of it
  if constexpr (CS > 1) cluster_sync_all();
}

}  // namespace dev
}  // namespace bsb
