// Shared-LHS interleaved sweep kernels for sm_100a.
//
// One thread owns one system (one column j of the interleaved n x m batch)
// and walks the forward and backward recurrences of the reference sweeps
// (tri_solver.cpp:24-47, pent_solver.cpp:19-62). Neighbouring threads own
// neighbouring columns, so every row access of a warp is one contiguous,
// coalesced segment, and every thread reads the same factor record for a
// row (a warp-uniform, L1-resident load).
//
// Two storage regimes for the forward intermediates (d-hat / g):
//   sweep_smem   - the CTA's whole W-system x n tile is staged in shared
//                  memory by TMA (one 2D box per R-row chunk, one mbarrier per
//                  chunk, all issued at CTA start), overwritten in place by the
//                  forward sweep, and the backward sweep streams x straight to
//                  HBM. HBM traffic: read b once, write x once.
//   sweep_global - in place in global memory (d-hat lands in L2 and is read
//                  back by the backward sweep). Any pitch/alignment; used when
//                  TMA's 16-byte stride rule fails or the tile does not fit.
//
// Arithmetic modes (template FAST):
//   exact - the reference's operation order with separately rounded
//           products/differences (__dmul_rn/__dsub_rn/...: nvcc cannot
//           contract them into FMAs). fp64 output is bitwise equal to the
//           reference CPU solver.
//   fast  - one fused multiply-add per row on the dependency chain, using
//           host-prescaled factor records.
//
// Boundary rows need no special-casing: the packed records carry signed
// zeros chosen so that the generic row formula reproduces the reference's
// peeled first/last rows bit for bit (see pack_* in solve.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace bsb {
namespace dev {

// ---- separately rounded arithmetic ----------------------------------------
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
// two fp32 systems at once. mul/add/sub as two scalar .rn operations: ptxas
// (12.9) contracts packed mul.rn.f32x2 + sub.rn.f32x2 into FFMA2 even with
// the explicit rounding (and __fmul2_rn/__fadd2_rn likewise), which would
// break the exact mode's separate roundings; scalar .rn is never contracted
__device__ __forceinline__ float2 mul_rn(float a, float2 b) { return make_float2(__fmul_rn(a, b.x), __fmul_rn(a, b.y)); }
__device__ __forceinline__ float2 mul_rn(float2 a, float b) { return make_float2(__fmul_rn(a.x, b), __fmul_rn(a.y, b)); }
__device__ __forceinline__ float2 add_rn(float2 a, float2 b) { return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y)); }
__device__ __forceinline__ float2 sub_rn(float2 a, float2 b) { return make_float2(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y)); }
// the fast mode's fused form (packed FFMA2)
__device__ __forceinline__ float2 fma_rn(float a, float2 b, float2 c) { return __ffma2_rn(make_float2(a, a), b, c); }

// ---- packed factor records (filled by solve.cu pack_*) ---------------------
// tri forward:  exact {a_i, m_i}          fast {a_i*m_i, m_i}
// tri backward: chat_i
// pent forward: exact {eps_i, beta_i, 1/alpha_i}   fast {eps_i/alpha_i, beta_i/alpha_i, 1/alpha_i}
// pent backward: {gamma_i, delta_i}
template <typename T>
struct alignas(2 * sizeof(T)) TriFwd {
  T a, m;
};
template <typename T>
struct alignas(4 * sizeof(T)) PentFwd {
  T e, b, ia, pad;
};
template <typename T>
struct alignas(2 * sizeof(T)) PentBwd {
  T g, d;
};

template <typename T, bool FAST>
__device__ __forceinline__ T tri_fwd(T d, T p1, const TriFwd<T>& f) {
  if constexpr (FAST) return fma_rn(-f.a, p1, mul_rn(d, f.m));
  else return mul_rn(sub_rn(d, mul_rn(f.a, p1)), f.m);  // (d - a*prev) * m
}
template <typename T, bool FAST>
__device__ __forceinline__ T tri_bwd(T dh, T q1, T c) {
  if constexpr (FAST) return fma_rn(-c, q1, dh);
  else return sub_rn(dh, mul_rn(c, q1));  // dhat - chat*next
}
template <typename T, bool FAST>
__device__ __forceinline__ T pent_fwd(T f, T g1, T g2, const PentFwd<T>& r) {
  if constexpr (FAST) return fma_rn(-r.b, g1, fma_rn(-r.e, g2, mul_rn(f, r.ia)));
  else return mul_rn(sub_rn(sub_rn(f, mul_rn(r.e, g2)), mul_rn(r.b, g1)), r.ia);  // ((f - e*g2) - b*g1) * ia
}
template <typename T, bool FAST>
__device__ __forceinline__ T pent_bwd(T g, T x1, T x2, const PentBwd<T>& r) {
  if constexpr (FAST) return fma_rn(-r.g, x1, fma_rn(-r.d, x2, g));
  else return sub_rn(g, add_rn(mul_rn(r.g, x1), mul_rn(r.d, x2)));  // g - (gamma*x1 + delta*x2)
}

// One sweep row for either band structure. s1/s2 carry the previous one/two
// values of the recurrence (zero-initialised before the first row).
template <typename T, bool PENT, bool FAST>
struct Rows {
  const void* fwd;
  const void* bwd;
  __device__ __forceinline__ T forward(int i, T d, T& s1, T& s2) const {
    T v;
    if constexpr (PENT) {
      const PentFwd<T> r = static_cast<const PentFwd<T>*>(fwd)[i];
      v = pent_fwd<T, FAST>(d, s1, s2, r);
    } else {
      const TriFwd<T> r = static_cast<const TriFwd<T>*>(fwd)[i];
      v = tri_fwd<T, FAST>(d, s1, r);
    }
    s2 = s1;
    s1 = v;
    return v;
  }
  __device__ __forceinline__ T backward(int i, T g, T& s1, T& s2) const {
    T v;
    if constexpr (PENT) {
      const PentBwd<T> r = static_cast<const PentBwd<T>*>(bwd)[i];
      v = pent_bwd<T, FAST>(g, s1, s2, r);
    } else {
      v = tri_bwd<T, FAST>(g, s1, static_cast<const T*>(bwd)[i]);
    }
    s2 = s1;
    s1 = v;
    return v;
  }
};

// ---- mbarrier / TMA primitives ---------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// 2D tiled TMA load of box {W, R} at (c0 = column, c1 = row) into smem,
// completing on bar; evict-first: every byte of b is read exactly once.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <typename T>
__device__ __forceinline__ void st_stream(T* p, T v) {
  __stcs(p, v);  // streaming store: x is written once and not re-read here
}

// ---- smem-resident regime --------------------------------------------------
// CTA = W threads = W consecutive systems; dynamic smem = ceil(n/R) chunks of
// R x W elements followed by one mbarrier per chunk.
template <typename T, int W, int R, bool PENT, bool FAST>
__global__ void __launch_bounds__(W) sweep_smem(const __grid_constant__ CUtensorMap tmap,
                                                T* __restrict__ x, int n, long long m, long long ld,
                                                const void* __restrict__ fwd,
                                                const void* __restrict__ bwd) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int chunks = (n + R - 1) / R;
  T* tile = reinterpret_cast<T*>(smem_raw);
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem_raw + static_cast<size_t>(chunks) * R * W * sizeof(T));
  const int t = threadIdx.x;
  const long long j0 = static_cast<long long>(blockIdx.x) * W;

  if (t == 0) {
    for (int c = 0; c < chunks; ++c) mbar_init(&bars[c], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (t == 0) {
    const uint64_t pol = policy_evict_first();
    constexpr uint32_t kBoxBytes = W * R * sizeof(T);  // OOB rows/cols are zero-filled
    for (int c = 0; c < chunks; ++c) {
      mbar_expect_tx(&bars[c], kBoxBytes);
      tma_load_2d(tile + static_cast<size_t>(c) * R * W, &tmap, static_cast<int>(j0), c * R,
                  &bars[c], pol);
    }
  }

  const Rows<T, PENT, FAST> rows{fwd, bwd};
  T* col = tile + t;

  // forward: d-hat / g over the staged b, in place in smem
  T s1 = T(0), s2 = T(0);
  for (int c = 0; c < chunks; ++c) {
    mbar_wait(&bars[c], 0);
    const int i0 = c * R;
    T* p = col + static_cast<size_t>(i0) * W;
    if (i0 + R <= n) {
#pragma unroll
      for (int r = 0; r < R; ++r) p[r * W] = rows.forward(i0 + r, p[r * W], s1, s2);
    } else {
      for (int r = 0; r < n - i0; ++r) p[r * W] = rows.forward(i0 + r, p[r * W], s1, s2);
    }
  }

  // backward: x streamed to HBM row by row (coalesced W-wide segments)
  const long long j = j0 + t;
  const bool live = j < m;
  T* out = x + j;
  s1 = T(0);
  s2 = T(0);
  for (int c = chunks - 1; c >= 0; --c) {
    const int i0 = c * R;
    const T* p = col + static_cast<size_t>(i0) * W;
    if (i0 + R <= n) {
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const T v = rows.backward(i0 + r, p[r * W], s1, s2);
        if (live) st_stream(out + static_cast<long long>(i0 + r) * ld, v);
      }
    } else {
      for (int r = n - i0 - 1; r >= 0; --r) {
        const T v = rows.backward(i0 + r, p[r * W], s1, s2);
        if (live) st_stream(out + static_cast<long long>(i0 + r) * ld, v);
      }
    }
  }
}

// ---- global (L2) regime ----------------------------------------------------
// One thread per system, in place; U-row blocks double-buffered in registers
// so the next block's loads are in flight while the current block computes.
// U: rows per register block (two blocks in flight). U = 8 when many systems
// share an SM; U = 32 for the few-long-systems regime (e.g. ADI axes), where
// each thread alone must cover HBM latency with its own prefetch.
// One system's column in place: rows [0, n) at col[i*ld], factor records of
// those rows at rows.fwd/rows.bwd index 0..n-1. The forward and backward
// halves are separate so the partitioned path (partition.cu) can hook them:
// `post(i, v)` sees each forward value; `pre(i, g)` adjusts each backward
// input; `out(i, v)` maps each backward value to what is stored (the
// recurrence carries v); s1/s2 carry the recurrence state in and out.
struct NoHook {
  template <typename T>
  __device__ __forceinline__ T operator()(int, T v) const { return v; }
};

// L2 prefetch (no register cost): PF > 0 pulls the rows PF blocks beyond the
// register double buffer into L2 so its loads pay L2, not HBM, latency
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

template <typename T, bool PENT, bool FAST, int U, typename Post = NoHook, int PF = 0>
__device__ __forceinline__ void column_forward(T* col, int n, long long ld, const Rows<T, PENT, FAST>& rows,
                                               T& s1, T& s2, const Post& post = Post{}) {
  T cur[U], nxt[U];
  const int full = n / U;  // number of complete U-row blocks
  if (full > 0) {
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = col[static_cast<long long>(u) * ld];
  }
  for (int b = 0; b < full; ++b) {
    const int i0 = b * U;
    if constexpr (PF > 0) {
      if (b + 1 + PF < full) {
#pragma unroll
        for (int u = 0; u < U; ++u) prefetch_l2(col + static_cast<long long>(i0 + (1 + PF) * U + u) * ld);
      }
    }
    if (b + 1 < full) {
#pragma unroll
      for (int u = 0; u < U; ++u) nxt[u] = col[static_cast<long long>(i0 + U + u) * ld];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cur[u] = rows.forward(i0 + u, cur[u], s1, s2);
      post(i0 + u, cur[u]);
      col[static_cast<long long>(i0 + u) * ld] = cur[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
  }
  for (int i = full * U; i < n; ++i) {
    T* p = col + static_cast<long long>(i) * ld;
    const T v = rows.forward(i, *p, s1, s2);
    post(i, v);
    *p = v;
  }
}

// backward over rows [0, n): the tail rows first (descending), then whole blocks
template <typename T, bool PENT, bool FAST, int U, typename Pre = NoHook, typename Out = NoHook, int PF = 0>
__device__ __forceinline__ void column_backward(T* col, int n, long long ld, const Rows<T, PENT, FAST>& rows,
                                                T& s1, T& s2, const Pre& pre = Pre{}, const Out& out = Out{}) {
  T cur[U], nxt[U];
  const int full = n / U;
  for (int i = n - 1; i >= full * U; --i) {
    T* p = col + static_cast<long long>(i) * ld;
    *p = out(i, rows.backward(i, pre(i, *p), s1, s2));
  }
  if (full > 0) {
    const int top = (full - 1) * U;
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = col[static_cast<long long>(top + u) * ld];
  }
  for (int b = full - 1; b >= 0; --b) {
    const int i0 = b * U;
    if constexpr (PF > 0) {
      if (b - 1 - PF >= 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) prefetch_l2(col + static_cast<long long>(i0 - (1 + PF) * U + u) * ld);
      }
    }
    if (b > 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) nxt[u] = col[static_cast<long long>(i0 - U + u) * ld];
    }
#pragma unroll
    for (int u = U - 1; u >= 0; --u) {
      cur[u] = rows.backward(i0 + u, pre(i0 + u, cur[u]), s1, s2);
      col[static_cast<long long>(i0 + u) * ld] = out(i0 + u, cur[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
  }
}

template <typename T, bool PENT, bool FAST, int U, int PF = 0>
__device__ __forceinline__ void column_sweep(T* col, int n, long long ld, const Rows<T, PENT, FAST>& rows) {
  T s1 = T(0), s2 = T(0);
  column_forward<T, PENT, FAST, U, NoHook, PF>(col, n, ld, rows, s1, s2);
  s1 = T(0);
  s2 = T(0);
  column_backward<T, PENT, FAST, U, NoHook, NoHook, PF>(col, n, ld, rows, s1, s2);
}

template <typename T, bool PENT, bool FAST, int U = 8, int PF = 0>
__global__ void __launch_bounds__(128) sweep_global(T* __restrict__ x, int n, long long m,
                                                    long long ld, const void* __restrict__ fwd,
                                                    const void* __restrict__ bwd) {
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  column_sweep<T, PENT, FAST, U, PF>(x + j, n, ld, Rows<T, PENT, FAST>{fwd, bwd});
}

// Few long systems (one warp per SM, e.g. the ADI axes): the same sweep with
// the factor records staged once into shared memory (fwd then bwd arrays,
// rec_f / rec_b bytes), so every row reads its record with a shared load
// instead of an L2 round trip; the RHS still streams through the register
// double buffer.
template <typename T, bool PENT, bool FAST, int U, int PF = 0>
__global__ void __launch_bounds__(128) sweep_global_rec(T* __restrict__ x, int n, long long m, long long ld,
                                                        const void* __restrict__ fwd, const void* __restrict__ bwd,
                                                        int rec_f, int rec_b) {
  extern __shared__ __align__(16) unsigned char srec[];
  {
    const uint4* sf = static_cast<const uint4*>(fwd);
    const uint4* sb = static_cast<const uint4*>(bwd);
    uint4* d = reinterpret_cast<uint4*>(srec);
    for (int i = threadIdx.x; i < rec_f / 16; i += blockDim.x) d[i] = sf[i];
    for (int i = threadIdx.x; i < rec_b / 16; i += blockDim.x) d[rec_f / 16 + i] = sb[i];
  }
  __syncthreads();
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  column_sweep<T, PENT, FAST, U, PF>(x + j, n, ld, Rows<T, PENT, FAST>{srec, srec + rec_f});
}

}  // namespace dev
}  // namespace bsb
