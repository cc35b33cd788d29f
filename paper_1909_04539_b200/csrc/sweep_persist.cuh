// Persistent shared-LHS sweep for sm_100a: smem tail + L2 head + TMA ring.
//
// Why: with one thread per system, a row costs one trip around the
// dependency chain (exact tri: DMUL->DADD->DMUL forward, DMUL->DADD backward,
// 8 cycles each on B200 = 40 cycles; pent 48). Sustaining ~1.2 rows/cycle/SM
// (80% of HBM) therefore needs >= ~60 systems in flight per SM, and every
// system in flight owns n forward intermediates. Shared memory alone holds
// only 48 systems at n = 512 fp64; the L2 (126 MB, ~850 KB per SM) is the
// larger on-chip store. So each system's rows are split:
//
//   head rows [0, H)   b streamed in by a 4-slot TMA ring; d-hat written in
//                      place to global (it stays in L2: the whole spilled
//                      working set is sized to a fraction of L2) and read
//                      back by the backward sweep with register prefetch.
//   tail rows [H, n)   TMA-staged in smem for the whole tile, overwritten
//                      in place; the backward sweep starts here.
//
// HBM traffic stays at "read b once, write x once" as long as the head
// d-hat survives in L2 between its write and its read (b and x use
// evict-first policies so they do not displace it).
//
// Organisation: one CTA per SM, `warps` independent warps; each warp owns a
// tile of 32 consecutive systems at a time and loops over tiles
// (tile += total warps). A warp is its own producer and consumer (lane 0
// issues its TMA loads), so the main loop has no CTA-wide barrier. The
// factor records are staged once per CTA into smem and read as warp-uniform
// broadcasts.
//
// The next tile's first ring chunks are fetched as soon as the ring drains
// (end of the forward head) and its tail chunks as soon as each tail chunk
// has been consumed by the backward sweep, so loads overlap the current
// tile's remaining compute.
#pragma once

#include "sweep_kernels.cuh"

namespace bsb {
namespace dev {

constexpr int kPW = 32;  // systems per warp tile (one lane per system)
constexpr int kRH = 16;  // rows per ring chunk (head)
constexpr int kKR = 4;   // ring slots
constexpr int kRT = 32;  // rows per tail chunk
constexpr int kRB = 16;  // backward-head register prefetch depth (rows)

template <typename T, bool PENT>
struct Recs {
  using Fwd = TriFwd<T>;
  using Bwd = T;
};
template <typename T>
struct Recs<T, true> {
  using Fwd = PentFwd<T>;
  using Bwd = PentBwd<T>;
};

__host__ __device__ constexpr size_t align128(size_t v) { return (v + 127) & ~size_t(127); }

// Shared-memory carve-up, identical on host (planning) and device.
struct PersistLayout {
  size_t fwd_off, bwd_off, warp_off, ring_bytes, tail_bytes, warp_stride, bar_off, total;
  __host__ __device__ static PersistLayout make(int n, int H, int TC, int warps, size_t elem, size_t fwd_rec,
                                                size_t bwd_rec) {
    PersistLayout L{};
    L.fwd_off = 0;
    L.bwd_off = align128(static_cast<size_t>(n) * fwd_rec);
    L.warp_off = L.bwd_off + align128(static_cast<size_t>(n) * bwd_rec);
    L.ring_bytes = H > 0 ? static_cast<size_t>(kKR) * kRH * kPW * elem : 0;
    L.tail_bytes = static_cast<size_t>(TC) * kRT * kPW * elem;
    L.warp_stride = L.ring_bytes + L.tail_bytes;
    L.bar_off = L.warp_off + L.warp_stride * warps;
    L.total = L.bar_off + static_cast<size_t>(warps) * (kKR + TC) * sizeof(uint64_t);
    return L;
  }
};

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// d-hat spill store / reload: keep L1 out of the way (nothing is re-read
// through it), default L2 priority so it outlives the evict-first streams.
template <typename T>
__device__ __forceinline__ void st_spill(T* p, T v) {
  if constexpr (sizeof(T) == 8)
    asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
  else
    asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
template <typename T>
__device__ __forceinline__ T ld_spill(const T* p) {
  T v;
  if constexpr (sizeof(T) == 8)
    asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  else
    asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}

template <typename T, bool PENT, bool FAST>
__device__ __forceinline__ T fwd_row(const typename Recs<T, PENT>::Fwd& r, T d, T& s1, T& s2) {
  T v;
  if constexpr (PENT) v = pent_fwd<T, FAST>(d, s1, s2, r);
  else v = tri_fwd<T, FAST>(d, s1, r);
  s2 = s1;
  s1 = v;
  return v;
}
template <typename T, bool PENT, bool FAST>
__device__ __forceinline__ T bwd_row(const typename Recs<T, PENT>::Bwd& r, T g, T& s1, T& s2) {
  T v;
  if constexpr (PENT) v = pent_bwd<T, FAST>(g, s1, s2, r);
  else v = tri_bwd<T, FAST>(g, s1, r);
  s2 = s1;
  s1 = v;
  return v;
}

template <typename T, bool PENT, bool FAST>
__global__ void __launch_bounds__(32 * 16, 1)
    sweep_persist(const __grid_constant__ CUtensorMap map_ring, const __grid_constant__ CUtensorMap map_tail,
                  T* __restrict__ x, int n, long long m, long long ld, int H, int TC, long long tiles,
                  const void* __restrict__ fwd_g, const void* __restrict__ bwd_g) {
  using FwdR = typename Recs<T, PENT>::Fwd;
  using BwdR = typename Recs<T, PENT>::Bwd;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const PersistLayout L = PersistLayout::make(n, H, TC, warps, sizeof(T), sizeof(FwdR), sizeof(BwdR));
  const FwdR* sf = reinterpret_cast<const FwdR*>(smem + L.fwd_off);
  const BwdR* sb = reinterpret_cast<const BwdR*>(smem + L.bwd_off);
  T* ring = reinterpret_cast<T*>(smem + L.warp_off + L.warp_stride * warp);
  T* tail = reinterpret_cast<T*>(smem + L.warp_off + L.warp_stride * warp + L.ring_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off) + warp * (kKR + TC);
  uint64_t* ring_bar = bars;
  uint64_t* tail_bar = bars + kKR;

  // stage the factor records once per CTA (16-byte words; both arrays are
  // 16-byte multiples in size because records are 8/16/32 bytes and the
  // per-array regions are 128-byte aligned and zero-padded by the copy)
  {
    const int nf = static_cast<int>((static_cast<size_t>(n) * sizeof(FwdR) + 15) / 16);
    const int nb = static_cast<int>((static_cast<size_t>(n) * sizeof(BwdR) + 15) / 16);
    const int4* gf = static_cast<const int4*>(fwd_g);
    const int4* gb = static_cast<const int4*>(bwd_g);
    int4* df = reinterpret_cast<int4*>(smem + L.fwd_off);
    int4* db = reinterpret_cast<int4*>(smem + L.bwd_off);
    for (int k = threadIdx.x; k < nf; k += blockDim.x) df[k] = gf[k];
    for (int k = threadIdx.x; k < nb; k += blockDim.x) db[k] = gb[k];
  }
  if (lane == 0) {
    for (int k = 0; k < kKR + TC; ++k) mbar_init(&bars[k], 1);
    fence_barrier_init();
  }
  __syncthreads();

  const long long G = static_cast<long long>(gridDim.x) * warps;
  long long tile = static_cast<long long>(blockIdx.x) * warps + warp;
  if (tile >= tiles) return;

  const int HC = H / kRH;  // head chunks per tile (H is a multiple of kRH)
  constexpr uint32_t kRingBytes = kRH * kPW * sizeof(T);
  constexpr uint32_t kTailBytes = kRT * kPW * sizeof(T);
  uint64_t pol = 0;
  if (lane == 0) pol = policy_evict_first();

  // The ring is a FIFO over this warp's concatenated head-chunk stream
  // (tile t0 chunks 0..HC-1, tile t0+G chunks 0..HC-1, ...): stream element
  // q lives in slot q % kKR and completes that slot's (q / kKR)-th phase.
  const long long first_tile = tile;
  long long issued = 0;  // next stream element to load (lane 0's view)
  auto issue_next_ring = [&]() {  // lane 0 only
    if (HC == 0) return;
    const long long t = first_tile + (issued / HC) * G;
    if (t >= tiles) return;
    const int c = static_cast<int>(issued % HC);
    const int slot = static_cast<int>(issued % kKR);
    mbar_expect_tx(&ring_bar[slot], kRingBytes);
    tma_load_2d(ring + static_cast<size_t>(slot) * kRH * kPW, &map_ring, static_cast<int>(t * kPW), c * kRH,
                &ring_bar[slot], pol);
    ++issued;
  };
  auto issue_tail = [&](long long t, int k) {  // lane 0 only
    mbar_expect_tx(&tail_bar[k], kTailBytes);
    tma_load_2d(tail + static_cast<size_t>(k) * kRT * kPW, &map_tail, static_cast<int>(t * kPW), H + k * kRT,
                &tail_bar[k], pol);
  };

  if (lane == 0) {  // prologue: fill the ring, stage the first tile's tail
    for (int q = 0; q < kKR; ++q) issue_next_ring();
    for (int k = 0; k < TC; ++k) issue_tail(tile, k);
  }
  long long consumed = 0;   // ring stream elements consumed (all lanes)
  uint32_t tail_phase = 0;  // parity of the current tile's tail loads

  for (; tile < tiles; tile += G) {
    const long long next = tile + G;
    const long long j = tile * kPW + lane;
    const bool live = j < m;
    T* const col = x + j;
    T s1 = T(0), s2 = T(0);

    // ---- forward, head rows: ring -> registers -> d-hat spilled in place
    {
      T* out = col;
      for (int c = 0; c < HC; ++c, ++consumed) {
        const int slot = static_cast<int>(consumed % kKR);
        mbar_wait(&ring_bar[slot], static_cast<uint32_t>((consumed / kKR) & 1));
        const T* src = ring + static_cast<size_t>(slot) * kRH * kPW + lane;
        const FwdR* f = sf + c * kRH;
#pragma unroll
        for (int r = 0; r < kRH; ++r) {
          const T v = fwd_row<T, PENT, FAST>(f[r], src[r * kPW], s1, s2);
          if (live) st_spill(out, v);
          out += ld;
        }
        __syncwarp();
        if (lane == 0) {
          fence_proxy_async_smem();  // generic reads of the slot before the async refill
          issue_next_ring();
        }
      }
    }

    // ---- forward, tail rows: in place in smem
    for (int k = 0; k < TC; ++k) {
      mbar_wait(&tail_bar[k], tail_phase);
      T* p = tail + static_cast<size_t>(k) * kRT * kPW + lane;
      const int i0 = H + k * kRT;
      const FwdR* f = sf + i0;
      if (i0 + kRT <= n) {
#pragma unroll
        for (int r = 0; r < kRT; ++r) p[r * kPW] = fwd_row<T, PENT, FAST>(f[r], p[r * kPW], s1, s2);
      } else {
        for (int r = 0; r < n - i0; ++r) p[r * kPW] = fwd_row<T, PENT, FAST>(f[r], p[r * kPW], s1, s2);
      }
    }
    tail_phase ^= 1u;

    // ---- backward, tail rows: smem -> x streamed to HBM
    s1 = T(0);
    s2 = T(0);
    for (int k = TC - 1; k >= 0; --k) {
      const T* p = tail + static_cast<size_t>(k) * kRT * kPW + lane;
      const int i0 = H + k * kRT;
      const BwdR* b = sb + i0;
      const int rows = (i0 + kRT <= n) ? kRT : n - i0;
      T* out = col + static_cast<long long>(i0 + rows - 1) * ld;
      if (rows == kRT) {
#pragma unroll
        for (int r = kRT - 1; r >= 0; --r) {
          const T v = bwd_row<T, PENT, FAST>(b[r], p[r * kPW], s1, s2);
          if (live) st_stream(out, v);
          out -= ld;
        }
      } else {
        for (int r = rows - 1; r >= 0; --r) {
          const T v = bwd_row<T, PENT, FAST>(b[r], p[r * kPW], s1, s2);
          if (live) st_stream(out, v);
          out -= ld;
        }
      }
      __syncwarp();
      if (lane == 0 && next < tiles) {
        fence_proxy_async_smem();
        issue_tail(next, k);
      }
    }

    // ---- backward, head rows: d-hat back from L2 with a kRB-row register prefetch
    if (H > 0) {
      T cur[kRB], nxt[kRB];
      T* top = col + static_cast<long long>(H - 1) * ld;  // row H-1
      {
        const T* q = top;
#pragma unroll
        for (int r = 0; r < kRB; ++r) {
          cur[r] = live ? ld_spill(q) : T(0);
          q -= ld;
        }
      }
      T* out = top;
      for (int i0 = H - 1; i0 >= 0; i0 -= kRB) {  // rows i0 .. i0-kRB+1 (H % kRB == 0)
        if (i0 - kRB >= 0) {
          const T* q = out - static_cast<long long>(kRB) * ld;
#pragma unroll
          for (int r = 0; r < kRB; ++r) {
            nxt[r] = live ? ld_spill(q) : T(0);
            q -= ld;
          }
        }
        const BwdR* b = sb + i0;
#pragma unroll
        for (int r = 0; r < kRB; ++r) {
          const T v = bwd_row<T, PENT, FAST>(b[-r], cur[r], s1, s2);
          if (live) st_stream(out, v);
          out -= ld;
        }
#pragma unroll
        for (int r = 0; r < kRB; ++r) cur[r] = nxt[r];
      }
    }
  }
}

}  // namespace dev
}  // namespace bsb
