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
//   head rows [0, H)   b streamed in by a 4-slot TMA ring; d-hat spilled to a
//                      compact per-warp scratch (H x 32 elements, reused by
//                      every tile of the warp, evict_last in L2, discarded
//                      without write-back at the end) and read back by the
//                      backward sweep with a register prefetch.
//   tail rows [H, n)   TMA-staged in smem for the whole tile, overwritten in
//                      place; the backward sweep starts here.
//
// HBM traffic stays at "read b once, write x once": b is loaded and x stored
// with evict-first policies, the scratch lives in L2.
//
// Organisation: one CTA per SM, `warps` (<= 8) independent warps; a warp
// owns a tile of 32 consecutive systems (one lane each) and loops over tiles
// (tile += total warps). A warp is its own producer and consumer (lane 0
// issues its TMA loads), so the main loop has no CTA-wide barrier. Factor
// records are staged once per CTA into smem and read as warp-uniform
// broadcasts. Every row loop is software-pipelined kD rows deep so the smem /
// L2 latency of the next rows overlaps the current row's dependency chain.
//
// Load scheduling: the ring is a FIFO over the warp's concatenated head-chunk
// stream, so the next tile's first head chunks load while the current tile is
// still computing. Tail slots are mapped in reverse order on alternate tiles:
// the backward sweep frees the slot of the last tail chunk first, and that
// slot receives the next tile's FIRST tail chunk, so the chunk the next
// forward sweep needs first has the longest lead time.
#pragma once

#include <type_traits>

#include "sweep_kernels.cuh"

namespace bsb {
namespace dev {

constexpr int kPW = 32;     // systems per warp tile (one lane per system)
constexpr int kRH = 16;     // rows per ring chunk (head)
constexpr int kKR = 4;      // ring slots
constexpr int kRT = 32;     // rows per tail chunk
constexpr int kD = 4;       // smem software-pipeline depth (rows)
constexpr int kMaxWarps = 8;
constexpr int kHAlign = kRH;  // spilled head rows come in whole ring chunks

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
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Scratch spill store / reload: no L1 allocation, evict_last in L2.
template <typename T>
__device__ __forceinline__ void st_spill(T* p, T v, uint64_t pol) {
  if constexpr (sizeof(T) == 8)
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
  else
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
template <typename T>
__device__ __forceinline__ T ld_spill(const T* p, uint64_t pol) {
  T v;
  if constexpr (sizeof(T) == 8)
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
  else
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// 1D bulk copy global -> smem completing on an mbarrier (size % 16 == 0).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// Drop a 128-byte L2 line without writing it back (the scratch is dead).
__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
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

// Forward over R consecutive smem rows p[r*kPW] (ascending), records f[r];
// results go to sink(r, v). Loads run kD rows ahead of the chain.
template <typename T, bool PENT, bool FAST, int R, typename Sink>
__device__ __forceinline__ void fwd_block(const T* p, const typename Recs<T, PENT>::Fwd* f, T& s1, T& s2,
                                          Sink&& sink) {
  using FwdR = typename Recs<T, PENT>::Fwd;
  constexpr int D = R < kD ? R : kD;
  T dq[D];
  FwdR fq[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    dq[k] = p[k * kPW];
    fq[k] = f[k];
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const T v = fwd_row<T, PENT, FAST>(fq[r % D], dq[r % D], s1, s2);
    if (r + D < R) {
      dq[r % D] = p[(r + D) * kPW];
      fq[r % D] = f[r + D];
    }
    sink(r, v);
  }
}

// Backward over R rows, descending: row r = R-1 .. 0 of p / b.
template <typename T, bool PENT, bool FAST, int R, typename Sink>
__device__ __forceinline__ void bwd_block(const T* p, const typename Recs<T, PENT>::Bwd* b, T& s1, T& s2,
                                          Sink&& sink) {
  using BwdR = typename Recs<T, PENT>::Bwd;
  constexpr int D = R < kD ? R : kD;
  T dq[D];
  BwdR bq[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    dq[k] = p[(R - 1 - k) * kPW];
    bq[k] = b[R - 1 - k];
  }
#pragma unroll
  for (int q = 0; q < R; ++q) {  // q-th processed row is r = R-1-q
    const T v = bwd_row<T, PENT, FAST>(bq[q % D], dq[q % D], s1, s2);
    if (q + D < R) {
      dq[q % D] = p[(R - 1 - q - D) * kPW];
      bq[q % D] = b[R - 1 - q - D];
    }
    sink(R - 1 - q, v);
  }
}

template <typename T, bool PENT, bool FAST>
__global__ void __launch_bounds__(32 * kMaxWarps, 1)
    sweep_persist(const __grid_constant__ CUtensorMap map_ring, const __grid_constant__ CUtensorMap map_tail,
                  T* __restrict__ x, int n, long long m, long long ld, int H, int TC, long long tiles,
                  const void* __restrict__ fwd_g, const void* __restrict__ bwd_g, T* __restrict__ scratch) {
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

  // stage the factor records once per CTA (16-byte words; device arrays are
  // padded to 256 bytes, smem regions to 128)
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

  const int HC = H / kRH;  // head chunks per tile (H is a multiple of kHAlign)
  constexpr uint32_t kRingBytes = kRH * kPW * sizeof(T);
  constexpr uint32_t kTailBytes = kRT * kPW * sizeof(T);
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  // this warp's scratch: H rows x 32 lanes, row-major (256-byte rows)
  T* const spill = scratch + (static_cast<long long>(blockIdx.x) * warps + warp) * H * kPW + lane;

  // Ring: a FIFO over this warp's stream of 16-row chunks. Per tile it
  // carries HC "load" elements (b, head chunks 0..HC-1, TMA tensor loads from
  // x) followed by HC "reload" elements (d-hat, head chunks HC-1..0, bulk
  // copies back from the scratch). Element q lives in slot q % kKR and
  // completes that slot's (q / kKR)-th phase. Lane 0 keeps kKR elements in
  // flight; a tile's reloads become issuable once its forward head is
  // written (fwd_done).
  long long iss_tile = tile;  // tile of the next element to issue
  int iss_k = 0;              // index of that element within its tile (0 .. 2HC-1)
  long long issued = 0;       // elements issued so far
  long long fwd_done = -1;    // last tile whose forward head sits in the scratch
  auto pump = [&](long long consumed_now) {  // lane 0 only
    while (HC > 0 && issued < consumed_now + kKR && iss_tile < tiles) {
      const int slot = static_cast<int>(issued % kKR);
      T* dst = ring + static_cast<size_t>(slot) * kRH * kPW;
      if (iss_k < HC) {
        mbar_expect_tx(&ring_bar[slot], kRingBytes);
        tma_load_2d(dst, &map_ring, static_cast<int>(iss_tile * kPW), iss_k * kRH, &ring_bar[slot], pol_stream);
      } else {
        if (iss_tile > fwd_done) break;
        const int c = 2 * HC - 1 - iss_k;
        mbar_expect_tx(&ring_bar[slot], kRingBytes);
        bulk_load(dst, spill - lane + static_cast<long long>(c) * kRH * kPW, kRingBytes, &ring_bar[slot], pol_keep);
      }
      ++issued;
      if (++iss_k == 2 * HC) {
        iss_k = 0;
        iss_tile += G;
      }
    }
  };
  // tail chunk k of the tile with iteration parity `par` lives in slot
  // par ? TC-1-k : k
  auto tail_slot = [&](int k, uint32_t par) { return par ? TC - 1 - k : k; };
  auto issue_tail = [&](long long t, int k, uint32_t par) {  // lane 0 only
    const int s = tail_slot(k, par);
    mbar_expect_tx(&tail_bar[s], kTailBytes);
    tma_load_2d(tail + static_cast<size_t>(s) * kRT * kPW, &map_tail, static_cast<int>(t * kPW), H + k * kRT,
                &tail_bar[s], pol_stream);
  };

  if (lane == 0) {  // prologue: fill the ring, stage the first tile's tail
    pump(0);
    for (int k = 0; k < TC; ++k) issue_tail(tile, k, 0);
  }
  long long consumed = 0;  // ring stream elements consumed (all lanes)
  uint32_t par = 0;        // tile iteration parity (tail slot mapping and barrier phase)

  // One tile. kFull: all 32 systems exist (every tile but possibly the last),
  // so the x stores need no per-lane guard.
  auto run_tile = [&](auto full_tag) {
    constexpr bool kFull = decltype(full_tag)::value;
    const long long next = tile + G;
    const long long j = tile * kPW + lane;
    const bool live = kFull || j < m;
    T* const col = x + (live ? j : 0);
    auto put = [&](T* q, T v) {
      if (kFull || live) st_stream(q, v);
    };
    T s1 = T(0), s2 = T(0);

    // ---- forward, head rows: ring -> registers -> d-hat to the L2 scratch
    for (int c = 0; c < HC; ++c, ++consumed) {
      const int slot = static_cast<int>(consumed % kKR);
      mbar_wait(&ring_bar[slot], static_cast<uint32_t>((consumed / kKR) & 1));
      const T* src = ring + static_cast<size_t>(slot) * kRH * kPW + lane;
      T* sp = spill + static_cast<long long>(c) * kRH * kPW;
      fwd_block<T, PENT, FAST, kRH>(src, sf + c * kRH, s1, s2,
                                    [&](int r, T v) { st_spill(sp + r * kPW, v, pol_keep); });
      __syncwarp();  // every lane has read the slot before lane 0 refills it
      if (lane == 0) pump(consumed + 1);
    }
    if (H > 0) {
      // this tile's head d-hat is in the scratch: make the generic stores
      // visible to the async proxy, then let the reloads go
      fence_proxy_async_global();
      __syncwarp();
      if (lane == 0) {
        fwd_done = tile;
        pump(consumed);
      }
    }

    // ---- forward, tail rows: in place in smem
    for (int k = 0; k < TC; ++k) {
      const int s = tail_slot(k, par);
      mbar_wait(&tail_bar[s], par);
      T* p = tail + static_cast<size_t>(s) * kRT * kPW + lane;
      const int i0 = H + k * kRT;
      const FwdR* f = sf + i0;
      if (i0 + kRT <= n) {
        fwd_block<T, PENT, FAST, kRT>(p, f, s1, s2, [&](int r, T v) { p[r * kPW] = v; });
      } else {
        for (int r = 0; r < n - i0; ++r) p[r * kPW] = fwd_row<T, PENT, FAST>(f[r], p[r * kPW], s1, s2);
      }
    }

    // ---- backward, tail rows: smem -> x streamed to HBM; each drained slot
    // immediately receives the next tile's chunk (reverse mapping)
    s1 = T(0);
    s2 = T(0);
    T* out = col + static_cast<long long>(n - 1) * ld;  // walks up one row per step
    for (int k = TC - 1; k >= 0; --k) {
      const int s = tail_slot(k, par);
      const T* p = tail + static_cast<size_t>(s) * kRT * kPW + lane;
      const int i0 = H + k * kRT;
      const BwdR* b = sb + i0;
      if (i0 + kRT <= n) {
        bwd_block<T, PENT, FAST, kRT>(p, b, s1, s2, [&](int, T v) {
          put(out, v);
          out -= ld;
        });
      } else {
        for (int r = n - i0 - 1; r >= 0; --r) {
          put(out, bwd_row<T, PENT, FAST>(b[r], p[r * kPW], s1, s2));
          out -= ld;
        }
      }
      __syncwarp();
      if (lane == 0 && next < tiles) issue_tail(next, TC - 1 - k, par ^ 1u);  // lands in slot s
    }

    // ---- backward, head rows: d-hat reloaded into the ring (bulk copies
    // issued since the forward head finished), smem -> x streamed to HBM
    for (int c = HC - 1; c >= 0; --c, ++consumed) {
      const int slot = static_cast<int>(consumed % kKR);
      mbar_wait(&ring_bar[slot], static_cast<uint32_t>((consumed / kKR) & 1));
      const T* src = ring + static_cast<size_t>(slot) * kRH * kPW + lane;
      bwd_block<T, PENT, FAST, kRH>(src, sb + c * kRH, s1, s2, [&](int, T v) {
        put(out, v);
        out -= ld;
      });
      __syncwarp();
      if (lane == 0) pump(consumed + 1);
    }
  };

  for (; tile < tiles; tile += G, par ^= 1u) {
    if ((tile + 1) * kPW <= m) run_tile(std::true_type{});
    else run_tile(std::false_type{});
  }

  // the scratch is dead: drop its L2 lines instead of writing them back
  if (H > 0) {
    __syncwarp();
    const char* base = reinterpret_cast<const char*>(spill - lane);
    const long long bytes = static_cast<long long>(H) * kPW * sizeof(T);
    for (long long off = static_cast<long long>(lane) * 128; off < bytes; off += 32 * 128) discard_l2_line(base + off);
  }
}

}  // namespace dev
}  // namespace bsb
