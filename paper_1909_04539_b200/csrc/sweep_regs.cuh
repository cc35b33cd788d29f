// Register-streamed head + smem tail sweep for sm_100a.
//
// Same split as sweep_stream.cuh (head rows [0, H) spilled to an L2 scratch,
// tail rows [H, n) resident in shared memory), but the head never touches
// shared memory: the forward sweep loads b straight into registers and the
// backward sweep reloads d-hat straight into registers, both through an
// NB-block x kRB-row register pipeline (loads issued (NB-1) blocks ahead).
// Shared memory then holds only the factor records and the tail, so at a
// given number of systems per SM the tail is longer and the L2 spill smaller
// than with smem rings (measured: spill volume beyond ~40 MB per GPU is what
// limits the ring version at n >= 512).
//
// b reaches L2 ahead of the register loads through TMA prefetches issued by
// each compute warp kRPD 16-row chunks ahead (crossing into the next group
// during the backward head sweep), so the register pipeline only has to
// cover L2 latency. One loader warp TMA-loads the tail chunks, into the slots
// the previous group's backward sweep freed (reverse order on alternate
// groups). HBM traffic: read b once, write x once.
#pragma once

#include "sweep_stream.cuh"

namespace bsb {
namespace dev {

constexpr int kRB = 8;    // rows per register block
constexpr int kRPD = 6;   // 16-row chunks of b prefetched into L2 ahead
constexpr int kRMaxWarps = 7;  // + loader = 8 warps (2 per SMSP): up to 255 registers per thread

struct RegsLayout {
  size_t fwd_off, bwd_off, tail_off, bar_off, total;
  __host__ __device__ static RegsLayout make(int n, int TC, int Wg, size_t elem, size_t fwd_rec, size_t bwd_rec) {
    RegsLayout L{};
    L.fwd_off = 0;
    L.bwd_off = align128(static_cast<size_t>(n) * fwd_rec);
    L.tail_off = L.bwd_off + align128(static_cast<size_t>(n) * bwd_rec);
    L.bar_off = L.tail_off + static_cast<size_t>(TC) * kSR * Wg * elem;
    L.total = L.bar_off + static_cast<size_t>(2 * TC) * sizeof(uint64_t);
    return L;
  }
};

template <typename T>
__device__ __forceinline__ T ld_hint(const T* p, uint64_t pol) {
  T v;
  if constexpr (sizeof(T) == 8)
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
  else
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}

template <typename T, bool PENT, bool FAST, int NB>
__global__ void __launch_bounds__(32 * (kRMaxWarps + 1), 1)
    sweep_regs(const __grid_constant__ CUtensorMap map_b, T* __restrict__ x, int n, long long m, long long ld, int H,
               int TC, long long groups, const void* __restrict__ fwd_g, const void* __restrict__ bwd_g,
               T* __restrict__ scratch) {
  using FwdR = typename Recs<T, PENT>::Fwd;
  using BwdR = typename Recs<T, PENT>::Bwd;
  using V1 = Vec<T, 1>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int P = static_cast<int>(blockDim.x >> 5) - 1;  // compute warps; warp P loads the tail
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int Wg = P * 32;
  const RegsLayout L = RegsLayout::make(n, TC, Wg, sizeof(T), sizeof(FwdR), sizeof(BwdR));
  const FwdR* sf = reinterpret_cast<const FwdR*>(smem + L.fwd_off);
  const BwdR* sb = reinterpret_cast<const BwdR*>(smem + L.bwd_off);
  T* tail = reinterpret_cast<T*>(smem + L.tail_off);
  uint64_t* t_full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* t_empty = t_full + TC;
  const int HB = H / kRB;              // register blocks in the head
  const int HC = H / kSR;              // 16-row chunks in the head (prefetch units)
  const int chunk = kSR * Wg;          // elements of one tail chunk (all warps)
  constexpr int kBlk = kSR * 32;       // elements of one warp's block of one tail chunk

  {  // factor records -> smem (16-byte words; device arrays padded to 256 B)
    const int nf = static_cast<int>((static_cast<size_t>(n) * sizeof(FwdR) + 15) / 16);
    const int nb = static_cast<int>((static_cast<size_t>(n) * sizeof(BwdR) + 15) / 16);
    const int4* gf = static_cast<const int4*>(fwd_g);
    const int4* gb = static_cast<const int4*>(bwd_g);
    int4* df = reinterpret_cast<int4*>(smem + L.fwd_off);
    int4* db = reinterpret_cast<int4*>(smem + L.bwd_off);
    for (int k = threadIdx.x; k < nf; k += blockDim.x) df[k] = gf[k];
    for (int k = threadIdx.x; k < nb; k += blockDim.x) db[k] = gb[k];
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < TC; ++k) {
      mbar_init(&t_full[k], 1);
      mbar_init(&t_empty[k], P);
    }
    fence_barrier_init();
  }
  __syncthreads();

  auto tail_slot = [TC](int k, uint32_t par) { return par ? TC - 1 - k : k; };

  // ----------------------------------------------------------- loader warp
  if (warp == P) {
    if (lane != 0) return;
    const uint64_t pol_b = policy_evict_first();
    const uint32_t c_bytes = static_cast<uint32_t>(chunk * sizeof(T));
    uint32_t it = 0;
    for (long long g = blockIdx.x; g < groups; g += gridDim.x, ++it) {
      const int c0 = static_cast<int>(g * Wg);
      const uint32_t par = it & 1u;
      for (int k = 0; k < TC; ++k) {
        const int s = tail_slot(k, par);
        if (it > 0) mbar_wait(&t_empty[s], (it - 1) & 1u);
        mbar_expect_tx(&t_full[s], c_bytes);
        for (int w = 0; w < P; ++w)
          tma_load_2d(tail + s * chunk + w * kBlk, &map_b, c0 + w * 32, H + k * kSR, &t_full[s], pol_b);
      }
    }
    return;
  }

  // --------------------------------------------------------- compute warps
  const uint64_t pol_keep = policy_evict_last();
  const uint64_t pol_b = policy_evict_first();
  const int wl = warp * kBlk + lane;
  V1* const tail_l = reinterpret_cast<V1*>(tail) + wl;
  // this warp's spill block: H rows x 32 lanes, reused by every group
  T* const spill = scratch + (static_cast<long long>(blockIdx.x) * P + warp) * H * 32 + lane;
  const int tfull = (n - H) / kSR;
  const int trem = (n - H) - tfull * kSR;
  uint32_t it = 0;
  long long g = blockIdx.x;

  auto prefetch_b = [&](long long grp, int c) {  // one 16-row chunk of this warp's 32 columns
    if (lane == 0) tma_prefetch_2d(&map_b, static_cast<int>(grp * Wg + warp * 32), c * kSR);
  };
  if (g < groups)
    for (int c = 0; c < HC && c < kRPD; ++c) prefetch_b(g, c);

  auto run_group = [&](auto full_tag) {
    constexpr bool kFull = decltype(full_tag)::value;
    const long long j = g * Wg + warp * 32 + lane;
    const bool live = kFull || j < m;
    const uint32_t par = it & 1u;
    const T* col = x + (live ? j : 0);
    T* out = x + (live ? j : 0) + static_cast<long long>(n - 1) * ld;
    auto put = [&](T v) {
      if (kFull || live) st_stream(out, v);
      out -= ld;
    };
    auto ld_b = [&](int row) -> T {
      if (kFull || live) return ld_hint(col + static_cast<long long>(row) * ld, pol_b);
      return T(0);
    };
    V1 s1{}, s2{};

    // ---- forward, head rows: b from L2 into registers, d-hat spilled to L2
    if (HB > 0) {
      T rb[NB][kRB];
#pragma unroll
      for (int u = 0; u < NB - 1; ++u)
        if (u < HB) {
#pragma unroll
          for (int r = 0; r < kRB; ++r) rb[u][r] = ld_b(u * kRB + r);
        }
      for (int c0 = 0; c0 < HB; c0 += NB) {
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int c = c0 + u;
          if (c >= HB) break;
          const int cl = c + NB - 1;
          if (cl < HB) {
#pragma unroll
            for (int r = 0; r < kRB; ++r) rb[(u + NB - 1) % NB][r] = ld_b(cl * kRB + r);
          }
          if ((c * kRB) % kSR == 0 && (c * kRB) / kSR + kRPD < HC) prefetch_b(g, (c * kRB) / kSR + kRPD);
          const FwdR* f = sf + c * kRB;
          T* sp = spill + c * kRB * 32;
#pragma unroll
          for (int r = 0; r < kRB; ++r) {
            const T v = fwd_row<T, PENT, FAST>(f[r], rb[u][r], s1.v[0], s2.v[0]);
            st_spill(sp + r * 32, v, pol_keep);
          }
        }
      }
    }

    // ---- forward, tail rows: in place in smem
    auto tslot = [&](int k) { return tail_l + tail_slot(k, par) * (chunk); };
    fwd_chunks<T, 1, PENT, FAST>(
        tfull, sf + H, s1, s2, tslot, [&](int k) { mbar_wait(&t_full[tail_slot(k, par)], par); }, [](int) {},
        [](int, int, V1* p, V1 v) { *p = v; });
    if (trem > 0) {
      mbar_wait(&t_full[tail_slot(tfull, par)], par);
      V1* p = tslot(tfull);
      const FwdR* f = sf + H + tfull * kSR;
      for (int r = 0; r < trem; ++r) p[r * kPR] = fwd_vec<T, 1, PENT, FAST>(f[r], p[r * kPR], s1, s2);
    }
    fence_proxy_async_smem();  // in-place smem writes before the TMA refills of these slots

    // ---- backward, tail rows: smem -> x; drained chunks go back to the loader
    s1 = V1{};
    s2 = V1{};
    auto tail_release = [&](int k) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_empty[tail_slot(k, par)]);
    };
    if (trem > 0) {
      const V1* p = tslot(tfull);
      const BwdR* b = sb + H + tfull * kSR;
      for (int r = trem - 1; r >= 0; --r) put(bwd_vec<T, 1, PENT, FAST>(b[r], p[r * kPR], s1, s2).v[0]);
      tail_release(tfull);
    }
    bwd_chunks<T, 1, PENT, FAST>(
        tfull, sb + H, s1, s2, [&](int k) -> const V1* { return tslot(k); }, [](int) {}, tail_release,
        [&](int, int, V1 v) { put(v.v[0]); });

    // ---- backward, head rows: d-hat back from L2 into registers, x to HBM
    if (HB > 0) {
      const long long gn = g + gridDim.x;  // this CTA's next group: get its first b chunks into L2
      if (gn < groups)
        for (int c = 0; c < HC && c < kRPD; ++c) prefetch_b(gn, c);
      T rb[NB][kRB];
#pragma unroll
      for (int u = 0; u < NB - 1; ++u)
        if (HB - 1 - u >= 0) {
#pragma unroll
          for (int r = 0; r < kRB; ++r) rb[u][r] = ld_spill(spill + ((HB - 1 - u) * kRB + r) * 32, pol_keep);
        }
      for (int c0 = HB - 1; c0 >= 0; c0 -= NB) {
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int c = c0 - u;
          if (c < 0) break;
          const int cl = c - (NB - 1);
          if (cl >= 0) {
#pragma unroll
            for (int r = 0; r < kRB; ++r)
              rb[(u + NB - 1) % NB][r] = ld_spill(spill + (cl * kRB + r) * 32, pol_keep);
          }
          const BwdR* b = sb + c * kRB;
#pragma unroll
          for (int q = 0; q < kRB; ++q) {
            const int r = kRB - 1 - q;
            put(bwd_row<T, PENT, FAST>(b[r], rb[u][r], s1.v[0], s2.v[0]));
          }
        }
      }
    }
  };
  for (; g < groups; g += gridDim.x, ++it) {
    if ((g + 1) * Wg <= m) run_group(std::true_type{});
    else run_group(std::false_type{});
  }

  // the scratch is dead: drop this warp's L2 lines instead of writing them back
  if (H > 0) {
    __syncwarp();
    const char* base = reinterpret_cast<const char*>(spill - lane);
    const long long bytes = static_cast<long long>(H) * 32 * sizeof(T);
    for (long long off = static_cast<long long>(lane) * 128; off < bytes; off += 32 * 128) discard_l2_line(base + off);
  }
}

}  // namespace dev
}  // namespace bsb
