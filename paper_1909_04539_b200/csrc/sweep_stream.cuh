// Warp-specialised streaming shared-LHS sweep for sm_100a (the default plan).
//
// Why this shape (measured, profiles/): one thread per system walks a
// dependent fp64 recurrence, so a row costs ~22 (tri) / ~36 (pent) cycles of
// one warp's time in the exact arithmetic mode (tools/microbench/rowcost.cu),
// and an SM must keep enough systems in flight to pull ~90% of HBM; every
// system in flight owns its n forward intermediates (4 KiB at n = 512 fp64).
// Each system's rows are therefore split:
//
//   head rows [0, H)   b arrives through a KB-slot TMA ring; the forward sweep
//                      spills d-hat to an L2 scratch (evict_last, dropped
//                      without write-back at the end); the backward sweep gets
//                      it back through the same ring (TMA bulk copies).
//   tail rows [H, n)   TMA-staged in shared memory, overwritten in place by
//                      the forward sweep; the backward sweep starts here.
//
// HBM traffic stays at "read b once, write x once". With no spill (H = 0,
// n <= ~256 fp64) this kernel runs at 92-97% of measured HBM bandwidth.
//
// Organisation: one CTA per SM, persistent over "groups" of Wg = 32 P
// consecutive systems. P compute warps (lane = system) walk a group in
// lockstep; one extra producer warp issues every TMA operation:
//
//   * smem tiles are per-warp [rows][32] blocks (256-byte rows), so every
//     row access in the sweeps is a compile-time offset from one base
//     register; a chunk of b is P TMA boxes {32 systems x kSR rows};
//   * the ring is a FIFO over the CTA's element stream: per group, HC head
//     chunks of b, then HC chunks of spilled d-hat in reverse order (one bulk
//     copy each, issued once every compute warp has published its spill);
//   * the producer keeps kSPD b chunks ahead of the ring in L2 with TMA
//     prefetches, crossing into the next group while the current one is in
//     its backward sweep, so ring loads pay L2 rather than HBM latency;
//   * tail chunks are loaded into the slots the previous group's backward
//     sweep frees, in reverse order on alternate groups so the chunk needed
//     first is the one freed first;
//   * the row loops are software-pipelined kSD rows deep ACROSS chunk
//     boundaries (the next chunk's barrier is waited on kSD rows early).
//
// Arithmetic: the row formulas of sweep_kernels.cuh (exact = the reference's
// operation order, bitwise equal; fast = one FMA per row on the chain).
#pragma once

#include "sweep_persist.cuh"

namespace bsb {
namespace dev {

constexpr int kSR = 16;        // rows per chunk (ring and tail)
constexpr int kSD = 4;         // software-pipeline depth (rows); divides kSR
constexpr int kPR = 32;        // vectors per row of a warp block (one per lane)
static_assert(kSR % kSD == 0, "pipeline depth must divide the chunk");
// V = systems per lane (adjacent columns): a warp covers 32 V systems.
__host__ __device__ constexpr int stream_max_warps(int V) { return V == 1 ? 8 : 4; }  // Wg <= 256 (TMA box)

// A lane's V systems (adjacent columns V l .. V l + V-1): one 8/16-byte
// access per row for all of them, and V independent dependency chains
// interleaved in one instruction stream.
template <typename T, int V>
struct alignas(V * sizeof(T)) Vec {
  T v[V];
};
template <typename T, int V, bool PENT, bool FAST>
__device__ __forceinline__ Vec<T, V> fwd_vec(const typename Recs<T, PENT>::Fwd& r, Vec<T, V> d, Vec<T, V>& s1,
                                             Vec<T, V>& s2) {
  Vec<T, V> o;
#pragma unroll
  for (int k = 0; k < V; ++k) o.v[k] = fwd_row<T, PENT, FAST>(r, d.v[k], s1.v[k], s2.v[k]);
  return o;
}
template <typename T, int V, bool PENT, bool FAST>
__device__ __forceinline__ Vec<T, V> bwd_vec(const typename Recs<T, PENT>::Bwd& r, Vec<T, V> g, Vec<T, V>& s1,
                                             Vec<T, V>& s2) {
  Vec<T, V> o;
#pragma unroll
  for (int k = 0; k < V; ++k) o.v[k] = bwd_row<T, PENT, FAST>(r, g.v[k], s1.v[k], s2.v[k]);
  return o;
}
template <typename T, int V>
__device__ __forceinline__ void st_spill_vec(Vec<T, V>* p, Vec<T, V> v, uint64_t pol) {
  if constexpr (V == 1) {
    st_spill(&p->v[0], v.v[0], pol);
  } else if constexpr (sizeof(T) == 8) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.v[0]),
                 "d"(v.v[1]), "l"(pol)
                 : "memory");
  } else {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.v[0]),
                 "f"(v.v[1]), "l"(pol)
                 : "memory");
  }
}
template <typename T, int V>
__device__ __forceinline__ void st_stream_vec(Vec<T, V>* p, Vec<T, V> v) {
  if constexpr (V == 1) st_stream(&p->v[0], v.v[0]);
  else if constexpr (sizeof(T) == 8) __stcs(reinterpret_cast<double2*>(p), make_double2(v.v[0], v.v[1]));
  else __stcs(reinterpret_cast<float2*>(p), make_float2(v.v[0], v.v[1]));
}

struct StreamLayout {
  size_t fwd_off, bwd_off, per_off, ck_off, bring_off, rring_off, tail_off, bar_off, total;
  // chunk: elements of one chunk (all warps) = kSR x Wg; per_arrays: fp64
  // arrays of n for the fused periodic correction (0, 2 tri, 4 pent);
  // ckpts: forward-state checkpoints per system (recompute tier: one per
  // recomputed segment after the first, two values each)
  __host__ __device__ static StreamLayout make(int n, int H, int TC, int Wg, int KB, int KR, size_t elem,
                                               size_t fwd_rec, size_t bwd_rec, int per_arrays = 0, int ckpts = 0) {
    StreamLayout L{};
    L.fwd_off = 0;
    L.bwd_off = align128(static_cast<size_t>(n) * fwd_rec);
    L.per_off = L.bwd_off + align128(static_cast<size_t>(n) * bwd_rec);
    L.ck_off = L.per_off + align128(static_cast<size_t>(per_arrays) * n * sizeof(double));
    L.bring_off = L.ck_off + align128(static_cast<size_t>(ckpts) * Wg * 2 * elem);
    const size_t chunk = static_cast<size_t>(kSR) * Wg * elem;
    L.rring_off = L.bring_off + (H > 0 ? static_cast<size_t>(KB) * chunk : 0);
    L.tail_off = L.rring_off + (H > 0 ? static_cast<size_t>(KR) * chunk : 0);
    L.bar_off = L.tail_off + static_cast<size_t>(TC) * chunk;
    // barriers, then one word for the TMEM base address
    L.total = L.bar_off + static_cast<size_t>(2 * KB + 2 * KR + 2 * TC + 2) * sizeof(uint64_t);
    return L;
  }
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}


// ---- Tensor Memory as a per-lane store for forward intermediates -----------------
// TMEM is 128 lanes x 512 columns x 32 bit per SM; with the .32x32b shape
// thread t of warp w (w < 4) reads/writes its own lane 32w + t, so each
// system owns up to 2 KB (256 fp64 rows) next to its registers: a third
// on-chip tier between shared memory and the L2 spill.
__device__ __forceinline__ void tmem_alloc_512(uint32_t* dst) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(dst)) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_512(uint32_t taddr) {  // the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 16 / 32 consecutive 32-bit columns of this lane. tcgen05.st is
// asynchronous; its data is visible to later tcgen05.ld after tmem_wait_st().
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31]) :: "memory");
}
// wait for this thread's TMEM loads; the registers are in/out operands so no
// consumer can be scheduled above the wait
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]) :: "memory");
}
// A piece of one lane's consecutive rows <-> raw 32-bit TMEM words: one
// whole 16-row chunk per .32x32b access (x32 for fp64, x16 for fp32; the
// 8-row x16 pieces for fp64 measured 10% slower at N = 512: twice the
// tcgen05 instructions and waits in the row loops). Row i of a TMEM region
// sits at column i * kColsPerRow.
#ifndef BSB_TMEM_PIECE_ROWS
#define BSB_TMEM_PIECE_ROWS 16
#endif
template <typename T>
struct TPiece {
  static constexpr int kWords = sizeof(T) == 8 ? 2 * BSB_TMEM_PIECE_ROWS : 16;
  static_assert(kWords == 16 || kWords == 32, "x16 / x32 accesses");
  static constexpr int kColsPerRow = static_cast<int>(sizeof(T)) / 4;
  static constexpr int kRows = kWords / kColsPerRow;
  uint32_t w[kWords];
  __device__ __forceinline__ void put(int r, T v) {
    if constexpr (sizeof(T) == 8) {
      w[2 * r] = static_cast<uint32_t>(__double2loint(v));
      w[2 * r + 1] = static_cast<uint32_t>(__double2hiint(v));
    } else {
      w[r] = __float_as_uint(v);
    }
  }
  __device__ __forceinline__ T get(int r) const {
    if constexpr (sizeof(T) == 8) return __hiloint2double(static_cast<int>(w[2 * r + 1]), static_cast<int>(w[2 * r]));
    else return __uint_as_float(w[r]);
  }
  // store, then wait for it: measured on B200 (N = 512, fp64) x32 + wait
  // 0.71 of roofline, x16 without the wait 0.64, x32 without it 0.49 — an
  // in-flight tcgen05.st pins its source registers, and the next piece's
  // gather into them stalls longer than the wait itself
  __device__ __forceinline__ void store(uint32_t taddr) const {
    if constexpr (kWords == 32) tmem_st32(taddr, w);
    else tmem_st16(taddr, w);
    tmem_wait_st();
  }
  __device__ __forceinline__ void load(uint32_t taddr) {
    if constexpr (kWords == 32) tmem_ld32(taddr, w);
    else tmem_ld16(taddr, w);
  }
  __device__ __forceinline__ void wait() { tmem_wait_ld(w); }
};
static_assert(kSR % TPiece<double>::kRows == 0 && kSR % TPiece<float>::kRows == 0, "pieces tile a chunk");

// Forward sweep over C consecutive kSR-row chunks in ascending row order,
// on this lane's pair of systems. base(c): the lane's row-0 pair of chunk c
// (row r at +r*kPR pairs); ready(c) blocks until chunk c may be read;
// release(c) is called once chunk c is no longer read; sink(c, r, p, v)
// consumes row r's result (p = its smem pair). f: the records of chunk 0's
// first row (chunk c at +c*kSR).
struct NoXf {};  // no input transform: the sweep consumes the staged rows as they are

// xf (optional): input transform xf(c, r, u, look) -> value fed to the
// recurrence for row r of chunk c, where look(k) (k = 1, 2) yields the raw
// row r+k of the stream (from the software pipeline, or extra(k') for the
// k'-th row past the stream's end). Used by the fused Crank-Nicolson step.
template <typename T, int V, bool PENT, bool FAST, typename Base, typename Ready, typename Release, typename Sink,
          typename Xf = NoXf, typename Extra = NoXf>
__device__ __forceinline__ void fwd_chunks(int C, const typename Recs<T, PENT>::Fwd* f, Vec<T, V>& s1, Vec<T, V>& s2,
                                           Base&& base, Ready&& ready, Release&& release, Sink&& sink,
                                           Xf&& xf = NoXf{}, Extra&& extra = NoXf{}) {
  using FwdR = typename Recs<T, PENT>::Fwd;
  constexpr bool kXf = !std::is_same<std::decay_t<Xf>, NoXf>::value;
  if (C <= 0) return;
  Vec<T, V> dq[kSD];
  FwdR fq[kSD];
  ready(0);
  Vec<T, V>* p = base(0);
#pragma unroll
  for (int k = 0; k < kSD; ++k) {
    dq[k] = p[k * kPR];
    fq[k] = f[k];
  }
  for (int c = 0; c < C; ++c) {
    const bool more = c + 1 < C;
    Vec<T, V>* pn = p;
    const FwdR* fc = f + c * kSR;
#pragma unroll
    for (int r = 0; r < kSR; ++r) {
      if (r == kSR - kSD && more) {
        ready(c + 1);
        pn = base(c + 1);
      }
      Vec<T, V> in = dq[r % kSD];
      if constexpr (kXf) {
        auto look = [&](int k) -> Vec<T, V> {
          if (r + k < kSR || more) return dq[(r + k) % kSD];
          return extra(r + k - kSR);
        };
        in = xf(c, r, in, look);
      }
      const Vec<T, V> v = fwd_vec<T, V, PENT, FAST>(fq[r % kSD], in, s1, s2);
      const int rn = r + kSD;
      if (rn < kSR) {
        dq[r % kSD] = p[rn * kPR];
        fq[r % kSD] = fc[rn];
      } else if (more) {
        dq[r % kSD] = pn[(rn - kSR) * kPR];
        fq[r % kSD] = fc[rn];
      }
      sink(c, r, p + r * kPR, v);
    }
    release(c);
    p = pn;
  }
}

// Backward sweep over chunks C-1 .. 0, rows descending. Same callbacks;
// b: the records of chunk 0's first row.
template <typename T, int V, bool PENT, bool FAST, typename Base, typename Ready, typename Release, typename Sink>
__device__ __forceinline__ void bwd_chunks(int C, const typename Recs<T, PENT>::Bwd* b, Vec<T, V>& s1, Vec<T, V>& s2,
                                           Base&& base, Ready&& ready, Release&& release, Sink&& sink) {
  using BwdR = typename Recs<T, PENT>::Bwd;
  if (C <= 0) return;
  Vec<T, V> dq[kSD];
  BwdR bq[kSD];
  ready(C - 1);
  const Vec<T, V>* p = base(C - 1);
  const BwdR* bc0 = b + (C - 1) * kSR;
#pragma unroll
  for (int k = 0; k < kSD; ++k) {
    dq[k] = p[(kSR - 1 - k) * kPR];
    bq[k] = bc0[kSR - 1 - k];
  }
  for (int c = C - 1; c >= 0; --c) {
    const bool more = c > 0;
    const Vec<T, V>* pn = p;
    const BwdR* bc = b + c * kSR;
#pragma unroll
    for (int q = 0; q < kSR; ++q) {  // q-th processed row is r = kSR-1-q
      if (q == kSR - kSD && more) {
        ready(c - 1);
        pn = base(c - 1);
      }
      const Vec<T, V> v = bwd_vec<T, V, PENT, FAST>(bq[q % kSD], dq[q % kSD], s1, s2);
      const int qn = q + kSD;
      if (qn < kSR) {
        dq[q % kSD] = p[(kSR - 1 - qn) * kPR];
        bq[q % kSD] = bc[kSR - 1 - qn];
      } else if (more) {
        dq[q % kSD] = pn[(2 * kSR - 1 - qn) * kPR];
        bq[q % kSD] = bc[kSR - 1 - qn];  // = records of chunk c-1, row 2kSR-1-qn
      }
      sink(c, kSR - 1 - q, v);
    }
    release(c);
    p = pn;
  }
}

// Ring cursor: slot index and mbarrier phase of the next element.
struct Cursor {
  uint32_t slot = 0, phase = 0;
  __device__ __forceinline__ void next(int K) {
    if (++slot == static_cast<uint32_t>(K)) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

// Fused periodic (cyclic) correction, PER = 1 (tri, rank 1) / 2 (pent,
// rank 2), fast mode: the correction needs y_0 (y_1), which the backward
// sweep produces last; but y = U^-1 d-hat, so y_0 = sum_k r0_k d-hat_k with
// r0 = U^-T e_0 (and r1 = U^-T e_1) fixed by the factor. The forward sweep
// accumulates these dot products, the correction coefficients are known
// when the backward sweep starts, and it emits x_i = y_i - w z_i directly:
// one pass, HBM traffic stays at read b once, write x once.
// per_g: r0 | z1 (tri) or r0 | r1 | z1 | z2 (pent), n each; pc: v_last,
// scale (tri) or the capacitance inverse (pent).
struct PerArgs {
  const double* arrays = nullptr;
  double pc[4] = {0.0, 0.0, 0.0, 0.0};
  // fused Crank-Nicolson (CN): x is the old field u (read through the tensor
  // map), out receives u_new; stencil coefficients s, 4s, 1-2s / 1-6s
  void* out = nullptr;
  double cn[3] = {0.0, 0.0, 0.0};
  // TMEM tier (kernel template TM): head chunks [rc_chunks, rc_chunks +
  // tmem_chunks) of each system live in Tensor Memory instead of the L2 spill
  int tmem_chunks = 0;
  // recompute tier (TM only): head chunks [0, rc_chunks) are not stored at
  // all. The forward sweep checkpoints its state every seg_chunks chunks; the
  // backward sweep re-streams b for one segment at a time (last first),
  // re-runs the forward recurrence from the checkpoint into TMEM (the same
  // operations on the same inputs: bitwise the same intermediates), and
  // sweeps back over it. Costs one extra read of b for those rows.
  int rc_chunks = 0;
  int seg_chunks = 0;
};

// TM: 0 = no TMEM tier; 1 = TMEM tier, up to 4 compute warps (one TMEM lane
// quadrant each, 512 columns); 2 = TMEM tier + recompute tier, up to 4
// compute warps; 3 = TMEM + recompute, up to 8 compute warps (warps w and
// w+4 share a lane quadrant, 256 columns each). The recompute code lives only
// in TM >= 2 instances: compiled into the plain TMEM kernel it pushes that
// kernel to 255 registers with spills (measured 0.71 -> 0.49 of roofline at
// N = 512).
__host__ __device__ constexpr int stream_tm_warps(int TM) { return TM == 3 ? 8 : 4; }
__host__ __device__ constexpr int stream_threads(int V, int TM) {
  return 32 * ((TM ? stream_tm_warps(TM) : stream_max_warps(V)) + 2);
}
// TMEM chunks (16 rows) a system can hold: 2 KB (1 KB with 8 warps) of lane storage
__host__ __device__ constexpr int stream_tmem_cap_chunks(int P, size_t elem) {
  return (P > 4 ? 256 : 512) * 4 / (kSR * static_cast<int>(elem));
}

template <typename T, int V, bool PENT, bool FAST, int PER = 0, bool CN = false, int TM = 0>
__global__ void __launch_bounds__(stream_threads(V, TM), 1)
    sweep_stream(const __grid_constant__ CUtensorMap map_b, T* __restrict__ x, int n, long long m, long long ld,
                 int H, int TC, int KB, int KR, int PD, int stagger_ns, long long groups,
                 const void* __restrict__ fwd_g, const void* __restrict__ bwd_g, T* __restrict__ scratch,
                 const PerArgs per, const __grid_constant__ CUtensorMap map_s) {
  static_assert(PER == 0 || (FAST && sizeof(T) == 8 && (PER == 2) == PENT), "fused periodic: fast fp64 only");
  static_assert(!CN || sizeof(T) == 8, "fused Crank-Nicolson: fp64 only");
  static_assert(!TM || V == 1, "TMEM tier: one system per lane");
  constexpr int kPerArrays = PER == 0 ? 0 : (PER == 1 ? 2 : 4);
  // recompute tier geometry (not with the fused CN stencil, whose look-ahead
  // crosses segment ends)
  constexpr bool kRC = TM >= 2 && !CN;
  const int RCc = kRC ? per.rc_chunks : 0;
  const int Lc = RCc > 0 ? per.seg_chunks : 1;
  const int nseg = (RCc + Lc - 1) / Lc;
  using FwdR = typename Recs<T, PENT>::Fwd;
  using BwdR = typename Recs<T, PENT>::Bwd;
  extern __shared__ __align__(128) unsigned char smem[];
  const int P = static_cast<int>(blockDim.x >> 5) - 2;  // compute warps; warp P loads b, warp P+1 reloads
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const StreamLayout L = StreamLayout::make(n, H, TC, P * 32 * V, KB, KR, sizeof(T), sizeof(FwdR), sizeof(BwdR),
                                           kPerArrays, nseg > 0 ? nseg - 1 : 0);
  const double* const spc = reinterpret_cast<const double*>(smem + L.per_off);  // staged per arrays
  const FwdR* sf = reinterpret_cast<const FwdR*>(smem + L.fwd_off);
  const BwdR* sb = reinterpret_cast<const BwdR*>(smem + L.bwd_off);
  T* bring = reinterpret_cast<T*>(smem + L.bring_off);
  T* rring = reinterpret_cast<T*>(smem + L.rring_off);
  T* tail = reinterpret_cast<T*>(smem + L.tail_off);
  uint64_t* b_full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* b_empty = b_full + KB;
  uint64_t* r_full = b_empty + KB;
  uint64_t* r_empty = r_full + KR;
  uint64_t* t_full = r_empty + KR;
  uint64_t* t_empty = t_full + TC;
  uint64_t* spilled = t_empty + TC;  // completes once per group when all warps' spills are published
  const int HC = H / kSR;
  const int RTc = TM ? per.tmem_chunks : 0;  // head chunks held in TMEM (after the recomputed ones)
  const int HS = HC - RCc - RTc;             // head chunks spilled to L2
  const int HT = RCc + RTc;                  // first spilled head chunk
  constexpr int kLW = 32 * V;      // systems per warp
  constexpr int kSBlk = kSR * kLW;  // elements of one warp's block of one chunk
  const int Wg = P * kLW;
  const int chunk = P * kSBlk;  // elements of one chunk (all warps)
  // this CTA's spill scratch: head chunks [HT, HC) x P warps x (kSR x 32V),
  // reused by every group; spill chunk c lives at (c - HT)
  T* const spill_cta = scratch + static_cast<long long>(blockIdx.x) * HS * chunk - static_cast<long long>(HT) * chunk;
  const bool use_tmem = TM && (RTc > 0 || RCc > 0);
  // the spill comes back through 2D TMA loads over the scratch viewed as
  // rows of 32 V elements (map_s, box {32 V, 16 P}): chunk c of this CTA
  // starts at this row
  auto spill_row = [&](int c) {
    return static_cast<int>((static_cast<long long>(blockIdx.x) * HS + (c - HT)) * P * kSR);
  };
  uint32_t& tmem_base_s = *reinterpret_cast<uint32_t*>(spilled + 1);  // written by tcgen05.alloc

  {  // factor records -> smem (16-byte words; device arrays padded to 256 B)
    const int nf = static_cast<int>((static_cast<size_t>(n) * sizeof(FwdR) + 15) / 16);
    const int nb = static_cast<int>((static_cast<size_t>(n) * sizeof(BwdR) + 15) / 16);
    const int4* gf = static_cast<const int4*>(fwd_g);
    const int4* gb = static_cast<const int4*>(bwd_g);
    int4* df = reinterpret_cast<int4*>(smem + L.fwd_off);
    int4* db = reinterpret_cast<int4*>(smem + L.bwd_off);
    for (int k = threadIdx.x; k < nf; k += blockDim.x) df[k] = gf[k];
    for (int k = threadIdx.x; k < nb; k += blockDim.x) db[k] = gb[k];
    if constexpr (PER != 0) {
      double* dp = reinterpret_cast<double*>(smem + L.per_off);
      for (int k = threadIdx.x; k < kPerArrays * n; k += blockDim.x) dp[k] = per.arrays[k];
    }
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < KB; ++k) {
      mbar_init(&b_full[k], 1);
      mbar_init(&b_empty[k], P);
    }
    for (int k = 0; k < KR; ++k) {
      mbar_init(&r_full[k], 1);
      mbar_init(&r_empty[k], P);
    }
    for (int k = 0; k < TC; ++k) {
      mbar_init(&t_full[k], 1);
      mbar_init(&t_empty[k], P);
    }
    mbar_init(spilled, P);
    fence_barrier_init();
  }
  // Every CTA runs the same phases (forward: no HBM traffic for x, backward:
  // x stores plus the next group's loads); odd CTAs start half a period late
  // so the two halves of the GPU interleave their bursts.
  if ((blockIdx.x & 1) && stagger_ns > 0) {
    for (int t = 0; t < stagger_ns; t += 1000) __nanosleep(1000);
  }
  if constexpr (TM != 0) {
    if (warp == 0 && use_tmem) tmem_alloc_512(&tmem_base_s);
    tmem_fence_before();
  }
  __syncthreads();
  uint32_t tmem_lane_base = 0;  // this warp's TMEM lane quadrant and first column
  if constexpr (TM != 0) {
    tmem_fence_after();
    tmem_lane_base = (use_tmem ? tmem_base_s : 0u) + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                     (TM == 3 ? static_cast<uint32_t>((warp >> 2) * 256) : 0u);
  }
  // the k-th recomputed chunk the backward sweep consumes: segments last to
  // first, chunks ascending within a segment (segment j = chunks [j Lc, ..))
  auto rc_chunk = [RCc, Lc, nseg](int k) {
    const int last_len = RCc - (nseg - 1) * Lc;
    if (k < last_len) return (nseg - 1) * Lc + k;
    k -= last_len;
    return (nseg - 2 - k / Lc) * Lc + k % Lc;
  };

  // tail chunk k of the group with iteration parity `par` lives in slot
  // par ? TC-1-k : k
  auto tail_slot = [TC](int k, uint32_t par) { return par ? TC - 1 - k : k; };
  const uint32_t c_bytes = static_cast<uint32_t>(chunk * sizeof(T));

  // ----------------------------------------------------- loader warp (b, tail)
  // Order per group g: the first min(KB, HC) head chunks (their slots were
  // freed by group g-1's forward head, so they load during g-1's tail and
  // backward sweeps), then g's tail (slots freed by g-1's backward tail),
  // then the remaining head chunks as g's own forward sweep drains the ring.
  if (warp == P) {
    if (lane != 0) return;
    const uint64_t pol_b = policy_evict_first();  // every byte of b is read once
    const uint64_t pol_keep = policy_evict_last();
    const long long my_groups = (groups - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int GB = HC + RCc;                    // b chunks per group: the head, then the recomputed segments
    const long long b_total = my_groups * GB;  // b chunks this CTA streams through the ring
    long long b_next = 0;                      // next b chunk (CTA-local index) to enter the ring
    long long b_pf = 0;                        // b chunks prefetched into L2 so far
    Cursor cur;
    uint32_t issued = 0;
    auto load_chunk = [&](T* dst, int c0, int row, uint64_t* bar) {
      mbar_expect_tx(bar, c_bytes);
      for (int w = 0; w < P; ++w) tma_load_2d(dst + w * kSBlk, &map_b, c0 + w * kLW, row, bar, pol_b);
    };
    auto prefetch = [&]() {
      while (b_pf < b_total && b_pf < b_next + PD) {
        const long long gi = b_pf / GB;
        const int k = static_cast<int>(b_pf - gi * GB);
        const int c = k < HC ? k : rc_chunk(k - HC);
        const int c0 = static_cast<int>((blockIdx.x + gi * gridDim.x) * Wg);
        for (int w = 0; w < P; ++w) tma_prefetch_2d(&map_b, c0 + w * kLW, c * kSR);
        ++b_pf;
      }
    };
    uint32_t it = 0;
    for (long long g = blockIdx.x; g < groups; g += gridDim.x, ++it) {
      const int c0 = static_cast<int>(g * Wg);
      const uint32_t par = it & 1u;
      const int pre = HC < KB ? HC : KB;
      auto load_tail = [&]() {
        for (int k = 0; k < TC; ++k) {
          const int s = tail_slot(k, par);
          if (it > 0) mbar_wait(&t_empty[s], (it - 1) & 1u);
          load_chunk(tail + s * chunk, c0, H + k * kSR, &t_full[s]);
        }
      };
      for (int c = 0; c < HC; ++c) {
        if (c == pre) load_tail();
        if (issued >= static_cast<uint32_t>(KB)) mbar_wait(&b_empty[cur.slot], cur.phase ^ 1u);
        load_chunk(bring + cur.slot * chunk, c0, c * kSR, &b_full[cur.slot]);
        cur.next(KB);
        ++issued;
        ++b_next;
        prefetch();
      }
      if (pre == HC) load_tail();
      if (KR == 0 && HS > 0) {  // unified ring: the spill comes back through the same FIFO
        mbar_wait(spilled, par);
        for (int c = HC - 1; c >= HT; --c) {
          if (issued >= static_cast<uint32_t>(KB)) mbar_wait(&b_empty[cur.slot], cur.phase ^ 1u);
          mbar_expect_tx(&b_full[cur.slot], c_bytes);
          tma_load_2d(bring + cur.slot * chunk, &map_s, 0, spill_row(c), &b_full[cur.slot], pol_keep);
          cur.next(KB);
          ++issued;
        }
      }
      for (int k = 0; k < RCc; ++k) {  // b again for the recomputed segments
        if (issued >= static_cast<uint32_t>(KB)) mbar_wait(&b_empty[cur.slot], cur.phase ^ 1u);
        load_chunk(bring + cur.slot * chunk, c0, rc_chunk(k) * kSR, &b_full[cur.slot]);
        cur.next(KB);
        ++issued;
        ++b_next;
        prefetch();
      }
    }
    return;
  }

  // ------------------------------------------------ reloader warp (spilled d-hat)
  if (warp == P + 1) {
    if (lane != 0 || HS <= 0 || KR == 0) return;
    const uint64_t pol_keep = policy_evict_last();
    Cursor cur;
    uint32_t issued = 0;
    uint32_t it = 0;
    for (long long g = blockIdx.x; g < groups; g += gridDim.x, ++it) {
      mbar_wait(spilled, it & 1u);  // every warp's head d-hat of this group is in the scratch
      for (int c = HC - 1; c >= HT; --c) {
        if (issued >= static_cast<uint32_t>(KR)) mbar_wait(&r_empty[cur.slot], cur.phase ^ 1u);
        mbar_expect_tx(&r_full[cur.slot], c_bytes);
        tma_load_2d(rring + cur.slot * chunk, &map_s, 0, spill_row(c), &r_full[cur.slot], pol_keep);
        cur.next(KR);
        ++issued;
      }
    }
    return;
  }

  // ------------------------------------------------------------ compute warps
  using P2 = Vec<T, V>;  // a lane's V systems
  const uint64_t pol_keep = policy_evict_last();
  const int wl = warp * (kSBlk / V) + lane;  // this lane's vector offset within a chunk
  const int cpairs = chunk / V;              // vectors per chunk
  P2* const bring_l = reinterpret_cast<P2*>(bring) + wl;
  P2* const rring_l = reinterpret_cast<P2*>(rring) + wl;
  P2* const tail_l = reinterpret_cast<P2*>(tail) + wl;
  P2* const spill_l = reinterpret_cast<P2*>(spill_cta) + wl;
  // recompute checkpoints: entry k of this lane at ck_l[k * ck_stride]
  Vec<T, 2>* const ck_l = reinterpret_cast<Vec<T, 2>*>(smem + L.ck_off) + warp * 32 + lane;
  const int ck_stride = Wg;
  const int tfull = (n - H) / kSR;  // full tail chunks (a partial one may follow)
  const int trem = (n - H) - tfull * kSR;
  Cursor bw, brl, rw, rrl;  // wait / release cursors of the two rings
  uint32_t it = 0;

  long long g = blockIdx.x;
  // Fused Crank-Nicolson: the forward sweep consumes f_i = (B u)_i, formed
  // from a register window of raw rows (u_{i-2}, u_{i-1} kept, u_{i+1},
  // u_{i+2} from the software pipeline). The wrap rows u_{n-2}, u_{n-1} that
  // row 0 needs are loaded from global one group ahead; u_0, u_1 (for the
  // last rows) are kept when they stream past.
  T* const xout = CN ? static_cast<T*>(per.out) : x;
  const uint64_t pol_wrap = policy_evict_first();
  auto load_wrap = [&](long long grp, P2& w1, P2& w2) {  // rows n-1, n-2 of this lane's columns
    const long long jj = grp * Wg + warp * kLW + V * lane;
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const bool ok = grp < groups && jj + q < m;
      w1.v[q] = ok ? ld_spill(x + static_cast<long long>(n - 1) * ld + jj + q, pol_wrap) : T(0);
      w2.v[q] = ok ? ld_spill(x + static_cast<long long>(n - 2) * ld + jj + q, pol_wrap) : T(0);
    }
  };
  P2 nw1{}, nw2{};  // next group's wrap rows
  if constexpr (CN) load_wrap(g, nw1, nw2);
  // One group. kFull: every column of the group exists (all groups but
  // possibly the last), so the x stores are unconditional 16-byte stores.
  auto run_group = [&](auto full_tag) {
    constexpr bool kFull = decltype(full_tag)::value;
    const long long j = g * Wg + warp * kLW + V * lane;  // this lane's first column
    const bool live2 = kFull || j + V - 1 < m;           // all V columns exist
    const bool live1 = kFull || j < m;                   // the first one does
    const uint32_t par = it & 1u;
    T* out = xout + (live1 ? j : 0) + static_cast<long long>(n - 1) * ld;
    auto put = [&](P2 v) {
      if (kFull) {
        st_stream_vec<T, V>(reinterpret_cast<P2*>(out), v);
      } else {
        if (live2) st_stream_vec<T, V>(reinterpret_cast<P2*>(out), v);
        else if (live1) st_stream(out, v.v[0]);
      }
      out -= ld;
    };
    P2 s1{}, s2{};
    TPiece<T> tbuf;  // TMEM tier staging (one piece of rows)
    using TP = TPiece<T>;
    // CN window: w1 = u_{i-1}, w2 = u_{i-2}; u0s/u1s = u_0, u_1 for the wrap
    P2 w1 = nw1, w2 = nw2, u0s{}, u1s{};
    auto stencil = [&](int row, P2 u, auto&& look) -> P2 {
      if constexpr (!CN) {
        return u;
      } else {
        const T cs = T(per.cn[0]), cs4 = T(per.cn[1]), cmid = T(per.cn[2]);
        const P2 d1 = look(1);
        P2 f;
        if constexpr (!PENT) {  // pde.cpp:85  o = s*(up + dn) + mid*mi
#pragma unroll
          for (int q = 0; q < V; ++q) f.v[q] = add_rn(mul_rn(cs, add_rn(w1.v[q], d1.v[q])), mul_rn(cmid, u.v[q]));
        } else {  // pde.cpp:108  o = -s*(u2 + d2) + s4*(u1 + d1) + mid*mi
          const P2 d2 = look(2);
#pragma unroll
          for (int q = 0; q < V; ++q)
            f.v[q] = add_rn(add_rn(mul_rn(-cs, add_rn(w2.v[q], d2.v[q])), mul_rn(cs4, add_rn(w1.v[q], d1.v[q]))),
                            mul_rn(cmid, u.v[q]));
        }
        if (row == 0) u0s = u;
        if (row == 1) u1s = u;
        w2 = w1;
        w1 = u;
        return f;
      }
    };
    // raw row `row` >= H of the old field (tail smem, or the wrap past n)
    auto tslot0 = [&](int k) { return tail_l + tail_slot(k, par) * cpairs; };
    auto raw_tail = [&](int row) -> P2 {
      if (row >= n) return row == n ? u0s : u1s;
      const int k = (row - H) / kSR;
      mbar_wait(&t_full[tail_slot(k, par)], par);
      return tslot0(k)[((row - H) - k * kSR) * kPR];
    };
    // fused periodic: y_0 (y_1) accumulated as dot products of the forward
    // outputs; correction coefficients w (tri) / t1, t2 (pent) per system
    P2 acc0{}, acc1{}, c1{}, c2{};
    auto accum = [&](int row, P2 v) {
      if constexpr (PER != 0) {
#pragma unroll
        for (int q = 0; q < V; ++q) {
          acc0.v[q] = fma_rn(T(spc[row]), v.v[q], acc0.v[q]);
          if constexpr (PER == 2) acc1.v[q] = fma_rn(T(spc[n + row]), v.v[q], acc1.v[q]);
        }
      }
    };
    auto emit = [&](int row, P2 y) {  // x_i = y_i - w z_i  (pent: - (z1_i t1 + z2_i t2))
      if constexpr (PER == 1) {
#pragma unroll
        for (int q = 0; q < V; ++q) y.v[q] = fma_rn(-c1.v[q], T(spc[n + row]), y.v[q]);
      } else if constexpr (PER == 2) {
#pragma unroll
        for (int q = 0; q < V; ++q)
          y.v[q] = fma_rn(-c1.v[q], T(spc[2 * n + row]), fma_rn(-c2.v[q], T(spc[3 * n + row]), y.v[q]));
      }
      put(y);
    };

    // ---- forward, head rows: b ring -> registers -> d-hat spilled to L2
    {
      uint32_t cs = 0;
      fwd_chunks<T, V, PENT, FAST>(
          HC, sf, s1, s2, [&](int) { return bring_l + cs * cpairs; },
          [&](int) {
            cs = bw.slot;
            mbar_wait(&b_full[bw.slot], bw.phase);
            bw.next(KB);
          },
          [&](int) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&b_empty[brl.slot]);
            brl.next(KB);
          },
          [&](int c, int r, P2*, P2 v) {
            if (kRC && c < RCc) {  // recompute tier: keep only the segment-start states
              if constexpr (kRC) {
                if (r == kSR - 1 && (c + 1) % Lc == 0 && c + 1 < RCc) ck_l[((c + 1) / Lc - 1) * ck_stride] = Vec<T, 2>{{s1.v[0], s2.v[0]}};
              }
            } else if (TM && c < HT) {  // TMEM tier: gather the chunk, one tcgen05.st per 16 rows
              if constexpr (TM != 0) {
                tbuf.put(r % TP::kRows, v.v[0]);
                if (r % TP::kRows == TP::kRows - 1)
                  tbuf.store(tmem_lane_base +
                             static_cast<uint32_t>(((c - RCc) * kSR + r - (TP::kRows - 1)) * TP::kColsPerRow));
              }
            } else {
              st_spill_vec<T, V>(spill_l + c * cpairs + r * kPR, v, pol_keep);
            }
            accum(c * kSR + r, v);
          },
          [&](int c, int r, P2 u, auto&& look) { return stencil(c * kSR + r, u, look); },
          [&](int k) { return raw_tail(H + k); });
    }
    if (HS > 0) {  // publish the spill to the async proxy (the reloader's bulk copies)
      fence_proxy_async_global();
      __syncwarp();
      if (lane == 0) mbar_arrive(spilled);
    }

    // ---- forward, tail rows: in place in smem
    auto tslot = [&](int k) { return tail_l + tail_slot(k, par) * cpairs; };
    fwd_chunks<T, V, PENT, FAST>(
        tfull, sf + H, s1, s2, tslot, [&](int k) { mbar_wait(&t_full[tail_slot(k, par)], par); }, [](int) {},
        [&](int c, int r, P2* p, P2 v) {
          *p = v;
          accum(H + c * kSR + r, v);
        },
        [&](int c, int r, P2 u, auto&& look) { return stencil(H + c * kSR + r, u, look); },
        [&](int k) { return raw_tail(H + tfull * kSR + k); });
    if (trem > 0) {
      mbar_wait(&t_full[tail_slot(tfull, par)], par);
      P2* p = tslot(tfull);
      const FwdR* f = sf + H + tfull * kSR;
      for (int r = 0; r < trem; ++r) {
        const int row = H + tfull * kSR + r;
        const P2 in = stencil(row, p[r * kPR], [&](int k) { return raw_tail(row + k); });
        p[r * kPR] = fwd_vec<T, V, PENT, FAST>(f[r], in, s1, s2);
        accum(row, p[r * kPR]);
      }
    }
    if constexpr (CN) load_wrap(g + gridDim.x, nw1, nw2);  // the next group's wrap rows, a group ahead
    fence_proxy_async_smem();  // in-place smem writes before the TMA refills of these slots
    if constexpr (PER == 1) {  // w = (y_0 + v_last y_{n-1}) * scale, y_{n-1} = d-hat_{n-1}
#pragma unroll
      for (int q = 0; q < V; ++q) c1.v[q] = T(per.pc[1]) * fma_rn(T(per.pc[0]), s1.v[q], acc0.v[q]);
    } else if constexpr (PER == 2) {  // y_{n-1} = g_{n-1}, y_{n-2} = g_{n-2} - gamma_{n-2} g_{n-1}
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const T yl = s1.v[q];
        const T yl2 = fma_rn(-T(sb[n - 2].g), s1.v[q], s2.v[q]);
        const T w1 = acc0.v[q] - yl, w2 = acc1.v[q] - yl2;
        c1.v[q] = fma_rn(T(per.pc[0]), w1, T(per.pc[1]) * w2);
        c2.v[q] = fma_rn(T(per.pc[2]), w1, T(per.pc[3]) * w2);
      }
    }

    // ---- backward, tail rows: smem -> x streamed to HBM; each drained chunk
    // goes back to the loader for the next group
    s1 = P2{};
    s2 = P2{};
    auto tail_release = [&](int k) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_empty[tail_slot(k, par)]);
    };
    if (trem > 0) {
      const P2* p = tslot(tfull);
      const BwdR* b = sb + H + tfull * kSR;
      for (int r = trem - 1; r >= 0; --r)
        emit(H + tfull * kSR + r, bwd_vec<T, V, PENT, FAST>(b[r], p[r * kPR], s1, s2));
      tail_release(tfull);
    }
    bwd_chunks<T, V, PENT, FAST>(
        tfull, sb + H, s1, s2, [&](int k) -> const P2* { return tslot(k); }, [](int) {}, tail_release,
        [&](int c, int r, P2 v) { emit(H + c * kSR + r, v); });

    // ---- backward, head rows: d-hat back through the reload ring (or, with
    // KR == 0, through the b ring: one FIFO), x to HBM
    {
      const bool uni = KR == 0;
      Cursor& cw = uni ? bw : rw;
      Cursor& cr = uni ? brl : rrl;
      P2* const ring_l = uni ? bring_l : rring_l;
      uint64_t* const full = uni ? b_full : r_full;
      uint64_t* const empty = uni ? b_empty : r_empty;
      const int K = uni ? KB : KR;
      uint32_t cs = 0;
      bwd_chunks<T, V, PENT, FAST>(
          HS, sb + HT * kSR, s1, s2, [&](int) -> const P2* { return ring_l + cs * cpairs; },
          [&](int) {
            cs = cw.slot;
            mbar_wait(&full[cw.slot], cw.phase);
            cw.next(K);
          },
          [&](int) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[cr.slot]);
            cr.next(K);
          },
          [&](int c, int r, P2 v) { emit((HT + c) * kSR + r, v); });
    }
    // ---- backward, TMEM rows: one tcgen05.ld per 16 rows, a chunk ahead.
    // nc chunks at TMEM columns [0, nc) hold rows [row0, row0 + 16 nc).
    auto tmem_bwd = [&](int nc, int row0) {
      if constexpr (TM != 0) {
        const int np = nc * (kSR / TP::kRows);  // pieces, processed last to first, one loaded ahead
        tmem_wait_st();  // this warp's stores of the region have landed
        TP cur, nxt;
        cur.load(tmem_lane_base + static_cast<uint32_t>((np - 1) * TP::kWords));
        cur.wait();
        for (int pc = np - 1; pc >= 0; --pc) {
          if (pc > 0) nxt.load(tmem_lane_base + static_cast<uint32_t>((pc - 1) * TP::kWords));
          const BwdR* b = sb + row0 + pc * TP::kRows;
#pragma unroll
          for (int q = 0; q < TP::kRows; ++q) {
            const int r = TP::kRows - 1 - q;
            P2 y;
            y.v[0] = bwd_row<T, PENT, FAST>(b[r], cur.get(r), s1.v[0], s2.v[0]);
            emit(row0 + pc * TP::kRows + r, y);
          }
          if (pc > 0) {
            nxt.wait();
            cur = nxt;
          }
        }
      }
    };
    if (TM && RTc > 0) tmem_bwd(RTc, RCc * kSR);
    // ---- backward, recomputed rows: per segment (last first) b comes back
    // through the b ring, the forward recurrence re-runs from the segment's
    // checkpoint into TMEM, and the backward sweep continues over it
    if constexpr (kRC) {
      for (int j = nseg - 1; j >= 0; --j) {
        const int cb = j * Lc;
        const int len = min(Lc, RCc - cb);
        P2 f1{}, f2{};
        if (j > 0) {
          const Vec<T, 2> ck = ck_l[(j - 1) * ck_stride];
          f1.v[0] = ck.v[0];
          f2.v[0] = ck.v[1];
        }
        uint32_t cs = 0;
        fwd_chunks<T, V, PENT, FAST>(
            len, sf + cb * kSR, f1, f2, [&](int) { return bring_l + cs * cpairs; },
            [&](int) {
              cs = bw.slot;
              mbar_wait(&b_full[bw.slot], bw.phase);
              bw.next(KB);
            },
            [&](int) {
              __syncwarp();
              if (lane == 0) mbar_arrive(&b_empty[brl.slot]);
              brl.next(KB);
            },
            [&](int c, int r, P2*, P2 v) {
              tbuf.put(r % TP::kRows, v.v[0]);
              if (r % TP::kRows == TP::kRows - 1)
                tbuf.store(tmem_lane_base + static_cast<uint32_t>((c * kSR + r - (TP::kRows - 1)) * TP::kColsPerRow));
            });
        tmem_bwd(len, cb * kSR);
      }
    }
  };
  for (; g < groups; g += gridDim.x, ++it) {
    if ((g + 1) * Wg <= m) run_group(std::true_type{});
    else run_group(std::false_type{});
  }

  // the scratch is dead: drop this warp's L2 lines instead of writing them back
  if (HS > 0) {
    __syncwarp();
    for (int c = HT; c < HC; ++c) {
      const char* base = reinterpret_cast<const char*>(spill_cta + static_cast<long long>(c) * chunk + warp * kSBlk);
      for (int off = lane * 128; off < kSBlk * static_cast<int>(sizeof(T)); off += 32 * 128)
        discard_l2_line(base + off);
    }
  }
  if constexpr (TM != 0) {  // every compute warp is done with TMEM: warp 0 frees it
    if (use_tmem) {
      tmem_fence_before();
      asm volatile("bar.sync 1, %0;" ::"r"(P * 32) : "memory");
      tmem_fence_after();
      if (warp == 0) tmem_dealloc_512(tmem_base_s);
    }
  }
}

}  // namespace dev
}  // namespace bsb
