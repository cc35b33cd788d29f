// Pipelined sequential shared-LHS sweep (sm_100a): the exact-mode kernel for
// many systems. Up to 512 rows every forward intermediate stays on chip;
// beyond, the last row chunks live in an L2 scratch tier.
//
// The exact mode must follow the reference's operation order
// (tri_solver.cpp:25-47, pent_solver.cpp:19-62): one sequential recurrence
// per system, so a system's n forward intermediates stay alive until its
// backward sweep, and the streaming kernel (sweep_stream.cuh) spills the
// rows that do not fit on chip to L2 (~20% throughput for any spill).
//
// Here each lane keeps ALL n rows of its system on chip — the first 256 in
// its TMEM lane (one lane quadrant per compute warp), the rest in shared
// memory — and the warp software-pipelines across groups exactly like
// sweep_spike.cuh: in step k it runs backward row chunk CL-1-k of group g and
// forward row chunk k of group g + 1 in ONE 16-row loop (two independent
// dependency chains interleaved in the instruction stream), and the forward
// chunk is stored into the storage slot the backward chunk has just been
// read from (slot p ? CL-1-k : k for group parity p), so the storage per lane
// stays n rows while both chains run. HBM traffic: read b once, write x once.
//
// P compute warps (32 P systems per group) + one TMA producer warp. The row
// formulas are sweep_kernels.cuh's (exact: bitwise equal to the reference).
#pragma once

#include "sweep_spike.cuh"

namespace bsb {
namespace dev {

constexpr int kPpR = 16;      // rows per chunk (one TMA box {32 x 16} per warp)
constexpr int kPpTmemRows = 256;  // rows per lane in TMEM (512 columns of fp64)
constexpr int kPpStage = 3;       // L2-tier chunks in flight per warp (cp.async staging slots)

// staging slots of the L2 tier: kPpStage when any chunk lives in L2
__host__ __device__ inline int pipe_stage_chunks(int n, int RT, int ST) {
  const int CL = n / kPpR;
  const int TT = CL < kPpTmemRows / kPpR ? CL : kPpTmemRows / kPpR;
  return CL - TT - RT - ST > 0 ? kPpStage : 0;
}

__device__ __forceinline__ void cp_async_16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct PipeLayout {
  size_t fwd_off, bwd_off, z_off, stor_off, stage_off, ring_off, bar_off, total;
  // n rows (multiple of 16), P compute warps, KB ring slots, ST shared-memory
  // storage chunks per lane (the first TT = min(n/16, 16) chunks live in
  // TMEM, then RT in registers, then ST in smem, the rest in the L2 scratch)
  // zw: doubles per row of the periodic correction's z (0, 1 tri, 2 pent);
  // DS: staging chunks of the L2 tier (pipe_stage_chunks)
  __host__ __device__ static PipeLayout make(int n, int P, int KB, size_t fwd_rec, size_t bwd_rec, int ST,
                                             int zw = 0, int DS = 0) {
    PipeLayout L{};
    L.fwd_off = 0;
    L.bwd_off = align128(static_cast<size_t>(n) * fwd_rec);
    L.z_off = L.bwd_off + align128(static_cast<size_t>(n) * bwd_rec);
    L.stor_off = L.z_off + align128(static_cast<size_t>(n) * zw * sizeof(double));
    // shared-memory slots: [ST][P warps][16 rows][32 lanes]
    L.stage_off = L.stor_off + static_cast<size_t>(ST) * P * kPpR * 32 * sizeof(double);
    L.ring_off = L.stage_off + static_cast<size_t>(DS) * P * kPpR * 32 * sizeof(double);
    L.bar_off = L.ring_off + static_cast<size_t>(KB) * P * kPpR * 32 * sizeof(double);
    L.total = L.bar_off + static_cast<size_t>(2 * KB + 1) * sizeof(uint64_t);
    return L;
  }
};

// One forward row (chain state fs1/fs2) and one backward row (bs1/bs2) of
// two different groups, written as interleaved stages so that each stage
// issues one operation of each chain: the chain-independent parts first
// (b - eps g2, delta x2), then the three dependent operations of each
// recurrence side by side. The operation order of each recurrence is the
// reference's (exact) or the FMA form (fast).
template <bool PENT, bool FAST, bool FW, bool BW, typename T = double>
__device__ __forceinline__ void pipe_rows(const typename Recs<Scalar<T>, PENT>::Fwd& fr, T d, T& fs1, T& fs2, T& fv,
                                          const typename Recs<Scalar<T>, PENT>::Bwd& br, T g, T& bs1, T& bs2,
                                          T& bv) {
  if constexpr (FAST) {
    if constexpr (FW) {
      if constexpr (PENT) fv = fma_rn(-fr.b, fs1, fma_rn(-fr.e, fs2, mul_rn(d, fr.ia)));
      else fv = fma_rn(-fr.a, fs1, mul_rn(d, fr.m));
    }
    if constexpr (BW) {
      if constexpr (PENT) bv = fma_rn(-br.g, bs1, fma_rn(-br.d, bs2, g));
      else bv = fma_rn(-br, bs1, g);
    }
  } else if constexpr (PENT) {
    T tf{}, xb{}, uf{}, ub{};
    if constexpr (FW) tf = sub_rn(d, mul_rn(fr.e, fs2));   // f - eps g2 (g2: one row old)
    if constexpr (BW) xb = mul_rn(br.d, bs2);              // delta x2 (x2: one row old)
    if constexpr (FW) uf = mul_rn(fr.b, fs1);              // chains: one op of each per stage
    if constexpr (BW) ub = mul_rn(br.g, bs1);
    if constexpr (FW) uf = sub_rn(tf, uf);
    if constexpr (BW) ub = add_rn(ub, xb);
    if constexpr (FW) fv = mul_rn(uf, fr.ia);              // ((f - eps g2) - beta g1) * ia
    if constexpr (BW) bv = sub_rn(g, ub);                  // g - (gamma x1 + delta x2)
  } else {
    T uf{}, ub{};
    if constexpr (FW) uf = mul_rn(fr.a, fs1);
    if constexpr (BW) ub = mul_rn(br, bs1);
    if constexpr (FW) uf = sub_rn(d, uf);
    if constexpr (BW) bv = sub_rn(g, ub);                  // dhat - chat next
    if constexpr (FW) fv = mul_rn(uf, fr.m);               // (d - a prev) * m
  }
  if constexpr (FW) {
    fs2 = fs1;
    fs1 = fv;
  }
  if constexpr (BW) {
    bs2 = bs1;
    bs1 = bv;
  }
}

// RT: storage chunks per lane held in REGISTERS (after the TMEM chunks; a
// lane's 16 x RT values in a statically indexed array, reached through a
// switch on the slot). With RT = 4 and 3 compute warps, 96 systems of 512
// rows fit on chip (TMEM 256 + registers 64 + shared memory 192 rows).
// PER: the periodic (Woodbury) correction fused, bitwise in exact mode. Its
// coefficients need y_0 (y_1) — the last values the backward sweep produces
// — so each group gets a first backward pass over its on-chip intermediates
// that keeps only y_{n-1}, y_{n-2}, y_1, y_0 (no memory traffic), then the
// interleaved second pass recomputes the same y (the same operations on the
// same values: the same bits) and stores x_i = y_i - w z_i in the reference's
// order (periodic.cpp:80-85, :189-203). z: z1 (and z2) of n doubles.
struct PipePer {
  const double* z1 = nullptr;
  const double* z2 = nullptr;
  double c[4] = {0.0, 0.0, 0.0, 0.0};  // tri: v_last, scale; pent: cap_inv
  // Crank-Nicolson step (template CN, with PER): b = the explicit periodic
  // stencil of the old field u (the tensor map's source), in the reference's
  // operation order (pde.cpp:85 / :108); x receives u_new. cn = s, 4s, mid
  const double* u = nullptr;
  double cn[3] = {0.0, 0.0, 0.0};
};

// T: double, or float2 = two fp32 systems per lane (packed FMUL2/FADD2 in
// the same operation order: the bits of the scalar fp32 sweep), stored and
// moved as 8-byte words exactly like fp64; x, m, ld then count pairs.
template <bool PENT, bool FAST, int P, int RT = 0, bool PER = false, bool CN = false, typename T = double>
__global__ void __launch_bounds__(32 * (P + 1), 1)
    sweep_pipe(const __grid_constant__ CUtensorMap map_b, double* __restrict__ x, int n, long long m, long long ld,
               int KB, int PD, long long groups, const void* __restrict__ fwd_g, const void* __restrict__ bwd_g,
               double* __restrict__ sink, int ST, double* __restrict__ scratch, PipePer per) {
  static_assert(std::is_same<T, double>::value || (!PER && !CN), "fp32 pairs: plain solves only");
  using FwdR = typename Recs<Scalar<T>, PENT>::Fwd;
  using BwdR = typename Recs<Scalar<T>, PENT>::Bwd;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int ZW = PER ? (PENT ? 2 : 1) : 0;
  const int DS = pipe_stage_chunks(n, RT, ST);
  const PipeLayout Ly = PipeLayout::make(n, P, KB, sizeof(FwdR), sizeof(BwdR), ST, ZW, DS);
  double* const sz = reinterpret_cast<double*>(smem + Ly.z_off);  // [n][ZW]
  const FwdR* sf = reinterpret_cast<const FwdR*>(smem + Ly.fwd_off);
  const BwdR* sb = reinterpret_cast<const BwdR*>(smem + Ly.bwd_off);
  double* stor = reinterpret_cast<double*>(smem + Ly.stor_off);
  double* ring = reinterpret_cast<double*>(smem + Ly.ring_off);
  double* stage = reinterpret_cast<double*>(smem + Ly.stage_off);  // [DS][P warps][16 rows][32 lanes]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Ly.bar_off);
  uint64_t* empty = full + KB;
  uint32_t& tmem_base_s = *reinterpret_cast<uint32_t*>(empty + KB);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int kBox = kPpR * 32;
  constexpr int kChunk = P * kBox;
  constexpr int Wg = 32 * P;
  const int CL = n / kPpR;
  const int TT = CL < kPpTmemRows / kPpR ? CL : kPpTmemRows / kPpR;  // chunks per lane in TMEM

  {  // factor records -> smem (16-byte words)
    const uint4* sfw = static_cast<const uint4*>(fwd_g);
    const uint4* sbw = static_cast<const uint4*>(bwd_g);
    uint4* df = reinterpret_cast<uint4*>(smem + Ly.fwd_off);
    uint4* db = reinterpret_cast<uint4*>(smem + Ly.bwd_off);
    const int wf = static_cast<int>((static_cast<size_t>(n) * sizeof(FwdR) + 15) / 16);
    const int wb = static_cast<int>((static_cast<size_t>(n) * sizeof(BwdR) + 15) / 16);
    for (int i = threadIdx.x; i < wf; i += blockDim.x) df[i] = sfw[i];
    for (int i = threadIdx.x; i < wb; i += blockDim.x) db[i] = sbw[i];
    if constexpr (PER) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        sz[ZW * i] = per.z1[i];
        if constexpr (PENT) sz[ZW * i + 1] = per.z2[i];
      }
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < KB; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], P);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_512(&tmem_base_s);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == P) {  // ---- producer: b chunks through the ring (one box per warp)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const long long my_groups = (groups - blockIdx.x + gridDim.x - 1) / gridDim.x;
      const long long total = my_groups * CL;
      long long pf = 0;
      int slot = 0;
      uint32_t phase = 0;
      for (long long t = 0; t < total; ++t) {
        for (; pf < total && pf < t + PD; ++pf) {
          const long long gi = pf / CL;
          const int c = static_cast<int>(pf - gi * CL);
          const int c0 = static_cast<int>((blockIdx.x + gi * gridDim.x) * Wg);
          for (int w = 0; w < P; ++w) tma_prefetch_2d(&map_b, c0 + w * 32, c * kPpR);
        }
        if (t >= KB) mbar_wait(&empty[slot], phase ^ 1u);
        const long long gi = t / CL;
        const int c = static_cast<int>(t - gi * CL);
        const int c0 = static_cast<int>((blockIdx.x + gi * gridDim.x) * Wg);
        mbar_expect_tx(&full[slot], kChunk * sizeof(double));
        for (int w = 0; w < P; ++w)
          tma_load_2d(ring + slot * kChunk + w * kBox, &map_b, c0 + w * 32, c * kPpR, &full[slot], pol);
        if (++slot == KB) {
          slot = 0;
          phase ^= 1u;
        }
      }
    }
    return;
  }

  // ---- compute warps: lane = one system of the warp's 32
  const uint32_t tlane = tmem_base_s + (static_cast<uint32_t>(32 * warp) << 16);
  // storage slot of chunk c of a group with parity p
  auto sidx = [&](uint32_t p, int c) { return p ? CL - 1 - c : c; };
  // tiers by slot: TMEM [0, TT), registers [TT, TT + RT), shared memory
  // [.., + ST), the L2 scratch [.., CL)
  const int TR = TT + RT;
  auto slot_smem = [&](int s) { return stor + (static_cast<size_t>(s - TR) * P + warp) * kBox + lane; };
  // L2 tier: this CTA's scratch, [GT chunks][P warps][16 rows][32 lanes]
  const int GT = CL - TR - ST;
  double* const scr = scratch + static_cast<long long>(blockIdx.x) * GT * P * kBox;
  auto slot_l2 = [&](int s) { return scr + (static_cast<long long>(s - TR - ST) * P + warp) * kBox + lane; };
  double rs[RT > 0 ? RT * kPpR : 1];  // register tier (static indices only)
  (void)rs;
  const uint64_t pol_keep = policy_evict_last();
  int slot = 0;
  uint32_t phase = 0;
  T fs1{}, fs2{};  // forward state (group being read)
  T bs1{}, bs2{};  // backward state (group being written)
  double wt1 = 0.0, wt2 = 0.0;  // periodic correction coefficients of the group being written
  long long step = 0;
  double* out = sink + lane;
  TPiece<double> cur;  // the backward chunk's 16 forward values

  // L2 tier: chunk c of the group being written (parity pw) -> staging slot
  // c % DS, as one cp.async group (empty when the chunk is not in L2), DS
  // chunks ahead of its use, so the L2 latency overlaps the row loops. A
  // lane copies 16-byte pieces of other lanes' words (the warp syncs).
  auto l2_prefetch = [&](uint32_t pw, int c) {
    if (GT > 0) {
      if (c >= 0 && sidx(pw, c) >= TR + ST) {
        const double* src = slot_l2(sidx(pw, c)) - lane;
        double* dst = stage + (static_cast<size_t>(c % DS) * P + warp) * kBox;
#pragma unroll
        for (int k = 0; k < kBox / 64; ++k) cp_async_16(dst + 2 * (lane + 32 * k), src + 2 * (lane + 32 * k));
      }
      cp_async_commit();
    }
  };
  // load the backward chunk c's values from slot s (TMEM: asynchronous, waited
  // in step(); L2 tier: from the staging slot when staged, else directly)
  auto bwd_load = [&](int s, int c, bool staged) {
    if (s < TT) {
      cur.load(tlane + static_cast<uint32_t>(s * TPiece<double>::kWords));
    } else if (s < TR) {
      if constexpr (RT > 0) {
        switch (s - TT) {
#define BSB_RS_LOAD(K)                                                      \
  case K:                                                                   \
    if constexpr (K < RT) {                                                 \
      _Pragma("unroll") for (int r = 0; r < kPpR; ++r) cur.put(r, rs[K * kPpR + r]); \
    }                                                                       \
    break;
          BSB_RS_LOAD(0) BSB_RS_LOAD(1) BSB_RS_LOAD(2) BSB_RS_LOAD(3)
#undef BSB_RS_LOAD
        }
      }
    } else if (s < TR + ST) {
      const double* q = slot_smem(s);
#pragma unroll
      for (int r = 0; r < kPpR; ++r) cur.put(r, q[r * 32]);
    } else if (staged) {
      cp_async_wait<kPpStage - 1>();  // DS - 1 younger groups may still be in flight
      __syncwarp();
      const double* q = stage + (static_cast<size_t>(c % DS) * P + warp) * kBox + lane;
#pragma unroll
      for (int r = 0; r < kPpR; ++r) cur.put(r, q[r * 32]);
    } else {  // this lane's own words, written by this lane one round earlier
      const double* q = slot_l2(s);
#pragma unroll
      for (int r = 0; r < kPpR; ++r) cur.put(r, ld_spill(q + r * 32, pol_keep));
    }
  };

  // One step: forward chunk kk of the group read (FW) and backward chunk c of
  // the group written (BW), rows interleaved; both use storage slot s.
  // CN halo: h1/h2 = u at the two rows above the chunk (carried; the wrap
  // rows n-2, n-1 for chunk 0, loaded a group ahead), la0/la1 = the two rows
  // below it (the next chunk's ring slot; rows 0, 1 past the last chunk)
  double h1 = 0.0, h2 = 0.0, la0 = 0.0, la1 = 0.0, nh1 = 0.0, nh2 = 0.0, nla0 = 0.0, nla1 = 0.0;
  auto u_at = [&](long long g, int row) -> double {
    if constexpr (CN) {
      row = row < 0 ? row + n : (row >= n ? row - n : row);
      long long j = g * Wg + warp * 32 + lane;
      j = j < m ? j : m - 1;
      return __ldg(per.u + static_cast<long long>(row) * ld + j);
    } else {
      return 0.0;
    }
  };
  auto halo_prefetch = [&](long long g) {
    if constexpr (CN) {
      nh2 = u_at(g, n - 2);
      nh1 = u_at(g, n - 1);
    }
  };

  auto run_step = [&](int kk, int c, int s, auto fw, auto bw, long long gr) {
    constexpr bool FW = decltype(fw)::value, BW = decltype(bw)::value;
    const double* blk = nullptr;
    double fin[CN ? kPpR : 1];  // CN: the stencil rows of this chunk
    (void)fin;
    (void)gr;
    if constexpr (FW) {
      mbar_wait(&full[slot], phase);
      blk = ring + slot * kChunk + warp * kBox + lane;
      if constexpr (CN) {
        if (kk == 0) {  // the wrap rows n-2, n-1 (loaded a group ahead)
          h2 = nh2;
          h1 = nh1;
        }
        if (kk + 1 < CL) {  // the next chunk's first two rows: the next ring slot (same warp box)
          const int ns = slot + 1 == KB ? 0 : slot + 1;
          mbar_wait(&full[ns], slot + 1 == KB ? phase ^ 1u : phase);
          const double* nbx = ring + ns * kChunk + warp * kBox + lane;
          la0 = nbx[0];
          la1 = nbx[32];
        } else {  // past the last row: rows 0, 1 of this group (kept from chunk 0)
          la0 = nla0;
          la1 = nla1;
        }
        double e[kPpR + 4];
        e[0] = h2;
        e[1] = h1;
#pragma unroll
        for (int r = 0; r < kPpR; ++r) e[r + 2] = blk[r * 32];
        e[kPpR + 2] = la0;
        e[kPpR + 3] = la1;
        if (kk == 0) {
          nla0 = e[2];
          nla1 = e[3];
        }
        const double cs = per.cn[0], cs4 = per.cn[1], cmid = per.cn[2];
#pragma unroll
        for (int r = 0; r < kPpR; ++r) {
          if constexpr (PENT) {  // pde.cpp:108
            const double t = add_rn(mul_rn(-cs, add_rn(e[r], e[r + 4])), mul_rn(cs4, add_rn(e[r + 1], e[r + 3])));
            fin[r] = add_rn(t, mul_rn(cmid, e[r + 2]));
          } else {  // pde.cpp:85
            fin[r] = add_rn(mul_rn(cs, add_rn(e[r + 1], e[r + 3])), mul_rn(cmid, e[r + 2]));
          }
        }
        h2 = e[kPpR];
        h1 = e[kPpR + 1];
      }
    }
    if constexpr (BW) {
      if (s < TT) cur.wait();
    }
    const FwdR* fc = sf + kk * kPpR;
    const BwdR* bc = sb + c * kPpR;
    TPiece<double> buf;
#pragma unroll
    for (int q = 0; q < kPpR; ++q) {
      const int r = kPpR - 1 - q;
      T fv{}, bv{};
      T din{};
      if constexpr (FW) {
        if constexpr (CN) din = fin[q];
        else din = from_word<T>(blk[q * 32]);
      }
      pipe_rows<PENT, FAST, FW, BW, T>(fc[q], din, fs1, fs2, fv, bc[r], BW ? from_word<T>(cur.get(r)) : T{}, bs1, bs2,
                                       bv);
      if constexpr (FW) buf.put(q, to_word(fv));
      if constexpr (BW) {
        if constexpr (PER) {  // x_i = y_i - w z_i (periodic.cpp:85 / :203)
          const int row = c * kPpR + r;
          if constexpr (PENT)
            bv = sub_rn(bv, add_rn(mul_rn(sz[2 * row], wt1), mul_rn(sz[2 * row + 1], wt2)));
          else
            bv = sub_rn(bv, mul_rn(wt1, sz[row]));
        }
        __stcs(out, to_word(bv));
        out -= step;
      }
    }
    if constexpr (FW) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == KB) {
        slot = 0;
        phase ^= 1u;
      }
      if (s < TT) {
        buf.store(tlane + static_cast<uint32_t>(s * TPiece<double>::kWords));
      } else if (s < TR) {
        if constexpr (RT > 0) {
          switch (s - TT) {
#define BSB_RS_STORE(K)                                                     \
  case K:                                                                   \
    if constexpr (K < RT) {                                                 \
      _Pragma("unroll") for (int r = 0; r < kPpR; ++r) rs[K * kPpR + r] = buf.get(r); \
    }                                                                       \
    break;
            BSB_RS_STORE(0) BSB_RS_STORE(1) BSB_RS_STORE(2) BSB_RS_STORE(3)
#undef BSB_RS_STORE
          }
        }
      } else if (s < TR + ST) {
        double* q = slot_smem(s);
#pragma unroll
        for (int r = 0; r < kPpR; ++r) q[r * 32] = buf.get(r);
      } else {
        double* q = slot_l2(s);
#pragma unroll
        for (int r = 0; r < kPpR; ++r) st_spill(q + r * 32, buf.get(r), pol_keep);
      }
    }
  };

  const long long my = (groups - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (my > 0) halo_prefetch(blockIdx.x);
  uint32_t p = 0;  // parity of the group being read
  for (long long i = 0; i <= my; ++i, p ^= 1u) {
    const long long g = blockIdx.x + i * gridDim.x;  // group read in this round (i < my)
    if (i > 0) {  // the group read last round is written this round: x from row n-1 down
      const long long j = (g - gridDim.x) * Wg + warp * 32 + lane;
      const bool live = j < m;
      step = live ? ld : 0;
      out = live ? x + static_cast<long long>(n - 1) * ld + j : sink + lane;
      bs1 = bs2 = T{};
      if constexpr (PER) {  // first backward pass: y_{n-1}, y_{n-2}, y_1, y_0 only
        double e0 = 0.0, e1 = 0.0, yl = 0.0, yl2 = 0.0;
        for (int c = CL - 1; c >= 0; --c) {
          const int s = sidx(p ^ 1u, c);
          bwd_load(s, c, false);
          if (s < TT) cur.wait();
          const BwdR* bc = sb + c * kPpR;
#pragma unroll
          for (int q = 0; q < kPpR; ++q) {
            const int r = kPpR - 1 - q;
            double fv = 0.0, bv = 0.0, d0 = 0.0, d1 = 0.0;
            pipe_rows<PENT, FAST, false, true>(sf[0], 0.0, d0, d1, fv, bc[r], cur.get(r), bs1, bs2, bv);
            if (c == CL - 1 && q == 0) yl = bv;   // y_{n-1}
            if (c == CL - 1 && q == 1) yl2 = bv;  // y_{n-2}
            if (c == 0 && r == 1) e1 = bv;        // y_1
            if (c == 0 && r == 0) e0 = bv;        // y_0
          }
        }
        if constexpr (PENT) {  // periodic.cpp:189-194
          const double w1 = sub_rn(e0, yl), w2 = sub_rn(e1, yl2);
          wt1 = add_rn(mul_rn(per.c[0], w1), mul_rn(per.c[1], w2));
          wt2 = add_rn(mul_rn(per.c[2], w1), mul_rn(per.c[3], w2));
        } else {  // periodic.cpp:80
          wt1 = mul_rn(add_rn(e0, mul_rn(per.c[0], yl)), per.c[1]);
        }
        bs1 = bs2 = T{};
      }
      for (int d = 0; d < DS; ++d) l2_prefetch(p ^ 1u, CL - 1 - d);
      bwd_load(sidx(p ^ 1u, CL - 1), CL - 1, true);
      __syncwarp();  // every lane has read the staging slot before it is refilled
      l2_prefetch(p ^ 1u, CL - 1 - DS);
    }
    fs1 = fs2 = T{};
    for (int kk = 0; kk < CL; ++kk) {
      const int c = CL - 1 - kk;
      const int s = sidx(p, kk);  // == sidx(p ^ 1, c)
      if (i > 0 && i < my) run_step(kk, c, s, std::true_type{}, std::true_type{}, g);
      else if (i < my) run_step(kk, c, s, std::true_type{}, std::false_type{}, g);
      else run_step(kk, c, s, std::false_type{}, std::true_type{}, g);
      if (CN && kk == 0 && i + 1 < my) halo_prefetch(g + gridDim.x);  // this group's halo is consumed
      if (i > 0 && c > 0) {  // next backward chunk (a different slot)
        bwd_load(sidx(p ^ 1u, c - 1), c - 1, true);
        __syncwarp();
        l2_prefetch(p ^ 1u, c - 1 - DS);
      }
    }
    __syncwarp();  // this warp's smem slot stores are visible to its own next-round loads
  }
  if (GT > 0) {  // the scratch is dead: drop this warp's lines instead of writing them back
    for (int s = TR + ST; s < CL; ++s)
      for (int r = lane; r < kPpR * 2; r += 32)  // 16 rows x 256 B = 32 lines of 128 B
        discard_l2_line(reinterpret_cast<const char*>(slot_l2(s) - lane) + r * 128);
  }
  tmem_fence_before();
  asm volatile("bar.sync 1, %0;" ::"r"(P * 32) : "memory");
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc_512(tmem_base_s);
  }
}

}  // namespace dev
}  // namespace bsb
