// Host side of the pipelined on-chip sequential sweep (sweep_pipe.cuh):
// plan (compute warps, ring depth) and launch.
#include <cuda_runtime.h>

#include <atomic>
#include <climits>
#include <cstdint>

#include "internal.hpp"
#include "sweep_pipe.cuh"

namespace bsb {

bool encode_tile_map(CUtensorMap* map, void* x, std::size_t elem, long long n, long long m, long long ld,
                     int box_w, int box_r);   // solve.cu
cudaError_t allow_max_smem(const void* kern);  // solve.cu
std::size_t max_smem_per_block();              // solve.cu
double* dead_lane_sink(int device);            // partition.cu
bandsolve_status cuda_fail(cudaError_t err, const char* what);  // solve.cu

namespace {

std::size_t fwd_rec(bool pent) { return pent ? sizeof(dev::PentFwd<double>) : sizeof(dev::TriFwd<double>); }
std::size_t bwd_rec(bool pent) { return pent ? sizeof(dev::PentBwd<double>) : sizeof(double); }

}  // namespace

// Compute warps (2..4) of the pipelined plan for this shape, 0 when it does
// not apply; *kb receives the ring depth, *rt the register chunks per lane
// (0 or 4, with 3 warps), *st the shared-memory chunks per lane (the rest
// beyond TMEM + registers + smem goes to the L2 scratch).
int pipe_warps(std::size_t n, std::size_t m, std::size_t ld, const void* x, bool pent, int sms, int* kb, int* rt,
               int* st, bool per) {
  const long long sel = tune_int("PIPE", -1);  // 0: never, 1: whenever it applies
  if (sel == 0 || tune_flag("PLAN")) return 0;
  // beyond 512 rows the last chunks live in the L2 tier (cp.async-staged a
  // few chunks ahead): measured 0.50-0.88 of the roofline at N = 4096..640
  // where the streaming kernel's spill / the two-pass sweep reached 0.43-0.68;
  // the limit in practice is the factor records in shared memory
  const std::size_t max_rows = static_cast<std::size_t>(tune_int("PIPE_MAX_N", 4096));
  if (n % dev::kPpR != 0 || n < 2 * dev::kPpR || n > max_rows) return 0;
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0 || ld % 2 != 0 || m % 2 != 0 ||
      m > static_cast<std::size_t>(INT_MAX) / 2)
    return 0;
  const std::size_t cap = max_smem_per_block();
  const int CL = static_cast<int>(n) / dev::kPpR;
  const int TT = std::min(CL, dev::kPpTmemRows / dev::kPpR);
  const int kmin = static_cast<int>(tune_int("PKB", 4));  // ring slots (tuning)
  const int rt_force = static_cast<int>(tune_int("PRT", -1));
  const int zw = per ? (pent ? 2 : 1) : 0;
  auto fits = [&](int P, int k, int ST, int RT) {
    return dev::PipeLayout::make(static_cast<int>(n), P, k, fwd_rec(pent), bwd_rec(pent), ST, zw,
                                 dev::pipe_stage_chunks(static_cast<int>(n), RT, ST))
               .total <= cap;
  };
  auto take = [&](int P, int RT, int ST) {
    int k = kmin;
    while (k < 10 && fits(P, k + 1, ST, RT)) ++k;
    *kb = k;
    *rt = RT;
    *st = ST;
    return P;
  };
  // 1) every row on chip: the most warps (chains) that fit, registers as a
  // fourth tier for 3 warps
  for (int P = 4; P >= 2; --P) {
    if (sel != 1 && m < static_cast<std::size_t>(sms) * 32 * P) continue;  // a full wave of groups
    for (int RT : {0, 4}) {
      if (RT > 0 && P != 3) continue;  // the only register-tier instance
      if (rt_force >= 0 && RT != rt_force) continue;
      const int ST = CL - TT - RT;
      if (ST < 0) continue;
      if (fits(P, kmin, ST, RT)) return take(P, RT, ST);
    }
  }
  // 2) the L2 tier: up to 1024 rows 3 warps with the register tier (pent
  // N = 1024: 0.63 vs 0.59 without it, 0.57 with 2 warps), beyond that 2
  // warps (less L2 scratch in flight: N = 2048 0.55 vs 0.50); PIPE_L2_P, PRT
  const int PL = static_cast<int>(
      std::min<long long>(4, std::max<long long>(2, tune_int("PIPE_L2_P", n <= 1024 ? 3 : 2))));
  const int RL = PL == 3 && rt_force != 0 ? 4 : 0;
  if (sel != 1 && m < static_cast<std::size_t>(sms) * 32 * PL) return 0;
  for (int ST = CL - TT - RL; ST >= 0; --ST)
    if (fits(PL, kmin, ST, RL)) return take(PL, RL, ST);
  return 0;
}

bandsolve_status pipe_solve_device(bool pent, bool fast, const void* fwd, const void* bwd, double* x, std::size_t n,
                                   std::size_t m, std::size_t ld, void* stream, int sms, bool* done,
                                   const PartPeriodic* per, const SpikeCN* cn, bool f32) {
  *done = false;
  if (cn && (!per || reinterpret_cast<uintptr_t>(cn->u) % 16 != 0)) return BANDSOLVE_OK;
  if (f32) {  // pairs of adjacent fp32 systems per lane (8-byte words), plain solves
    if (per || cn || m % 4 != 0 || ld % 4 != 0) return BANDSOLVE_OK;
    m /= 2;
    ld /= 2;
  }
  int KB = 0, RT = 0, ST = 0;
  const int P = pipe_warps(n, m, ld, x, pent, sms, &KB, &RT, &ST, per != nullptr);
  if (P == 0) return BANDSOLVE_OK;
  int device = 0;
  if (cudaGetDevice(&device) != cudaSuccess) {
    cudaGetLastError();
    return BANDSOLVE_OK;
  }
  double* sink = dead_lane_sink(device);
  if (!sink) return fail(BANDSOLVE_ERR_INTERNAL, "pipe scratch");
  CUtensorMap map;
  // the tensor map reads b (in place: x; Crank-Nicolson: the old field u)
  if (!encode_tile_map(&map, cn ? const_cast<double*>(cn->u) : x, sizeof(double), static_cast<long long>(n),
                       static_cast<long long>(m), static_cast<long long>(ld), 32, dev::kPpR))
    return BANDSOLVE_OK;
  using Kern = decltype(&dev::sweep_pipe<true, false, 2, 0, false, false>);
#define BSB_PIPE_SET(PP, RR, PR, CC)                                                                        \
  {{dev::sweep_pipe<false, false, PP, RR, PR, CC>, dev::sweep_pipe<false, true, PP, RR, PR, CC>},          \
   {dev::sweep_pipe<true, false, PP, RR, PR, CC>, dev::sweep_pipe<true, true, PP, RR, PR, CC>}}
#define BSB_PIPE_WARPS(PR, CC) \
  {BSB_PIPE_SET(2, 0, PR, CC), BSB_PIPE_SET(3, 0, PR, CC), BSB_PIPE_SET(4, 0, PR, CC), BSB_PIPE_SET(3, 4, PR, CC)}
  // [plain, periodic, CN step][2 warps, 3 warps, 4 warps, 3 warps + register tier][pent][fast]
  static const Kern kerns[3][4][2][2] = {BSB_PIPE_WARPS(false, false), BSB_PIPE_WARPS(true, false),
                                         BSB_PIPE_WARPS(true, true)};
#undef BSB_PIPE_WARPS
#undef BSB_PIPE_SET
  // fp32 pairs: [2 warps, 3 warps, 4 warps, 3 warps + register tier][pent][fast]
#define BSB_PIPE_F2(PP, RR)                                                                                 \
  {{dev::sweep_pipe<false, false, PP, RR, false, false, float2>,                                           \
    dev::sweep_pipe<false, true, PP, RR, false, false, float2>},                                           \
   {dev::sweep_pipe<true, false, PP, RR, false, false, float2>, dev::sweep_pipe<true, true, PP, RR, false, false, float2>}}
  static const Kern kf2[4][2][2] = {BSB_PIPE_F2(2, 0), BSB_PIPE_F2(3, 0), BSB_PIPE_F2(4, 0), BSB_PIPE_F2(3, 4)};
#undef BSB_PIPE_F2
  const int ki = RT > 0 ? 3 : P - 2;
  const int vi = f32 ? 3 : cn ? 2 : per ? 1 : 0;
  const Kern kern = f32 ? kf2[ki][pent][fast] : kerns[vi][ki][pent][fast];
  static std::atomic<uint64_t> configured[64];
  std::atomic<uint64_t>& done_attr = configured[vi * 16 + ki * 4 + (pent ? 2 : 0) + (fast ? 1 : 0)];
  const uint64_t bit = device < 64 ? (1ull << device) : 0;
  if (!(bit && (done_attr.load(std::memory_order_relaxed) & bit))) {
    if (cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern)); e != cudaSuccess)
      return fail(BANDSOLVE_ERR_INTERNAL, std::string("pipe attributes: ") + cudaGetErrorString(e));
    if (bit) done_attr.fetch_or(bit, std::memory_order_relaxed);
  }
  const int Wg = 32 * P;
  const long long groups = (static_cast<long long>(m) + Wg - 1) / Wg;
  const std::size_t smem =
      dev::PipeLayout::make(static_cast<int>(n), P, KB, fwd_rec(pent), bwd_rec(pent), ST, per ? (pent ? 2 : 1) : 0,
                            dev::pipe_stage_chunks(static_cast<int>(n), RT, ST))
          .total;
  dev::PipePer pp;
  if (per) {
    pp.z1 = per->z1;
    pp.z2 = per->z2;
    for (int q = 0; q < 4; ++q) pp.c[q] = per->c[q];
  }
  if (cn) {
    pp.u = cn->u;
    for (int q = 0; q < 3; ++q) pp.cn[q] = cn->c[q];
  }
  const int CL = static_cast<int>(n) / dev::kPpR;
  const int GT = CL - std::min(CL, dev::kPpTmemRows / dev::kPpR) - RT - ST;
  const long long grid = std::min<long long>(sms, groups);
  auto s = static_cast<cudaStream_t>(stream);
  double* scratch = nullptr;  // the L2 tier: per CTA, GT chunks x P warps x 4 KiB
  if (GT > 0) {
    const std::size_t bytes = static_cast<std::size_t>(grid) * GT * P * dev::kPpR * 32 * sizeof(double);
    if (cudaError_t e = pool_malloc_async(reinterpret_cast<void**>(&scratch), bytes, s); e != cudaSuccess)
      return cuda_fail(e, "pipe scratch");
  }
  const int PD = static_cast<int>(tune_int("SPD", 4));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid), 1, 1);
  cfg.blockDim = dim3(32 * (P + 1), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = tune_flag("NO_PDL") ? 0 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, map, x, static_cast<int>(n), static_cast<long long>(m),
                                     static_cast<long long>(ld), KB, PD, groups, fwd, bwd, sink, ST, scratch, pp);
  note_launches(1);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (scratch) cudaFreeAsync(scratch, s);
  if (e != cudaSuccess) return fail(BANDSOLVE_ERR_INTERNAL, std::string("pipe launch: ") + cudaGetErrorString(e));
  *done = true;
  return BANDSOLVE_OK;
}

}  // namespace bsb
