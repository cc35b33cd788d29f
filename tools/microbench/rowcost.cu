// Microbenchmark: cycles per row-step of the smem-resident sweep loops
// (fwd_block / bwd_block of sweep_persist.cuh) for one warp per SMSP, by
// arithmetic variant. Tells how far the compiled row loop is from the pure
// dependency-chain bound (8-cycle DP latency x chain length).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1909_04539_b200/csrc -o rowcost rowcost.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "sweep_persist.cuh"

using namespace bsb::dev;

template <bool PENT, bool FAST>
__global__ void rowcost(double* out, long long* cyc, int reps) {
  using FwdR = typename Recs<double, PENT>::Fwd;
  using BwdR = typename Recs<double, PENT>::Bwd;
  __shared__ FwdR sf[64];
  __shared__ BwdR sb[64];
  __shared__ double tile[4][40 * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < 64; k += blockDim.x) {
    if constexpr (PENT) {
      sf[k] = FwdR{0.01, 0.02, 0.9, 0.0};
      sb[k] = BwdR{0.01, 0.02};
    } else {
      sf[k] = FwdR{0.01, 0.9};
      sb[k] = 0.01;
    }
  }
  for (int k = threadIdx.x; k < 40 * 32; k += 32) tile[warp][k] = 0.5;
  __syncthreads();
  double* p = &tile[warp][lane];
  double s1 = 0, s2 = 0, acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    fwd_block<double, PENT, FAST, 32>(p, sf, s1, s2, [&](int i, double v) { p[i * kPW] = v; });
    bwd_block<double, PENT, FAST, 32>(p + 8 * kPW, sb, s1, s2, [&](int, double v) { acc += v; });
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc + s1 + s2;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <bool PENT, bool FAST>
void run(double* d, long long* c, const char* name) {
  const int reps = 2000;
  for (int warps : {1, 4}) {
    rowcost<PENT, FAST><<<1, 32 * warps>>>(d, c, reps);
    cudaDeviceSynchronize();
    long long cyc = 0;
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("%-12s warps=%d : %.1f cycles per row-step (fwd+bwd avg)\n", name, warps, cyc / (64.0 * reps));
  }
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&c, 8);
  run<false, false>(d, c, "tri exact");
  run<false, true>(d, c, "tri fast");
  run<true, false>(d, c, "pent exact");
  run<true, true>(d, c, "pent fast");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
