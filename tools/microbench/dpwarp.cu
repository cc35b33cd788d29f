// Microbenchmark: fp64 dependent-op latency for FULL warps (1..16 warps in one
// CTA on one SM) and per-SM fp64 issue throughput. The single-thread latency
// (dplat.cu) understates what a 32-lane warp sees if the DP pipe is narrower
// than a warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dpwarp dpwarp.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP, int ILP>
__global__ void chain(double* out, long long* cyc, double a, double b, int iters) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = out[threadIdx.x] + k;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < ILP; ++k) {
        if (OP == 0) x[k] = __dadd_rn(x[k], a);
        if (OP == 1) x[k] = __dmul_rn(x[k], a);
        if (OP == 2) x[k] = __fma_rn(x[k], a, b);
      }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int OP, int ILP>
void run(double* d, long long* c, const char* name) {
  const int iters = 4096;
  for (int warps : {1, 2, 4, 8, 16}) {
    chain<OP, ILP><<<1, 32 * warps>>>(d, c, 1.0000001, 0.5, iters);
    cudaDeviceSynchronize();
    long long cyc = 0;
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    const double ops = 8.0 * iters;  // dependent ops per chain
    printf("%s ilp=%d warps=%2d : %.2f cycles per dependent op, %.2f warp-instr/cycle/SM\n", name, ILP, warps,
           cyc / ops, warps * ILP * ops / cyc);
  }
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&c, 8);
  cudaMemset(d, 0, 1 << 20);
  run<0, 1>(d, c, "dadd");
  run<1, 1>(d, c, "dmul");
  run<2, 1>(d, c, "dfma");
  run<2, 2>(d, c, "dfma");
  run<2, 4>(d, c, "dfma");
  return 0;
}
