// Microbenchmark: fp64 dependent-op latency and device facts on the box.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dplat dplat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void lat_kernel(double* out, long long* cyc, double a, double b, int iters) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) x = __dadd_rn(x, a);
      if (OP == 1) x = __dmul_rn(x, a);
      if (OP == 2) x = __fma_rn(x, a, b);
      if (OP == 3) x = __fmul_rn((float)x, (float)a);
      if (OP == 4) x = __dmul_rn(__dsub_rn(b, __dmul_rn(a, x)), a);  // tri fwd chain (3 ops)
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

// throughput: many independent chains per thread, full SM occupancy
__global__ void tput_kernel(double* out, double a, double b, int iters) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b); x3 = __fma_rn(x3, a, b);
    x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b); x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk = 0, memclk = 0, busw = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0);
  cudaDeviceGetAttribute(&busw, cudaDevAttrGlobalMemoryBusWidth, 0);
  printf("name=%s cc=%d.%d sms=%d l2=%d B smem/sm=%zu smem/block_optin=%zu regs/sm=%d maxthr/sm=%d clk_khz=%d memclk_khz=%d busw=%d gmem=%zu persistL2max=%d\n",
         p.name, p.major, p.minor, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerMultiprocessor,
         p.sharedMemPerBlockOptin, p.regsPerMultiprocessor, p.maxThreadsPerMultiProcessor, clk, memclk, busw,
         p.totalGlobalMem, p.persistingL2CacheMaxSize);
  double* d; long long* c; cudaMalloc(&d, 1 << 24); cudaMalloc(&c, 8);
  cudaMemset(d, 0, 1 << 24);
  const char* names[] = {"dadd", "dmul", "dfma", "fmul", "tri_fwd_chain(3op)"};
  for (int op = 0; op < 5; ++op) {
    long long cyc = 0;
    int iters = 1000;
    for (int rep = 0; rep < 2; ++rep) {
      if (op == 0) lat_kernel<0><<<1, 1>>>(d, c, 1e-9, 0.5, iters);
      if (op == 1) lat_kernel<1><<<1, 1>>>(d, c, 1.0000001, 0.5, iters);
      if (op == 2) lat_kernel<2><<<1, 1>>>(d, c, 0.999, 0.5, iters);
      if (op == 3) lat_kernel<3><<<1, 1>>>(d, c, 1.0000001, 0.5, iters);
      if (op == 4) lat_kernel<4><<<1, 1>>>(d, c, 0.3, 0.5, iters);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("lat %-20s %.2f cycles/op-chain-step\n", names[op], (double)cyc / (iters * 16));
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 20000;
  tput_kernel<<<blocks, threads>>>(d, 0.999, 0.5, 100);
  cudaEventRecord(e0);
  tput_kernel<<<blocks, threads>>>(d, 0.999, 0.5, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 8 * (double)iters * blocks * threads;
  printf("dfma throughput %.2f TFLOP/s\n", flops / ms / 1e9);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
