// Memory-pattern microbenchmark for the interleaved sweep (no arithmetic):
// how fast can the chip stream an n x m interleaved fp64 batch when each
// CTA owns a W-column strip for all n rows?
//   tma   : TMA 2D boxes {W, 32} for the whole strip into smem, then STG back
//   ldg   : thread per column, rows streamed with LDG (unroll 8) then STG
//   rowcp : fully coalesced row-major copy (reference point)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pattern pattern.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int W>
__global__ void __launch_bounds__(W) tma_strip(const __grid_constant__ CUtensorMap map, double* x, int n, long m) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int R = 32, chunks = (n + R - 1) / R;
  double* tile = (double*)sm;
  uint64_t* bars = (uint64_t*)(sm + (size_t)chunks * R * W * 8);
  const int t = threadIdx.x;
  const long j0 = (long)blockIdx.x * W;
  if (t == 0) {
    for (int c = 0; c < chunks; ++c) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[c])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  if (t == 0) {
    for (int c = 0; c < chunks; ++c) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[c])), "r"(W * R * 8));
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(tile + (size_t)c * R * W)), "l"((uint64_t)&map), "r"((int)j0), "r"(c * R), "r"(su32(&bars[c])) : "memory");
    }
  }
  double acc = 0;
  for (int c = 0; c < chunks; ++c) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                   : "=r"(ok) : "r"(su32(&bars[c])) : "memory");
    for (int r = 0; r < R && c * R + r < n; ++r) acc += tile[(c * R + r) * W + t];
  }
  for (int i = n - 1; i >= 0; --i) __stcs(x + (long)i * m + j0 + t, tile[i * W + t] + acc * 0.0);
}

__global__ void ldg_strip(double* x, int n, long m) {
  const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double* c = x + j;
  for (int i = 0; i < n; i += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = c[(long)(i + u) * m];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[(long)(i + u) * m] = v[u] * 1.0000001;
  }
}

__global__ void rowcp(const double4* a, double4* b, long count) {
  for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < count; k += (long)gridDim.x * blockDim.x) b[k] = a[k];
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 512;
  const long m = argc > 2 ? atol(argv[2]) : (1l << 20);
  const size_t bytes = (size_t)n * m * 8;
  double *x, *y;
  cudaMalloc(&x, bytes);
  cudaMalloc(&y, bytes);
  cudaMemset(x, 0, bytes);
  cudaMemset(y, 0, bytes);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch, const char* name, double traffic) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s n=%d m=%ld  %.3f ms  %.0f GB/s  err=%s\n", name, n, m, ms / reps, traffic / (ms / reps * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  auto run_tma = [&](auto kern, int W, int promo) {
    CUtensorMap map;
    cuuint64_t gd[2] = {(cuuint64_t)m, (cuuint64_t)n};
    cuuint64_t gs[1] = {(cuuint64_t)m * 8};
    cuuint32_t box[2] = {(cuuint32_t)W, 32};
    cuuint32_t es[2] = {1, 1};
    encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int chunks = (n + 31) / 32;
    size_t smem = (size_t)chunks * 32 * W * 8 + chunks * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, W, smem);
    char name[64];
    snprintf(name, sizeof name, "tma W=%d promo=%d occ=%d", W, promo, occ);
    if (smem > 232448) { printf("%s: tile too big\n", name); return; }
    timeit([&] { kern<<<(unsigned)((m + W - 1) / W), W, smem>>>(map, x, n, m); }, name, 2.0 * bytes);
  };
  for (int promo = 0; promo <= 3; ++promo) {
    run_tma(tma_strip<8>, 8, promo);
    run_tma(tma_strip<16>, 16, promo);
    run_tma(tma_strip<32>, 32, promo);
  }
  timeit([&] { ldg_strip<<<(unsigned)((m + 127) / 128), 128>>>(x, n, m); }, "ldg strip 128thr", 2.0 * bytes);
  timeit([&] { rowcp<<<148 * 8, 512>>>((const double4*)x, (double4*)y, (long)(bytes / 32)); }, "row-major copy", 2.0 * bytes);
  return 0;
}
