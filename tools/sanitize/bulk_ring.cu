// Minimal full/empty mbarrier ring, the protocol of sweep_stream.cuh's reload
// ring: one producer lane fills KR slots with a 1D bulk copy
// (cp.async.bulk ... mbarrier::complete_tx) or, with -DTENSOR, a 2D TMA
// tensor load; P consumer warps wait on full[s], read the slot, __syncwarp,
// and lane 0 arrives on empty[s]. Checks the data; used to tell a racecheck
// report on this protocol from a real race (tools/gpu_sanitize.sh).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

constexpr int KR = 2, P = 4, CH = 16 * 32;  // slot = P warp blocks of 16 x 32 doubles
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}

__global__ void ring(const __grid_constant__ CUtensorMap map, const double* src, int chunks, double* out) {
  __shared__ alignas(128) double slot[KR][P * CH];
  __shared__ alignas(8) uint64_t full[KR], empty[KR];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < KR; ++s) { init(&full[s], 1); init(&empty[s], P); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == P) {
    if (lane == 0)
      for (int c = 0; c < chunks; ++c) {
        const int s = c % KR;
        if (c >= KR) wait(&empty[s], ((c / KR) - 1) & 1);
        expect(&full[s], P * CH * 8);
#ifdef TENSOR
        for (int w = 0; w < P; ++w)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       :: "r"(su32(&slot[s][w * CH])), "l"(&map), "r"(0), "r"((c * P + w) * 16), "r"(su32(&full[s])) : "memory");
#else
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(su32(&slot[s][0])), "l"(src + static_cast<long long>(c) * P * CH), "r"(P * CH * 8), "r"(su32(&full[s])) : "memory");
#endif
      }
    return;
  }
  double acc = 0.0;
  for (int c = 0; c < chunks; ++c) {
    const int s = c % KR;
    wait(&full[s], (c / KR) & 1);
    for (int r = 0; r < 16; ++r) acc += slot[s][warp * CH + r * 32 + lane];
    __syncwarp();
    if (lane == 0) arrive(&empty[s]);
  }
  out[warp * 32 + lane] = acc;
}

int main() {
  const int chunks = 64;
  const size_t n = static_cast<size_t>(chunks) * P * CH;
  double *src, *out;
  cudaMalloc(&src, n * 8);
  cudaMalloc(&out, P * 32 * 8);
  double* h = new double[n];
  for (size_t i = 0; i < n; ++i) h[i] = static_cast<double>(i % 1000);
  cudaMemcpy(src, h, n * 8, cudaMemcpyHostToDevice);
  CUtensorMap map{};
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  const cuuint64_t gdim[2] = {32, static_cast<cuuint64_t>(n / 32)}, gstr[1] = {32 * 8};
  const cuuint32_t box[2] = {32, 16}, es[2] = {1, 1};
  reinterpret_cast<Enc>(fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, src, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  ring<<<1, (P + 1) * 32>>>(map, src, chunks, out);
  double o[P * 32];
  cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int w = 0; w < P; ++w)
    for (int l = 0; l < 32; ++l) {
      double want = 0.0;
      for (int c = 0; c < chunks; ++c)
        for (int r = 0; r < 16; ++r) want += h[static_cast<size_t>(c) * P * CH + w * CH + r * 32 + l];
      if (o[w * 32 + l] != want) ++bad;
    }
  printf("%s ring: %s (%s)\n",
#ifdef TENSOR
         "tensor",
#else
         "bulk",
#endif
         bad ? "WRONG" : "data ok", cudaGetErrorString(cudaGetLastError()));
  return bad != 0;
}
