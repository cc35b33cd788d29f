// Minimal interface exchange of the cluster spike kernel (sweep_spike.cuh,
// CS > 1): each CTA of a 2-CTA cluster writes its values into a
// double-buffered shared-memory slot, every warp arrives (release.cluster) on
// a per-parity mbarrier in every CTA of the cluster, waits on its own
// (acquire.cluster), then reads the other CTA's slot with ld.shared::cluster.
// With -DHWBAR the same exchange uses barrier.cluster instead. Checks the
// data; used to tell a racecheck report on this protocol from a real race.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

constexpr int kW = 4, kIters = 64;
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __cluster_dims__(2, 1, 1) xch(int* bad) {
  __shared__ double slot[2][kW * 32];
  __shared__ alignas(8) uint64_t bar[2];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int p = 0; p < 2; ++p) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[p])), "r"(2 * kW));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t phase = 0;
  (void)phase;
  for (int it = 0; it < kIters; ++it) {
    const int p = it & 1;
    slot[p][warp * 32 + lane] = rank * 1000.0 + it * 10.0 + warp + lane * 0.001;
#ifdef HWBAR
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
#else
    asm volatile("fence.acq_rel.cluster;" ::: "memory");
    __syncwarp();
    if (lane < 2) {
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su32(&bar[p])), "r"(lane));
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                   : "=r"(ok) : "r"(su32(&bar[p])), "r"((phase >> p) & 1u) : "memory");
    phase ^= 1u << p;
#endif
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(su32(&slot[p][warp * 32 + lane])), "r"(rank ^ 1u));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    if (v != (rank ^ 1u) * 1000.0 + it * 10.0 + warp + lane * 0.001) atomicAdd(bad, 1);
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
  int* bad;
  cudaMalloc(&bad, sizeof(int));
  cudaMemset(bad, 0, sizeof(int));
  xch<<<2, 32 * kW>>>(bad);
  int h = -1;
  cudaMemcpy(&h, bad, sizeof h, cudaMemcpyDeviceToHost);
  printf("%s cluster exchange: %s (%s)\n",
#ifdef HWBAR
         "barrier.cluster",
#else
         "mbarrier",
#endif
         h ? "WRONG" : "data ok", cudaGetErrorString(cudaGetLastError()));
  return h != 0;
}
