// Handshake microbenchmark (debug tool): the producer -> MMA -> producer
// mbarrier round trip of the CTA-pair GEMM pipeline, with no loads and no
// MMAs, so the cost per k-block of the synchronisation alone is visible.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hs tools/hs_bench.cu -lcuda
//   mode 0: MMA thread releases stages with tcgen05.commit (multicast to both CTAs)
//   mode 1: plain remote mbarrier arrives instead of tcgen05.commit
//   mode 2: like 0, the producer's lane 0 alone (no __syncwarp)
//   mode 3: like 0, only the leader's producer arrives (local), count 1
//   mode 4: everything CTA-local (leader only; plain local arrives)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0, 1, 0, "
        "P;\n}\n"
        : "=r"(done)
        : "r"(su32(b)), "r"(ph)
        : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void arrive_cl(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}

template <int S>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    hs(int nk, int mode, long long* out) {
  __shared__ uint64_t full[S], empty[S];
  __shared__ uint32_t tslot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { init(&full[s], mode >= 3 ? 1 : 2); init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tslot)));
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const long long t0 = clock64();
  if (warp == 0) {
    int s = 0; uint32_t ph = 0;
    for (int kb = 0; kb < nk; ++kb) {
      if (mode == 2 && lane != 0) break;
      if (mode >= 3 && rank != 0) break;
      wait(&empty[s], ph ^ 1);
      if (lane == 0) {
        if (mode >= 3)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
        else
          arrive_cl(mapa(su32(&full[s]), 0));
      }
      if (mode != 2) __syncwarp();
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    int s = 0; uint32_t ph = 0;
    for (int kb = 0; kb < nk; ++kb) {
      wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (mode == 4) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
      } else if (mode == 1) {
        arrive_cl(mapa(su32(&empty[s]), 0));
        arrive_cl(mapa(su32(&empty[s]), 1));
      } else {
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
            " [%0], %1;" ::"r"(su32(&empty[s])), "h"(static_cast<uint16_t>(3))
            : "memory");
      }
      if (++s == S) { s = 0; ph ^= 1; }
    }
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tslot));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int nk = 24 * 100;
  for (int mode = 0; mode < 5; ++mode) {
    for (int grid : {1, 7}) {
      cudaMemset(d, 0, 148 * sizeof(long long));
      auto k = grid == 1 ? hs<1> : grid == 2 ? hs<2> : grid == 7 ? hs<7> : hs<14>;
      k<<<148, 128>>>(nk, mode, d);
      k<<<148, 128>>>(nk, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("mode %d stages %3d: %s  %.1f cycles per k-block\n", mode, grid, cudaGetErrorString(e),
             double(h[0]) / nk);
    }
  }
  return 0;
}
