// CTA-pair tcgen05 MMA rate microbenchmark (debug tool): the GEMM pipeline's
// producer / MMA handshake with real M=256 x N=BN x K=16 MMAs on zeroed
// smem operands (no loads), cycles per 64-deep k-block vs the floor 2*BN.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench tools/mma_bench.cu
//   mode 0: full handshake per k-block (producer arrive -> MMA wait -> commit)
//   mode 1: MMA thread alone (no full waits; commit per k-block)
//   mode 2: MMA thread alone, one commit per 8 k-blocks
#include <cstdint>
#include <cstdio>
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
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(su32(b)), "h"(static_cast<uint16_t>(3))
      : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}

constexpr int S = 6;
template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mb(int nk, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int kA = 128 * 64 * 2, kB = (BN / 2) * 64 * 2, kSt = kA + kB;
  __shared__ uint64_t full[S], empty[S], done;
  __shared__ uint32_t tslot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < S * kSt / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { init(&full[s], 2); init(&empty[s], 1); }
    init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const long long t0 = clock64();
  if (warp == 0 && mode == 0) {
    int s = 0; uint32_t ph = 0;
    for (int kb = 0; kb < nk; ++kb) {
      wait(&empty[s], ph ^ 1);
      if (lane == 0) arrive_cl(mapa(su32(&full[s]), 0));
      __syncwarp();
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    constexpr uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(256 >> 4) << 24);
    const uint32_t base = su32(sm);
    int s = 0; uint32_t ph = 0;
    for (int kb = 0; kb < nk; ++kb) {
      if (mode == 0) wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t da = sdesc(base + s * kSt, 16, 1024), db = sdesc(base + s * kSt + kA, 16, 1024);
#pragma unroll
      for (int k = 0; k < 4; ++k) mma(tmem, da + 2 * k, db + 2 * k, id, (kb | k) != 0);
      if (mode != 2 || (kb % 8) == 7) commit(&empty[s]);
      if (++s == S) { s = 0; ph ^= 1; }
    }
    commit(&done);
    wait(&done, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
}

template <int BN>
void run(long long* d, int mode) {
  constexpr int smem = S * (128 * 64 * 2 + (BN / 2) * 64 * 2) + 1024;
  cudaFuncSetAttribute(mb<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int nk = 2400;
  mb<BN><<<148, 128, smem>>>(nk, mode, d);
  mb<BN><<<148, 128, smem>>>(nk, mode, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double c = double(h[0]) / nk;
  printf("BN %3d mode %d: %s  %.1f cycles per k-block (floor %d, %.0f%%)\n", BN, mode,
         cudaGetErrorString(e), c, 2 * BN, 100.0 * 2 * BN / c);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  for (int mode = 0; mode < 3; ++mode) {
    run<128>(d, mode);
    run<192>(d, mode);
    run<256>(d, mode);
  }
  return 0;
}
