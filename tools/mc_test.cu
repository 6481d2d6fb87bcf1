// Multicast + cta_group::2 TMA completion semantics probe (debug tool).
// 4-CTA cluster = two CTA pairs.  CTA r loads 64 rows x 64 bf16 (8 KB) into
// smem offset (r >> 1) * 8 KB of CTAs r and r ^ 2; pair leaders (0, 2) expect
// 32 KB on their `full` barrier.  mode 0: barrier operand = the pair leader's
// barrier (mapa rank & ~1); mode 1: the CTA's own barrier address.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mc_test tools/mc_test.cu -lcuda
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__global__ void __cluster_dims__(4, 1, 1) probe(const __grid_constant__ CUtensorMap m, int mode,
                                                int* out) {
  __shared__ __align__(1024) uint16_t buf[128 * 64];
  __shared__ uint64_t full;
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) buf[i] = 0xFFFF;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
    if ((r & 1) == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full)), "r"(32768));
    uint32_t bar = su32(&full);
    if (mode == 0) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(bar), "r"(r & ~1u));
    const uint16_t mask = static_cast<uint16_t>((1u << r) | (1u << (r ^ 2u)));
    const int row = static_cast<int>(r & 1) * 128 + static_cast<int>(r >> 1) * 64;
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        ".multicast::cluster.cta_group::2 [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(su32(buf) + (r >> 1) * 8192),
        "l"(&m), "r"(bar), "r"(0), "r"(row), "h"(mask)
        : "memory");
  }
  // the non-leaders' halves land in their own smem but are signalled on the
  // leader; the leader waits (bounded) and reports
  int done = 0;
  if ((r & 1) == 0 && threadIdx.x == 0) {
    for (long it = 0; it < 20000000 && !done; ++it) {
      uint32_t d;
      asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\nselp.u32 %0, 1, 0, P;\n}\n"
                   : "=r"(d) : "r"(su32(&full)) : "memory");
      done = d;
    }
    out[blockIdx.x * 4 + 0] = done;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  // wait a little for stragglers, then check the data: row i of this CTA's
  // 128-row block should hold global row (r & 1) * 128 + i (value = row)
  for (volatile int spin = 0; spin < 100000; ++spin) {}
  if (threadIdx.x == 0) {
    int bad = 0;
    for (int i = 0; i < 128; ++i) {
      // 128B swizzle: element 0 of row i sits in 16-byte chunk (0 ^ (i & 7))
      const uint16_t v = buf[i * 64 + ((i & 7) * 8)];
      if (v != static_cast<uint16_t>((r & 1) * 128 + i)) ++bad;
    }
    out[blockIdx.x * 4 + 1] = bad;
  }
}

int main() {
  const int rows = 256, cols = 64;
  uint16_t h[rows * cols];
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) h[i * cols + j] = static_cast<uint16_t>(i);
  void* d;
  cudaMalloc(&d, sizeof(h));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
  CUresult cr = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", cr); return 1; }
  int* out;
  cudaMalloc(&out, 16 * sizeof(int));
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(out, 0xff, 16 * sizeof(int));
    probe<<<4, 128>>>(m, mode, out);
    cudaError_t e = cudaDeviceSynchronize();
    int ho[16];
    cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %s\n", mode, mode == 0 ? "leader barrier" : "own barrier", cudaGetErrorString(e));
    for (int b = 0; b < 4; ++b) printf("  CTA %d: leader-done %d  bad rows %d\n", b, ho[b * 4], ho[b * 4 + 1]);
  }
  return 0;
}
