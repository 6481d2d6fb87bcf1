// tma_bw.cu -- per-SM TMA load throughput into an mbarrier ring (no MMA), the
// operand path of the tcgen05 GEMMs: one CTA per SM, a producer warp issues
// 2D tensor-map boxes of 64 bf16 columns (128 B rows, 128B swizzle) x R rows
// into an S-stage ring, a consumer warp waits on each stage and frees it.
// Footprint small (L2-resident) or large (HBM).  Prints GB/s and B/clk/SM.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/tma_bw.cu -lcuda -o /tmp/tma_bw
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}\n" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mb_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes));
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)));
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

struct Args {
  CUtensorMap map;
  int rows_box;   // R rows per box
  int boxes;      // boxes per stage
  int stages;
  int iters;      // stages per CTA
  int rows_total;
};

__global__ void __launch_bounds__(64, 1) bench(const __grid_constant__ Args a) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024 - (su32(raw) & 1023)) & 1023);
  const int stage_bytes = a.rows_box * 128 * a.boxes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + a.stages * stage_bytes);
  uint64_t* empty = full + a.stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x / 32;
  if (warp == 0 && threadIdx.x == 0) {
    int s = 0; uint32_t ph = 0;
    int row = (blockIdx.x * 977) % a.rows_total;
    for (int i = 0; i < a.iters; ++i) {
      mb_wait(&empty[s], ph ^ 1);
      mb_arrive_tx(&full[s], stage_bytes);
      for (int b = 0; b < a.boxes; ++b) {
        tma2d(sm + s * stage_bytes + b * a.rows_box * 128, &a.map, &full[s], 64 * (b & 1), row);
        row += a.rows_box;
        if (row + a.rows_box > a.rows_total) row = 0;
      }
      if (++s == a.stages) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1 && threadIdx.x == 32) {
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < a.iters; ++i) {
      mb_wait(&full[s], ph);
      mb_arrive(&empty[s]);
      if (++s == a.stages) { s = 0; ph ^= 1; }
    }
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                           const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                           const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (size_t mb : {16, 2048}) {
    const int cols = 128;  // bf16 row of 256 B; boxes take 64-column halves
    const size_t rows_total = (mb << 20) / (cols * 2);
    void* buf; cudaMalloc(&buf, mb << 20); cudaMemset(buf, 1, mb << 20);
    for (int R : {64, 128, 256}) {
      for (int boxes : {1, 2, 3}) {
        for (int stages : {4, 8}) {
          const int stage_bytes = R * 128 * boxes;
          if (stage_bytes * stages > 200 * 1024) continue;
          Args a{};
          cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), rows_total};
          cuuint64_t str[1] = {static_cast<cuuint64_t>(cols) * 2};
          cuuint32_t box[2] = {64, static_cast<cuuint32_t>(R)}, es[2] = {1, 1};
          enc(&a.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          a.rows_box = R; a.boxes = boxes; a.stages = stages;
          a.rows_total = static_cast<int>(rows_total);
          a.iters = static_cast<int>((256ll << 20) / (stage_bytes * (long long)sms)) + 8;
          const int smem = stage_bytes * stages + 2048;
          bench<<<sms, 64, smem>>>(a);
          cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
          cudaEventRecord(e0);
          bench<<<sms, 64, smem>>>(a);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          const double bytes = static_cast<double>(stage_bytes) * a.iters * sms;
          const double gbs = bytes / ms / 1e6;
          printf("footprint %5zu MB box %3d rows x %d/stage, %d stages (%3d KB in flight): %7.0f GB/s  %5.1f B/clk/SM  err=%s\n",
                 mb, R, boxes, stages, stage_bytes * stages / 1024, gbs,
                 gbs * 1e9 / (sms * (clk * 1e3)), cudaGetErrorString(cudaGetLastError()));
        }
      }
    }
    cudaFree(buf);
  }
  return 0;
}
