// l2bw.cu -- measure L2->SM read bandwidth (footprint << L2) and HBM read
// bandwidth (footprint >> L2) with 16-byte loads.  nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a tools/l2bw.cu -o /tmp/l2bw && /tmp/l2bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const uint4* __restrict__ p, size_t n16, int iters, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
      uint4 v;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if (acc.x == 0x12345678) sink[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* buf; uint4* sink;
  size_t big = (size_t)4 << 30;
  cudaMalloc(&buf, big); cudaMalloc(&sink, 64);
  cudaMemset(buf, 1, big);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t mb : {8, 24, 48, 96, 4096}) {
    size_t bytes = mb << 20, n16 = bytes / 16;
    int iters = mb >= 1024 ? 2 : (int)(8192 / mb);
    for (int bps : {4, 8}) {
      rd<<<sms * bps, 512>>>(buf, n16, 1, sink);
      cudaEventRecord(a);
      rd<<<sms * bps, 512>>>(buf, n16, iters, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("footprint %5zu MB blocks/SM %d: %.0f GB/s\n", mb, bps, (double)bytes * iters / ms / 1e6);
    }
  }
  return 0;
}
