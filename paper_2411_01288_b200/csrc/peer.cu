// peer.cu -- peer-shareable buffers, CUDA IPC handles and a device-side
// barrier over peer flags: the plumbing of the fused GEMM -> reduce-scatter
// (hxm_moe_forward_tp / hxm_moe_backward_tp, include/hexamoe.h).
//
// One process per GPU: every rank cudaMalloc's its own receive buffer and
// flag array, exports IPC handles, and maps its peers' (NVLink P2P between
// GPUs of one node; the same mechanism between processes on one GPU).  The
// ESMM epilogues then reduce rows straight into the owners' buffers.
#include <cstring>

#include "common.cuh"

namespace hxm {
namespace {

// Rank `rank` publishes `epoch` into slot [rank] of every rank's flag array
// and waits until all slots of its own array reach `epoch`.  Release /
// acquire at system scope order the reductions issued before (by kernels
// earlier in the stream, completed) against the owners' reads after.
__global__ void peer_barrier_kernel(hxm_peer_flags f, int32_t epoch) {
  const int i = threadIdx.x;
  if (i >= f.n_ranks) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(f.ptrs[i] + f.rank), "r"(epoch)
               : "memory");
  const int32_t* mine = f.ptrs[f.rank] + i;
  const long long t0 = clock64();
  while (true) {
    int32_t v;
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
    if (v >= epoch) break;
    if (clock64() - t0 > (1ll << 36)) __trap();  // a peer never arrived: fail, do not hang
  }
}

}  // namespace
}  // namespace hxm

using namespace hxm;

extern "C" {

hxm_status hxm_peer_malloc(size_t bytes, void** ptr) {
  if (!ptr) return invalid_arg("peer_malloc: null out pointer");
  HXM_TRY_CUDA(cudaMalloc(ptr, bytes > 0 ? bytes : 1));
  HXM_TRY_CUDA(cudaMemset(*ptr, 0, bytes > 0 ? bytes : 1));
  return HXM_OK;
}

hxm_status hxm_peer_free(void* ptr) {
  HXM_TRY_CUDA(cudaFree(ptr));
  return HXM_OK;
}

hxm_status hxm_ipc_get_handle(void* ptr, unsigned char handle[64]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  HXM_TRY_CUDA(cudaIpcGetMemHandle(&h, ptr));
  std::memcpy(handle, &h, 64);
  return HXM_OK;
}

hxm_status hxm_ipc_open_handle(const unsigned char handle[64], void** ptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  HXM_TRY_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return HXM_OK;
}

hxm_status hxm_ipc_close_handle(void* ptr) {
  HXM_TRY_CUDA(cudaIpcCloseMemHandle(ptr));
  return HXM_OK;
}

hxm_status hxm_peer_barrier(const hxm_peer_flags* f, int32_t epoch, hxm_stream_t stream) {
  if (!f || f->n_ranks < 1 || f->n_ranks > HXM_MAX_PEERS || f->rank < 0 || f->rank >= f->n_ranks)
    return invalid_arg("peer_barrier: bad flag table");
  for (int r = 0; r < f->n_ranks; ++r)
    if (!f->ptrs[r]) return invalid_arg("peer_barrier: null flag array");
  peer_barrier_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*f, epoch);
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

}  // extern "C"
