// umma_impl.cuh -- the tcgen05 GEMM kernel templates and their host-side
// helpers, shared by umma.cu (the ESMM / ESTMM launchers) and esfk.cu (the
// one-launch ESFK).  Everything is in an anonymous namespace: each
// translation unit instantiates what it launches.
#pragma once
#include <cuda.h>

#include <cstring>

#include "kernels.cuh"

namespace hxm {

namespace {

constexpr int BM = 128;  // UMMA M (rows per tile, TMEM lanes)
constexpr int BK = 64;   // one 128-byte swizzle atom of bf16 per k-block
constexpr int UK = 16;   // UMMA K for kind::f16
// Epilogue warps per CTA: 8 (two per TMEM lane group), or 16 for the
// stash-writing MODE 1 / 2 kernels at BN = 256, whose epilogue (activation,
// F' multiply, column sums, TMA stores) is the bottleneck at K = 384 and needs
// more warps to hide its latencies.  Threads = producer + MMA + epilogue.
__host__ __device__ constexpr int epi_warps(int bn, int mode) {
  return (mode == 1 || mode == 2 || mode == 3) && bn == 256 ? 16 : 8;
}
constexpr uint32_t kTmemCols = 512;
constexpr int kABytes = BM * BK * 2;  // 16 KB

// ------------------------------------------------------------- PTX layer --
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Debug timeline (build with -DHXM_TRACE_BUILD, run with HXM_TRACE=<label>,
// read with tools/trace_kernel.py): per-CTA item timestamps and barrier
// wait totals.  Compiled out otherwise.
#ifdef HXM_TRACE_BUILD
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif
// HXM_DEBUG_NOLOAD knobs (operand loads / stores / MMAs skipped) without the
// timeline: -DHXM_DBG_BUILD (python tools/trace_build.py --dbg)
#if defined(HXM_DBG_BUILD) || defined(HXM_TRACE_BUILD)
constexpr bool kDbg = true;
#else
constexpr bool kDbg = false;
#endif
#define TRACE(item, slot)                                                              \
  do {                                                                                 \
    if (kTrace && p.trace && (item) < 64)                                              \
      p.trace[(static_cast<size_t>(blockIdx.x) * 64 + (item)) * 8 + (slot)] = gtime(); \
  } while (0)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
// Blocking phase wait.  A pipeline bug must not hang the GPU: after 2^28
// failed polls (seconds) without progress the kernel traps, which surfaces as
// a CUDA error on the host instead of a wedged device.  (A clock64 deadline
// in the poll loop measurably slowed the pipeline hand-offs.)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done;
  asm volatile(
      "{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(done)
      : "r"(a), "r"(parity)
      : "memory");
  if (done) return;
  uint32_t n = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) return;
    // every failed try_wait suspends the thread for up to a hardware time
    // limit first, so 2^28 of them are many seconds
    if (++n == (1u << 28)) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                       int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                       int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                       int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// 4 rows (r0..r3, -1 = out of bounds -> zero fill) x 64 columns from col.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int col, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// TMA tile store smem -> global (bulk-group completion)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map),
      "r"(c0), "r"(c1), "r"(smem_u32(src))
      : "memory");
}
// the same store with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, const void* src, int c0,
                                                  int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint"
      " [%0, {%1, %2}], [%3], %4;" ::"l"(map),
      "r"(c0), "r"(c1), "r"(smem_u32(src)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// named barrier among a subset of warps (id 0 is __syncthreads)
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// ---- CTA-pair (cluster of 2) helpers ----------------------------------------
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of the same smem offset in CTA rank 0
__device__ __forceinline__ uint32_t mapa0(uint32_t local) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(local));
  return r;
}
// Arrival on the leader's barrier (the epilogues' accumulator release).
// Default (cta-scope) semantics, as in CUTLASS's ClusterBarrier: what it
// orders is TMEM traffic, which the tcgen05 fences cover; a .cluster-scope
// release/acquire would make ptxas emit MEMBAR / CCTL.IVALL on every spin.
__device__ __forceinline__ void mbar_arrive_cl(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity);
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
  mbar_wait(bar, parity);
}
// TMA loads whose completion is signalled on the leader CTA's barrier
__device__ __forceinline__ void tma_2d_cg2(void* dst, const CUtensorMap* map, uint32_t bar, int c0,
                                           int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d_cg2(void* dst, const CUtensorMap* map, uint32_t bar, int c0,
                                           int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                       int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_5d_cg2(void* dst, const CUtensorMap* map, uint32_t bar, int c0,
                                           int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_4d_cg2(void* dst, const CUtensorMap* map, uint32_t bar, int c0,
                                           int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// arrive on the barrier at this smem offset in BOTH CTAs of the pair
__device__ __forceinline__ void umma_commit_cg2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

// One 64-deep k-block: four K=16 UMMAs (descriptors advanced in their low
// words, which hold the start address) and the commit that frees the stage,
// in one asm statement so the issuing thread converts its operands to
// uniform registers once per k-block.  first = 1: the item's first k-block
// (overwrite the accumulator).  skip = 1 (debug): commit only.
template <int CG>
__device__ __forceinline__ void umma_kblock(uint32_t tmem_d, uint32_t a_lo, uint32_t a_hi,
                                            uint32_t a_step, uint32_t b_lo, uint32_t b_hi,
                                            uint32_t b_step, uint32_t idesc, uint32_t first,
                                            uint64_t* bar, uint32_t skip = 0) {
  if constexpr (CG == 2) {
    asm volatile(
        "{\n"
        ".reg .pred p0, p1, sk;\n"
        ".reg .b64 da, db;\n"
        ".reg .b32 al, bl;\n"
        "setp.ne.b32 p0, %8, 0;\n"
        "setp.eq.b32 p1, %8, %8;\n"
        "setp.ne.b32 sk, %10, 0;\n"
        "@sk bra.uni DONE%=;\n"
        "mov.b64 da, {%1, %2};\n"
        "mov.b64 db, {%4, %5};\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %7, p0;\n"
        "add.u32 al, %1, %3;\n"
        "add.u32 bl, %4, %6;\n"
        "mov.b64 da, {al, %2};\n"
        "mov.b64 db, {bl, %5};\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %7, p1;\n"
        "add.u32 al, al, %3;\n"
        "add.u32 bl, bl, %6;\n"
        "mov.b64 da, {al, %2};\n"
        "mov.b64 db, {bl, %5};\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %7, p1;\n"
        "add.u32 al, al, %3;\n"
        "add.u32 bl, bl, %6;\n"
        "mov.b64 da, {al, %2};\n"
        "mov.b64 db, {bl, %5};\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %7, p1;\n"
        "DONE%=:\n"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%9], %11;\n"
        "}\n" ::"r"(tmem_d),
        "r"(a_lo), "r"(a_hi), "r"(a_step), "r"(b_lo), "r"(b_hi), "r"(b_step), "r"(idesc),
        "r"(first ? 0u : 1u), "r"(smem_u32(bar)), "r"(skip), "h"(static_cast<uint16_t>(3))
        : "memory");
  } else {
    asm volatile(
        "{\n"
        ".reg .pred p0, p1, sk;\n"
        ".reg .b64 da, db;\n"
        ".reg .b32 al, bl;\n"
        "setp.ne.b32 p0, %8, 0;\n"
        "setp.eq.b32 p1, %8, %8;\n"
        "setp.ne.b32 sk, %10, 0;\n"
        "@sk bra.uni DONE%=;\n"
        "mov.b64 da, {%1, %2};\n"
        "mov.b64 db, {%4, %5};\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %7, p0;\n"
        "add.u32 al, %1, %3;\n"
        "add.u32 bl, %4, %6;\n"
        "mov.b64 da, {al, %2};\n"
        "mov.b64 db, {bl, %5};\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %7, p1;\n"
        "add.u32 al, al, %3;\n"
        "add.u32 bl, bl, %6;\n"
        "mov.b64 da, {al, %2};\n"
        "mov.b64 db, {bl, %5};\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %7, p1;\n"
        "add.u32 al, al, %3;\n"
        "add.u32 bl, bl, %6;\n"
        "mov.b64 da, {al, %2};\n"
        "mov.b64 db, {bl, %5};\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %7, p1;\n"
        "DONE%=:\n"
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n"
        "}\n" ::"r"(tmem_d),
        "r"(a_lo), "r"(a_hi), "r"(a_step), "r"(b_lo), "r"(b_hi), "r"(b_step), "r"(idesc),
        "r"(first ? 0u : 1u), "r"(smem_u32(bar)), "r"(skip)
        : "memory");
  }
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

// same load without the completion wait (pair with tmem_wait)
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}
// Reductions into ANOTHER GPU's memory (fused reduce-scatter over NVLink):
// several GPUs add into the same owner row, so the atomics must be morally
// strong across devices -- system scope, not the default .gpu scope.
__device__ __forceinline__ void red_add_v4_sys(float* p, float a, float b, float c, float d) {
  asm volatile("red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a),
               "f"(b), "f"(c), "f"(d)
               : "memory");
}

// UMMA shared-memory descriptor (sm100): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version=1 [46,48), layout SWIZZLE_128B=2 [61,64).
// layout 2 = SWIZZLE_128B, 4 = SWIZZLE_64B.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                          uint64_t layout = 2) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}
// Instruction descriptor kind::f16: D=f32, A=B=bf16, majors, N>>3, M>>4.
__host__ __device__ constexpr uint32_t idesc_bf16(int n, int a_mn, int b_mn, int m = BM) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// ---- packed fp32x2 math (FFMA2 / FMUL2 on sm_100): two lanes per issue ----
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
        "l"(*reinterpret_cast<uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
// Read-only loads of optional operands (bias pointers that may be null):
// asm volatile so the compiler cannot speculate them above the null check
// (an __ldg was hoisted above `if (bias)` in one build: a fault at address 0)
__device__ __forceinline__ float4 ldg_nc_v4(const float4* ptr) {
  float4 r;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(ptr));
  return r;
}
__device__ __forceinline__ float ldg_nc(const float* ptr) {
  float r;
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(r) : "l"(ptr));
  return r;
}
__device__ __forceinline__ float tanh_approx(float u) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return t;
}
// F and F' of two values at once (tensor.cpp:39-53, 62-72); GELU-tanh with
// one tanh.approx per value shared by F and F', the rest in f32x2 ops:
// with s = (1 + tanh u) / 2,  F = x s  and  F' = s + 2 u'(x) F (1 - s)
// (1 - tanh^2 u = 4 s (1 - s)): 9 packed ops per pair.
template <int ACT>
__device__ __forceinline__ void act_pair(float2 x, float2& f, float2& df) {
  if constexpr (ACT == HXM_ACT_GELU) {
    constexpr float k0 = 0.7978845608028654f, k1 = 0.7978845608028654f * 0.044715f;
    const float2 x2 = f2_mul(x, x);
    const float2 u = f2_mul(x, f2_fma(f2(k1), x2, f2(k0)));
    const float2 t = make_float2(tanh_approx(u.x), tanh_approx(u.y));
    const float2 s = f2_fma(t, f2(0.5f), f2(0.5f));
    f = f2_mul(x, s);
    const float2 du2 = f2_fma(f2(6.f * k1), x2, f2(2.f * k0));  // 2 u'(x)
    const float2 oms = f2_fma(s, f2(-1.f), f2(1.f));
    df = f2_fma(du2, f2_mul(f, oms), s);
  } else if constexpr (ACT == HXM_ACT_RELU) {
    f = make_float2(x.x > 0.f ? x.x : 0.f, x.y > 0.f ? x.y : 0.f);
    df = make_float2(x.x > 0.f ? 1.f : 0.f, x.y > 0.f ? 1.f : 0.f);
  } else {
    f = x;
    df = f2(1.f);
  }
}

struct UParams {
  CUtensorMap tmA;  // ESMM A / ESTMM X1
  CUtensorMap tmB;  // ESMM W / ESTMM X2
  CUtensorMap tmO1;  // MODE 1/2: dense bf16 stash output(s), 32-col x 128-row boxes
  CUtensorMap tmO2;
  CUtensorMap tmO1s;  // the same outputs, 32 x 32 boxes (segment-end slices)
  CUtensorMap tmO2s;
  CUtensorMap tmY;  // MODE 2: F'(y1) stash, 32 x 128 boxes
  RowMap amap;      // gather map of A (ESMM rows / ESTMM X1 rows)
  RowMap bmap;      // ESTMM X2 rows
  int a_gather, b_gather, b_kmajor;
  int dbg_noload;
  unsigned long long* trace;  // debug timeline (HXM_TRACE), null normally
  int b_sw64;  // CG = 2, MN-major B halves of 32-column multiples: 64B-swizzled boxes
  // shard-major weights (data-centric TP cache, hxm_layer_desc.weight_shards):
  // W is [P][E][..] with the H axis split into P slices of w_shard_h; the B
  // map gains a shard dimension.  w_shard_k: the split H axis is K (else N).
  int w_shard_h;
  int w_shard_k;
  int bias_shard_h;  // MODE 1: b1 is [P][E][h] (0: E x N)
  int stream_k;      // MODE 0, reduction epilogue: equal k-block ranges per cluster
  int n_experts;
  int l2hint;  // MODE 1/2: L2 eviction-priority hints on the stash stores
  int reverse; // walk the work items last to first
  int trans_out;         // whole-tile ESTMM: store out[e] transposed
  int n_peer;            // EPI_ATOMIC: > 0 -> row t reduces into peer[t / peer_rows]
  int peer_dim;          // ESTMM: 0 = output rows, 1 = output columns split over peers
  long long peer_rows;
  float* peer[HXM_MAX_PEERS];
  int K, N, M;  // ESMM: K=d1, N=d2 ; ESTMM: M=d1, N=d2
  int n_nt, n_mt;
  const SegTile* tiles;
  const int32_t* n_tiles;
  int epi, act;
  const float* bias;
  float* out_f32;
  RowMap omap;
  void* out1;
  void* out2;
  const void* y1s;
  float* colsum;  // MODE 2: per-(tile, lane group) column sums of the output
  float* est_out;
  const char* label;
};

// B operand box of one k-block: W[e] (MN-major, 4D view / 5D shard-major)
// or W^T use (K-major, 3D view / 4D shard-major).  `nb` = this CTA's first B
// column, k0 = the k-block's first K row.
template <int CG>
__device__ __forceinline__ void load_w_box(const UParams& p, void* sb, uint64_t* bar_local,
                                           uint32_t bar_lead, int k0, int nb, int e) {
  const int bw = p.b_sw64 ? 32 : 64;
  const int h = p.w_shard_h;
  if (p.b_kmajor) {
    if (h == 0) {
      if constexpr (CG == 2) tma_3d_cg2(sb, &p.tmB, bar_lead, k0, nb, e);
      else tma_3d(sb, &p.tmB, bar_local, k0, nb, e);
    } else {
      const int c0 = p.w_shard_k ? k0 % h : k0, c1 = p.w_shard_k ? nb : nb % h;
      const int sh = p.w_shard_k ? k0 / h : nb / h;
      if constexpr (CG == 2) tma_4d_cg2(sb, &p.tmB, bar_lead, c0, c1, e, sh);
      else tma_4d(sb, &p.tmB, bar_local, c0, c1, e, sh);
    }
  } else {
    if (h == 0) {
      if constexpr (CG == 2) tma_4d_cg2(sb, &p.tmB, bar_lead, 0, k0, nb / bw, e);
      else tma_4d(sb, &p.tmB, bar_local, 0, k0, nb / bw, e);
    } else {
      const int c1 = p.w_shard_k ? k0 % h : k0, c2 = (p.w_shard_k ? nb : nb % h) / bw;
      const int sh = p.w_shard_k ? k0 / h : nb / h;
      if constexpr (CG == 2) tma_5d_cg2(sb, &p.tmB, bar_lead, 0, c1, c2, e, sh);
      else tma_5d(sb, &p.tmB, bar_local, 0, c1, c2, e, sh);
    }
  }
}

// Division by a kernel-uniform divisor without the ~25-instruction integer
// division sequence (work item -> tile, column block), as CUTLASS FastDivmod:
// q = umulhi(n, m) >> s for n < 2^31.
struct FastDiv {
  uint32_t d, m, s;
  __device__ __forceinline__ explicit FastDiv(uint32_t div) : d(div), m(0), s(0) {
    if (div > 1) {
      const uint32_t l = 32 - __clz(div - 1);  // ceil(log2(div))
      const uint32_t pw = 31 + l;
      m = static_cast<uint32_t>(((1ull << pw) + div - 1) / div);
      s = pw - 32;
    }
  }
  __device__ __forceinline__ int div(int n) const {
    return d == 1 ? n : static_cast<int>(__umulhi(static_cast<uint32_t>(n), m) >> s);
  }
  __device__ __forceinline__ int mod(int n) const { return n - div(n) * static_cast<int>(d); }
};

// CG = CTAs per UMMA (cta_group): with CG = 2 a CTA pair runs M = 256 tiles,
// each CTA holding 128 rows of A / D and half (BN/2) of the B columns.
template <int BN, int CG = 1, int MODE = 0, int EW = 8>
struct Cfg {
  static constexpr int kBBytes = (BN / CG) * BK * 2;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kEW = EW;
  static constexpr int kGroups = kEW / 4;  // column groups of 4 warps (one per lane group)
  // MODE 1 / 2 staging per column group: MODE 1: kOutBufs output boxes (two
  // 8 KB boxes F', F each); MODE 2: a kYRing-deep ring of 8 KB F'(y1) boxes,
  // each overwritten in place by its chunk's g_y1 (a thread reads its own
  // row of F' before writing that row of g_y1) and TMA-stored from there;
  // 16 epilogue warps trade depth for the extra groups.
  static constexpr int kOutBufs = kEW == 16 ? 1 : 2;
  static constexpr int kYRing = kEW == 16 ? 2 : 3;
  static constexpr int kOutBox = MODE == 1 ? 16384 : 8192;
  static constexpr int kGroupBytes =
      MODE == 1 ? kOutBufs * kOutBox : MODE == 2 ? kYRing * 8192 : 4 * 2048;
  // 227 KB opt-in smem = stages + epilogue staging + 1 KB alignment slack +
  // barriers.  Staging: 2 KB per epilogue warp (MODE 0 / 3).
  static constexpr int kStaging = kGroups * kGroupBytes;
  // MODE 1: the item's bias columns (BN floats), shared by a column group's warps
  static constexpr int kBias = MODE == 1 ? BN * 4 : 0;
  // MODE 2 with 16 warps: per-warp F'(y1) slices and barriers (HXM_PW_EPI)
#ifndef HXM_PW_EPI
#define HXM_PW_EPI 1
#endif
  static constexpr bool kPW2 = HXM_PW_EPI && MODE == 2 && EW == 16;
  static constexpr int kDbars = (kPW2 ? kEW : kGroups) * kYRing;
  static constexpr int kBars = kPW2 ? 512 : 256;
  static constexpr int kBudget = 232448 - 1024 - kBars - kStaging - kBias;
  static constexpr int kStages = kBudget / kStage > 8 ? 8 : kBudget / kStage;
  static constexpr int kSmem =
      kStages * kStage + kStaging + kBias + 1024 /*align*/ + kBars /*barriers*/;
};

// MODE: 0 = ESMM, fp32 write / accumulate / reduce epilogue; 1 = ESMM with
// bias + activation into the bf16 stash (y1, y2); 2 = ESMM times F'(y1) into
// the bf16 g_y1 stash; 3 = ESTMM.  One instantiation per mode keeps each
// epilogue's register footprint to what it uses.
//
// CG = 2 (dense operands only): clusters of 2 CTAs; the leader (rank 0)
// issues tcgen05.mma.cta_group::2 with M = 256; both CTAs' TMA loads signal
// the leader's full barrier; commits multicast to both CTAs' empty / tfull
// barriers; both CTAs' epilogues arrive on the leader's tempty barrier.
//
// The body is a device function over a "virtual grid" of n_clusters
// clusters, so one launch can also run two operators side by side on
// disjoint clusters (esfk_kernel below: ESMM grad-x tiles + ESTMM grad-W
// tiles, es_ops.cpp:210-247).
template <int BN, int MODE, int CG = 1, int ACT = -1, int EW = 8>
__device__ __forceinline__ void umma_body(const UParams& p, const int cluster,
                                          const int n_clusters) {
  constexpr bool ESTMM = MODE == 3;
  using C = Cfg<BN, CG, MODE, EW>;
  uint32_t rank = 0;
  if constexpr (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (128B-swizzle atoms); pointer arithmetic on the
  // __shared__ array keeps the address space visible to the compiler, so
  // staging accesses compile to LDS/STS rather than generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* staging = smem + C::kStages * C::kStage;
  float* bias_s = reinterpret_cast<float*>(staging + C::kStaging);  // MODE 1
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + C::kStaging + C::kBias);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* dbar = tempty + 2;  // MODE 2: F'(y1) box loads, [group][ring slot]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dbar + C::kDbars);

  // warp index broadcast from lane 0: ptxas then knows it is warp-uniform and
  // keeps what derives from it (roles, TMEM lane group, column group, staging
  // slices, TMA-store coordinates) in uniform registers (CUTLASS's
  // canonical_warp_idx_sync)
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0);
  const int lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);  // CG = 2: the leader's producer expects both CTAs' bytes
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], C::kEW * CG);
    }
    for (int b = 0; b < C::kDbars; ++b) mbar_init(&dbar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  // the leader CTA's copies of the shared barriers (CG = 2)
  const uint32_t full_lead = CG == 2 ? mapa0(smem_u32(full)) : smem_u32(full);
  const uint32_t tempty_lead = CG == 2 ? mapa0(smem_u32(tempty)) : smem_u32(tempty);

  // PDL: everything above overlapped the previous kernel; from here on the
  // kernel reads what earlier kernels wrote (tile tables, operands)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n_items = *p.n_tiles;
  const int per_item = ESTMM ? p.n_mt * p.n_nt : p.n_nt;
  const int total = n_items * per_item;
  const FastDiv fdi(static_cast<uint32_t>(per_item));  // work item -> (tile, rem)
  // p.reverse: walk the items last to first, so a kernel that consumes the
  // previous kernel's output starts on the rows written last (L2-resident)
  auto wmap = [&](int wl) { return p.reverse ? total - 1 - wl : wl; };
  // Work units of this cluster: (work item wl, k-blocks [lo, hi)).  Default:
  // whole items wl = cluster, cluster + n_clusters, ... (round-robin: the
  // pairs that work on the two N-tiles of an M-tile run side by side and
  // share its A rows' HBM reads in L2).  Stream-K tail (MODE 0 with a
  // reduction epilogue, p.stream_k): the full waves stay round-robin, the
  // items of the last partial wave are flattened into (item, k-block) space
  // and cut into n_clusters equal contiguous ranges, so no cluster idles
  // through a partial wave; a tail item cut between two clusters is reduced
  // twice (red.add), its bias added by the part holding k-block 0.
  // hi = -1: the item's own length (ESTMM chunks).
  struct Unit {
    int wl, lo, hi;
    bool ok;
  };
  const int nk_all = ESTMM ? 1 : p.K / BK;  // (stream_k is never set for ESTMM)
  const int full_waves = p.stream_k ? total / n_clusters : 0;
  const int tail0 = full_waves * n_clusters;  // first tail item
  const long long tail_kb = p.stream_k ? static_cast<long long>(total - tail0) * nk_all : 0;
  const int sk_g0 = static_cast<int>(tail_kb * cluster / n_clusters);
  const int sk_g1 = static_cast<int>(tail_kb * (cluster + 1) / n_clusters);
  auto unit_at = [&](int i) -> Unit {
    if (!p.stream_k) {
      const int wl = cluster + i * n_clusters;
      return Unit{wl, 0, ESTMM ? -1 : nk_all, wl < total};
    }
    if (i < full_waves) return Unit{cluster + i * n_clusters, 0, nk_all, true};
    const int j = i - full_waves;
    const int it = sk_g0 / nk_all + j;  // tail-relative item
    const int lo = j == 0 ? sk_g0 % nk_all : 0;
    const int base = it * nk_all;
    const int hi = sk_g1 - base < nk_all ? sk_g1 - base : nk_all;
    return Unit{tail0 + it, lo, hi, base + lo < sk_g1};
  };

  if (warp == 0) {
    // ================================ TMA producer =======================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmB) : "memory");
    }
    int s = 0;
    uint32_t ph = 0;
    int pit_ = 0;
    for (int ui = 0;; ++ui, ++pit_) {
      const Unit u = unit_at(ui);
      if (!u.ok) break;
      const int w = wmap(u.wl);
      const SegTile t = p.tiles[fdi.div(w)];
      const int rem = fdi.mod(w);
      if (!ESTMM) {
        const int n0 = rem * BN;
        const int nk = u.hi;
        int rows[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int q = t.begin + 4 * lane + i;
          rows[i] = (p.a_gather && q < t.end) ? p.amap(q) : -1;
        }
        unsigned long long pw = 0;
        for (int kb = u.lo; kb < nk; ++kb) {
          const long long tp0 = (kTrace && p.trace) ? clock64() : 0;
          mbar_wait(&empty[s], ph ^ 1);
          if (kTrace && p.trace) pw += clock64() - tp0;
          if (kTrace && p.trace && lane == 0 && kb == nk - 1 && pit_ < 64) p.trace[(static_cast<size_t>(blockIdx.x) * 64 + pit_) * 8 + 7] = pw;
          uint8_t* sa = smem + s * C::kStage;
          uint8_t* sb = sa + kABytes;
          if constexpr (CG == 2) {
            // dense only: this CTA's 128 rows of A and BN/2 columns of B,
            // completion counted on the leader's full barrier
            if (elect_one()) {
              const uint32_t fb = full_lead + 8u * s;
              if (kDbg && (p.dbg_noload & 1)) {  // debug: no operand loads
                if (rank == 0) mbar_arrive(&full[s]);
              } else if (kDbg && (p.dbg_noload & 24)) {  // debug: A only (8) / B only (16)
                if (rank == 0) mbar_arrive_tx(&full[s], 2 * ((p.dbg_noload & 8) ? kABytes : C::kBBytes));
                const int nb = n0 + static_cast<int>(rank) * (BN / 2);
                if (p.dbg_noload & 8) tma_2d_cg2(sa, &p.tmA, fb, kb * BK, t.begin + static_cast<int>(rank) * BM);
                else load_w_box<2>(p, sb, nullptr, fb, kb * BK, nb, t.expert);
              } else {
                // the leader expects both CTAs' bytes; the peer's loads
                // only complete_tx on it (no second remote arrive)
                if (rank == 0) mbar_arrive_tx(&full[s], 2 * C::kStage);
                tma_2d_cg2(sa, &p.tmA, fb, kb * BK, t.begin + static_cast<int>(rank) * BM);
                const int nb = n0 + static_cast<int>(rank) * (BN / 2);
                // all of this CTA's swizzle-atom column chunks in one box
                load_w_box<2>(p, sb, nullptr, fb, kb * BK, nb, t.expert);
              }
            }
          } else {
            const bool el = elect_one();
            if (el) mbar_arrive_tx(&full[s], C::kStage);
            __syncwarp();
            if (p.a_gather) {
              tma_gather4(sa + lane * 512, &p.tmA, &full[s], kb * BK, rows[0], rows[1], rows[2],
                          rows[3]);
            } else if (el) {
              tma_2d(sa, &p.tmA, &full[s], kb * BK, t.begin);
            }
            if (el) load_w_box<1>(p, sb, &full[s], 0u, kb * BK, n0, t.expert);
          }
          __syncwarp();
          if (++s == C::kStages) { s = 0; ph ^= 1; }
        }
      } else {
        const int mt = rem / p.n_nt, nt = rem % p.n_nt;
        const int m0 = mt * BM * CG + static_cast<int>(rank) * BM;
        const int n0 = nt * BN + static_cast<int>(rank) * (BN / CG);
        const int nk = (t.end - t.begin + BK - 1) / BK;
        for (int kb = 0; kb < nk; ++kb) {
          const int p0 = t.begin + kb * BK;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * C::kStage;
          uint8_t* sb = sa + kABytes;
          if constexpr (CG == 2) {  // dense only (host guarantees)
            if (elect_one()) {
              const uint32_t fb = full_lead + 8u * s;
              if (kDbg && (p.dbg_noload & 1)) {  // debug: no operand loads
                if (rank == 0) mbar_arrive(&full[s]);
              } else {
                if (rank == 0) mbar_arrive_tx(&full[s], 2 * C::kStage);
                // both 64-column chunks of A, all chunks of B: one 3D box each
                tma_3d_cg2(sa, &p.tmA, fb, 0, p0, m0 / 64);
                tma_3d_cg2(sb, &p.tmB, fb, 0, p0, n0 / (p.b_sw64 ? 32 : 64));
              }
            }
            __syncwarp();
            if (++s == C::kStages) { s = 0; ph ^= 1; }
            continue;
          }
          const bool el = elect_one();
          if (el) mbar_arrive_tx(&full[s], C::kStage);
          __syncwarp();
          // A = X1^T: two 64-column chunks of the 64 k-rows
          if (p.a_gather) {
            const int rg = lane % 16, ch = lane / 16;
            int r[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int q = p0 + 4 * rg + i;
              r[i] = q < t.end ? p.amap(q) : -1;
            }
            tma_gather4(sa + ch * 8192 + rg * 512, &p.tmA, &full[s], m0 + 64 * ch, r[0], r[1],
                        r[2], r[3]);
          } else if (el) {
            tma_3d(sa, &p.tmA, &full[s], 0, p0, m0 / 64);
          }
          // B = X2: BN/64 chunks of the 64 k-rows
          if (p.b_gather) {
            for (int g = lane; g < (BN / 64) * 16; g += 32) {
              const int rg = g % 16, ch = g / 16;
              int r[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int q = p0 + 4 * rg + i;
                r[i] = q < t.end ? p.bmap(q) : -1;
              }
              tma_gather4(sb + ch * 8192 + rg * 512, &p.tmB, &full[s], n0 + 64 * ch, r[0], r[1],
                          r[2], r[3]);
            }
          } else if (el) {
            tma_3d(sb, &p.tmB, &full[s], 0, p0, n0 / 64);
          }
          __syncwarp();
          if (++s == C::kStages) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ==========================
    constexpr uint32_t kIdescEsmmMN = idesc_bf16(BN, 0, 1, BM * CG);
    constexpr uint32_t kIdescEsmmK = idesc_bf16(BN, 0, 0, BM * CG);
    constexpr uint32_t kIdescEst = idesc_bf16(BN, 1, 1, BM * CG);
    // One thread issues everything; descriptors are built once and advanced
    // by adding to the start-address field, so a k-block costs ~a dozen
    // instructions (the tensor pipe needs a new UMMA every 64-128 cycles).
    // CG = 2: only the leader CTA issues; its descriptors address the same
    // smem offsets in both CTAs.
    if (rank == 0) {  // the whole warp walks the loop (uniform); one elected lane issues
      const uint32_t idesc = ESTMM ? kIdescEst : (p.b_kmajor ? kIdescEsmmK : kIdescEsmmMN);
      // per UMMA_K (16) step, in 16-byte descriptor units: K-major = 32 B
      // inside the swizzle atom; MN-major = 16 k-rows = 2 x 1024 B
      const bool a_mn = ESTMM, b_mn = ESTMM || !p.b_kmajor;
      // SW64 MN-major B: 32-column atoms, 4 KB per 64 k-rows, 512 B per 8 rows
      const bool sw64 = b_mn && p.b_sw64;
      const uint32_t a_step = a_mn ? 128u : 2u, b_step = b_mn ? (sw64 ? 64u : 128u) : 2u;
      const uint32_t base = smem_u32(smem);
      const uint64_t da0 = a_mn ? sdesc(base, 8192, 1024) : sdesc(base, 16, 1024);
      const uint64_t db0 = !b_mn ? sdesc(base + kABytes, 16, 1024)
                           : sw64 ? sdesc(base + kABytes, 4096, 512, 4)
                                  : sdesc(base + kABytes, 8192, 1024);
      const uint32_t a_lo = static_cast<uint32_t>(da0), a_hi = static_cast<uint32_t>(da0 >> 32);
      const uint32_t b_lo = static_cast<uint32_t>(db0), b_hi = static_cast<uint32_t>(db0 >> 32);
      constexpr uint32_t kStageUnits = C::kStage >> 4;
      static_assert(BK / UK == 4, "umma_kblock issues four K=16 UMMAs per k-block");
      const uint32_t skip = kDbg && (p.dbg_noload & 4) ? 1u : 0u;
      int s = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      int it_ = 0;
      for (int ui = 0;; ++ui, ++it_) {
        const Unit u = unit_at(ui);
        if (!u.ok) break;
        const int w = wmap(u.wl);
        const int nk = ESTMM ? (p.tiles[fdi.div(w)].end - p.tiles[fdi.div(w)].begin + BK - 1) / BK
                             : u.hi;
        if (lane == 0) TRACE(it_, 0);
        if constexpr (CG == 2) mbar_wait_cl(&tempty[acc], aph ^ 1);
        else mbar_wait(&tempty[acc], aph ^ 1);
        if (lane == 0) TRACE(it_, 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        unsigned long long wsum = 0;
        for (int kb = u.lo; kb < nk; ++kb) {
          const long long tw0 = (kTrace && p.trace) ? clock64() : 0;
          if constexpr (CG == 2) mbar_wait_cl(&full[s], ph);
          else mbar_wait(&full[s], ph);
          if (kTrace && p.trace) wsum += clock64() - tw0;
          tc_fence_after();
          const uint32_t so = static_cast<uint32_t>(s) * kStageUnits;
          if (elect_one())
            umma_kblock<CG>(d, a_lo + so, a_hi, a_step, b_lo + so, b_hi, b_step, idesc, kb == u.lo,
                            &empty[s], skip);
          __syncwarp();
          if (++s == C::kStages) { s = 0; ph ^= 1; }
        }
        if (elect_one()) {
          if constexpr (CG == 2) umma_commit_cg2(&tfull[acc]);
          else umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (lane == 0) TRACE(it_, 2);
        if (kTrace && p.trace && lane == 0 && it_ < 64) p.trace[(static_cast<size_t>(blockIdx.x) * 64 + it_) * 8 + 6] = wsum;
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
    __syncwarp();
  } else {
    // ================================ epilogue ============================
    // kEW warps: warp w reads TMEM lane group (w % 4) -- the hardware rule --
    // and column group (w - 2) / 4 of the accumulator (HB columns), so
    // kEW / 4 warps per SMSP overlap TMEM loads, math and global traffic.
    // fp32 outputs: each 32-row x 32-column chunk is transposed through a
    // per-warp staging tile so stores / reductions cover row segments.
    constexpr int HB = BN / C::kGroups;
    const int lg = warp & 3;
    const int half = (warp - 2) / 4;  // column group
    uint8_t* stg = staging + (warp - 2) * 2048;
    // accumulator drained by this warp: arrive on the (leader's) tempty
    auto release_acc = [&](int a) {
      if constexpr (CG == 2) mbar_arrive_cl(tempty_lead + 8u * a);
      else mbar_arrive(&tempty[a]);
    };
    int acc = 0;
    uint32_t aph = 0;
    int dchunk = 0;  // MODE 1/2: running chunk count of this group (buffers / phases)
    constexpr int kYRing = C::kYRing;  // MODE 2: F'(y1) boxes in flight per group
    constexpr bool bwd = MODE == 2;
    constexpr bool dense_out = MODE == 1 || MODE == 2;
    // MODE 1 with 16 epilogue warps (one output box per column group):
    // per-warp staging slices and stores (HXM_PW_EPI=0 at build time: the
    // column group's box is stored by one thread after a group barrier).
    // MODE 2 with 16 warps (kPW2): each warp also loads its own 32-row
    // slices of the F'(y1) boxes (own barriers), so the g_y1 chunk needs no
    // group barrier either.
    constexpr bool kPW = HXM_PW_EPI && MODE == 1 && C::kOutBufs == 1;
    constexpr bool kPW2 = C::kPW2;
    constexpr int kNch = HB / 32;  // 32-column chunks per warp per tile
    const bool elect = ((warp - 2) & 3) == 0 && lane == 0;
    // this group's staging: kOutBufs output boxes, then (MODE 2) the F'(y1)
    // ring (8 KB per box: 128 rows x 32 bf16)
    uint8_t* hstage = staging + half * C::kGroupBytes;
    // ESMM: the next work item's tile and this lane's output row are loaded
    // one item ahead, so an epilogue that finds its accumulator already full
    // does not wait on the tile table / index latency.
    auto tile_at = [&](int wi) { return wi < total ? p.tiles[fdi.div(wi)] : SegTile{0, 0, 0, 0}; };
    // MODE 0: this lane's token-order output row.  MODE 1/2 only need to
    // know pads, which the layer's tile flags carry (no index load).
    auto orow_of = [&](const SegTile& tt) {
      const int qq = tt.begin + static_cast<int>(rank) * BM + lg * 32 + lane;
      if (dense_out && (tt.flags & 4)) return qq - tt.begin < (tt.flags >> 8) ? 0 : -1;
      if (qq >= tt.end) return -1;
      if (p.omap.kind == MAP_SLOT) {  // issued where written (asm volatile: not sunk)
        int sv;
        asm volatile("ld.global.nc.b32 %0, [%1];"
                     : "=r"(sv)
                     : "l"(static_cast<const int32_t*>(p.omap.v) + qq));
        return sv < 0 ? -1 : sv % p.omap.n;
      }
      return p.omap(qq);
    };
    int ep_it = 0;
    const Unit u0 = unit_at(0);
    SegTile t_cur = ESTMM || !u0.ok ? SegTile{0, 0, 0, 0} : tile_at(wmap(u0.wl));
    int orow_cur = ESTMM ? -1 : orow_of(t_cur);
    // MODE 1 bias: the column group's HB bias floats of the current item sit
    // in smem; lane l < HB / 4 of lane-group warp lg owns entry lg * HB / 4 + l,
    // loads the next item's value during this item (latency hidden) and
    // writes it once the group is past this item's last read (the chunk
    // barriers order writes and reads)
    constexpr int kBq = HB / 4;
    float* gbias = bias_s + half * HB;
    const bool bias_smem = MODE == 1 && p.bias != nullptr;
    auto bias_at = [&](const SegTile& tt, int ww) {
      const int col = fdi.mod(ww) * BN + half * HB + lg * kBq + lane;
      const int hb = p.bias_shard_h;
      return ldg_nc(p.bias + (hb == 0 ? static_cast<int64_t>(tt.expert) * p.N + col
                                     : (static_cast<int64_t>(col / hb) * p.n_experts + tt.expert) *
                                               hb + col % hb));
    };
    if (bias_smem && lane < kBq && u0.ok) gbias[lg * kBq + lane] = bias_at(t_cur, wmap(u0.wl));
    int y_iss = 0;  // MODE 2 (elected thread): global F'(y1) chunks issued so far
    for (int ui = 0;; ++ui) {
      const Unit u = unit_at(ui);
      if (!u.ok) break;
      const int w = wmap(u.wl);
      const SegTile t = ESTMM ? p.tiles[fdi.div(w)] : t_cur;
      const int rem = fdi.mod(w);
      if (!ESTMM) {
        const Unit u_nx = unit_at(ui + 1);
        const bool has_nx = u_nx.ok;
        const int w_nx = has_nx ? wmap(u_nx.wl) : 0;
        const SegTile t_nx = has_nx ? tile_at(w_nx) : SegTile{0, 0, 0, 0};  // prefetch
        int orow_nx = -1;
        float bias_nx = 0.f;  // loaded during the last chunk (short register lifetime)
        const int n0 = rem * BN + half * HB;
        const int orow = orow_cur;
        const int N = p.N;
        // dense bf16 outputs (MODE 1/2): the 4 warps of a column half stage a
        // 128-row x 32-column box per chunk (double-buffered) and one elected
        // thread TMA-stores it; MODE 2 TMA-loads the matching F'(y1) boxes two
        // chunks ahead.  The layer's segments end on 64-row boundaries, so
        // every 32-row warp slice is entirely valid or entirely past the end.
        const int qbase = t.begin + static_cast<int>(rank) * BM;  // row 0 of the box
        const int rows_here = t.end - qbase;
        auto ybox = [&](int gchunk) { return hstage + (gchunk % kYRing) * 8192; };
        auto ybar = [&](int gchunk) {
          return &dbar[(kPW2 ? warp - 2 : half) * kYRing + gchunk % kYRing];
        };
        // F'(y1) boxes stream kYRing - 1 chunks ahead of the math, across the
        // item boundary (the next item's first boxes load during this item's
        // last chunk); a box goes into the slot of the chunk before the one
        // being computed, which every thread has left at that chunk's barrier
        const int chunk0 = dchunk;  // this item's first global chunk
        auto y_issue_to = [&](int limit) {
          if (limit > chunk0 + (has_nx ? 2 : 1) * kNch) limit = chunk0 + (has_nx ? 2 : 1) * kNch;
          for (; y_iss < limit; ++y_iss) {
            const int c = y_iss - chunk0;
            const bool nx = c >= kNch;
            const int col = (nx ? fdi.mod(w_nx) * BN + half * HB : n0) + 32 * (nx ? c - kNch : c);
            const int row = (nx ? t_nx.begin : t.begin) + static_cast<int>(rank) * BM;
            if constexpr (kPW2) {  // this warp's 32 rows (tmO2s: the F' stash, 32 x 32)
              mbar_arrive_tx(ybar(y_iss), 2048);
              tma_2d(ybox(y_iss) + lg * 2048, &p.tmO2s, ybar(y_iss), col, row + lg * 32);
            } else {
              mbar_arrive_tx(ybar(y_iss), 8192);
              tma_2d(ybox(y_iss), &p.tmY, ybar(y_iss), col, row);
            }
          }
        };
        const bool y_issuer = kPW2 ? lane == 0 : elect;
        if (bwd && y_issuer) y_issue_to(chunk0 + (kNch < kYRing - 1 ? kNch : kYRing - 1));
        // MODE 0 bias of this warp's HB columns: every lane reads the same 32
        // floats per chunk (uniform-address LDG.128, one broadcast transaction
        // each, L1-resident) and adds them in f32x2 (MODE 1: from smem, below)
        const bool has_bias = p.bias && !bwd && !dense_out && u.lo == 0;  // stream-K: once
        const float4* bias4 =
            has_bias ? reinterpret_cast<const float4*>(p.bias + static_cast<int64_t>(t.expert) * N + n0)
                     : nullptr;
        // the group's bias entries for this item (written by all four
        // warps at the previous item's end / before the loop) are complete
        if (bias_smem) named_bar_sync(1 + half, 128);
        if (warp == 2 && lane == 0) TRACE(ep_it, 3);
        if constexpr (CG == 2) mbar_wait_cl(&tfull[acc], aph);
        else mbar_wait(&tfull[acc], aph);
        if (warp == 2 && lane == 0) TRACE(ep_it, 4);
        tc_fence_after();
        if (kDbg && !dense_out && (p.dbg_noload & 32)) {  // debug: no epilogue work
          tc_fence_before();
          __syncwarp();
          if (lane == 0) release_acc(acc);
          t_cur = t_nx;
          orow_cur = has_nx ? orow_of(t_nx) : -1;
          if (++acc == 2) { acc = 0; aph ^= 1; }
          continue;
        }
        const uint32_t taddr =
            tmem + (static_cast<uint32_t>(lg * 32) << 16) + acc * BN + half * HB;
        // 8 epilogue warps double-buffer the TMEM loads (the next chunk's
        // load overlaps this chunk's math); 16 warps hide the latency with
        // each other and keep the 32 registers (their budget is 112)
        constexpr bool kTmemDB = EW == 8;
        uint32_t rbuf[kTmemDB ? 2 : 1][32];
        tmem_ld32_async(taddr, rbuf[0]);
        tmem_wait();
        if (HB == 32) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) release_acc(acc);
        }
#pragma unroll
        for (int c0 = 0; c0 < HB; c0 += 32) {
          uint32_t (&r)[32] = rbuf[kTmemDB ? (c0 / 32) & 1 : 0];
          if constexpr (kTmemDB) {
            // next chunk's TMEM load overlaps this chunk's math
            if (c0 + 32 < HB) tmem_ld32_async(taddr + c0 + 32, rbuf[((c0 / 32) + 1) & 1]);
          } else if (c0 > 0) {
            tmem_ld32_async(taddr + c0, rbuf[0]);
            tmem_wait();
            if (c0 + 32 >= HB) {  // last TMEM load landed: free the accumulator
              tc_fence_before();
              __syncwarp();
              if (lane == 0) release_acc(acc);
            }
          }
          // the next item's output row (its tile was loaded at this item's start)
          if (c0 == 0 && has_nx) orow_nx = orow_of(t_nx);
          if (c0 + 32 >= HB && bias_smem && has_nx && lane < kBq) bias_nx = bias_at(t_nx, w_nx);
          const int n = n0 + c0;
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          if (has_bias) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 b = ldg_nc_v4(bias4 + (c0 + i) / 4);
              const float2 lo = f2_fma(make_float2(v[i], v[i + 1]), f2(1.f), make_float2(b.x, b.y));
              const float2 hi = f2_fma(make_float2(v[i + 2], v[i + 3]), f2(1.f), make_float2(b.z, b.w));
              v[i] = lo.x; v[i + 1] = lo.y; v[i + 2] = hi.x; v[i + 3] = hi.y;
            }
          }
          if (dense_out) {
            // MODE 1 stores its padding slots' rows unmasked: their x_s rows
            // are zero (prologue), so y1 = b1 gives finite F, F' that fwd2
            // drops and that meet zero g_y_s rows in the backward.  MODE 2
            // masks them: the fused gb1 column sums read the whole staged box,
            // including rows past the segment end
            const bool pad = orow < 0;
            const int hrow = lg * 32 + lane;  // this thread's row in the 128-row box
            const int swz = (hrow >> 1) & 3;  // TMA 64B swizzle: chunk ^= (row >> 1) & 3
            uint8_t* obox = bwd ? ybox(dchunk) : hstage + (dchunk % C::kOutBufs) * C::kOutBox;
            // MODE 1: the chunk's math (bias + F, F' packed to bf16) before
            // the box barrier, overlapping the previous store's smem read
            uint32_t o1[16], o2[16];
            if (!bwd) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                float2 f, df, x = make_float2(v[2 * i], v[2 * i + 1]);
                if (bias_smem) {  // uniform-address LDS: broadcast
                  const float2 b = *reinterpret_cast<const float2*>(gbias + c0 + 2 * i);
                  x = f2_fma(x, f2(1.f), b);
                }
                // activation fixed at compile time (MODE 1 instantiations)
                act_pair<ACT>(x, f, df);
                o1[i] = pack_bf16(df.x, df.y);
                o2[i] = pack_bf16(f.x, f.y);
              }
            }
            // (1) the store that last used this box has read its smem, and
            //     every thread is past the previous chunk's F'(y1) reads
            //     (MODE 2: the previous chunk's box is the slot the next F'
            //     load refills, so its store must have read it)
            if constexpr (kPW || kPW2) {
              // per-warp staging: this warp's 32-row slices of the group's
              // boxes, stored by its own lane 0 -- no group barrier per chunk
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              __syncwarp();
            } else {
              if (elect) {
                if constexpr (C::kOutBufs == 2 && !bwd)
                  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                else
                  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              }
              named_bar_sync(1 + half, 128);
            }
            if (bwd && y_issuer) y_issue_to(dchunk + kYRing);  // F'(y1) kYRing-1 chunks ahead
            uint4 dv[4];
            if (bwd) {  // this row's F'(y1) chunk from the staged box
              mbar_wait(ybar(dchunk), (dchunk / kYRing) & 1);
              const uint8_t* src = ybox(dchunk) + hrow * 64;
#pragma unroll
              for (int j = 0; j < 4; ++j)
                dv[j] = *reinterpret_cast<const uint4*>(src + ((j ^ swz) * 16));
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (!bwd) {
                // stash = (F'(y1), F(y1)): everything the backward needs
                *reinterpret_cast<uint4*>(obox + hrow * 64 + ((j ^ swz) * 16)) =
                    make_uint4(o1[4 * j], o1[4 * j + 1], o1[4 * j + 2], o1[4 * j + 3]);
                *reinterpret_cast<uint4*>(obox + 8192 + hrow * 64 + ((j ^ swz) * 16)) =
                    make_uint4(o2[4 * j], o2[4 * j + 1], o2[4 * j + 2], o2[4 * j + 3]);
              } else {
                // g_y1 = g_y2 * F'(y1)
                uint32_t a1[4];
                const __nv_bfloat16* yb = reinterpret_cast<const __nv_bfloat16*>(&dv[j]);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float2 g = f2_mul(make_float2(v[8 * j + 2 * i], v[8 * j + 2 * i + 1]),
                                          __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(yb)[i]));
                  a1[i] = pad ? 0u : pack_bf16(g.x, g.y);
                }
                *reinterpret_cast<uint4*>(obox + hrow * 64 + ((j ^ swz) * 16)) =
                    make_uint4(a1[0], a1[1], a1[2], a1[3]);
              }
            }
            // (2) box complete -> one TMA store per output (or per valid
            //     32-row slice at a segment end), one bulk group per chunk
            fence_async_smem();
            if constexpr (kPW2) {
              __syncwarp();
              if (lane == 0 && lg * 32 < rows_here && !(kDbg && (p.dbg_noload & 2))) {
                if (p.l2hint)
                  tma_store_2d_hint(&p.tmO1s, obox + lg * 2048, n, qbase + lg * 32,
                                    policy_evict_last());
                else
                  tma_store_2d(&p.tmO1s, obox + lg * 2048, n, qbase + lg * 32);
                bulk_commit();
              }
            } else if constexpr (kPW) {
              __syncwarp();
              if (lane == 0 && lg * 32 < rows_here && !(kDbg && (p.dbg_noload & 2))) {
                const int row = qbase + lg * 32;
                if (p.l2hint) {
                  tma_store_2d_hint(&p.tmO1s, obox + lg * 2048, n, row, policy_evict_first());
                  tma_store_2d_hint(&p.tmO2s, obox + 8192 + lg * 2048, n, row, policy_evict_last());
                } else {
                  tma_store_2d(&p.tmO1s, obox + lg * 2048, n, row);
                  tma_store_2d(&p.tmO2s, obox + 8192 + lg * 2048, n, row);
                }
                bulk_commit();
              }
            } else {
            named_bar_sync(1 + half, 128);
            if (elect && !(kDbg && (p.dbg_noload & 2))) {
              if (rows_here >= BM) {
                // L2 policy: what the NEXT kernel reads stays (MODE 1: F(y1)
                // for ESMM fwd2; MODE 2: g_y1 for ESTMM gW1 / ESMM gx), what
                // is read only much later goes first (MODE 1: F'(y1))
                if (p.l2hint) {
                  if (!bwd) {
                    tma_store_2d_hint(&p.tmO1, obox, n, qbase, policy_evict_first());
                    tma_store_2d_hint(&p.tmO2, obox + 8192, n, qbase, policy_evict_last());
                  } else {
                    tma_store_2d_hint(&p.tmO1, obox, n, qbase, policy_evict_last());
                  }
                } else {
                  tma_store_2d(&p.tmO1, obox, n, qbase);
                  if (!bwd) tma_store_2d(&p.tmO2, obox + 8192, n, qbase);
                }
              } else {
                for (int sl = 0; sl * 32 < rows_here; ++sl) {
                  tma_store_2d(&p.tmO1s, obox + sl * 2048, n, qbase + sl * 32);
                  if (!bwd) tma_store_2d(&p.tmO2s, obox + 8192 + sl * 2048, n, qbase + sl * 32);
                }
              }
              bulk_commit();
            }
            }  // !kPW
            if (bwd && p.colsum) {
              // fused gb1 (ESS of g_y1, es_ops.cpp:86-102): column sums of the
              // bf16 values this warp just staged (its own 32 rows, so only
              // __syncwarp ordering).  Lane (rsub, cq) reads 16-byte column
              // chunk cq of rows rsub + 8i (4 x LDS.128, conflict-free),
              // sums them in f32x2, reduces the 8 row groups by shuffles;
              // lanes 0..3 write this warp's 32 column sums: one
              // deterministic partial row per (tile, CTA, lane group).
              __syncwarp();
              const int cq = lane & 3, rsub = lane >> 2;
              float2 cs[4] = {f2(0.f), f2(0.f), f2(0.f), f2(0.f)};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int r = lg * 32 + rsub + 8 * i;
                const uint4 q4 = *reinterpret_cast<const uint4*>(obox + r * 64 +
                                                                 ((cq ^ ((r >> 1) & 3)) * 16));
                const uint32_t w4[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  cs[k] = f2_fma(make_float2(__uint_as_float(w4[k] << 16),
                                             __uint_as_float(w4[k] & 0xffff0000u)),
                                 f2(1.f), cs[k]);
              }
#pragma unroll
              for (int o = 4; o < 32; o <<= 1)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  cs[k].x += __shfl_xor_sync(0xffffffffu, cs[k].x, o);
                  cs[k].y += __shfl_xor_sync(0xffffffffu, cs[k].y, o);
                }
              if (lane < 4) {
                float* dst = p.colsum + ((static_cast<int64_t>(fdi.div(w)) * CG + rank) * 4 + lg) * N +
                             n + cq * 8;
                reinterpret_cast<float4*>(dst)[0] = make_float4(cs[0].x, cs[0].y, cs[1].x, cs[1].y);
                reinterpret_cast<float4*>(dst)[1] = make_float4(cs[2].x, cs[2].y, cs[3].x, cs[3].y);
              }
            }
            ++dchunk;
          } else {
            // fp32 rows scattered to token order: two 16-column halves through
            // a 2 KB per-warp staging tile (32 rows x 64 B, 16-byte chunks
            // XOR-swizzled by (row >> 1) & 3: conflict-free both ways), so a
            // store / reduction instruction covers 8 row segments of 64 B
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              __syncwarp();
#pragma unroll
              for (int j = 0; j < 4; ++j)
                *reinterpret_cast<float4*>(stg + lane * 64 + ((j ^ ((lane >> 1) & 3)) * 16)) =
                    make_float4(v[16 * h2 + 4 * j], v[16 * h2 + 4 * j + 1], v[16 * h2 + 4 * j + 2],
                                v[16 * h2 + 4 * j + 3]);
              __syncwarp();
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int rr = i * 8 + lane / 4, cc = lane % 4;
                const int orr = __shfl_sync(0xffffffffu, orow, rr);
                const float4 val =
                    *reinterpret_cast<const float4*>(stg + rr * 64 + ((cc ^ ((rr >> 1) & 3)) * 16));
                if (orr < 0 || (kDbg && (p.dbg_noload & 2))) continue;
                if (MODE == 0 && p.n_peer > 0) {
                  // fused reduce-scatter: the token's owner rank, over peer memory
                  const int owner = static_cast<int>(orr / p.peer_rows);
                  float* o = p.peer[owner] + (orr - owner * p.peer_rows) * N + n + 16 * h2 + cc * 4;
                  // system-scope atomics (several GPUs add into one owner row);
                  // ordering against the owner's reads: the epilogue's closing
                  // fence.sc.sys + hxm_peer_barrier (release / acquire, .sys)
                  red_add_v4_sys(o, val.x, val.y, val.z, val.w);
                  continue;
                }
                float* o = p.out_f32 + static_cast<int64_t>(orr) * N + n + 16 * h2 + cc * 4;
                if (p.epi == EPI_WRITE) {
                  *reinterpret_cast<float4*>(o) = val;
                } else if (p.epi == EPI_ACCUM) {
                  float4 c = *reinterpret_cast<float4*>(o);
                  c.x += val.x; c.y += val.y; c.z += val.z; c.w += val.w;
                  *reinterpret_cast<float4*>(o) = c;
                } else {
                  red_add_v4(o, val.x, val.y, val.z, val.w);
                }
              }
            }
          }
          if (kTmemDB && c0 + 32 < HB) {
            tmem_wait();
            if (c0 + 64 >= HB) {  // last TMEM load landed: free the accumulator
              tc_fence_before();
              __syncwarp();
              if (lane == 0) release_acc(acc);
            }
          }
        }
        // every warp of the group is past this item's last bias read (the
        // last chunk's barrier): stage the next item's bias
        if constexpr (kPW) {
          if (bias_smem && has_nx) named_bar_sync(1 + half, 128);
        }
        if (bias_smem && has_nx && lane < kBq) gbias[lg * kBq + lane] = bias_nx;
        t_cur = t_nx;
        orow_cur = orow_nx;
        if (warp == 2 && lane == 0) TRACE(ep_it, 5);
      } else {
        const int mt = rem / p.n_nt, nt = rem % p.n_nt;
        // first output row of this warp (CG = 2: this CTA's half of 256)
        const int m0 = mt * BM * CG + static_cast<int>(rank) * BM + lg * 32;
        const int n0 = nt * BN + half * HB;
        const bool split = t.flags & 1;
        const bool empty_seg = t.end <= t.begin;
        float* obase = p.est_out + static_cast<int64_t>(t.expert) * p.M * p.N;
        if constexpr (CG == 2) mbar_wait_cl(&tfull[acc], aph);
        else mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t taddr =
            tmem + (static_cast<uint32_t>(lg * 32) << 16) + acc * BN + half * HB;
#pragma unroll
        for (int c0 = 0; c0 < HB; c0 += 32) {
          uint32_t r[32];
          if (!empty_seg) {
            tmem_ld32(taddr + c0, r);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = 0u;
          }
          if (c0 + 32 == HB) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) release_acc(acc);
          }
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(stg + lane * 64 + ((j ^ ((lane >> 1) & 3)) * 16)) =
                  make_uint4(r[16 * h2 + 4 * j], r[16 * h2 + 4 * j + 1], r[16 * h2 + 4 * j + 2],
                             r[16 * h2 + 4 * j + 3]);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int rr = i * 8 + lane / 4, cc = lane % 4;
              const float4 val =
                  *reinterpret_cast<const float4*>(stg + rr * 64 + ((cc ^ ((rr >> 1) & 3)) * 16));
              if (m0 + rr >= p.M || (kDbg && (p.dbg_noload & 2))) continue;
              if (p.n_peer > 0) {
                // fused reduce-scatter of the weight gradient along H to the
                // shard owners: rows (peer_dim 0, gW2) or columns (1, gW1)
                const int64_t m = m0 + rr, n = n0 + c0 + 16 * h2 + cc * 4;
                const int64_t span = p.peer_rows;
                float* o;
                if (p.peer_dim == 0) {
                  const int owner = static_cast<int>(m / span);
                  o = p.peer[owner] + (t.expert * span + (m - owner * span)) * p.N + n;
                } else {
                  const int owner = static_cast<int>(n / span);
                  o = p.peer[owner] + (t.expert * static_cast<int64_t>(p.M) + m) * span +
                      (n - owner * span);
                }
                if (!empty_seg) red_add_v4_sys(o, val.x, val.y, val.z, val.w);
                continue;
              }
              float* o = obase + static_cast<int64_t>(m0 + rr) * p.N + n0 + c0 + 16 * h2 + cc * 4;
              if (split && !empty_seg) red_add_v4(o, val.x, val.y, val.z, val.w);
              else *reinterpret_cast<float4*>(o) = val;
            }
          }
        }
      }
      ++ep_it;
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
    if (lane == 0) bulk_wait0();  // this warp's TMA stores are complete
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();  // pair done with TMEM
  if constexpr (MODE == 0 || MODE == 3) {
    // peer reductions (ordered before this point by the barrier above) made
    // visible system-wide before the kernel ends; hxm_peer_barrier's .sys
    // release / acquire then orders them before the owners' reads
    if (threadIdx.x == 0 && p.n_peer > 0) asm volatile("fence.sc.sys;" ::: "memory");
  }
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(kTmemCols));
  }
}

template <int BN, int MODE, int CG = 1, int ACT = -1, int EW = 8>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
    umma_kernel(const __grid_constant__ UParams p) {
  umma_body<BN, MODE, CG, ACT, EW>(p, blockIdx.x / CG, gridDim.x / CG);
}

// ESFK (es_ops.cpp:210-247) as ONE persistent launch: clusters [0, split)
// walk the grad-x ESMM tiles (MODE 0, W read K-major as W^T), clusters
// [split, n) the grad-W ESTMM chunks (MODE 3) of the same expert-sorted
// operands -- the reference's combined work list, partitioned by cluster so
// each side keeps its own smem ring / TMEM pipeline.  (grad-b, the ESS part
// of the list, is fused into the operand gather that precedes this launch.)
template <int BN0, int BN3, int CG, int EW>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
    esfk_kernel(const __grid_constant__ UParams p0, const __grid_constant__ UParams p3,
                const int split) {
  const int cl = blockIdx.x / CG, ncl = gridDim.x / CG;
  if (cl < split) umma_body<BN0, 0, CG, -1, EW>(p0, cl, split);
  else umma_body<BN3, 3, CG, -1, EW>(p3, cl - split, ncl - split);
}

// ----------------------------------------------------------- host side ---
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// bf16 tensor of `rank` dims (dims[0] innermost, element counts), row pitch
// strides in bytes for dims 1.., box sizes, 128B (default) or 64B swizzle,
// OOB -> zeros.
bool make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
              const uint64_t* strides_bytes, const uint32_t* box,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeFn enc = encoder();
  if (!enc) return false;
  cuuint64_t gd[5], gs[4];
  cuuint32_t bx[5], es[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
  }
  for (int i = 0; i + 1 < rank; ++i) gs[i] = strides_bytes[i];
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), gd, gs,
                   bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int pick_bn(int64_t n) {
  for (int bn : {256, 192, 128, 64})
    if (n % bn == 0) return bn;
  return 0;
}
// CTA-pair tiles: an MN-major B half must be whole swizzle atoms -- 64
// columns (128B swizzle), or 32 columns with 64B-swizzled boxes (BN = 192)
int pick_bn2(int64_t n, bool b_mn) {
  static const int bn_max = [] {  // HXM_BN2_MAX: experiment override
    const char* e = std::getenv("HXM_BN2_MAX");
    return e ? std::atoi(e) : 256;
  }();
  for (int bn : {256, 192, 128, 64})
    if (bn <= bn_max && n % bn == 0 && (!b_mn || bn >= 128)) return bn;
  return 0;
}
bool bn2_sw64(int bn, bool b_mn) { return b_mn && (bn / 2) % 64 != 0; }

unsigned long long* g_trace = nullptr;
unsigned long long* trace_buffer_for(const char* label) {
  const char* want = std::getenv("HXM_TRACE");
  if (!want || !label || std::strcmp(want, label) != 0) return nullptr;
  if (!g_trace) {
    cudaMalloc(&g_trace, 148 * 64 * 8 * sizeof(unsigned long long));
  }
  cudaMemset(g_trace, 0, 148 * 64 * 8 * sizeof(unsigned long long));
  return g_trace;
}

template <int BN, int MODE, int CG, int ACT = -1, int EW = 8>
hxm_status launch_bn_ew(const UParams& prm_in, int max_work, cudaStream_t st) {
  UParams prm = prm_in;
  prm.trace = kTrace ? trace_buffer_for(prm_in.label) : nullptr;
  {
    static const bool hint = [] {
      const char* e = std::getenv("HXM_L2HINT");
      return !(e && e[0] == '0');
    }();
    prm.l2hint = hint;
  }
  // debug decomposition (HXM_DEBUG_NOLOAD bits: 1 = no operand loads, 2 = no
  // epilogue stores, 4 = no MMAs); results are garbage, timing only
  if (kDbg) { const char* e = std::getenv("HXM_DEBUG_NOLOAD"); prm.dbg_noload = e ? std::atoi(e) : 0; }
  using C = Cfg<BN, CG, MODE, EW>;
  auto kern = umma_kernel<BN, MODE, CG, ACT, EW>;
  constexpr int kThreads = 64 + 32 * EW;
  static bool attr_set[64] = {false};  // kernel attributes are per device
  int dev = 0;
  HXM_TRY_CUDA(cudaGetDevice(&dev));
  dev = dev < 64 ? dev : 63;
  if (!attr_set[dev]) {
    HXM_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr_set[dev] = true;
  }
  const int sms = sm_count();
  if (sms <= 0) return invalid_arg("tcgen05 path: no CUDA device");
  // persistent: one CTA (CG = 1) or CTA pair (CG = 2) per SM (pair)
  const int grid = std::max(1, std::min(sms / CG, max_work)) * CG;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  // programmatic dependent launch: this grid's CTAs may start (barrier
  // init, TMEM alloc, tensor-map prefetch) while the previous kernel in the
  // stream drains; griddepcontrol.wait in the kernel orders the data
  if (pdl_on()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if constexpr (CG == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  HXM_TRY_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

// 16 epilogue warps where epi_warps() asks for them (HXM_EPI16=0: always 8)
bool rev_on() {
  static const bool on = [] {
    const char* e = std::getenv("HXM_REVERSE");
    return !(e && e[0] == '0');
  }();
  return on;
}

int epi16_mode() {  // HXM_EPI16: 0 = never, 2 = always, default = short K only
  static const int m = [] {
    const char* e = std::getenv("HXM_EPI16");
    return e ? std::atoi(e) : 1;
  }();
  return m;
}
template <int BN, int MODE, int CG, int ACT = -1>
hxm_status launch_bn(const UParams& prm, int max_work, cudaStream_t st) {
  // only where the epilogue bounds the kernel: short K (<= 512, e.g. c2's
  // D = 384); at long K the MMA bounds it and 8 warps keep more ring stages
  if constexpr (epi_warps(BN, MODE) == 16) {
    const int m = epi16_mode();
    if constexpr (MODE == 3) {
      // ESTMM: the store-heavy epilogue (a full fp32 gW tile per item) bounds
      // items with few tokens (skewed routing); neutral for the others
      if (m != 0) return launch_bn_ew<BN, MODE, CG, ACT, 16>(prm, max_work, st);
    } else if (m == 2 || (m == 1 && prm.K <= 512)) {
      return launch_bn_ew<BN, MODE, CG, ACT, 16>(prm, max_work, st);
    }
  }
  return launch_bn_ew<BN, MODE, CG, ACT, 8>(prm, max_work, st);
}

template <int MODE, int CG, int ACT = -1>
hxm_status launch_bn_any(int bn, const UParams& prm, int max_work, cudaStream_t st) {
  switch (bn) {
    case 256: return launch_bn<256, MODE, CG, ACT>(prm, max_work, st);
    case 192: return launch_bn<192, MODE, CG, ACT>(prm, max_work, st);
    case 128: return launch_bn<128, MODE, CG, ACT>(prm, max_work, st);
    default: return launch_bn<64, MODE, CG, ACT>(prm, max_work, st);
  }
}
// the forward activation epilogue is specialised per activation
template <int CG>
hxm_status launch_fwd_act(int act, int bn, const UParams& prm, int max_work, cudaStream_t st) {
  if (act == HXM_ACT_GELU) return launch_bn_any<1, CG, HXM_ACT_GELU>(bn, prm, max_work, st);
  if (act == HXM_ACT_RELU) return launch_bn_any<1, CG, HXM_ACT_RELU>(bn, prm, max_work, st);
  return launch_bn_any<1, CG, HXM_ACT_IDENTITY>(bn, prm, max_work, st);
}

// rows of the tensor behind a row map: gathered sources are bounded by the
// largest valid row (n_rows), dense sorted buffers by the padded bound.

// tensor maps and epilogue parameters of an ESMM launch (CG, bn chosen by the caller)
hxm_status prep_esmm(const EsmmArgs& a, const int CG, const int bn, UParams& prm_out) {
  const bool gather = a.amap.kind != MAP_DENSE;
  UParams& prm = prm_out;
  prm = UParams{};
  // A: gathered token rows (n_rows = a_rows) or the dense sorted stash
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(a.d1), static_cast<uint64_t>(a.a_rows)};
    const uint64_t strides[1] = {static_cast<uint64_t>(a.d1) * 2};
    const uint32_t box[2] = {64, gather ? 1u : 128u};
    if (!make_map(&prm.tmA, a.a, 2, dims, strides, box))
      return invalid_arg("umma_esmm: cannot encode the A tensor map");
  }
  // B: W[e] (E x d1 x d2, MN-major) or W^T use (E x d2 x d1, K-major).
  // Shard-major weights (a.w_shards = P > 1): the split H axis (K when
  // a.w_split_k, else N) is [P][E][..h..], one more map dimension (the shard)
  // outermost; a box never straddles two shards (h % 64 == 0 for K, h % the
  // CTA's B width for N -- checked here).
  {
    const int64_t E = a.n_experts;
    const int64_t P = a.w_shards > 1 ? a.w_shards : 1;
    const bool sk = P > 1 && a.w_split_k, sn = P > 1 && !a.w_split_k;
    const int64_t hk = sk ? a.d1 / P : a.d1;  // K rows per shard (or all)
    const int64_t hn = sn ? a.d2 / P : a.d2;  // N columns per shard (or all)
    if (P > 1) {
      const int64_t hsplit = sk ? a.d1 : a.d2;
      if (hsplit % P != 0 || (hsplit / P) % 64 != 0 || (sn && (hsplit / P) % (bn / CG) != 0))
        return invalid_arg("umma_esmm: shard-major weights need H / P a multiple of 64 and of "
                           "the CTA's B tile width");
      prm.w_shard_h = static_cast<int>(hsplit / P);
      prm.w_shard_k = sk ? 1 : 0;
    }
    if (!a.w_trans) {
      // (atom column, k row, atom chunk, expert[, shard]): one box carries
      // every swizzle-atom column chunk of this CTA's B for a k-block
      const bool sw64 = CG == 2 && bn2_sw64(bn, true);
      const uint64_t bw = sw64 ? 32 : 64;
      const uint64_t dims[5] = {bw, static_cast<uint64_t>(hk), static_cast<uint64_t>(hn) / bw,
                                static_cast<uint64_t>(E), static_cast<uint64_t>(P)};
      const uint64_t strides[4] = {static_cast<uint64_t>(hn) * 2, bw * 2,
                                   static_cast<uint64_t>(hk * hn) * 2,
                                   static_cast<uint64_t>(E * hk * hn) * 2};
      const uint32_t box[5] = {static_cast<uint32_t>(bw), 64,
                               static_cast<uint32_t>((bn / CG) / static_cast<int>(bw)), 1, 1};
      if (!make_map(&prm.tmB, a.w, P > 1 ? 5 : 4, dims, strides, box,
                    sw64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
        return invalid_arg("umma_esmm: cannot encode the W tensor map");
      prm.b_sw64 = sw64;
    } else {
      // (k, n row, expert[, shard]) of W stored N x K per expert
      const uint64_t dims[4] = {static_cast<uint64_t>(hk), static_cast<uint64_t>(hn),
                                static_cast<uint64_t>(E), static_cast<uint64_t>(P)};
      const uint64_t strides[3] = {static_cast<uint64_t>(hk) * 2,
                                   static_cast<uint64_t>(hk * hn) * 2,
                                   static_cast<uint64_t>(E * hk * hn) * 2};
      const uint32_t box[4] = {64, static_cast<uint32_t>(bn / CG), 1, 1};  // this CTA's B rows
      if (!make_map(&prm.tmB, a.w, P > 1 ? 4 : 3, dims, strides, box))
        return invalid_arg("umma_esmm: cannot encode the W^T tensor map");
    }
  }
  prm.amap = a.amap;
  prm.a_gather = gather;
  prm.b_kmajor = a.w_trans;
  prm.K = static_cast<int>(a.d1);
  prm.N = static_cast<int>(a.d2);
  prm.n_nt = static_cast<int>(a.d2 / bn);
  prm.n_mt = 1;
  prm.tiles = a.tiles;
  prm.n_tiles = a.n_tiles;
  prm.label = a.label;
  prm.reverse = a.reverse && rev_on();
  if (a.peer) {
    if (a.epi != EPI_ATOMIC || a.peer->n_ranks < 1 || a.peer->n_ranks > HXM_MAX_PEERS ||
        a.peer->rows_per_rank < 1)
      return invalid_arg("esmm: peer rows need the reduction epilogue and 1..8 ranks");
    prm.n_peer = a.peer->n_ranks;
    prm.peer_rows = a.peer->rows_per_rank;
    for (int r = 0; r < prm.n_peer; ++r) prm.peer[r] = a.peer->ptrs[r];
  }
  prm.epi = a.epi;
  prm.act = a.act;
  prm.n_experts = static_cast<int>(a.n_experts);
  {
    // stream-K tail for the reduction epilogue (fwd2 / gx), HXM_STREAMK=1:
    // off by default -- a split tail item adds a third fp32 partial to its y /
    // g_x rows, so with k = 2 the result would no longer be bit-reproducible
    // (two addends onto zero commute exactly), and the measured gain is small
    // (profiles/r2_notes.md)
    static const bool sk = [] {
      const char* e = std::getenv("HXM_STREAMK");
      return e && e[0] == '1';
    }();
    prm.stream_k = (sk && a.epi == EPI_ATOMIC) ? 1 : 0;
  }
  prm.bias_shard_h = a.epi == EPI_FWD_ACT && a.w_shards > 1 ? static_cast<int>(a.d2 / a.w_shards) : 0;
  prm.bias = a.bias;
  prm.out_f32 = a.out_f32;
  prm.omap = a.omap;
  prm.out1 = a.out1;
  prm.out2 = a.out2;
  prm.y1s = a.y1s;
  prm.colsum = a.epi == EPI_BWD_ACT ? a.colsum : nullptr;
  if (a.epi == EPI_FWD_ACT || a.epi == EPI_BWD_ACT) {
    // dense bf16 stash outputs (same row space as the dense A operand):
    // 32 x 32 boxes stored by TMA from the epilogue's 64B-swizzled staging
    const uint64_t dims[2] = {static_cast<uint64_t>(a.d2), static_cast<uint64_t>(a.a_rows)};
    const uint64_t strides[1] = {static_cast<uint64_t>(a.d2) * 2};
    const uint32_t box[2] = {32, 128}, box_s[2] = {32, 32};
    const auto sw = CU_TENSOR_MAP_SWIZZLE_64B;
    bool ok = make_map(&prm.tmO1, a.out1, 2, dims, strides, box, sw) &&
              make_map(&prm.tmO1s, a.out1, 2, dims, strides, box_s, sw);
    if (a.epi == EPI_FWD_ACT)
      ok = ok && make_map(&prm.tmO2, a.out2, 2, dims, strides, box, sw) &&
           make_map(&prm.tmO2s, a.out2, 2, dims, strides, box_s, sw);
    else  // MODE 2: the F'(y1) stash, 32 x 128 boxes (and 32 x 32 per-warp slices in tmO2s)
      ok = ok && make_map(&prm.tmY, a.y1s, 2, dims, strides, box, sw) &&
           make_map(&prm.tmO2s, a.y1s, 2, dims, strides, box_s, sw);
    if (!ok) return invalid_arg("umma_esmm: cannot encode the stash tensor maps");
  }
  return HXM_OK;
}

// tensor maps and epilogue parameters of an ESTMM launch
hxm_status prep_estmm(const EstmmArgs& a, const int CG, const int bn, UParams& prm_out) {
  const bool ga = a.m1.kind != MAP_DENSE, gb = a.m2.kind != MAP_DENSE;
  UParams& prm = prm_out;
  prm = UParams{};
  // dense operands: 3D views (atom column, row, atom chunk) so one box
  // carries every column chunk of a k-block; gathered ones: 2D row maps
  {
    bool ok;
    if (ga) {
      const uint64_t dims[2] = {static_cast<uint64_t>(a.d1), static_cast<uint64_t>(a.x1_rows)};
      const uint64_t strides[1] = {static_cast<uint64_t>(a.d1) * 2};
      const uint32_t box[2] = {64, 1};
      ok = make_map(&prm.tmA, a.x1, 2, dims, strides, box);
    } else {
      const uint64_t dims[3] = {64, static_cast<uint64_t>(a.x1_rows),
                                static_cast<uint64_t>(a.d1) / 64};
      const uint64_t strides[2] = {static_cast<uint64_t>(a.d1) * 2, 128};
      const uint32_t box[3] = {64, 64, BM / 64};
      ok = make_map(&prm.tmA, a.x1, 3, dims, strides, box);
    }
    if (!ok) return invalid_arg("umma_estmm: cannot encode the X1 tensor map");
  }
  {
    const bool sw64 = CG == 2 && bn2_sw64(bn, true);
    bool ok;
    if (gb) {
      const uint64_t dims[2] = {static_cast<uint64_t>(a.d2), static_cast<uint64_t>(a.x2_rows)};
      const uint64_t strides[1] = {static_cast<uint64_t>(a.d2) * 2};
      const uint32_t box[2] = {64, 1};
      ok = make_map(&prm.tmB, a.x2, 2, dims, strides, box);
    } else {
      const uint64_t bw = sw64 ? 32 : 64;
      const uint64_t dims[3] = {bw, static_cast<uint64_t>(a.x2_rows),
                                static_cast<uint64_t>(a.d2) / bw};
      const uint64_t strides[2] = {static_cast<uint64_t>(a.d2) * 2, bw * 2};
      const uint32_t box[3] = {static_cast<uint32_t>(bw), 64,
                               static_cast<uint32_t>((bn / CG) / static_cast<int>(bw))};
      ok = make_map(&prm.tmB, a.x2, 3, dims, strides, box,
                    sw64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
    }
    if (!ok) return invalid_arg("umma_estmm: cannot encode the X2 tensor map");
    prm.b_sw64 = sw64;
  }
  prm.amap = a.m1;
  prm.bmap = a.m2;
  prm.a_gather = ga;
  prm.b_gather = gb;
  prm.M = static_cast<int>(a.d1);
  prm.N = static_cast<int>(a.d2);
  prm.n_mt = static_cast<int>(ceil_div(a.d1, BM * CG));
  prm.n_nt = static_cast<int>(a.d2 / bn);
  prm.tiles = a.tiles;
  prm.n_tiles = a.n_tiles;
  prm.est_out = a.out;
  prm.label = a.label;
  prm.reverse = a.reverse && rev_on();
  if (a.peer) {  // gW reduce-scattered to the owners' H-shards
    const int64_t span = a.peer->rows_per_rank, ext = a.peer_dim == 0 ? a.d1 : a.d2;
    if (a.peer->n_ranks < 1 || a.peer->n_ranks > HXM_MAX_PEERS || span < 1 ||
        span * a.peer->n_ranks != ext || span % 4 != 0)
      return invalid_arg("estmm: peer shards must split the H extent evenly (multiple of 4)");
    prm.n_peer = a.peer->n_ranks;
    prm.peer_rows = span;
    prm.peer_dim = a.peer_dim;
    for (int r = 0; r < prm.n_peer; ++r) prm.peer[r] = a.peer->ptrs[r];
  }
  return HXM_OK;
}

}  // namespace
}  // namespace hxm
