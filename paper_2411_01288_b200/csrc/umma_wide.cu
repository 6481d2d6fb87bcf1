// umma_wide.cu -- the K = H reduction GEMMs of the layer (ESMM fwd2:
// y += F(y1) W2 + b2, and ESMM gx: g_x += g_y1 W1^T; es_ops.cpp:47-81 in
// accumulate mode over the k choices) on CTA pairs that own the WHOLE
// 256 x 384 output tile when the output width is 384 (c2's D).
//
// Why: with 256 x 192 tiles (umma.cu) every A row block (the H-wide stash)
// is streamed from L2 twice, once per N-half, and the kernels sit at the L2
// throughput cap with the operand ring starved (profiles/r1b_notes.md 4, 15,
// 23; the LTS cap is path-independent, B300_MICROARCH.md).  One pair per
// 256 x 384 tile reads A once: per 64-deep k-block a CTA loads 16 KB of A +
// 24 KB of B for two MMAs (N = 256 and N = 128, both cta_group::2) instead
// of 2 x (16 + 12) KB -- 29 % fewer L2 bytes per FLOP.
//
// TMEM: the tile needs 384 accumulator columns, so the accumulator cannot be
// double-buffered whole.  It is split: the N = 256 part always lives in
// columns [0, 256), the N = 128 part alternates between [256, 384) and
// [384, 512).  The epilogue drains the 256-column part first and releases
// it, so the next tile's MMAs start while the epilogue still drains the
// 128-column part of the previous one.
//
// Column mapping: CTA r loads B columns [192 r, 192 r + 192) as one box;
// MMA1 (N = 256) covers CTA0's first 128 and CTA1's first 128 columns, MMA2
// (N = 128) the last 64 of each.  Epilogue column group g (4 warps, one per
// TMEM lane group) drains lo columns [128 g, 128 g + 128) and hi columns
// [64 g, 64 g + 64), i.e. exactly the global columns [192 g, 192 g + 192).
#include "umma_impl.cuh"

namespace hxm {
namespace {

constexpr int kWideN = 384;                       // output columns per tile
constexpr int kWideBHalf = kWideN / 2;            // B columns per CTA
constexpr int kWideBBytes = kWideBHalf * BK * 2;  // 24 KB
constexpr int kWideStage = kABytes + kWideBBytes; // 40 KB
constexpr int kWideEW = 8;                        // epilogue warps per CTA
constexpr int kWideStaging = kWideEW * 2048;
constexpr int kWideStages = (232448 - 1024 - 256 - kWideStaging) / kWideStage;  // 5
constexpr int kWideSmem = kWideStages * kWideStage + kWideStaging + 1024 + 256;
constexpr int kWideThreads = 64 + 32 * kWideEW;

// One 64-deep k-block of the wide tile: four K = 16 steps of MMA1 (N = 256,
// accumulator d_lo) and MMA2 (N = 128, accumulator d_hi), then the commit
// that frees the stage (multicast to both CTAs of the pair).
__device__ __forceinline__ void wide_kblock(uint32_t d_lo, uint32_t d_hi, uint32_t a_lo,
                                            uint32_t a_hi, uint32_t a_step, uint32_t b_lo,
                                            uint32_t b_hi, uint32_t b_step, uint32_t b2_off,
                                            uint32_t idesc1, uint32_t idesc2, uint32_t first,
                                            uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred p0, p1;\n"
      ".reg .b64 da, db, db2;\n"
      ".reg .b32 al, bl, b2l;\n"
      "setp.ne.b32 p0, %11, 0;\n"
      "setp.eq.b32 p1, %11, %11;\n"
      "mov.b32 al, %2;\n"
      "mov.b32 bl, %5;\n"
      "add.u32 b2l, %5, %8;\n"
      "mov.b64 da, {al, %3};\n"
      "mov.b64 db, {bl, %6};\n"
      "mov.b64 db2, {b2l, %6};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %9, p0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%1], da, db2, %10, p0;\n"
      "add.u32 al, al, %4;\n"
      "add.u32 bl, bl, %7;\n"
      "add.u32 b2l, b2l, %7;\n"
      "mov.b64 da, {al, %3};\n"
      "mov.b64 db, {bl, %6};\n"
      "mov.b64 db2, {b2l, %6};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %9, p1;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%1], da, db2, %10, p1;\n"
      "add.u32 al, al, %4;\n"
      "add.u32 bl, bl, %7;\n"
      "add.u32 b2l, b2l, %7;\n"
      "mov.b64 da, {al, %3};\n"
      "mov.b64 db, {bl, %6};\n"
      "mov.b64 db2, {b2l, %6};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %9, p1;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%1], da, db2, %10, p1;\n"
      "add.u32 al, al, %4;\n"
      "add.u32 bl, bl, %7;\n"
      "add.u32 b2l, b2l, %7;\n"
      "mov.b64 da, {al, %3};\n"
      "mov.b64 db, {bl, %6};\n"
      "mov.b64 db2, {b2l, %6};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %9, p1;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%1], da, db2, %10, p1;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%12], %13;\n"
      "}\n" ::"r"(d_lo),
      "r"(d_hi), "r"(a_lo), "r"(a_hi), "r"(a_step), "r"(b_lo), "r"(b_hi), "r"(b_step),
      "r"(b2_off), "r"(idesc1), "r"(idesc2), "r"(first ? 0u : 1u), "r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

__global__ void __launch_bounds__(kWideThreads, 1)
    umma_wide_kernel(const __grid_constant__ UParams p) {
  constexpr int CG = 2;
  uint32_t rank = 0;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int cluster = blockIdx.x / CG, n_clusters = gridDim.x / CG;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* staging = smem + kWideStages * kWideStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + kWideStaging);
  uint64_t* empty = full + kWideStages;
  uint64_t* tfull = empty + kWideStages;   // [2] by tile parity
  uint64_t* tempty_lo = tfull + 2;         // [1] the N = 256 accumulator
  uint64_t* tempty_hi = tempty_lo + 1;     // [2] the two N = 128 slots
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_hi + 2);
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0);  // warp-uniform
  const int lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWideStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty_hi[a], kWideEW * CG);
    }
    mbar_init(tempty_lo, kWideEW * CG);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  const uint32_t full_lead = mapa0(smem_u32(full));
  const uint32_t tlo_lead = mapa0(smem_u32(tempty_lo));
  const uint32_t thi_lead = mapa0(smem_u32(tempty_hi));

  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int total = *p.n_tiles;  // one work item per 256-row tile (N = 384 whole)
  auto wmap = [&](int wl) { return p.reverse ? total - 1 - wl : wl; };
  const int nk = p.K / BK;

  if (warp == 0) {
    // ================================ TMA producer =======================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmB) : "memory");
    }
    int s = 0;
    uint32_t ph = 0;
    for (int wl = cluster; wl < total; wl += n_clusters) {
      const SegTile t = p.tiles[wmap(wl)];
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * kWideStage;
        uint8_t* sb = sa + kABytes;
        if (elect_one()) {
          const uint32_t fb = full_lead + 8u * s;
          if (rank == 0) mbar_arrive_tx(&full[s], 2 * kWideStage);
          tma_2d_cg2(sa, &p.tmA, fb, kb * BK, t.begin + static_cast<int>(rank) * BM);
          load_w_box<2>(p, sb, nullptr, fb, kb * BK, static_cast<int>(rank) * kWideBHalf,
                        t.expert);
        }
        __syncwarp();
        if (++s == kWideStages) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ==========================
    if (rank == 0) {
      const bool b_mn = !p.b_kmajor;
      const uint32_t idesc1 = idesc_bf16(256, 0, b_mn ? 1 : 0, BM * CG);
      const uint32_t idesc2 = idesc_bf16(128, 0, b_mn ? 1 : 0, BM * CG);
      const uint32_t base = smem_u32(smem);
      const uint64_t da0 = sdesc(base, 16, 1024);
      const uint64_t db0 = b_mn ? sdesc(base + kABytes, 8192, 1024) : sdesc(base + kABytes, 16, 1024);
      const uint32_t a_lo = static_cast<uint32_t>(da0), a_hi = static_cast<uint32_t>(da0 >> 32);
      const uint32_t b_lo = static_cast<uint32_t>(db0), b_hi = static_cast<uint32_t>(db0 >> 32);
      const uint32_t a_step = 2u, b_step = b_mn ? 128u : 2u;
      // MMA2's B: the CTA's last 64 columns (MN-major: the third 8 KB atom
      // column chunk) or rows 128..191 (K-major): 16 KB in, in 16-B units
      const uint32_t b2_off = 16384u >> 4;
      constexpr uint32_t kStageUnits = kWideStage >> 4;
      int s = 0, it = 0;
      uint32_t ph = 0, lo_ph = 0, hi_ph[2] = {0, 0};
      for (int wl = cluster; wl < total; wl += n_clusters, ++it) {
        const int hs = it & 1;
        mbar_wait(tempty_lo, lo_ph ^ 1);
        mbar_wait(&tempty_hi[hs], hi_ph[hs] ^ 1);
        lo_ph ^= 1;
        hi_ph[hs] ^= 1;
        tc_fence_after();
        const uint32_t d_lo = tmem, d_hi = tmem + 256 + 128 * hs;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t so = static_cast<uint32_t>(s) * kStageUnits;
          if (elect_one())
            wide_kblock(d_lo, d_hi, a_lo + so, a_hi, a_step, b_lo + so, b_hi, b_step, b2_off,
                        idesc1, idesc2, kb == 0, &empty[s]);
          __syncwarp();
          if (++s == kWideStages) { s = 0; ph ^= 1; }
        }
        if (elect_one()) umma_commit_cg2(&tfull[it & 1]);
        __syncwarp();
      }
    }
    __syncwarp();
  } else {
    // ================================ epilogue ============================
    const int lg = warp & 3;
    const int g = (warp - 2) / 4;  // column group: global columns [192 g, 192 g + 192)
    uint8_t* stg = staging + (warp - 2) * 2048;
    const int N = p.N;
    uint32_t tf_ph[2] = {0, 0};
    int it = 0;
    for (int wl = cluster; wl < total; wl += n_clusters, ++it) {
      const int w = wmap(wl);
      const SegTile t = p.tiles[w];
      const int hs = it & 1;
      // this lane's token-order output row
      int orow = -1;
      {
        const int qq = t.begin + static_cast<int>(rank) * BM + lg * 32 + lane;
        if (qq < t.end) orow = p.omap(qq);
      }
      const float* bias = p.bias ? p.bias + static_cast<int64_t>(t.expert) * N : nullptr;
      mbar_wait(&tfull[it & 1], tf_ph[it & 1]);
      tf_ph[it & 1] ^= 1;
      tc_fence_after();
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(lg * 32) << 16);
      // one 32-column chunk (TMEM registers r) -> bias -> fp32 rows scattered
      // to token order through the per-warp swizzled staging tile (8 row
      // segments of 64 B per reduction instruction)
      auto emit = [&](const uint32_t (&r)[32], const int gcol) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (bias) {
          const float4* b4 = reinterpret_cast<const float4*>(bias + gcol);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b = ldg_nc_v4(b4 + i / 4);
            v[i] += b.x; v[i + 1] += b.y; v[i + 2] += b.z; v[i + 3] += b.w;
          }
        }
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
            if (orr < 0) continue;
            const int n = gcol + 16 * h2 + cc * 4;
            if (p.n_peer > 0) {
              const int owner = static_cast<int>(orr / p.peer_rows);
              float* o = p.peer[owner] + (orr - owner * p.peer_rows) * N + n;
              red_add_v4_sys(o, val.x, val.y, val.z, val.w);
            } else {
              red_add_v4(p.out_f32 + static_cast<int64_t>(orr) * N + n, val.x, val.y, val.z,
                         val.w);
            }
          }
        }
      };
      // the lo accumulator (4 chunks) is loaded into registers at once and
      // released before any of it is reduced, so the next tile's MMAs start
      // after ~4 TMEM loads instead of after the whole lo epilogue
      {
        uint32_t rl[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32_async(lane_base + 128 * g + 32 * c, rl[c]);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cl(tlo_lead);
#pragma unroll
        for (int c = 0; c < 4; ++c) emit(rl[c], 192 * g + 32 * c);
      }
      {
        uint32_t rh[2][32];
#pragma unroll
        for (int c = 0; c < 2; ++c)
          tmem_ld32_async(lane_base + 256 + 128 * hs + 64 * g + 32 * c, rh[c]);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cl(thi_lead + 8u * hs);
#pragma unroll
        for (int c = 0; c < 2; ++c) emit(rh[c], 192 * g + 128 + 32 * c);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (threadIdx.x == 0 && p.n_peer > 0) asm volatile("fence.sc.sys;" ::: "memory");
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}


// ---------------------------------------------------------------------------
// ESTMM (es_ops.cpp:106-128) with the same whole-tile scheme: out[e] (M x 384)
// = X1^T X2 over one K chunk of the expert's positions, a CTA pair per 256
// rows of M (each CTA 128), the whole N = 384 in one accumulator (N = 256 +
// N = 128 MMAs, TMEM split as above).  Against 256 x 192 pair tiles the X1
// rows (A, MN-major) are streamed once per M tile instead of twice, and
// against the single-CTA 128 x 256 tiles gW1 needs (M = D_i = 384 does not
// tile in pairs) both operands are read once per 256 x 384 tile: computing
// gW1 as (g_y1^T x_s)^T puts H on M, and the transposed store is coalesced
// along the TMEM lanes (consecutive h).
// Work item w: K chunk w / n_mt, M tile w % n_mt.  Empty chunks write zeros;
// split chunks (flags & 1) reduce with red.add into the zeroed slices.
// one 32-column chunk (output columns gcol..+31) of this lane's row m of a
// whole-tile ESTMM item; an empty chunk (no positions) stores zeros.  `wrow`
// = the out[e] slice offset of the warp's first row (TRANS: of row m);
// offsets inside one expert's slice fit 32 bits.
template <bool TRANS>
__device__ __forceinline__ void est_emit(const UParams& p, const uint32_t (&r)[32], const int gcol,
                                         float* wbase, const int ld, uint8_t* stg,
                                         const int lane, const bool split, const bool empty_seg) {
  if constexpr (TRANS) {
    // out[e] is N x M (row length ld = M): for each column the warp's 32
    // lanes write 32 consecutive m -- one coalesced 128-byte segment per store
    float* o = wbase + gcol * ld;
    if (split || p.n_peer > 0) {
      if (empty_seg) return;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (p.n_peer > 0)
          asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(o + j * ld),
                       "f"(__uint_as_float(r[j])) : "memory");
        else
          asm volatile("red.global.add.f32 [%0], %1;" ::"l"(o + j * ld),
                       "f"(__uint_as_float(r[j])) : "memory");
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) o[j * ld] = empty_seg ? 0.f : __uint_as_float(r[j]);
    }
  } else {
    // out[e] is M x N (row length ld = N): rows through the per-warp
    // swizzled staging tile (8 row segments of 64 B per instruction)
    if (empty_seg && (split || p.n_peer > 0)) return;
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
        float4 val =
            *reinterpret_cast<const float4*>(stg + rr * 64 + ((cc ^ ((rr >> 1) & 3)) * 16));
        float* o = wbase + rr * ld + gcol + 16 * h2 + cc * 4;
        if (p.n_peer > 0) red_add_v4_sys(o, val.x, val.y, val.z, val.w);
        else if (split) red_add_v4(o, val.x, val.y, val.z, val.w);
        else {
          if (empty_seg) val = make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<float4*>(o) = val;
        }
      }
    }
  }
}

template <bool TRANS>
__global__ void __launch_bounds__(kWideThreads, 1)
    umma_wide_estmm_kernel(const __grid_constant__ UParams p) {
  constexpr int CG = 2;
  uint32_t rank = 0;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int cluster = blockIdx.x / CG, n_clusters = gridDim.x / CG;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* staging = smem + kWideStages * kWideStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + kWideStaging);
  uint64_t* empty = full + kWideStages;
  uint64_t* tfull = empty + kWideStages;   // [2] by item parity
  uint64_t* tempty_lo = tfull + 2;         // [1] the N = 256 accumulator
  uint64_t* tempty_hi = tempty_lo + 1;     // [2] the two N = 128 slots
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_hi + 2);
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0);  // warp-uniform
  const int lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWideStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty_hi[a], kWideEW * CG);
    }
    mbar_init(tempty_lo, kWideEW * CG);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t full_lead = mapa0(smem_u32(full));
  const uint32_t tlo_lead = mapa0(smem_u32(tempty_lo));
  const uint32_t thi_lead = mapa0(smem_u32(tempty_hi));

  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n_mt = p.n_mt;
  const int total = *p.n_tiles * n_mt;
  auto wmap = [&](int wl) { return p.reverse ? total - 1 - wl : wl; };

  if (warp == 0) {
    // ================================ TMA producer =======================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmB) : "memory");
    }
    int s = 0;
    uint32_t ph = 0;
    for (int wl = cluster; wl < total; wl += n_clusters) {
      const int w = wmap(wl);
      const SegTile t = p.tiles[w / n_mt];
      const int m0 = (w % n_mt) * (BM * CG) + static_cast<int>(rank) * BM;
      const int nk = (t.end - t.begin + BK - 1) / BK;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * kWideStage;
        uint8_t* sb = sa + kABytes;
        if (elect_one()) {
          const uint32_t fb = full_lead + 8u * s;
          if (rank == 0) mbar_arrive_tx(&full[s], 2 * kWideStage);
          const int p0 = t.begin + kb * BK;
          // A = X1^T: this CTA's 128 M columns of the 64 positions; B = X2:
          // this CTA's 192 of the 384 N columns
          tma_3d_cg2(sa, &p.tmA, fb, 0, p0, m0 / 64);
          tma_3d_cg2(sb, &p.tmB, fb, 0, p0, static_cast<int>(rank) * (kWideBHalf / 64));
        }
        __syncwarp();
        if (++s == kWideStages) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ==========================
    if (rank == 0) {
      const uint32_t idesc1 = idesc_bf16(256, 1, 1, BM * CG);
      const uint32_t idesc2 = idesc_bf16(128, 1, 1, BM * CG);
      const uint32_t base = smem_u32(smem);
      const uint64_t da0 = sdesc(base, 8192, 1024);            // MN-major, 64-col atoms 8 KB apart
      const uint64_t db0 = sdesc(base + kABytes, 8192, 1024);
      const uint32_t a_lo = static_cast<uint32_t>(da0), a_hi = static_cast<uint32_t>(da0 >> 32);
      const uint32_t b_lo = static_cast<uint32_t>(db0), b_hi = static_cast<uint32_t>(db0 >> 32);
      const uint32_t step = 128u;  // 16 k rows of 128 B per K = 16
      const uint32_t b2_off = 16384u >> 4;  // the CTA's third 64-column atom
      constexpr uint32_t kStageUnits = kWideStage >> 4;
      int s = 0, it = 0;
      uint32_t ph = 0, lo_ph = 0, hi_ph[2] = {0, 0};
      for (int wl = cluster; wl < total; wl += n_clusters, ++it) {
        const int w = wmap(wl);
        const SegTile t = p.tiles[w / n_mt];
        const int nk = (t.end - t.begin + BK - 1) / BK;
        const int hs = it & 1;
        mbar_wait(tempty_lo, lo_ph ^ 1);
        mbar_wait(&tempty_hi[hs], hi_ph[hs] ^ 1);
        lo_ph ^= 1;
        hi_ph[hs] ^= 1;
        tc_fence_after();
        const uint32_t d_lo = tmem, d_hi = tmem + 256 + 128 * hs;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t so = static_cast<uint32_t>(s) * kStageUnits;
          if (elect_one())
            wide_kblock(d_lo, d_hi, a_lo + so, a_hi, step, b_lo + so, b_hi, step, b2_off, idesc1,
                        idesc2, kb == 0, &empty[s]);
          __syncwarp();
          if (++s == kWideStages) { s = 0; ph ^= 1; }
        }
        if (elect_one()) umma_commit_cg2(&tfull[it & 1]);
        __syncwarp();
      }
    }
    __syncwarp();
  } else {
    // ================================ epilogue ============================
    const int lg = warp & 3;
    const int g = (warp - 2) / 4;  // column group: output columns [192 g, 192 g + 192)
    uint8_t* stg = staging + (warp - 2) * 2048;
    const int64_t M = p.M, N = p.N;
    uint32_t tf_ph[2] = {0, 0};
    int it = 0;
    for (int wl = cluster; wl < total; wl += n_clusters, ++it) {
      const int w = wmap(wl);
      const SegTile t = p.tiles[w / n_mt];
      const int hs = it & 1;
      const bool split = t.flags & 1;
      const bool empty_seg = t.end <= t.begin;
      const int64_t m = static_cast<int64_t>(w % n_mt) * (BM * CG) + rank * BM + lg * 32 + lane;
      float* obase = p.est_out + static_cast<int64_t>(t.expert) * M * N;
      mbar_wait(&tfull[it & 1], tf_ph[it & 1]);
      tf_ph[it & 1] ^= 1;
      tc_fence_after();
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(lg * 32) << 16);
      // base of this warp's rows (TRANS: of this lane's row m, column 0):
      // out[e], or the owner's H-shard when the gradient is reduce-scattered
      // (H = m split in spans: [E][span][N] rows / [E][N][span] columns)
      float* wbase;
      int ld;
      {
        const int64_t mw = TRANS ? m : m - lane;
        if (p.n_peer > 0) {
          const int64_t span = p.peer_rows;
          const int owner = static_cast<int>(mw / span);
          const int64_t ml = mw - owner * span;
          wbase = TRANS ? p.peer[owner] + t.expert * N * span + ml
                        : p.peer[owner] + (t.expert * span + ml) * N;
          ld = static_cast<int>(TRANS ? span : N);
        } else {
          wbase = TRANS ? obase + mw : obase + mw * N;
          ld = static_cast<int>(TRANS ? M : N);
        }
      }
      auto emit = [&](const uint32_t (&r)[32], const int gcol) {
        est_emit<TRANS>(p, r, gcol, wbase, ld, stg, lane, split, empty_seg);
      };
      {
        // (an empty chunk's accumulator is never written: the loads return
        // stale values, which est_emit replaces by zeros)
        uint32_t rl[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32_async(lane_base + 128 * g + 32 * c, rl[c]);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cl(tlo_lead);
#pragma unroll
        for (int c = 0; c < 4; ++c) emit(rl[c], 192 * g + 32 * c);
      }
      {
        uint32_t rh[2][32];
#pragma unroll
        for (int c = 0; c < 2; ++c)
          tmem_ld32_async(lane_base + 256 + 128 * hs + 64 * g + 32 * c, rh[c]);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cl(thi_lead + 8u * hs);
#pragma unroll
        for (int c = 0; c < 2; ++c) emit(rh[c], 192 * g + 128 + 32 * c);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (threadIdx.x == 0 && p.n_peer > 0) asm volatile("fence.sc.sys;" ::: "memory");
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

}  // namespace

bool umma_wide_ok(const EsmmArgs& a) {
  static const bool on = [] {
    const char* e = std::getenv("HXM_WIDE");
    return !(e && e[0] == '0');
  }();
  return on && a.epi == EPI_ATOMIC && a.tile_rows == kUmma2Rows && a.d2 == kWideN &&
         a.amap.kind == MAP_DENSE && a.d1 % BK == 0;
}

hxm_status umma_wide_esmm(const EsmmArgs& a, cudaStream_t st) {
  if (a.max_tiles <= 0) return HXM_OK;
  UParams prm{};
  HXM_RETURN_IF(prep_esmm(a, 2, kWideN, prm));
  prm.stream_k = 0;
  static bool attr_set[64] = {false};
  int dev = 0;
  HXM_TRY_CUDA(cudaGetDevice(&dev));
  dev = dev < 64 ? dev : 63;
  if (!attr_set[dev]) {
    HXM_TRY_CUDA(cudaFuncSetAttribute(umma_wide_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kWideSmem));
    attr_set[dev] = true;
  }
  const int sms = sm_count();
  if (sms <= 0) return invalid_arg("tcgen05 path: no CUDA device");
  const int grid = std::max(1, std::min(sms / 2, a.max_tiles)) * 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kWideThreads);
  cfg.dynamicSmemBytes = kWideSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_on()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = 2;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  cfg.attrs = attr;
  cfg.numAttrs = na;
  HXM_TRY_CUDA(cudaLaunchKernelEx(&cfg, umma_wide_kernel, prm));
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}


bool umma_wide_estmm_ok(const EstmmArgs& a) {
  static const bool on = [] {
    const char* e = std::getenv("HXM_WIDE_EST");
    return !(e && e[0] == '0');
  }();
  const char* cp = std::getenv("HXM_CTA_PAIR");
  const bool pair_ok = !(cp && cp[0] == '0');
  // peer shards: a warp's 32 rows must belong to one owner (row-major out)
  const bool peer_ok = !a.peer || a.trans_out || a.peer->rows_per_rank % 32 == 0;
  return on && pair_ok && peer_ok && a.m1.kind == MAP_DENSE && a.m2.kind == MAP_DENSE &&
         a.d2 == kWideN && a.d1 % (BM * 2) == 0 && a.d1 > 0;
}

hxm_status umma_wide_estmm(const EstmmArgs& a, cudaStream_t st) {
  if (a.max_tiles <= 0) return HXM_OK;
  if (!umma_wide_estmm_ok(a)) return invalid_arg("umma_wide_estmm: unsupported shape");
  UParams prm{};
  HXM_RETURN_IF(prep_estmm(a, 2, kWideN, prm));
  // prep_estmm encodes B boxes for 256 x 192 pair tiles; this kernel takes
  // the CTA's 192 columns as three 64-column atoms (128B swizzle)
  {
    const uint64_t dims[3] = {64, static_cast<uint64_t>(a.x2_rows),
                              static_cast<uint64_t>(a.d2) / 64};
    const uint64_t strides[2] = {static_cast<uint64_t>(a.d2) * 2, 128};
    const uint32_t box[3] = {64, 64, static_cast<uint32_t>(kWideBHalf / 64)};
    if (!make_map(&prm.tmB, a.x2, 3, dims, strides, box))
      return invalid_arg("umma_wide_estmm: cannot encode the X2 tensor map");
    prm.b_sw64 = 0;
  }
  prm.n_mt = static_cast<int>(a.d1 / (BM * 2));
  prm.trans_out = a.trans_out;
  static bool attr_set[64] = {false};
  int dev = 0;
  HXM_TRY_CUDA(cudaGetDevice(&dev));
  dev = dev < 64 ? dev : 63;
  void (*kern)(UParams) = a.trans_out ? umma_wide_estmm_kernel<true> : umma_wide_estmm_kernel<false>;
  if (!attr_set[dev]) {
    HXM_TRY_CUDA(cudaFuncSetAttribute(umma_wide_estmm_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kWideSmem));
    HXM_TRY_CUDA(cudaFuncSetAttribute(umma_wide_estmm_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kWideSmem));
    attr_set[dev] = true;
  }
  const int sms = sm_count();
  if (sms <= 0) return invalid_arg("tcgen05 path: no CUDA device");
  const int work = a.max_tiles * prm.n_mt;
  const int grid = std::max(1, std::min(sms / 2, work)) * 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kWideThreads);
  cfg.dynamicSmemBytes = kWideSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_on()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = 2;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  cfg.attrs = attr;
  cfg.numAttrs = na;
  HXM_TRY_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

}  // namespace hxm
