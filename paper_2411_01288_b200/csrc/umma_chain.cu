// umma_chain.cu -- the layer forward's two ESMMs as ONE persistent tcgen05
// kernel (moe_layer.cpp:56-63: y1 = x W1 + b1, y2 = F(y1), y += y2 W2 + b2),
// for the 384-wide layers (c2: d_in = d_out = 384).
//
// Why: fwd1 writes the H-wide stash F(y1) and fwd2 streams it straight back
// in (100 MB each way at c2), and both run at K = 384 / N = 384 widths whose
// per-tile epilogue and operand latencies leave each kernel well short of
// its roofline (profiles/r1b_notes.md 4, 5, 15).  Chained, every 256-row
// tile (a CTA pair, cta_group::2) walks the hidden dimension in 128-column
// chunks:
//
//   GEMM1(c):  acc1[256 x 128]  = x_s[256 x D_i] . W1[e][:, chunk c]
//   epilogue:  + b1, F and F' in f32x2; F' -> stash (global); F -> smem in
//              the UMMA K-major layout, TMA-stored to the F stash from there
//   GEMM2(c):  acc2[256 x 384] += F_c[256 x 128] . W2[e][chunk c, :]
//
// and the y epilogue (+ b2, fp32 reductions into token order) runs once per
// tile.  The F chunk never round-trips through HBM for the second GEMM.
//
// Shared memory (per CTA, 128 rows): x_s tile resident for the whole tile
// (D_i / 64 atoms of 16 KB), the F chunk (2 x 16 KB: GEMM2's A operand, the
// TMA-store source, and the y epilogue's staging), a ring of 24 KB weight
// stages (W1: 192 K rows x 64 columns; W2: 64 K rows x this CTA's 192
// columns), the chunk bias.  TMEM (512 columns): acc2 = [0, 384) (N = 256 and
// N = 128 MMAs as in umma_wide.cu), acc1 = [384, 512).
//
// Issue order on the tensor pipe: GEMM1(0), then per chunk c >= 1: GEMM1(c),
// GEMM2(c - 1) -- GEMM1(c) runs while the epilogue turns acc1(c - 1) into F,
// GEMM2(c - 1) while the epilogue waits for acc1(c).
//
// Ring order (producer = MMA consumption): W1(0), {W1(c), W2(c-1)} for
// c = 1.., W2(last); the next tile's x_s rows load once GEMM1(last) is done.
//
// The backward's g_y1 -> g_x pair (moe_layer.cpp:105-108, 118) is the same
// chain with the roles of the weights swapped (BWD = true):
//
//   GEMM1(c):  acc1 = g_y_s[256 x D_o] . W2[e]^T[:, chunk c]   (B K-major)
//   epilogue:  g_y1 = acc1 * F'(y1) (the stash chunk, read from global),
//              pads masked; g_y1 -> smem -> TMA store to the g_y1 stash (the
//              ESTMM gW1 operand); fused gb1 column sums (ESS of g_y1,
//              es_ops.cpp:86-102) as deterministic per-(tile, CTA, lane
//              group) partials, the layout colsum_combine reduces
//   GEMM2(c):  acc2 += g_y1_c . W1[e]^T[chunk c, :]             (B K-major)
//   out:       g_x rows (fp32 reductions into token order)
#include "umma_impl.cuh"

namespace hxm {
namespace {

constexpr int kChNC = 128;                       // hidden columns per chunk
constexpr int kChN2 = 384;                       // output width (d_out)
constexpr int kChMaxA = 6;                       // x_s atoms (d_in <= 384)
constexpr int kChStage = 24576;                  // one ring stage
constexpr int kChStages = 4;
constexpr int kChEW = 16;                        // epilogue warps
constexpr int kChThreads = 64 + 32 * kChEW;      // 576
constexpr int kChA1 = kChMaxA * kABytes;         // 96 KB
constexpr int kChF = 2 * kABytes;                // 32 KB
constexpr int kChBias = 2 * 4 * 32 * 4;          // 1 KB: [slot][column group][32]
constexpr int kChBars = 256;
constexpr int kChSmem = kChA1 + kChF + kChStages * kChStage + kChBias + kChBars + 1024;
static_assert(kChSmem <= 232448, "chain smem");

struct ChainParams {
  CUtensorMap tmA;   // GEMM1 A rows (x_s / g_y_s): (K1, rows), box 64 x 128
  CUtensorMap tmW1;  // W1 as (64, d_in, H / 64, E), box 64 x 192 x 1
  CUtensorMap tmW2;  // W2 as (64, H, d_out / 64, E), box 64 x 64 x 3
  CUtensorMap tmF;   // bf16 chunk output stash (F / g_y1): (H, rows), box 64 x 128
  CUtensorMap tmFs;  // the same, box 64 x 32 (segment-end slices)
  CUtensorMap tmD;   // F'(y1) stash (H, rows), box 64 x 128
  CUtensorMap tmDs;  // F'(y1) stash, box 64 x 32
  int fp_tma;        // F' through the chunk buffer by TMA (1) or per-row global access (0)
  __nv_bfloat16* dact;  // F'(y1) stash, row stride H: written (forward) / read (backward)
  const float* b1;      // forward: E x H
  const float* b2;      // forward: E x 384 or null
  float* y;             // y (forward) / g_x (backward): rows x 384, token order via omap
  float* colsum;        // backward: gb1 column-sum partials
  RowMap omap;
  const SegTile* tiles;
  const int32_t* n_tiles;
  int H, n_a1, n_g1;  // n_a1 = K1 / 64 atoms, n_g1 = K1 / 192 GEMM1 stages per chunk
  unsigned long long* trace;  // HXM_CHAIN_TRACE=1: per-CTA wait totals (cycles), else null
};
// trace slots per CTA (clock64 cycles): MMA waits on acc1_empty / full (GEMM1)
// / f_full / full (GEMM2) / acc2_empty / a1full; producer waits on empty /
// a1empty; epilogue (warp 2, lane 0) waits on acc1_full, chunk math, B1,
// f_empty, F write + B2, acc2_full, y epilogue; CTA total
constexpr int kChTrace = 20;
#define CH_T0() const long long _t0 = (TR && p.trace) ? clock64() : 0
#define CH_ACC(var) do { if (TR && p.trace) var += clock64() - _t0; } while (0)

// Four K = 16 UMMAs of one 64-deep k-block, no commit (GEMM1: three k-blocks
// share a ring stage; the stage is released by one commit after the third).
__device__ __forceinline__ void mma4_cg2(uint32_t d, uint32_t a_lo, uint32_t a_hi,
                                         uint32_t b_lo, uint32_t b_hi, uint32_t b_step,
                                         uint32_t idesc, uint32_t first) {
  asm volatile(
      "{\n"
      ".reg .pred p0, p1;\n"
      ".reg .b64 da, db;\n"
      ".reg .b32 al, bl;\n"
      "setp.ne.b32 p0, %7, 0;\n"
      "setp.eq.b32 p1, %7, %7;\n"
      "mov.b64 da, {%1, %2};\n"
      "mov.b64 db, {%3, %4};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %6, p0;\n"
      "add.u32 al, %1, 2;\n"
      "add.u32 bl, %3, %5;\n"
      "mov.b64 da, {al, %2};\n"
      "mov.b64 db, {bl, %4};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %6, p1;\n"
      "add.u32 al, al, 2;\n"
      "add.u32 bl, bl, %5;\n"
      "mov.b64 da, {al, %2};\n"
      "mov.b64 db, {bl, %4};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %6, p1;\n"
      "add.u32 al, al, 2;\n"
      "add.u32 bl, bl, %5;\n"
      "mov.b64 da, {al, %2};\n"
      "mov.b64 db, {bl, %4};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %6, p1;\n"
      "}\n" ::"r"(d),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(b_step), "r"(idesc), "r"(first ? 0u : 1u)
      : "memory");
}

// The two N-parts of GEMM2's k-block (N = 256 into acc2 lo, N = 128 into acc2
// hi), four K = 16 steps, then the stage commit -- umma_wide.cu's k-block.
__device__ __forceinline__ void mma_wide_cg2(uint32_t d_lo, uint32_t d_hi, uint32_t a_lo,
                                             uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                                             uint32_t b_step, uint32_t b2_off, uint32_t idesc1,
                                             uint32_t idesc2, uint32_t first, uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred p0, p1;\n"
      ".reg .b64 da, db, db2;\n"
      ".reg .b32 al, bl, b2l;\n"
      "setp.ne.b32 p0, %10, 0;\n"
      "setp.eq.b32 p1, %10, %10;\n"
      "mov.b32 al, %2;\n"
      "mov.b32 bl, %4;\n"
      "add.u32 b2l, %4, %7;\n"
      "mov.b64 da, {al, %3};\n"
      "mov.b64 db, {bl, %5};\n"
      "mov.b64 db2, {b2l, %5};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %8, p0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%1], da, db2, %9, p0;\n"
      "add.u32 al, al, 2;\n"
      "add.u32 bl, bl, %6;\n"
      "add.u32 b2l, b2l, %6;\n"
      "mov.b64 da, {al, %3};\n"
      "mov.b64 db, {bl, %5};\n"
      "mov.b64 db2, {b2l, %5};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %8, p1;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%1], da, db2, %9, p1;\n"
      "add.u32 al, al, 2;\n"
      "add.u32 bl, bl, %6;\n"
      "add.u32 b2l, b2l, %6;\n"
      "mov.b64 da, {al, %3};\n"
      "mov.b64 db, {bl, %5};\n"
      "mov.b64 db2, {b2l, %5};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %8, p1;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%1], da, db2, %9, p1;\n"
      "add.u32 al, al, 2;\n"
      "add.u32 bl, bl, %6;\n"
      "add.u32 b2l, b2l, %6;\n"
      "mov.b64 da, {al, %3};\n"
      "mov.b64 db, {bl, %5};\n"
      "mov.b64 db2, {b2l, %5};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %8, p1;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%1], da, db2, %9, p1;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%11], %12;\n"
      "}\n" ::"r"(d_lo),
      "r"(d_hi), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(b_step), "r"(b2_off),
      "r"(idesc1), "r"(idesc2), "r"(first ? 0u : 1u), "r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

// The F chunk is written by threads (generic proxy) and read by the leader's
// tcgen05.mma (async proxy) in both CTAs: every writer fences with
// fence.proxy.async.shared::cta, the chunk barrier collects them, and one
// thread per CTA arrives on the leader's f_full with the default (cta-scope)
// semantics -- CUTLASS's ClusterBarrier pattern for thread-produced UMMA
// operands.  A .release.cluster arrive would also wait for the thread's
// outstanding global stores (MEMBAR): measured at ~3 us per chunk.
template <int ACT, bool BWD, bool TR>
__global__ void __launch_bounds__(kChThreads, 1)
    umma_chain_kernel(const __grid_constant__ ChainParams p) {
  constexpr int CG = 2;
  uint32_t rank = 0;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int cluster = blockIdx.x / CG, n_clusters = gridDim.x / CG;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA1 = smem;
  uint8_t* sF = sA1 + kChA1;
  uint8_t* ring = sF + kChF;
  float* bias_s = reinterpret_cast<float*>(ring + kChStages * kChStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(bias_s) + kChBias);
  uint64_t* empty = full + kChStages;
  uint64_t* a1full = empty + kChStages;
  uint64_t* a1empty = a1full + 1;
  uint64_t* acc1_full = a1empty + 1;
  uint64_t* acc1_empty = acc1_full + 1;
  uint64_t* f_full = acc1_empty + 1;
  uint64_t* f_empty = f_full + 1;
  uint64_t* acc2_full = f_empty + 1;
  uint64_t* acc2_empty = acc2_full + 1;
  uint64_t* fp_full = acc2_empty + 1;  // backward: F'(y1) chunk landed in the F buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fp_full + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kChStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(a1full, 1);
    mbar_init(a1empty, 1);
    mbar_init(acc1_full, 1);
    mbar_init(acc1_empty, kChEW * CG);
    mbar_init(f_full, CG);
    mbar_init(f_empty, 1);
    mbar_init(acc2_full, 1);
    mbar_init(acc2_empty, kChEW * CG);
    mbar_init(fp_full, 1);
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
  const uint32_t a1full_lead = mapa0(smem_u32(a1full));
  const uint32_t acc1e_lead = mapa0(smem_u32(acc1_empty));
  const uint32_t ffull_lead = mapa0(smem_u32(f_full));
  const uint32_t acc2e_lead = mapa0(smem_u32(acc2_empty));

  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int total = *p.n_tiles;
  const int nC = p.H / kChNC;

  if (warp == 0) {
    // ================================ TMA producer =======================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmW1) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmW2) : "memory");
    }
    int s = 0;
    uint32_t ph = 0, a1ph = 0;
    long long tpe = 0, tpa = 0;
    const int rk = static_cast<int>(rank);
    // GEMM1's B for chunk c, 192 K rows per stage.  Forward: W1[e][k][h]
    // (MN-major, this CTA's 64 hidden columns).  Backward: W2[e][h][d] read
    // as W2^T (K-major: this CTA's 64 hidden rows, three 64-deep K atoms).
    auto stage_w1 = [&](int c, int e) {
      for (int j = 0; j < p.n_g1; ++j) {
        {
          CH_T0();
          mbar_wait(&empty[s], ph ^ 1);
          CH_ACC(tpe);
        }
        if (elect_one()) {
          if (rank == 0) mbar_arrive_tx(&full[s], 2 * kChStage);
          if (BWD)
            tma_4d_cg2(ring + s * kChStage, &p.tmW2, full_lead + 8u * s, 0,
                       c * kChNC + 64 * rk, 3 * j, e);
          else
            tma_4d_cg2(ring + s * kChStage, &p.tmW1, full_lead + 8u * s, 0, 192 * j,
                       (c * kChNC) / 64 + rk, e);
        }
        __syncwarp();
        if (++s == kChStages) { s = 0; ph ^= 1; }
      }
    };
    // GEMM2's B for chunk c, 64 K (hidden) rows per stage.  Forward: W2[e][h][d]
    // (MN-major, this CTA's 192 output columns).  Backward: W1[e][d][h] read as
    // W1^T (K-major: this CTA's 192 output rows of one 64-deep K atom).
    auto stage_w2 = [&](int c, int e) {
      for (int j = 0; j < 2; ++j) {
        {
          CH_T0();
          mbar_wait(&empty[s], ph ^ 1);
          CH_ACC(tpe);
        }
        if (elect_one()) {
          if (rank == 0) mbar_arrive_tx(&full[s], 2 * kChStage);
          if (BWD)
            tma_4d_cg2(ring + s * kChStage, &p.tmW1, full_lead + 8u * s, 0, 192 * rk,
                       (c * kChNC) / 64 + j, e);
          else
            tma_4d_cg2(ring + s * kChStage, &p.tmW2, full_lead + 8u * s, 0, c * kChNC + 64 * j,
                       3 * rk, e);
        }
        __syncwarp();
        if (++s == kChStages) { s = 0; ph ^= 1; }
      }
    };
    for (int wl = cluster; wl < total; wl += n_clusters) {
      const SegTile t = p.tiles[wl];
      // x_s rows of this tile: once the previous tile's last GEMM1 is done
      {
        CH_T0();
        mbar_wait(a1empty, a1ph ^ 1);
        CH_ACC(tpa);
      }
      a1ph ^= 1;
      if (elect_one()) {
        if (rank == 0) mbar_arrive_tx(a1full, 2 * p.n_a1 * kABytes);
        for (int j = 0; j < p.n_a1; ++j)
          tma_2d_cg2(sA1 + j * kABytes, &p.tmA, a1full_lead, 64 * j,
                     t.begin + static_cast<int>(rank) * BM);
      }
      __syncwarp();
      stage_w1(0, t.expert);
      for (int c = 1; c < nC; ++c) {
        stage_w1(c, t.expert);
        stage_w2(c - 1, t.expert);
      }
      stage_w2(nC - 1, t.expert);
    }
    if (TR && p.trace && lane == 0) {
      p.trace[blockIdx.x * kChTrace + 6] = tpe;
      p.trace[blockIdx.x * kChTrace + 7] = tpa;
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ==========================
    if (rank == 0) {
      // A K-major everywhere; B MN-major (forward) or K-major (backward: W^T)
      constexpr int bmn = BWD ? 0 : 1;
      const uint32_t idesc1 = idesc_bf16(kChNC, 0, bmn, BM * CG);
      const uint32_t idesc_lo = idesc_bf16(256, 0, bmn, BM * CG);
      const uint32_t idesc_hi = idesc_bf16(128, 0, bmn, BM * CG);
      const uint64_t da1 = sdesc(smem_u32(sA1), 16, 1024);
      const uint64_t dF = sdesc(smem_u32(sF), 16, 1024);
      const uint64_t db = BWD ? sdesc(smem_u32(ring), 16, 1024) : sdesc(smem_u32(ring), 8192, 1024);
      // per K = 16 step: 16 MN-major rows of 128 B, or 32 B inside a K-major atom
      constexpr uint32_t b_step = BWD ? 2u : 128u;
      const uint32_t a1_lo = static_cast<uint32_t>(da1), a1_hi = static_cast<uint32_t>(da1 >> 32);
      const uint32_t f_lo = static_cast<uint32_t>(dF), f_hi = static_cast<uint32_t>(dF >> 32);
      const uint32_t b_lo = static_cast<uint32_t>(db), b_hi = static_cast<uint32_t>(db >> 32);
      constexpr uint32_t kStageU = kChStage >> 4;
      constexpr uint32_t kAtomU = kABytes >> 4;  // 16 KB
      const uint32_t d_acc1 = tmem + 384, d_lo = tmem, d_hi = tmem + 256;
      int s = 0;
      uint32_t ph = 0, a1ph = 0, e1ph = 0, ffph = 0, e2ph = 0;
      long long tw[6] = {0, 0, 0, 0, 0, 0};
      auto gemm1 = [&](int c, bool last) {
        {
          CH_T0();
          mbar_wait(acc1_empty, e1ph ^ 1);
          CH_ACC(tw[0]);
        }
        e1ph ^= 1;
        tc_fence_after();
        for (int j = 0; j < p.n_g1; ++j) {
          {
            CH_T0();
            mbar_wait(&full[s], ph);
            CH_ACC(tw[1]);
          }
          tc_fence_after();
          if (elect_one()) {
            const uint32_t so = static_cast<uint32_t>(s) * kStageU;
#pragma unroll
            for (int kb = 0; kb < 3; ++kb)
              mma4_cg2(d_acc1, a1_lo + (3 * j + kb) * kAtomU, a1_hi, b_lo + so + kb * 512u, b_hi,
                       b_step, idesc1, j == 0 && kb == 0);
            umma_commit_cg2(&empty[s]);
          }
          __syncwarp();
          if (++s == kChStages) { s = 0; ph ^= 1; }
        }
        if (elect_one()) {
          umma_commit_cg2(acc1_full);
          if (last) umma_commit_cg2(a1empty);  // x_s tile free for the next tile
        }
        __syncwarp();
        (void)c;
      };
      auto gemm2 = [&](int c, bool last) {
        {
          CH_T0();
          mbar_wait(f_full, ffph);  // both CTAs' F chunk written
          CH_ACC(tw[2]);
        }
        ffph ^= 1;
        if (c == 0) {
          CH_T0();
          mbar_wait(acc2_empty, e2ph ^ 1);  // the previous tile's y epilogue drained acc2
          CH_ACC(tw[4]);
          e2ph ^= 1;
        }
        tc_fence_after();
        for (int j = 0; j < 2; ++j) {
          {
            CH_T0();
            mbar_wait(&full[s], ph);
            CH_ACC(tw[3]);
          }
          tc_fence_after();
          if (elect_one())
            mma_wide_cg2(d_lo, d_hi, f_lo + j * kAtomU, f_hi,
                         b_lo + static_cast<uint32_t>(s) * kStageU, b_hi, b_step, 16384u >> 4,
                         idesc_lo, idesc_hi, c == 0 && j == 0, &empty[s]);
          __syncwarp();
          if (++s == kChStages) { s = 0; ph ^= 1; }
        }
        if (elect_one()) {
          umma_commit_cg2(f_empty);
          if (last) umma_commit_cg2(acc2_full);
        }
        __syncwarp();
      };
      for (int wl = cluster; wl < total; wl += n_clusters) {
        {
          CH_T0();
          mbar_wait(a1full, a1ph);
          CH_ACC(tw[5]);
        }
        a1ph ^= 1;
        tc_fence_after();
        gemm1(0, nC == 1);
        for (int c = 1; c < nC; ++c) {
          gemm1(c, c == nC - 1);
          gemm2(c - 1, false);
        }
        gemm2(nC - 1, true);
      }
      if (TR && p.trace && lane == 0)
        for (int i = 0; i < 6; ++i) p.trace[blockIdx.x * kChTrace + i] = tw[i];
    }
    __syncwarp();
  } else {
    // ================================ epilogue ============================
    const int ew = warp - 2;      // 0..15
    const int lg = warp & 3;      // TMEM lane group (hardware rule: warp % 4)
    const int cg = ew >> 2;       // column group: 32 columns of each chunk
    const int r = lg * 32 + lane; // this thread's row of the CTA's 128
    const bool elect = ew == 0 && lane == 0;
    const int H = p.H;
    uint32_t f1ph = 0, feph = 0, f2ph = 0, fpph = 0;
    int gch = 0;  // running chunk count (bias slots)
    long long te[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long tk0 = (TR && p.trace) ? clock64() : 0;
    long long tmark = 0;
    auto mark = [&](int slot) {
      if (TR && p.trace) {
        const long long now = clock64();
        te[slot] += now - tmark;
        tmark = now;
      }
    };
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(lg * 32) << 16);
    uint8_t* stg = sF + ew * 2048;
    // chunk bias: warp lg == 0 of each column group stages the group's 32
    // floats of the NEXT chunk (slot (gch + 1) & 1) between the chunk's two
    // barriers; everyone reads the current slot before the first barrier
    auto bias_val = [&](int e, int c) {
      return BWD ? 0.f : ldg_nc(p.b1 + static_cast<int64_t>(e) * H + c * kChNC + cg * 32 + lane);
    };
    {
      const int wl0 = cluster;
      if (!BWD && lg == 0 && wl0 < total)
        bias_s[(0 * 4 + cg) * 32 + lane] = bias_val(p.tiles[wl0].expert, 0);
      named_bar_sync(1, 32 * kChEW);
    }
    for (int wl = cluster; wl < total; wl += n_clusters) {
      const SegTile t = p.tiles[wl];
      const int nwl = wl + n_clusters;
      const int next_e = nwl < total ? p.tiles[nwl].expert : -1;
      const int qbase = t.begin + static_cast<int>(rank) * BM;
      const int rows_here = t.end - qbase;  // >= 128: whole box; 32-row slices otherwise
      const bool slice_ok = lg * 32 < rows_here;
      int orow = -1;
      {
        const int qq = qbase + r;
        if (qq < t.end) orow = p.omap(qq);
      }
      __nv_bfloat16* dact_row = p.dact + static_cast<int64_t>(qbase + r) * H + cg * 32;
      if (TR && p.trace) tmark = clock64();
      for (int c = 0; c < nC; ++c, ++gch) {
        // backward: pull the next chunk's F'(y1) boxes into L2 (the in-place
        // TMA load below then waits on an L2 hit, not on HBM)
        if (BWD && p.fp_tma && elect) {
          const bool more = c + 1 < nC;
          if (more || nwl < total) {
            const int pc = more ? (c + 1) * kChNC : 0;
            const int pr = more ? qbase : p.tiles[nwl].begin + static_cast<int>(rank) * BM;
            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(&p.tmD),
                         "r"(pc), "r"(pr) : "memory");
            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(&p.tmD),
                         "r"(pc + 64), "r"(pr) : "memory");
          }
        }
        // next chunk's bias value (this tile's next chunk, or the next tile's first)
        float bnext = 0.f;
        const bool wr_bias = !BWD && lg == 0 && (c + 1 < nC || next_e >= 0);
        if (wr_bias) bnext = bias_val(c + 1 < nC ? t.expert : next_e, c + 1 < nC ? c + 1 : 0);
        // backward: this row's F'(y1) chunk, loaded before the accumulator wait
        uint4 dv[4] = {};
        if (BWD && !p.fp_tma && slice_ok) {
          const __nv_bfloat16* src = dact_row + c * kChNC;
#pragma unroll
          for (int j = 0; j < 2; ++j)
            asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=r"(dv[2 * j].x), "=r"(dv[2 * j].y), "=r"(dv[2 * j].z), "=r"(dv[2 * j].w),
                           "=r"(dv[2 * j + 1].x), "=r"(dv[2 * j + 1].y), "=r"(dv[2 * j + 1].z),
                           "=r"(dv[2 * j + 1].w)
                         : "l"(src + 16 * j));
        }
        mark(7);
        mbar_wait(acc1_full, f1ph);
        mark(0);
        f1ph ^= 1;
        tc_fence_after();
        uint32_t rr[32];
        tmem_ld32_async(lane_base + 384 + cg * 32, rr);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cl(acc1e_lead);
        uint32_t o1[16], o2[16];  // forward: F', F; backward: o2 = g_y1
        if constexpr (!BWD) {
          const float* bs = bias_s + ((gch & 1) * 4 + cg) * 32;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 b = *reinterpret_cast<const float2*>(bs + 2 * i);
            float2 f, df;
            act_pair<ACT>(f2_fma(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])),
                                 f2(1.f), b),
                          f, df);
            o1[i] = pack_bf16(df.x, df.y);
            o2[i] = pack_bf16(f.x, f.y);
          }
          // F' straight to the stash (this row's 64 bytes of the chunk)
          // (two 256-bit stores: whole 32-byte sectors, no partial-sector writes)
          if (!p.fp_tma && slice_ok) {
            __nv_bfloat16* dst = dact_row + c * kChNC;
#pragma unroll
            for (int j = 0; j < 2; ++j)
              asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + 16 * j),
                           "r"(o1[8 * j]), "r"(o1[8 * j + 1]), "r"(o1[8 * j + 2]), "r"(o1[8 * j + 3]),
                           "r"(o1[8 * j + 4]), "r"(o1[8 * j + 5]), "r"(o1[8 * j + 6]), "r"(o1[8 * j + 7])
                           : "memory");
          }
        } else if (!p.fp_tma) {
          // g_y1 = (g_y W2^T) * F'(y1); padding slots and rows past the
          // segment end are zero (they feed the gb1 sums and GEMM2)
          const bool pad = orow < 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const __nv_bfloat162* yb = reinterpret_cast<const __nv_bfloat162*>(&dv[j]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 g = f2_mul(make_float2(__uint_as_float(rr[8 * j + 2 * i]),
                                                  __uint_as_float(rr[8 * j + 2 * i + 1])),
                                      __bfloat1622float2(yb[i]));
              o2[4 * j + i] = pad ? 0u : pack_bf16(g.x, g.y);
            }
          }
          (void)o1;
        }
        // (B1) the F buffer is free: the previous chunk's TMA store has read
        // it (elected thread) and GEMM2 of the previous chunk is done
        mark(1);
        if (elect) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        named_bar_sync(1, 32 * kChEW);
        mark(2);
        mbar_wait(f_empty, feph ^ 1);
        mark(3);
        feph ^= 1;
        uint8_t* const frow = sF + (cg >> 1) * kABytes + r * 128;
        if (p.fp_tma) {
          if constexpr (!BWD) {
            // F' through the (now free) chunk buffer: one TMA store per
            // 64-column box instead of per-row global stores
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int j0 = (cg & 1) * 4 + j;
              *reinterpret_cast<uint4*>(frow + ((j0 ^ (r & 7)) << 4)) =
                  make_uint4(o1[4 * j], o1[4 * j + 1], o1[4 * j + 2], o1[4 * j + 3]);
            }
            fence_async_smem();
            named_bar_sync(4, 32 * kChEW);
            if (elect) {
              const int col = c * kChNC;
              if (rows_here >= BM) {
                tma_store_2d(&p.tmD, sF, col, qbase);
                tma_store_2d(&p.tmD, sF + kABytes, col + 64, qbase);
              } else {
                for (int sl = 0; sl * 32 < rows_here; ++sl) {
                  tma_store_2d(&p.tmDs, sF + sl * 4096, col, qbase + sl * 32);
                  tma_store_2d(&p.tmDs, sF + kABytes + sl * 4096, col + 64, qbase + sl * 32);
                }
              }
              bulk_commit();
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            named_bar_sync(5, 32 * kChEW);
          } else {
            // F'(y1) chunk of this CTA's 128 rows into the chunk buffer (the
            // rows past a segment end are loaded too and masked below)
            if (elect) {
              mbar_arrive_tx(fp_full, 2 * kABytes);
              tma_2d(sF, &p.tmD, fp_full, c * kChNC, qbase);
              tma_2d(sF + kABytes, &p.tmD, fp_full, c * kChNC + 64, qbase);
            }
            mbar_wait(fp_full, fpph);
            fpph ^= 1;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int j0 = (cg & 1) * 4 + j;
              dv[j] = *reinterpret_cast<const uint4*>(frow + ((j0 ^ (r & 7)) << 4));
            }
            const bool pad = orow < 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const __nv_bfloat162* yb = reinterpret_cast<const __nv_bfloat162*>(&dv[j]);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 g = f2_mul(make_float2(__uint_as_float(rr[8 * j + 2 * i]),
                                                    __uint_as_float(rr[8 * j + 2 * i + 1])),
                                        __bfloat1622float2(yb[i]));
                o2[4 * j + i] = pad ? 0u : pack_bf16(g.x, g.y);
              }
            }
          }
        }
        {
          uint8_t* fa = sF + (cg >> 1) * kABytes + r * 128;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int j0 = (cg & 1) * 4 + j;
            *reinterpret_cast<uint4*>(fa + ((j0 ^ (r & 7)) << 4)) =
                make_uint4(o2[4 * j], o2[4 * j + 1], o2[4 * j + 2], o2[4 * j + 3]);
          }
        }
        if constexpr (BWD) {
          if (p.colsum) {
            // fused gb1: column sums of the bf16 g_y1 values this warp just
            // wrote (its own 32 rows: __syncwarp ordering).  Lane (rsub, cq)
            // sums 8 columns of rows rsub + 8i in f32x2, the 8 row groups
            // reduce by shuffles; lanes 0..3 write the warp's 32 sums: one
            // deterministic partial row per (tile, CTA, lane group), the
            // order of umma_impl.cuh's MODE 2 epilogue
            __syncwarp();
            const int cq = lane & 3, rsub = lane >> 2;
            float2 cs[4] = {f2(0.f), f2(0.f), f2(0.f), f2(0.f)};
            const uint8_t* fb = sF + (cg >> 1) * kABytes;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int rw = lg * 32 + rsub + 8 * i;
              const int j0 = (cg & 1) * 4 + cq;
              const uint4 q4 = *reinterpret_cast<const uint4*>(fb + rw * 128 + ((j0 ^ (rw & 7)) << 4));
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
              float* dst = p.colsum + ((static_cast<int64_t>(wl) * CG + rank) * 4 + lg) * H +
                           c * kChNC + cg * 32 + cq * 8;
              reinterpret_cast<float4*>(dst)[0] = make_float4(cs[0].x, cs[0].y, cs[1].x, cs[1].y);
              reinterpret_cast<float4*>(dst)[1] = make_float4(cs[2].x, cs[2].y, cs[3].x, cs[3].y);
            }
          }
        }
        if (wr_bias) bias_s[(((gch + 1) & 1) * 4 + cg) * 32 + lane] = bnext;
        fence_async_smem();
        named_bar_sync(2, 32 * kChEW);
        if (elect) {
          const int col = c * kChNC;
          if (rows_here >= BM) {
            tma_store_2d(&p.tmF, sF, col, qbase);
            tma_store_2d(&p.tmF, sF + kABytes, col + 64, qbase);
          } else {
            for (int sl = 0; sl * 32 < rows_here; ++sl) {
              tma_store_2d(&p.tmFs, sF + sl * 4096, col, qbase + sl * 32);
              tma_store_2d(&p.tmFs, sF + kABytes + sl * 4096, col + 64, qbase + sl * 32);
            }
          }
          bulk_commit();
          mbar_arrive_cl(ffull_lead);
        }
        mark(4);
      }
      // ---- y epilogue: acc2 (+ b2) reduced into token order ---------------
      if (TR && p.trace) tmark = clock64();
      mbar_wait(acc2_full, f2ph);
      mark(5);
      f2ph ^= 1;
      tc_fence_after();
      if (elect) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      named_bar_sync(3, 32 * kChEW);  // F buffer free: staging for the fp32 rows
      // (the backward's g_x has no bias: compiled out, not just skipped)
      const float* bias2 = (!BWD && p.b2) ? p.b2 + static_cast<int64_t>(t.expert) * kChN2 : nullptr;
      auto emit = [&](const uint32_t (&q)[32], const int gcol) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(q[i]);
        if (!BWD && bias2) {
          const float4* b4 = reinterpret_cast<const float4*>(bias2 + gcol);
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
            const int rw = i * 8 + lane / 4, cc = lane % 4;
            const int orr = __shfl_sync(0xffffffffu, orow, rw);
            const float4 val =
                *reinterpret_cast<const float4*>(stg + rw * 64 + ((cc ^ ((rw >> 1) & 3)) * 16));
            if (orr < 0) continue;
            red_add_v4(p.y + static_cast<int64_t>(orr) * kChN2 + gcol + 16 * h2 + cc * 4, val.x,
                       val.y, val.z, val.w);
          }
        }
      };
      // acc2 columns of this warp: lo [64 cg, 64 cg + 64) and hi [32 cg, 32 cg + 32);
      // lo column a holds output a (a < 128) or a + 64, hi column b output
      // 128 + b (b < 64) or 256 + b (the pair's B halves, umma_wide.cu)
      {
        uint32_t q[32];
        int a = 64 * cg;
        tmem_ld32(lane_base + a, q);
        emit(q, a < 128 ? a : a + 64);
        a += 32;
        tmem_ld32(lane_base + a, q);
        emit(q, a < 128 ? a : a + 64);
        const int b = 32 * cg;
        tmem_ld32(lane_base + 256 + b, q);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cl(acc2e_lead);
        emit(q, b < 64 ? 128 + b : 256 + b);
      }
      mark(6);
    }
    if (elect) bulk_wait0();
    if (TR && p.trace && warp == 2 && lane == 0) {
      for (int i = 0; i < 7; ++i) p.trace[blockIdx.x * kChTrace + 8 + i] = te[i];
      p.trace[blockIdx.x * kChTrace + 15] = clock64() - tk0;
      p.trace[blockIdx.x * kChTrace + 16] = te[7];
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

unsigned long long* g_chain_trace[2] = {nullptr, nullptr};
unsigned long long* chain_trace_buf(bool bwd) {
  static const bool on = [] {
    const char* e = std::getenv("HXM_CHAIN_TRACE");
    return e && e[0] == '1';
  }();
  if (!on) return nullptr;
  if (!g_chain_trace[bwd]) {
    void* ptr = nullptr;
    if (cudaMalloc(&ptr, 1024 * kChTrace * 8) != cudaSuccess) return nullptr;
    cudaMemset(ptr, 0, 1024 * kChTrace * 8);
    g_chain_trace[bwd] = static_cast<unsigned long long*>(ptr);
  }
  return g_chain_trace[bwd];
}

// Opt-in (HXM_CHAIN=1 forward, HXM_CHAIN_BWD=1 backward): measured on c2
// the chains are bit-identical but not faster than the two-kernel paths they
// replace (forward -1 %, backward +2.5 % step time) -- the stash epilogues,
// not HBM, bound these GEMMs (profiles/r2_notes.md 5-8)
bool chain_on(bool bwd) {
  static const bool fwd_on = [] {
    const char* e = std::getenv("HXM_CHAIN");
    return e && e[0] == '1';
  }();
  static const bool bwd_on = [] {
    const char* e = std::getenv("HXM_CHAIN_BWD");
    return e && e[0] == '1';
  }();
  return bwd ? bwd_on : fwd_on;
}

}  // namespace

bool umma_chain_ok(bool bwd, int64_t d_in, int64_t hidden, int64_t d_out, int tile_rows) {
  // GEMM2's output width is 384 (acc2 = TMEM [0, 384)); GEMM1's K is whole
  // 192-row weight stages and fits the resident A tile (<= 6 atoms)
  const int64_t k1 = bwd ? d_out : d_in, n2 = bwd ? d_in : d_out;
  return chain_on(bwd) && tile_rows == kUmma2Rows && n2 == kChN2 && k1 % 192 == 0 &&
         k1 <= 64 * kChMaxA && hidden % kChNC == 0 && hidden > 0;
}

hxm_status umma_chain(const ChainArgs& a, cudaStream_t st) {
  if (!umma_chain_ok(a.bwd, a.d_in, a.hidden, a.d_out, kUmma2Rows))
    return invalid_arg("chained layer GEMMs: unsupported shape");
  if (a.max_tiles <= 0) return HXM_OK;
  ChainParams prm{};
  const uint64_t E = static_cast<uint64_t>(a.n_experts);
  const uint64_t Di = static_cast<uint64_t>(a.d_in), H = static_cast<uint64_t>(a.hidden),
                 Do = static_cast<uint64_t>(a.d_out), R = static_cast<uint64_t>(a.rows);
  const uint64_t K1 = a.bwd ? Do : Di;
  {
    const uint64_t dims[2] = {K1, R};
    const uint64_t strides[1] = {K1 * 2};
    const uint32_t box[2] = {64, 128};
    if (!make_map(&prm.tmA, a.a, 2, dims, strides, box))
      return invalid_arg("chained layer GEMMs: cannot encode the A map");
  }
  {
    const uint64_t dims[4] = {64, Di, H / 64, E};
    const uint64_t strides[3] = {H * 2, 128, Di * H * 2};
    const uint32_t box[4] = {64, 192, 1, 1};
    if (!make_map(&prm.tmW1, a.w1, 4, dims, strides, box))
      return invalid_arg("chained layer GEMMs: cannot encode the W1 map");
  }
  {
    const uint64_t dims[4] = {64, H, Do / 64, E};
    const uint64_t strides[3] = {Do * 2, 128, H * Do * 2};
    const uint32_t box[4] = {64, 64, 3, 1};
    if (!make_map(&prm.tmW2, a.w2, 4, dims, strides, box))
      return invalid_arg("chained layer GEMMs: cannot encode the W2 map");
  }
  {
    const uint64_t dims[2] = {H, R};
    const uint64_t strides[1] = {H * 2};
    const uint32_t box[2] = {64, 128};
    const uint32_t box_s[2] = {64, 32};
    if (!make_map(&prm.tmF, a.chunk_out, 2, dims, strides, box) ||
        !make_map(&prm.tmFs, a.chunk_out, 2, dims, strides, box_s))
      return invalid_arg("chained layer GEMMs: cannot encode the stash map");
    if (!make_map(&prm.tmD, a.dact, 2, dims, strides, box) ||
        !make_map(&prm.tmDs, a.dact, 2, dims, strides, box_s))
      return invalid_arg("chained layer GEMMs: cannot encode the F' stash map");
  }
  {
    // F' by TMA through the chunk buffer: the backward's default (per-row
    // loads of the stash throttle the LSU); the forward stores F' per row
    // (faster there: the extra store / read-back barrier pair costs more)
    static const int fpt = [] {
      const char* e = std::getenv("HXM_CHAIN_FPT");
      return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    prm.fp_tma = fpt >= 0 ? fpt : (a.bwd ? 1 : 0);
  }
  prm.dact = static_cast<__nv_bfloat16*>(a.dact);
  prm.b1 = a.bwd ? nullptr : a.b1;
  prm.b2 = a.bwd ? nullptr : a.b2;
  prm.y = a.out;
  prm.colsum = a.bwd ? a.colsum : nullptr;
  prm.omap = a.omap;
  prm.tiles = a.tiles;
  prm.n_tiles = a.n_tiles;
  prm.H = static_cast<int>(H);
  prm.n_a1 = static_cast<int>(K1 / 64);
  prm.n_g1 = static_cast<int>(K1 / 192);
  prm.trace = chain_trace_buf(a.bwd);
  using Kern = void (*)(ChainParams);
  int ai = a.bwd ? 3 : a.act == HXM_ACT_GELU ? 0 : a.act == HXM_ACT_RELU ? 1 : 2;
  const Kern kerns[4] = {umma_chain_kernel<HXM_ACT_GELU, false, false>,
                         umma_chain_kernel<HXM_ACT_RELU, false, false>,
                         umma_chain_kernel<HXM_ACT_IDENTITY, false, false>,
                         umma_chain_kernel<-1, true, false>};
  const Kern tkerns[4] = {umma_chain_kernel<HXM_ACT_GELU, false, true>, nullptr, nullptr,
                          umma_chain_kernel<-1, true, true>};
  const Kern kern = prm.trace && tkerns[ai] ? tkerns[ai] : kerns[ai];
  if (kern == tkerns[ai]) ai += 4;
  static bool attr_set[64][8] = {};
  int dev = 0;
  HXM_TRY_CUDA(cudaGetDevice(&dev));
  dev = dev < 64 ? dev : 63;
  if (!attr_set[dev][ai]) {
    HXM_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kChSmem));
    attr_set[dev][ai] = true;
  }
  const int sms = sm_count();
  if (sms <= 0) return invalid_arg("tcgen05 path: no CUDA device");
  const int grid = std::max(1, std::min(sms / 2, a.max_tiles)) * 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kChThreads);
  cfg.dynamicSmemBytes = kChSmem;
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

// debug: the per-CTA wait totals of the last chained launch (HXM_CHAIN_TRACE=1)
extern "C" int hxm_debug_chain_trace(int bwd, unsigned long long* out, int n_ctas) {
  unsigned long long* b = hxm::g_chain_trace[bwd ? 1 : 0];
  if (!b) return -1;
  return cudaMemcpy(out, b, static_cast<size_t>(n_ctas) * hxm::kChTrace * 8,
                    cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -1;
}
