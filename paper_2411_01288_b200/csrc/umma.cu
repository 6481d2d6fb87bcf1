// umma.cu -- tcgen05 (5th-gen tensor core) expert-specific GEMMs for sm_100a:
// bf16 operands staged by TMA (tile and tile::gather4), fp32 accumulators in
// TMEM, one persistent warp-specialised kernel per operator.
//
//   ESMM  (es_ops.cpp:47-81):   out[p] = A[row(p)] . W[e] (+ b[e]) over 128-row
//          segment tiles of one expert; A rows gathered by TMA gather4 straight
//          from the token-order tensor (no dispatch copy), or read as dense
//          tiles from the expert-sorted stash.  W read MN-major (W[e] is D1 x D2
//          row-major) or K-major (W^T use: no transpose_experts copy).
//   ESTMM (es_ops.cpp:106-128): out[e] = X1^T X2 over the expert's token
//          positions (K = tokens, variable), both operands MN-major, split-K
//          over <= kEstmmChunk-position chunks with fp32 red.add for split
//          experts.
//
// Warp roles (320 threads): warp 0 = TMA producer (all 32 lanes issue gather4),
// warp 1 = TMEM allocator + single-thread tcgen05.mma issuer, warps 2..9 =
// epilogue (TMEM -> registers -> bias / activation / stores).  Pipelines:
// smem ring full/empty (TMA <-> MMA) and a double-buffered TMEM accumulator
// full/empty (MMA <-> epilogue), so tile i's epilogue overlaps tile i+1's MMA.
#include "umma_impl.cuh"

namespace hxm {

bool umma_supports_esmm(int64_t d1, int64_t d2) {
  return d1 > 0 && d2 > 0 && d1 % 64 == 0 && d2 % 64 == 0 && d1 < (1 << 30) && d2 < (1 << 30);
}
bool umma_supports_estmm(int64_t d1, int64_t d2) { return umma_supports_esmm(d1, d2); }
int umma_pick_bn(int64_t n) { return pick_bn(n); }
int umma_pick_bn2(int64_t n, bool b_mn) { return pick_bn2(n, b_mn); }
bool umma2_supports_esmm(int64_t d1, int64_t d2, bool w_trans) {
  return umma_supports_esmm(d1, d2) && pick_bn2(d2, !w_trans) > 0;
}

hxm_status umma_esmm(const EsmmArgs& a, cudaStream_t st) {
  if (a.max_tiles <= 0) return HXM_OK;
  // 384-wide reduction GEMMs (c2's fwd2 / gx): whole-tile CTA pairs
  if (umma_wide_ok(a)) return umma_wide_esmm(a, st);
  const int CG = a.tile_rows == kUmma2Rows ? 2 : 1;
  if (a.tile_rows != kUmmaRows && CG == 1)
    return invalid_arg("umma_esmm: tiles must have 128 (or 256) rows");
  const bool gather = a.amap.kind != MAP_DENSE;
  if (CG == 2 && (gather || !umma2_supports_esmm(a.d1, a.d2, a.w_trans)))
    return invalid_arg("umma_esmm: 256-row (CTA-pair) tiles need dense A and BN | N");
  const int bn = CG == 2 ? pick_bn2(a.d2, !a.w_trans) : pick_bn(a.d2);
  UParams prm{};
  HXM_RETURN_IF(prep_esmm(a, CG, bn, prm));
  const int work = a.max_tiles * prm.n_nt;
  if (CG == 2) {
    if (a.epi == EPI_FWD_ACT) return launch_fwd_act<2>(a.act, bn, prm, work, st);
    if (a.epi == EPI_BWD_ACT) return launch_bn_any<2, 2>(bn, prm, work, st);
    return launch_bn_any<0, 2>(bn, prm, work, st);
  }
  if (a.epi == EPI_FWD_ACT) return launch_fwd_act<1>(a.act, bn, prm, work, st);
  if (a.epi == EPI_BWD_ACT) return launch_bn_any<2, 1>(bn, prm, work, st);
  return launch_bn_any<0, 1>(bn, prm, work, st);
}

hxm_status umma_estmm(const EstmmArgs& a, cudaStream_t st) {
  if (a.max_tiles <= 0) return HXM_OK;
  // 384-wide outputs (c2's gW2, and gW1 computed transposed): whole-tile pairs
  if (umma_wide_estmm_ok(a)) return umma_wide_estmm(a, st);
  if (a.trans_out) return invalid_arg("umma_estmm: transposed output needs the whole-tile kernel");
  const bool ga = a.m1.kind != MAP_DENSE, gb = a.m2.kind != MAP_DENSE;
  // CTA pairs (M = 256 output rows per pair) when both operands are dense
  // and the output rows tile evenly
  const char* env = std::getenv("HXM_CTA_PAIR");  // 0: single-CTA tiles everywhere
  const bool pair_ok = !(env && env[0] == '0');
  const int CG = (pair_ok && !ga && !gb && a.d1 % 256 == 0 && pick_bn2(a.d2, true) > 0) ? 2 : 1;
  const int bn = CG == 2 ? pick_bn2(a.d2, true) : pick_bn(a.d2);
  UParams prm{};
  HXM_RETURN_IF(prep_estmm(a, CG, bn, prm));
  const int work = a.max_tiles * prm.n_mt * prm.n_nt;
  if (CG == 2) return launch_bn_any<3, 2>(bn, prm, work, st);
  return launch_bn_any<3, 1>(bn, prm, work, st);
}

}  // namespace hxm

extern "C" void hxm_debug_trace(unsigned long long* out) {
  if (hxm::g_trace)
    cudaMemcpy(out, hxm::g_trace, 148 * 64 * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}
