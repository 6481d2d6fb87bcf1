// ops.cu -- C ABI of the operator-level API (replaces es_ops.hpp:37-65).
//
// Each call validates shapes on the host in the reference's order
// (es_ops.cpp:140-165 for esmm, 180-186 ess, 193-201 estmm, 210-221 esfk),
// cuts the caller's ReIndex into segment tiles on the device (no host sync,
// N' is read from idx[E] by the tiler), then launches the expert-specific
// kernels.
#include "kernels.cuh"
#include "routing.cuh"

namespace hxm {

int esmm_tile_rows(hxm_dtype dt, int64_t d1, int64_t d2) {
  return (dt == HXM_BF16 && umma_supports_esmm(d1, d2)) ? kUmmaRows : kSimtRows;
}

hxm_status launch_esmm(hxm_dtype dt, const EsmmArgs& a, cudaStream_t st) {
  ProfScope ps(st, a.label ? a.label : "esmm", a.work, WORK_FLOP, a.bytes);
  if (a.tile_rows == kUmmaRows || a.tile_rows == kUmma2Rows) {
    if (dt != HXM_BF16 || !umma_supports_esmm(a.d1, a.d2))
      return invalid_arg("esmm: 128-row tiles need the tcgen05 kernel");
    return umma_esmm(a, st);
  }
  if (a.tile_rows > kSimtRows) return invalid_arg("esmm: bad tile rows");
  if (a.peer) return invalid_arg("esmm: the fused reduce-scatter needs the tcgen05 path");
  return simt_esmm(dt, a, st);
}

hxm_status launch_estmm(hxm_dtype dt, const EstmmArgs& a, cudaStream_t st) {
  ProfScope ps(st, a.label ? a.label : "estmm", a.work, WORK_FLOP, a.bytes);
  if (a.peer) {  // owners zero their shards; every tile reduces
    if (dt != HXM_BF16 || !umma_supports_estmm(a.d1, a.d2))
      return invalid_arg("estmm: the fused reduce-scatter needs the tcgen05 path");
    return umma_estmm(a, st);
  }
  if (!a.skip_zero_split)
    HXM_RETURN_IF(zero_split_experts(a.tiles, a.n_tiles, a.max_tiles, a.d1 * a.d2, a.out, st));
  if (dt == HXM_BF16 && umma_supports_estmm(a.d1, a.d2)) return umma_estmm(a, st);
  return simt_estmm(dt, a, st);
}

namespace {

struct OpWs {
  SegTile* tiles;
  int32_t* tile_off;
  int32_t* n_tiles;
  SegTile* ktiles;  // estmm chunks
  int32_t* ktile_off;
  int32_t* n_ktiles;
  SegTile* ktiles64;  // bf16 ESTMM chunks over the relayout
  SegTile* etiles;  // ess tiles
  int32_t* etile_off;
  int32_t* n_etiles;
  float* partial;
  void* sorted;  // bf16 ESMM: the expert-sorted copy of the A rows (np_bound x d1)
  void* sorted2;   // bf16 ESTMM: the second operand, 64-position relayout
  int32_t* idx64;  // bf16 ESTMM: segment offsets of the relayout
  int64_t bound64;
  int max_tiles, max_ktiles, max_etiles, max_ktiles64;
};

OpWs carve(Arena& ar, int64_t np_bound, int64_t E, int64_t d1, int64_t d2) {
  OpWs w{};
  w.max_tiles = static_cast<int>(max_tiles(np_bound, E, kSimtRows));
  w.max_ktiles = static_cast<int>(max_tiles(np_bound, E, kEstmmSplit));
  w.max_etiles = static_cast<int>(max_tiles(np_bound, E, kEssRows));
  w.tiles = ar.take<SegTile>(w.max_tiles);
  w.tile_off = ar.take<int32_t>(E + 1);
  w.n_tiles = ar.take<int32_t>(1);
  w.ktiles = ar.take<SegTile>(w.max_ktiles);
  w.ktile_off = ar.take<int32_t>(E + 1);
  w.n_ktiles = ar.take<int32_t>(1);
  w.etiles = ar.take<SegTile>(w.max_etiles);
  w.etile_off = ar.take<int32_t>(E + 1);
  w.n_etiles = ar.take<int32_t>(1);
  w.partial = ar.take<float>(static_cast<size_t>(w.max_etiles) * std::max(d1, d2));
  // 2-byte rows: only the bf16 tcgen05 path sorts its operands.  The ESTMM
  // relayout pads every segment to 64 positions: at most np_bound + 63 E rows.
  w.bound64 = np_bound + 63 * E;
  w.sorted = ar.take<char>(static_cast<size_t>(std::max<int64_t>(w.bound64, 1)) *
                           std::max(d1, d2) * 2);
  // (both widths: hxm_esfk runs the ESMM with d1 and d2 swapped on one workspace)
  w.sorted2 = ar.take<char>(static_cast<size_t>(std::max<int64_t>(w.bound64, 1)) *
                            std::max(d1, d2) * 2);
  w.idx64 = ar.take<int32_t>(E + 1);
  w.max_ktiles64 = static_cast<int>(max_tiles(w.bound64, E, kEstmmSplit));
  w.ktiles64 = ar.take<SegTile>(w.max_ktiles64);
  return w;
}

bool valid_dtype(hxm_dtype dt) { return dt == HXM_F32 || dt == HXM_BF16; }

}  // namespace
}  // namespace hxm

using namespace hxm;

extern "C" {

size_t hxm_op_workspace_bytes(int64_t n, int64_t E, int64_t np_bound, int64_t d1,
                              int64_t d2) {
  (void)n;
  Arena ar(nullptr, 0);
  carve(ar, np_bound, E, d1, d2);
  // the same workspace also serves hxm_esfk's expert-sorted layout
  return std::max(ar.used, esfk_ws_bytes(np_bound, E, d1, d2));
}

hxm_status hxm_esmm(hxm_dtype dt, const void* x, int64_t n, int64_t d1, const void* w,
                    int64_t E, int64_t d2, int w_trans, const float* bias,
                    const int64_t* v, const int64_t* idx, int64_t np_bound,
                    hxm_out_mode mode, float* dest, void* ws, size_t ws_bytes,
                    hxm_stream_t stream) {
  if (!valid_dtype(dt)) return invalid_arg("esmm: unknown dtype");
  // es_ops.cpp:143 check_reindex is structural; v/idx live on the device
  if (!v || !idx || E < 1) return shape_error("es-ops: malformed re-index vector");
  if (n < 0 || d1 < 0 || d2 < 0) return shape_error("esmm: negative extent");
  if (!dest) {  // es_ops.cpp:156-161
    return invalid_arg(mode == HXM_ACCUMULATE ? "esmm: Accumulate mode requires a destination"
                                              : "esmm: destination is null");
  }
  if (n > 0x7fffffffLL || np_bound > 0x7fffffffLL) return invalid_arg("esmm: n too large");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Arena ar(ws, ws_bytes);
  OpWs o = carve(ar, np_bound, E, d1, d2);
  if (ar.overflow) return invalid_arg("esmm: workspace too small");
  if (n == 0 || d2 == 0) return HXM_OK;
  const int rows = esmm_tile_rows(dt, d1, d2);
  HXM_RETURN_IF(launch_tiles<int64_t>(idx, E, rows, false, o.tiles, o.tile_off, o.n_tiles, st));
  EsmmArgs a{};
  a.a = x;
  a.amap = map_v64(v);
  a.a_rows = n;
  if (rows == kUmmaRows) {
    // tcgen05 path: one bandwidth-bound gather of the routed rows into
    // expert-sorted order, then dense TMA tiles (a TMA gather4 request per
    // 4 rows is request-rate bound); rows past a segment's end
    // belong to the next expert and are masked by the epilogue's row map
    HXM_RETURN_IF(launch_gather_rows64(dt, x, map_v64(v), d1, idx, static_cast<int>(E),
                                       np_bound, o.sorted, st));
    a.a = o.sorted;
    a.amap = map_dense();
    a.a_rows = std::max<int64_t>(np_bound, 1);
  }
  a.n_experts = E;
  a.w = w;
  a.w_trans = w_trans;
  a.d1 = d1;
  a.d2 = d2;
  a.bias = bias;
  a.tiles = o.tiles;
  a.n_tiles = o.n_tiles;
  a.max_tiles = static_cast<int>(max_tiles(np_bound, E, rows));
  a.tile_rows = rows;
  a.epi = mode == HXM_ACCUMULATE ? EPI_ACCUM : EPI_WRITE;
  a.out_f32 = dest;
  a.omap = map_v64(v);
  return launch_esmm(dt, a, st);
}

hxm_status hxm_ess(hxm_dtype dt, const void* x, int64_t n, int64_t d, const int64_t* v,
                   const int64_t* idx, int64_t E, int64_t np_bound, float* out, void* ws,
                   size_t ws_bytes, hxm_stream_t stream) {
  if (!valid_dtype(dt)) return invalid_arg("ess: unknown dtype");
  if (!v || !idx || E < 1) return shape_error("es-ops: malformed re-index vector");
  if (n < 0 || d < 0) return shape_error("ess: negative extent");
  if (!out) return invalid_arg("ess: output is null");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Arena ar(ws, ws_bytes);
  OpWs o = carve(ar, np_bound, E, d, d);
  if (ar.overflow) return invalid_arg("ess: workspace too small");
  if (d == 0) return HXM_OK;
  HXM_RETURN_IF(launch_tiles<int64_t>(idx, E, kEssRows, false, o.etiles, o.etile_off,
                                      o.n_etiles, st));
  EssArgs a{};
  a.x = x;
  a.map = map_v64(v);
  a.d = d;
  a.tiles = o.etiles;
  a.n_tiles = o.n_etiles;
  a.tile_off = o.etile_off;
  a.max_tiles = o.max_etiles;
  a.n_experts = static_cast<int>(E);
  a.partial = o.partial;
  a.out = out;
  return launch_ess(dt, a, st);
}

hxm_status hxm_estmm(hxm_dtype dt, const void* x1, const void* x2, int64_t n, int64_t d1,
                     int64_t d2, const int64_t* v, const int64_t* idx, int64_t E,
                     int64_t np_bound, float* out, void* ws, size_t ws_bytes,
                     hxm_stream_t stream) {
  if (!valid_dtype(dt)) return invalid_arg("estmm: unknown dtype");
  if (!v || !idx || E < 1) return shape_error("es-ops: malformed re-index vector");
  if (n < 0 || d1 < 0 || d2 < 0) return shape_error("estmm: negative extent");
  if (!out) return invalid_arg("estmm: output is null");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Arena ar(ws, ws_bytes);
  OpWs o = carve(ar, np_bound, E, d1, d2);
  if (ar.overflow) return invalid_arg("estmm: workspace too small");
  if (d1 == 0 || d2 == 0) return HXM_OK;
  if (dt == HXM_BF16 && umma_supports_estmm(d1, d2)) {
    // tcgen05 path: both operands gathered into a 64-position segment
    // layout (one bandwidth-bound pass), then dense TMA tiles instead of a
    // gather4 request per 4 rows
    HXM_RETURN_IF(launch_estmm_relayout(x1, d1, x2, d2, v, idx, static_cast<int>(E), o.bound64,
                                        o.idx64, o.sorted, o.sorted2, st));
    HXM_RETURN_IF(launch_tiles<int32_t>(o.idx64, E, kEstmmChunk, true, o.ktiles64, o.ktile_off,
                                        o.n_ktiles, st, kEstmmSplit));
    EstmmArgs a{};
    a.x1 = o.sorted;
    a.m1 = map_dense();
    a.x2 = o.sorted2;
    a.m2 = map_dense();
    a.x1_rows = o.bound64;
    a.x2_rows = o.bound64;
    a.d1 = d1;
    a.d2 = d2;
    a.tiles = o.ktiles64;
    a.n_tiles = o.n_ktiles;
    a.max_tiles = o.max_ktiles64;
    a.n_experts = static_cast<int>(E);
    a.out = out;
    return launch_estmm(dt, a, st);
  }
  HXM_RETURN_IF(launch_tiles<int64_t>(idx, E, kEstmmChunk, true, o.ktiles, o.ktile_off,
                                      o.n_ktiles, st));
  EstmmArgs a{};
  a.x1 = x1;
  a.m1 = map_v64(v);
  a.x2 = x2;
  a.m2 = map_v64(v);
  a.x1_rows = n;
  a.x2_rows = n;
  a.d1 = d1;
  a.d2 = d2;
  a.tiles = o.ktiles;
  a.n_tiles = o.n_ktiles;
  a.max_tiles = o.max_ktiles;
  a.n_experts = static_cast<int>(E);
  a.out = out;
  return launch_estmm(dt, a, st);
}

hxm_status hxm_esfk(hxm_dtype dt, const void* x, const void* g, int64_t n, int64_t d1,
                    int64_t d2, const void* w_t, int w_transposed, const int64_t* v,
                    const int64_t* idx, int64_t E, int64_t np_bound, float* grad_x,
                    float* grad_b, float* grad_w, void* ws, size_t ws_bytes,
                    hxm_stream_t stream) {
  // es_ops.cpp:210-221 checks (structure / token counts are the host
  // wrapper's; here: extents and buffers)
  if (!valid_dtype(dt)) return invalid_arg("esfk: unknown dtype");
  if (!v || !idx || E < 1) return shape_error("es-ops: malformed re-index vector");
  if (n < 0 || d1 < 0 || d2 < 0) return shape_error("esfk: negative extent");
  if (!grad_x || !grad_b || !grad_w || !w_t) return invalid_arg("esfk: null tensor");
  if (n > 0x7fffffffLL || np_bound > 0x7fffffffLL) return invalid_arg("esfk: n too large");
  if (n > 0 && (!x || !g)) return invalid_arg("esfk: null tensor");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (d1 == 0 || d2 == 0) return HXM_OK;
  // the reference's combined work list (grad-x tiles, grad-b tiles, grad-W
  // tiles) as one device work list: bf16 -> gather/ESS prologue + one
  // tcgen05 launch running grad-x and grad-W side by side (esfk.cu); fp32 ->
  // one SIMT launch (simt.cu)
  if (dt == HXM_BF16 && esfk_umma_ok(d1, d2)) {
    if (ws_bytes < esfk_ws_bytes(np_bound, E, d1, d2)) return invalid_arg("esfk: workspace too small");
    return umma_esfk(x, g, n, d1, d2, w_t, w_transposed, v, idx, E, np_bound, grad_x, grad_b,
                     grad_w, ws, ws_bytes, st);
  }
  ProfScope ps(st, "esfk_simt", 6.0 * n * d1 * d2, WORK_FLOP);
  return simt_esfk(dt, x, g, n, d1, d2, w_t, w_transposed, v, idx, E, np_bound, grad_x, grad_b,
                   grad_w, st);
}

}  // extern "C"
