// layer.cu -- MoE layer forward / backward on the device.
//
// Replaces moekit::moe_forward / moe_backward (reference
// core/src/moe_layer.cpp:30-122).  Semantics kept exactly:
//   y      = sum_i ESMM(F(ESMM(x, W1, b1, R_i)), W2, b2, R_i)   (b2 once per choice)
//   gb2    = sum_i ESS(g_y, R_i)             gW2 = sum_i ESTMM(y2_i, g_y, R_i)
//   g_y2_i = ESMM(g_y, W2^T, R_i)            g_y1_i = g_y2_i * F'(y1_i)
//   gb1    = sum_i ESS(g_y1_i, R_i)          gW1 = sum_i ESTMM(x, g_y1_i, R_i)
//   gx     = sum_i ESMM(g_y1_i, W1^T, R_i)
// B200-first changes (not a transliteration):
//  * the k choices share ONE expert-grouped index over k*N (token, choice)
//    slots (hxm::build_reindex_slots), so each expert's weights are streamed
//    once per layer and every GEMM is one launch;
//  * the stash y1/y2 and g_y1 live in expert-sorted row order (padded to 64
//    positions per expert, pads written as zero rows), so only x and g_y --
//    which arrive in token order -- are gathered; the sorted operands are
//    read with dense tiles;
//  * W^T is never materialised (transpose_experts, moe_layer.cpp:91-92): the
//    GEMM reads W K-major;
//  * y and gx accumulate over choices with fp32 reductions into zeroed
//    buffers (the memory-efficient scheme, moe_layer.cpp:61-63).
#include <memory>

#include "kernels.cuh"
#include "routing.cuh"

namespace hxm {

int esmm_tile_rows(hxm_dtype dt, int64_t d1, int64_t d2);

namespace {

constexpr int64_t kSortedBlk = 64;  // internal segment padding (UMMA K-step)

struct LayerWs {
  int32_t* v;     // combined index, slot ids
  int32_t* idx;   // E+1
  void* rws;      // reindex scratch
  size_t rws_bytes;
  SegTile* tiles_a;  // ESMM tiles over in=D_i (both GEMMs share rows)
  int32_t* tiles_a_off;
  int32_t* n_tiles_a;
  SegTile* ktiles;  // ESTMM chunks
  int32_t* ktiles_off;
  int32_t* n_ktiles;
  SegTile* etiles;  // ESS tiles
  int32_t* etiles_off;
  int32_t* n_etiles;
  float* partial;
  int32_t* done;  // bwd prologue: per-expert ESS arrival counters
  void* xs;   // x in expert-sorted slot order (forward stash)
  void* gys;  // g_y in expert-sorted slot order (backward scratch)
  void* y1s;
  void* y2s;
  void* g1s;
  float* colsum;  // tcgen05 path: per-(tile, CTA) column sums of g_y1 (fused gb1)
  int64_t bound;
  int max_tiles_a, max_ktiles, max_etiles;
  int rows_a;
};

size_t esize(int32_t dt) { return dt == HXM_BF16 ? 2 : 4; }
// partial rows of the fused gb1 column sums per tile
int colsum_parts(int rows_a) { return rows_a >= kUmmaRows ? (rows_a / kUmmaRows) * 4 : 1; }

LayerWs carve(Arena& ar, const hxm_layer_desc& d) {
  LayerWs w{};
  const int64_t slots = d.k * d.n_tokens;
  // expert-specific: every slot plus < 64 pad rows per expert; conventional
  // baseline: exactly `capacity` rows per expert
  w.bound = d.capacity > 0 ? d.n_experts * static_cast<int64_t>(d.capacity)
                           : slots + d.n_experts * (kSortedBlk - 1);
  const hxm_dtype dt = static_cast<hxm_dtype>(d.dtype);
  // all four layer GEMMs share one tile table, so they must agree on the
  // tile rows: 128 (tcgen05) when every shape is TMA-describable
  const bool umma = dt == HXM_BF16 && umma_supports_esmm(d.d_in, d.hidden) &&
                    umma_supports_esmm(d.hidden, d.d_out) &&
                    umma_supports_esmm(d.d_out, d.hidden) &&
                    umma_supports_esmm(d.hidden, d.d_in);
  // 256-row tiles on CTA pairs (cta_group::2) when every layer GEMM's B
  // splits into whole halves; HXM_CTA_PAIR=0 forces single-CTA tiles
  const char* env = std::getenv("HXM_CTA_PAIR");
  const bool pair_ok = !(env && env[0] == '0');
  const bool umma2 = umma && pair_ok && umma2_supports_esmm(d.d_in, d.hidden, false) &&
                     umma2_supports_esmm(d.hidden, d.d_out, false) &&
                     umma2_supports_esmm(d.d_out, d.hidden, true) &&
                     umma2_supports_esmm(d.hidden, d.d_in, true);
  w.rows_a = umma2 ? kUmma2Rows : (umma ? kUmmaRows : kSimtRows);
  w.v = ar.take<int32_t>(w.bound);
  w.idx = ar.take<int32_t>(d.n_experts + 1);
  w.rws_bytes = reindex_ws_bytes(slots, d.n_experts);
  w.rws = ar.take<char>(w.rws_bytes);
  w.max_tiles_a = static_cast<int>(max_tiles(w.bound, d.n_experts, kSimtRows));
  w.tiles_a = ar.take<SegTile>(w.max_tiles_a);
  w.tiles_a_off = ar.take<int32_t>(d.n_experts + 1);
  w.n_tiles_a = ar.take<int32_t>(1);
  w.max_ktiles = static_cast<int>(max_tiles(w.bound, d.n_experts, kEstmmSplit));
  w.ktiles = ar.take<SegTile>(w.max_ktiles);
  w.ktiles_off = ar.take<int32_t>(d.n_experts + 1);
  w.n_ktiles = ar.take<int32_t>(1);
  w.max_etiles = static_cast<int>(max_tiles(w.bound, d.n_experts, kEssRows));
  w.etiles = ar.take<SegTile>(w.max_etiles);
  w.etiles_off = ar.take<int32_t>(d.n_experts + 1);
  w.n_etiles = ar.take<int32_t>(1);
  w.done = ar.take<int32_t>(d.n_experts);
  w.partial = ar.take<float>(static_cast<size_t>(w.max_etiles) * std::max(d.hidden, d.d_out));
  const size_t stash = static_cast<size_t>(w.bound) * d.hidden * esize(d.dtype);
  w.xs = ar.take<char>(static_cast<size_t>(w.bound) * d.d_in * esize(d.dtype));
  w.gys = ar.take<char>(static_cast<size_t>(w.bound) * d.d_out * esize(d.dtype));
  w.y1s = ar.take<char>(stash);
  w.y2s = ar.take<char>(stash);
  w.g1s = ar.take<char>(stash);
  const char* fuse = std::getenv("HXM_FUSE_GB1");  // 0: separate ESS pass for gb1
  // fused gb1 column sums: tcgen05 (per tile, CTA and TMEM lane group) or the
  // dense fp32 SIMT kernel (one partial row per 64-row tile)
  const bool simt_cs = w.rows_a == kSimtRows && dt == HXM_F32 && d.hidden % 4 == 0 &&
                       d.d_out % 4 == 0;
  if ((w.rows_a >= kUmmaRows || simt_cs) && !(fuse && fuse[0] == '0'))
    w.colsum = ar.take<float>(static_cast<size_t>(max_tiles(w.bound, d.n_experts, w.rows_a)) *
                              colsum_parts(w.rows_a) * d.hidden);
  return w;
}

hxm_status check_desc(const hxm_layer_desc* d) {
  if (!d) return invalid_arg("moe layer: null descriptor");
  if (d->dtype != HXM_F32 && d->dtype != HXM_BF16) return invalid_arg("moe layer: unknown dtype");
  if (d->activation < 0 || d->activation > 2) return invalid_arg("moe layer: unknown activation");
  if (d->k < 1) return shape_error("RoutingChoice: expected k assignment vectors");
  if (d->k > d->n_experts) return invalid_arg("RoutingChoice: k exceeds expert count");
  if (d->n_tokens < 0 || d->d_in < 1 || d->hidden < 1 || d->d_out < 1)
    return shape_error("moe layer: extents must be positive");
  if (d->k * d->n_tokens + d->n_experts * kSortedBlk > 0x7fffffffLL)
    return invalid_arg("moe layer: k*N exceeds int32 slot range");
  if (d->capacity < 0 || d->capacity % kSortedBlk != 0)
    return invalid_arg("moe layer: capacity must be 0 or a positive multiple of 64");
  if (static_cast<int64_t>(d->capacity) * d->n_experts > 0x7fffffffLL)
    return invalid_arg("moe layer: capacity * E exceeds int32 row range");
  if (d->weight_shards < 0 || d->weight_shards > 64)
    return invalid_arg("moe layer: weight_shards must be 0..64");
  return HXM_OK;
}

// shard-major weights: every GEMM that reads W must keep its boxes inside
// one shard (h % 64 for the K-split uses; h % the CTA's B width for the
// N-split ones) -- the tile widths are those the tcgen05 launchers pick
bool shards_ok(const hxm_layer_desc& d, const LayerWs& w, int64_t P) {
  if (P <= 1) return true;
  if (w.rows_a < kUmmaRows || d.hidden % P != 0) return false;
  const int64_t h = d.hidden / P;
  if (h % 64 != 0) return false;
  const int CG = w.rows_a == kUmma2Rows ? 2 : 1;
  // N = H for fwd1 (W1, MN-major) and bwd_act (W2^T, K-major)
  const int bn_f = CG == 2 ? umma_pick_bn2(d.hidden, true) : umma_pick_bn(d.hidden);
  const int bn_b = CG == 2 ? umma_pick_bn2(d.hidden, false) : umma_pick_bn(d.hidden);
  return bn_f > 0 && bn_b > 0 && h % (bn_f / CG) == 0 && h % (bn_b / CG) == 0;
}

// stash export: sorted row p (slot s = choice*N + t) -> token-order fp32
template <class T>
__global__ void export_kernel(const int32_t* v, const int32_t* idx, int E, int64_t n,
                              int choice, int64_t H, const T* y1s, const T* y2s, float* y1,
                              float* y2) {
  const int64_t np = idx[E];
  for (int64_t p = blockIdx.x; p < np; p += gridDim.x) {
    const int s = v[p];
    if (s < 0 || s / n != choice) continue;
    const int64_t t = s % n;
    for (int64_t h = threadIdx.x; h < H; h += blockDim.x) {
      y1[t * H + h] = to_f32(y1s[p * H + h]);
      y2[t * H + h] = to_f32(y2s[p * H + h]);
    }
  }
}

}  // namespace
}  // namespace hxm

using namespace hxm;

extern "C" {

size_t hxm_layer_workspace_bytes(const hxm_layer_desc* d) {
  if (check_desc(d) != HXM_OK) return 0;
  Arena ar(nullptr, 0);
  carve(ar, *d);
  return ar.used;
}

int hxm_layer_path(const hxm_layer_desc* d) {
  if (check_desc(d) != HXM_OK) return -1;
  Arena ar(nullptr, 0);
  const LayerWs w = carve(ar, *d);
  return w.rows_a == kUmma2Rows ? 2 : (w.rows_a == kUmmaRows ? 1 : 0);
}

int hxm_layer_weight_shards_ok(const hxm_layer_desc* d, int32_t n_shards) {
  if (check_desc(d) != HXM_OK) return 0;
  Arena ar(nullptr, 0);
  const LayerWs w = carve(ar, *d);
  return shards_ok(*d, w, n_shards) ? 1 : 0;
}

uint64_t hxm_layer_forward_macs(const hxm_layer_desc* d) {
  // rows the GEMMs compute per weight: every routed slot (expert-specific)
  // or E x capacity (conventional baseline, padding included)
  const uint64_t rows = d->capacity > 0 ? static_cast<uint64_t>(d->n_experts) * d->capacity
                                        : static_cast<uint64_t>(d->k) * d->n_tokens;
  return rows * (d->d_in * d->hidden + d->hidden * d->d_out);
}

}  // extern "C"

namespace hxm {
namespace {
hxm_status check_peer(const hxm_peer_rows* pr, const hxm_layer_desc* d, const LayerWs& w,
                      const char* what) {
  if (!pr) return HXM_OK;
  if (pr->n_ranks < 1 || pr->n_ranks > HXM_MAX_PEERS || pr->rows_per_rank < 1 ||
      pr->rows_per_rank * pr->n_ranks < d->n_tokens)
    return invalid_arg(std::string(what) + ": peer rows must cover the N tokens on 1..8 ranks");
  for (int r = 0; r < pr->n_ranks; ++r)
    if (!pr->ptrs[r]) return invalid_arg(std::string(what) + ": null peer buffer");
  if (w.rows_a < kUmmaRows)
    return invalid_arg(std::string(what) + ": the fused reduce-scatter needs the bf16 tcgen05 path");
  return HXM_OK;
}
// data-centric gW shard tables: H split evenly over 1..8 ranks in spans of a
// multiple of 4 columns, every rank's shard mapped -- checked before the
// first launch so a bad table leaves no partial results behind
hxm_status check_shards(const hxm_peer_rows* pr, const hxm_layer_desc* d, const LayerWs& w,
                        const char* what) {
  if (!pr) return HXM_OK;
  const int64_t span = pr->rows_per_rank;
  if (pr->n_ranks < 1 || pr->n_ranks > HXM_MAX_PEERS || span < 1 ||
      span * pr->n_ranks != d->hidden || span % 4 != 0)
    return invalid_arg(std::string(what) +
                       ": peer shards must split H evenly over 1..8 ranks (span % 4 == 0)");
  for (int r = 0; r < pr->n_ranks; ++r)
    if (!pr->ptrs[r]) return invalid_arg(std::string(what) + ": null peer shard");
  if (w.rows_a < kUmmaRows)
    return invalid_arg(std::string(what) + ": the fused reduce-scatter needs the bf16 tcgen05 path");
  return HXM_OK;
}
}  // namespace

// y (or, with `yp`, the owners' peer rows) = the layer forward
hxm_status layer_forward(const hxm_layer_desc* d, const void* x, const void* w1,
                         const float* b1, const void* w2, const float* b2,
                         const int32_t* assignments, float* y, const hxm_peer_rows* yp,
                         void* ws, size_t ws_bytes, int32_t* status, hxm_stream_t stream) {
  HXM_RETURN_IF(check_desc(d));
  const bool tok = d->n_tokens > 0;  // token tensors may be empty (null) when N == 0
  if ((tok && (!x || !assignments || (!y && !yp))) || !w1 || !b1 || !w2 || (d->add_b2 && !b2))
    return invalid_arg("moe_forward: null tensor");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Arena ar(ws, ws_bytes);
  LayerWs w = carve(ar, *d);
  if (ar.overflow) return invalid_arg("moe_forward: workspace too small");
  if (!shards_ok(*d, w, d->weight_shards))
    return invalid_arg("moe_forward: shard-major weights unsupported for this shape");
  HXM_RETURN_IF(check_peer(yp, d, w, "moe_forward_tp"));
  const hxm_dtype dt = static_cast<hxm_dtype>(d->dtype);
  const int64_t N = d->n_tokens, E = d->n_experts, slots = d->k * N;
  // (0) one cooperative launch: routing validation, the k-choice slot index
  // (v, idx), its three tilings (ESMM tiles, ESTMM chunks, ESS tiles -- the
  // backward reuses them from the stash), y = 0 and the expert-sorted copy of
  // x, so every later GEMM reads dense tiles
  {
    FwdPrologue pro{};
    pro.a = assignments;
    pro.n_slots = slots;
    pro.n_tok = N;
    pro.k = static_cast<int>(d->k);
    pro.E = static_cast<int>(E);
    pro.blk = kSortedBlk;
    pro.capacity = d->capacity;
    pro.v = w.v;
    pro.idx = w.idx;
    pro.s0 = {w.rows_a, 0, w.tiles_a, w.tiles_a_off, w.n_tiles_a};
    pro.s1 = {kEstmmChunk, 1, w.ktiles, w.ktiles_off, w.n_ktiles, kEstmmSplit};
    pro.s2 = {kEssRows, 0, w.etiles, w.etiles_off, w.n_etiles};
    pro.x = N > 0 ? x : nullptr;
    pro.xs = w.xs;
    pro.row_bytes = d->d_in * static_cast<int64_t>(esize(d->dtype));
    pro.unit = (pro.row_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0) ? 16
               : (pro.row_bytes % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 4 == 0) ? 4 : 2;
    pro.y = y;
    pro.y_elems = yp ? 0 : N * d->d_out;  // peer rows: each owner zeroes its own
    pro.status = status;
    pro.zero_i32 = w.done;
    pro.zero_n = static_cast<int>(E);
    pro.ws = w.rws;
    pro.ws_bytes = w.rws_bytes;
    // algorithmic bytes: assignments read twice, v written, every routed
    // slot's x row read and written once, y zeroed
    const double bytes = 8.0 * slots + 4.0 * w.bound +
                         2.0 * static_cast<double>(slots) * pro.row_bytes + 4.0 * N * d->d_out;
    ProfScope ps(st, "fwd_prologue", bytes, WORK_BYTES);
    HXM_RETURN_IF(launch_fwd_prologue(pro, st));
  }
  if (N == 0) return HXM_OK;
  // the cache fill of shard-major weights overlapped the index build
  if (d->weights_ready)
    HXM_TRY_CUDA(cudaStreamWaitEvent(st, reinterpret_cast<cudaEvent_t>(d->weights_ready), 0));
  const RowMap slot = map_slot(w.v, N);
  // (1) y1 = x W1 + b1 ; y2 = F(y1)          (moe_layer.cpp:56-57)
  EsmmArgs a1{};
  a1.a = w.xs;
  a1.amap = map_dense();
  a1.a_rows = w.bound;
  a1.n_experts = E;
  a1.w = w1;
  a1.w_trans = 0;
  a1.w_shards = static_cast<int>(d->weight_shards);  // W1 [P][E][D_i][h]: N (H) split
  a1.w_split_k = 0;
  a1.d1 = d->d_in;
  a1.d2 = d->hidden;
  a1.bias = b1;
  a1.tiles = w.tiles_a;
  a1.n_tiles = w.n_tiles_a;
  a1.max_tiles = static_cast<int>(max_tiles(w.bound, E, w.rows_a));
  a1.tile_rows = w.rows_a;
  a1.epi = EPI_FWD_ACT;
  const double kn = static_cast<double>(slots);
  a1.label = "esmm_fwd1";
  a1.work = 2.0 * kn * d->d_in * d->hidden;
  const double es_ = static_cast<double>(esize(d->dtype));
  const double wbytes = static_cast<double>(E) * d->d_in * d->hidden * es_;  // W1
  const double w2bytes = static_cast<double>(E) * d->hidden * d->d_out * es_;
  // x_s read, W1 read, the two stash outputs written (real slots)
  a1.bytes = kn * d->d_in * es_ + wbytes + 2.0 * kn * d->hidden * es_;
  a1.act = d->activation;
  a1.omap = slot;
  a1.out1 = w.y1s;
  a1.out2 = w.y2s;
  if (dt == HXM_BF16 && d->weight_shards <= 1 && !yp &&
      umma_chain_ok(false, d->d_in, d->hidden, d->d_out, w.rows_a)) {
    // (1) + (2) as one chained launch: the F(y1) chunks feed the second GEMM
    // from shared memory (umma_chain.cu); the stash is written as before
    ChainArgs c{};
    c.bwd = false;
    c.a = w.xs;
    c.rows = w.bound;
    c.w1 = w1;
    c.b1 = b1;
    c.w2 = w2;
    c.b2 = d->add_b2 ? b2 : nullptr;
    c.n_experts = E;
    c.d_in = d->d_in;
    c.hidden = d->hidden;
    c.d_out = d->d_out;
    c.tiles = w.tiles_a;
    c.n_tiles = w.n_tiles_a;
    c.max_tiles = a1.max_tiles;
    c.act = d->activation;
    c.dact = w.y1s;
    c.chunk_out = w.y2s;
    c.out = y;
    c.omap = slot;
    // x_s, W1, W2 read; F', F written; y (fp32) written once
    const double bytes = a1.bytes + w2bytes + 4.0 * N * d->d_out;
    ProfScope ps(st, "esmm_fwd_chain", a1.work + 2.0 * kn * d->hidden * d->d_out, WORK_FLOP,
                 bytes);
    return umma_chain(c, st);
  }
  HXM_RETURN_IF(launch_esmm(dt, a1, st));
  // (2) y += y2 W2 + b2 over all choices     (moe_layer.cpp:61-63)
  EsmmArgs a2 = a1;
  a2.a = w.y2s;
  a2.amap = map_dense();
  a2.a_rows = w.bound;
  a2.w = w2;
  a2.w_split_k = 1;  // W2 [P][E][h][D_o]: K (H) split
  a2.d1 = d->hidden;
  a2.d2 = d->d_out;
  a2.bias = d->add_b2 ? b2 : nullptr;
  a2.epi = EPI_ATOMIC;
  a2.label = "esmm_fwd2";
  a2.work = 2.0 * kn * d->hidden * d->d_out;
  // y2 read, W2 read, y (fp32) written once
  a2.bytes = kn * d->hidden * es_ + w2bytes + 4.0 * N * d->d_out;
  a2.out_f32 = y;
  a2.peer = yp;  // fused reduce-scatter into the token owners' rows
  a2.omap = slot;
  a2.reverse = 1;  // y2 rows written last by fwd1 are still in L2
  a2.out1 = a2.out2 = nullptr;
  return launch_esmm(dt, a2, st);
}

hxm_status layer_backward(const hxm_layer_desc* d, const void* x, const void* w1,
                          const void* w2, const void* g_y, void* ws, size_t ws_bytes,
                          float* gw1, float* gb1, float* gw2, float* gb2, float* gx,
                          const hxm_peer_rows* gxp, hxm_stream_t stream,
                          const hxm_peer_rows* gw1p = nullptr,
                          const hxm_peer_rows* gw2p = nullptr) {
  HXM_RETURN_IF(check_desc(d));
  const bool tok = d->n_tokens > 0;  // token tensors may be empty (null) when N == 0
  if ((tok && (!x || !g_y || (!gx && !gxp))) || !w1 || !w2 || (!gw1 && !gw1p) || !gb1 ||
      (!gw2 && !gw2p) || (d->add_b2 && !gb2))
    return invalid_arg("moe_backward: null tensor");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Arena ar(ws, ws_bytes);
  LayerWs w = carve(ar, *d);
  if (ar.overflow) return invalid_arg("moe_backward: workspace too small");
  if (!shards_ok(*d, w, d->weight_shards))
    return invalid_arg("moe_backward: shard-major weights unsupported for this shape");
  HXM_RETURN_IF(check_peer(gxp, d, w, "moe_backward_tp"));
  HXM_RETURN_IF(check_shards(gw1p, d, w, "moe_backward_dc gW1"));
  HXM_RETURN_IF(check_shards(gw2p, d, w, "moe_backward_dc gW2"));
  const hxm_dtype dt = static_cast<hxm_dtype>(d->dtype);
  const int64_t N = d->n_tokens, E = d->n_experts;
  const int64_t Di = d->d_in, H = d->hidden, Do = d->d_out;
  // tile tables were built by hxm_moe_forward (they live in the stash)
  const RowMap slot = map_slot(w.v, N > 0 ? N : 1);
  // (4) gb2 = sum_i ESS(g_y, R_i)             (moe_layer.cpp:103)
  EssArgs es{};
  es.x = g_y;
  es.map = slot;
  es.d = Do;
  es.tiles = w.etiles;
  es.n_tiles = w.n_etiles;
  es.tile_off = w.etiles_off;
  es.max_tiles = w.max_etiles;
  es.n_experts = static_cast<int>(E);
  es.partial = w.partial;
  es.out = d->add_b2 ? gb2 : nullptr;
  es.copy_out = w.gys;  // fused: expert-sorted copy of g_y
  const double kn = static_cast<double>(d->k * N);
  const double esz = static_cast<double>(esize(d->dtype));
  es.label = "ess_gb2";
  es.work = kn * Do * esz + static_cast<double>(E) * Do * 4.0;
  {
    // one launch: gx = 0, split experts' gW slices = 0, and the
    // gb2 ESS fused with the expert-sorted copy of g_y
    BwdPrologue bp{};
    bp.label = "bwd_prologue";
    bp.es = es;
    bp.gx = gx;
    bp.gx_elems = gxp ? 0 : N * Di;  // peer rows: each owner zeroes its own
    bp.ktiles = w.ktiles;
    bp.n_ktiles = w.n_ktiles;
    bp.gw2 = gw2p ? nullptr : gw2;  // peer shards are zeroed by their owners
    bp.gw2_slice = H * Do;
    bp.gw1 = gw1p ? nullptr : gw1;
    bp.gw1_slice = Di * H;
    bp.done = w.done;
    // algorithmic bytes: g_y read once per routed slot, its sorted copy
    // written, gb2 written, gx zeroed (split-expert zeroing is data-dependent)
    bp.work = 2.0 * kn * Do * esz + static_cast<double>(E) * Do * 4.0 + 4.0 * N * Di;
    HXM_RETURN_IF(launch_bwd_prologue(dt, bp, st));
  }
  es.copy_out = nullptr;
  // (5) gW2 = sum_i ESTMM(y2_i, g_y, R_i)     (moe_layer.cpp:104)
  EstmmArgs t2{};
  t2.x1 = w.y2s;
  t2.m1 = map_dense();
  t2.x2 = w.gys;
  t2.m2 = map_dense();
  t2.x1_rows = w.bound;
  t2.x2_rows = w.bound;
  t2.d1 = H;
  t2.d2 = Do;
  t2.tiles = w.ktiles;
  t2.n_tiles = w.n_ktiles;
  t2.max_tiles = w.max_ktiles;
  t2.n_experts = static_cast<int>(E);
  t2.out = gw2;
  t2.skip_zero_split = 1;  // done by the backward prologue
  t2.peer = gw2p;          // data-centric: rows (H) reduce-scattered to the owners
  t2.peer_dim = 0;
  t2.label = "estmm_gw2";
  t2.work = 2.0 * kn * H * Do;
  // y2 and the sorted g_y read, gW2 (fp32) written
  t2.bytes = kn * (H + Do) * esz + 4.0 * E * H * Do;
  // HXM_BWD_CONC=1: gW2 (and later gb1 combine + gW1) on the side stream,
  // beside bwd_act / gx on the main stream -- independent GEMMs whose
  // persistent grids can then fill each other's tails (graph branches)
  static const bool conc = [] {
    const char* e = std::getenv("HXM_BWD_CONC");
    return e && e[0] == '1';
  }();
  const bool use_conc = conc && w.colsum != nullptr;
  std::unique_ptr<SideBranch> branch_gw2;  // joined on every return path
  if (use_conc) {
    const SideStream side = side_stream(st);
    branch_gw2.reset(new SideBranch(st, side));
    if (!branch_gw2->ok()) {
      set_error("moe_backward: side-stream fork failed");
      return HXM_ERR_CUDA;
    }
    HXM_RETURN_IF(launch_estmm(dt, t2, side.st));
  } else {
    HXM_RETURN_IF(launch_estmm(dt, t2, st));
  }
  // (6,7) g_y1 = (g_y W2^T) * F'(y1)          (moe_layer.cpp:105-108)
  EsmmArgs b6{};
  b6.a = w.gys;
  b6.amap = map_dense();
  b6.a_rows = w.bound;
  b6.n_experts = E;
  b6.w = w2;
  b6.w_trans = 1;  // W2 is E x H x Do; use W2[e]^T (Do x H)
  b6.w_shards = static_cast<int>(d->weight_shards);  // N (H) split
  b6.w_split_k = 0;
  b6.d1 = Do;
  b6.d2 = H;
  b6.tiles = w.tiles_a;
  b6.n_tiles = w.n_tiles_a;
  b6.max_tiles = static_cast<int>(max_tiles(w.bound, E, w.rows_a));
  b6.tile_rows = w.rows_a;
  b6.epi = EPI_BWD_ACT;
  b6.label = "esmm_bwd_act";
  b6.work = 2.0 * kn * Do * H;
  // sorted g_y, W2 and F'(y1) read, g_y1 written
  b6.bytes = kn * (Do + 2.0 * H) * esz + static_cast<double>(E) * H * Do * esz;
  b6.act = d->activation;
  b6.omap = slot;
  b6.out1 = w.g1s;
  b6.y1s = w.y1s;
  // (8) gb1 = sum_i ESS(g_y1_i, R_i)          (moe_layer.cpp:116)
  // tcgen05 path: fused into the g_y1 epilogue (column sums of the stored
  // bf16 tile per (tile, CTA)), then a deterministic per-expert combine
  b6.colsum = w.colsum;
  // fp32: the fused sums need the dense SIMT kernel (aligned, 4-wide rows)
  if (b6.colsum && w.rows_a < kUmmaRows && !simt_dense_esmm_ok(dt, b6)) b6.colsum = nullptr;
  // (6,7) + (10) chained (umma_chain.cu): the g_y1 chunks feed the g_x GEMM
  // from shared memory; g_y1 is still stashed for gW1 and its gb1 column sums
  // are fused as above
  const bool chain = dt == HXM_BF16 && d->weight_shards <= 1 && !gxp &&
                     umma_chain_ok(true, Di, H, Do, w.rows_a);
  if (chain) {
    ChainArgs c{};
    c.bwd = true;
    c.a = w.gys;
    c.rows = w.bound;
    c.w1 = w1;
    c.w2 = w2;
    c.n_experts = E;
    c.d_in = Di;
    c.hidden = H;
    c.d_out = Do;
    c.tiles = w.tiles_a;
    c.n_tiles = w.n_tiles_a;
    c.max_tiles = b6.max_tiles;
    c.act = d->activation;
    c.dact = w.y1s;
    c.chunk_out = w.g1s;
    c.out = gx;
    c.colsum = w.colsum;
    c.omap = slot;
    // sorted g_y, W2, F'(y1) and W1 read, g_y1 written, gx (fp32) written
    const double bytes = b6.bytes + static_cast<double>(E) * Di * H * esz + 4.0 * N * Di;
    ProfScope ps(st, "esmm_bwd_chain", b6.work + 2.0 * kn * H * Di, WORK_FLOP, bytes);
    HXM_RETURN_IF(umma_chain(c, st));
  } else {
    HXM_RETURN_IF(launch_esmm(dt, b6, st));
  }
  std::unique_ptr<SideBranch> branch;  // joined on every return path
  const char* se = std::getenv("HXM_SIDE");
  const bool use_side = !(se && se[0] == '0');
  if (b6.colsum && !use_side) {
    const int parts = colsum_parts(w.rows_a);
    HXM_RETURN_IF(launch_colsum_combine(
        w.colsum, w.tiles_a_off, static_cast<int>(E), parts, H, gb1, st, "gb1_combine",
        (static_cast<double>(max_tiles(w.bound, E, w.rows_a)) * parts + E) * H * 4.0));
  } else if (b6.colsum) {
    // the gb1 combine is independent of gW1 / gx: it runs on the side
    // stream beside them (a parallel branch of the captured graph)
    const SideStream side = side_stream(st);
    branch.reset(new SideBranch(st, side));
    if (!branch->ok()) {
      set_error("moe_backward: side-stream fork failed");
      return HXM_ERR_CUDA;
    }
    const int parts = colsum_parts(w.rows_a);  // per tile: CTAs x TMEM lane groups (tcgen05)
    HXM_RETURN_IF(launch_colsum_combine(
        w.colsum, w.tiles_a_off, static_cast<int>(E), parts, H, gb1, side.st, "gb1_combine",
        (static_cast<double>(max_tiles(w.bound, E, w.rows_a)) * parts + E) * H * 4.0));
  } else {
    es.x = w.g1s;
    es.map = map_dense();
    es.d = H;
    es.out = gb1;
    es.label = "ess_gb1";
    es.work = kn * H * esz + static_cast<double>(E) * H * 4.0;
    HXM_RETURN_IF(launch_ess(dt, es, st));
  }
  // (9) gW1 = sum_i ESTMM(x, g_y1_i, R_i)     (moe_layer.cpp:117)
  EstmmArgs t1 = t2;
  t1.x1 = w.xs;
  t1.m1 = map_dense();
  t1.x2 = w.g1s;
  t1.m2 = map_dense();
  t1.x1_rows = w.bound;
  t1.x2_rows = w.bound;
  t1.d1 = Di;
  t1.d2 = H;
  t1.out = gw1;
  t1.reverse = 1;  // g_y1 rows written last by bwd_act are still in L2
  t1.peer = gw1p;  // data-centric: columns (H) reduce-scattered to the owners
  t1.peer_dim = 1;
  t1.label = "estmm_gw1";
  t1.work = 2.0 * kn * Di * H;
  t1.bytes = kn * (Di + H) * esz + 4.0 * E * Di * H;
  {
    // D_i = 384 (c2): compute gW1 as (g_y1^T x_s)^T on the whole-tile kernel
    // -- H on M (CTA pairs of 256 rows), the 384 columns of D_i in one
    // accumulator, stored transposed (umma_wide.cu)
    EstmmArgs sw = t1;
    sw.x1 = w.g1s;
    sw.x2 = w.xs;
    sw.d1 = H;
    sw.d2 = Di;
    sw.trans_out = 1;
    sw.peer_dim = 0;  // the owners' H spans are now rows of the computed tile
    if (dt == HXM_BF16 && umma_wide_estmm_ok(sw)) t1 = sw;
  }
  if (use_conc && branch) {
    HXM_RETURN_IF(launch_estmm(dt, t1, side_stream(st).st));
  } else {
    HXM_RETURN_IF(launch_estmm(dt, t1, st));
  }
  // (10) gx += g_y1_i W1^T                    (moe_layer.cpp:118)
  EsmmArgs b10 = b6;
  b10.a = w.g1s;
  b10.amap = map_dense();
  b10.a_rows = w.bound;
  b10.w = w1;
  b10.w_trans = 1;  // W1 is E x Di x H; use W1[e]^T (H x Di)
  b10.w_split_k = 1;  // K (H) split
  b10.d1 = H;
  b10.d2 = Di;
  b10.epi = EPI_ATOMIC;
  b10.label = "esmm_bwd_gx";
  b10.work = 2.0 * kn * H * Di;
  // g_y1 and W1 read, gx (fp32) written
  b10.bytes = kn * H * esz + static_cast<double>(E) * Di * H * esz + 4.0 * N * Di;
  b10.out_f32 = gx;
  b10.peer = gxp;  // fused reduce-scatter into the token owners' rows
  b10.out1 = nullptr;
  b10.y1s = nullptr;
  if (!chain) HXM_RETURN_IF(launch_esmm(dt, b10, st));
  if (branch) HXM_TRY_CUDA(branch->join());
  if (branch_gw2) HXM_TRY_CUDA(branch_gw2->join());
  return HXM_OK;
}

}  // namespace hxm

extern "C" {

hxm_status hxm_moe_forward(const hxm_layer_desc* d, const void* x, const void* w1,
                           const float* b1, const void* w2, const float* b2,
                           const int32_t* assignments, float* y, void* ws, size_t ws_bytes,
                           int32_t* status, hxm_stream_t stream) {
  return layer_forward(d, x, w1, b1, w2, b2, assignments, y, nullptr, ws, ws_bytes, status,
                       stream);
}

hxm_status hxm_moe_forward_tp(const hxm_layer_desc* d, const void* x, const void* w1,
                              const float* b1, const void* w2, const float* b2,
                              const int32_t* assignments, const hxm_peer_rows* y_rows, void* ws,
                              size_t ws_bytes, int32_t* status, hxm_stream_t stream) {
  if (!y_rows) return invalid_arg("moe_forward_tp: null peer rows");
  return layer_forward(d, x, w1, b1, w2, b2, assignments, nullptr, y_rows, ws, ws_bytes,
                       status, stream);
}

hxm_status hxm_moe_backward(const hxm_layer_desc* d, const void* x, const void* w1,
                            const void* w2, const void* g_y, void* ws, size_t ws_bytes,
                            float* gw1, float* gb1, float* gw2, float* gb2, float* gx,
                            hxm_stream_t stream) {
  return layer_backward(d, x, w1, w2, g_y, ws, ws_bytes, gw1, gb1, gw2, gb2, gx, nullptr,
                        stream);
}

hxm_status hxm_moe_backward_tp(const hxm_layer_desc* d, const void* x, const void* w1,
                               const void* w2, const void* g_y, void* ws, size_t ws_bytes,
                               float* gw1, float* gb1, float* gw2, float* gb2,
                               const hxm_peer_rows* gx_rows, hxm_stream_t stream) {
  if (!gx_rows) return invalid_arg("moe_backward_tp: null peer rows");
  return layer_backward(d, x, w1, w2, g_y, ws, ws_bytes, gw1, gb1, gw2, gb2, nullptr, gx_rows,
                        stream);
}

hxm_status hxm_moe_backward_dc(const hxm_layer_desc* d, const void* x, const void* w1,
                               const void* w2, const void* g_y, void* ws, size_t ws_bytes,
                               const hxm_peer_rows* gw1_shards, float* gb1,
                               const hxm_peer_rows* gw2_shards, float* gb2, float* gx,
                               hxm_stream_t stream) {
  if (!gw1_shards || !gw2_shards) return invalid_arg("moe_backward_dc: null peer shards");
  return layer_backward(d, x, w1, w2, g_y, ws, ws_bytes, nullptr, gb1, nullptr, gb2, gx,
                        nullptr, stream, gw1_shards, gw2_shards);
}

hxm_status hxm_moe_stash_export(const hxm_layer_desc* d, const void* ws, int64_t choice,
                                float* y1, float* y2, hxm_stream_t stream) {
  HXM_RETURN_IF(check_desc(d));
  if (choice < 0 || choice >= d->k) return invalid_arg("stash_export: choice out of range");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Arena ar(const_cast<void*>(ws), SIZE_MAX);
  LayerWs w = carve(ar, *d);
  const int64_t N = d->n_tokens;
  if (N == 0) return HXM_OK;
  const int grid = static_cast<int>(std::min<int64_t>(4096, w.bound));
  if (d->dtype == HXM_BF16)
    export_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        w.v, w.idx, static_cast<int>(d->n_experts), N, static_cast<int>(choice), d->hidden,
        static_cast<const __nv_bfloat16*>(w.y1s), static_cast<const __nv_bfloat16*>(w.y2s), y1,
        y2);
  else
    export_kernel<float><<<grid, 256, 0, st>>>(w.v, w.idx, static_cast<int>(d->n_experts), N,
                                               static_cast<int>(choice), d->hidden,
                                               static_cast<const float*>(w.y1s),
                                               static_cast<const float*>(w.y2s), y1, y2);
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

}  // extern "C"
