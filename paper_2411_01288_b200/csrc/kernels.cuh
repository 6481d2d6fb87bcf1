// kernels.cuh -- argument blocks and launchers of the expert-specific kernels.
//
// ESMM  (es_ops.cpp:47-81)   : grouped per-expert GEMM over segment tiles.
// ESTMM (es_ops.cpp:106-128) : per-expert transposed GEMM, K = the expert's
//                              tokens (variable), split-K over segment chunks.
// ESS   (es_ops.cpp:86-102)  : per-expert segmented column sums.
// bf16 runs on the tcgen05 tensor cores (umma.cu); fp32 runs on fp32 FMA
// (simt.cu).  Both consume the same argument blocks.
#pragma once
#include "common.cuh"

namespace hxm {

// Row map: padded position p -> source/destination row, -1 = padding slot.
enum MapKind : int { MAP_V64 = 0, MAP_SLOT = 1, MAP_DENSE = 2 };
struct RowMap {
  int kind;
  int n;  // tokens per choice (MAP_SLOT)
  const void* v;
  __device__ __forceinline__ int operator()(int64_t p) const {
    if (kind == MAP_V64) return static_cast<int>(static_cast<const int64_t*>(v)[p]);
    if (kind == MAP_SLOT) {
      const int s = static_cast<const int32_t*>(v)[p];
      return s < 0 ? -1 : s % n;
    }
    return static_cast<int>(p);
  }
};
inline RowMap map_v64(const int64_t* v) { return RowMap{MAP_V64, 0, v}; }
inline RowMap map_slot(const int32_t* v, int64_t n) {
  return RowMap{MAP_SLOT, static_cast<int>(n), v};
}
inline RowMap map_dense() { return RowMap{MAP_DENSE, 0, nullptr}; }

enum EpiMode : int {
  EPI_WRITE = 0,    // out_f32[omap(p)]  = acc + bias          (esmm write)
  EPI_ACCUM = 1,    // out_f32[omap(p)] += acc + bias          (esmm accumulate)
  EPI_ATOMIC = 2,   // red.add out_f32[omap(p)], acc (+bias)   (k-merged y, gx)
  EPI_FWD_ACT = 3,  // y1 = acc + bias: out1[p] = F'(y1), out2[p] = F(y1)  (stash)
  EPI_BWD_ACT = 4   // out1[p] = acc * y1s[p]  (y1s holds F'(y1))         (g_y1)
};

struct EsmmArgs {
  const char* label;  // profiling region name (nullable)
  double work;        // algorithmic FLOP (GEMMs) or bytes (ESS) of the launch
  double bytes;       // GEMMs: algorithmic HBM bytes (operands once, outputs once)
  const void* a;  // A rows, K = d1 columns
  RowMap amap;
  int64_t a_rows;  // rows of the tensor behind `a` (TMA bounds)
  int64_t n_experts;
  const void* w;  // w_trans == 0: E x d1 x d2 ; 1: E x d2 x d1 (use W^T)
  int w_trans;
  int64_t d1, d2;
  const float* bias;  // E x d2 or null
  const SegTile* tiles;
  const int32_t* n_tiles;
  int max_tiles;
  int tile_rows;  // rows per segment tile (kSimtRows or kUmmaRows)
  int epi;
  int act;
  float* out_f32;  // WRITE / ACCUM / ATOMIC destination, rows via omap
  RowMap omap;     // scatter map, or the pad-detection map for dense outputs
  void* out1;      // FWD_ACT / BWD_ACT dense outputs (dtype), row stride d2
  void* out2;
  const void* y1s;  // BWD_ACT: pre-activation stash (dtype), row stride d2
  int reverse;      // tcgen05: work items last to first (see umma.cu)
  const hxm_peer_rows* peer;  // EPI_ATOMIC: rows reduced into their owners' buffers
  float* colsum;    // BWD_ACT (tcgen05): per-(tile, CTA, lane group) column sums of out1,
                    // [((tile * CG + cta) * 4 + group) x d2] -> colsum_combine
  int w_shards;     // > 1: w (and, for FWD_ACT, bias) shard-major [P][E][..]: the H axis
  int w_split_k;    // split in P slices -- K (d1) when set, else N (d2); tcgen05 only
};

struct EstmmArgs {
  const char* label;  // profiling region name (nullable)
  double work;        // algorithmic FLOP (GEMMs) or bytes (ESS) of the launch
  double bytes;       // algorithmic HBM bytes (operands once, outputs once)
  const void* x1;  // rows via m1, d1 columns
  RowMap m1;
  const void* x2;  // rows via m2, d2 columns
  RowMap m2;
  int64_t x1_rows, x2_rows;  // rows of the tensors behind x1 / x2
  int64_t d1, d2;
  const SegTile* tiles;  // K chunks (split flag / empty flag)
  const int32_t* n_tiles;
  int max_tiles;
  int n_experts;
  float* out;  // E x d1 x d2
  int reverse;      // tcgen05: work items last to first
  const hxm_peer_rows* peer;  // tcgen05: reduce-scatter to H-shard owners (out unused)
  int peer_dim;               // 0: d1 (rows) is the split H extent, 1: d2 (columns)
  int skip_zero_split;  // split experts' slices already zeroed by the caller
  int trans_out;        // tcgen05 whole-tile kernel: out[e] stored d2 x d1 (out = (X1^T X2)^T)
};

struct EssArgs {
  const char* label;  // profiling region name (nullable)
  double work;        // algorithmic FLOP (GEMMs) or bytes (ESS) of the launch
  const void* x;
  RowMap map;
  int64_t d;
  const SegTile* tiles;  // <= kEssRows positions each
  const int32_t* n_tiles;
  const int32_t* tile_off;  // E+1
  int max_tiles;
  int n_experts;
  float* partial;  // max_tiles x d
  float* out;      // E x d, or null: no reduction (copy only)
  void* copy_out;  // optional: rows also copied to expert-sorted order
                   // (copy_out[p] = x[map(p)], padding slots -> zero rows)
};

// dst[p] = src[map(p)] for p < idx[E] (padding slots -> zero rows): the
// expert-sorted copy of a token-order tensor, bandwidth-bound (operator ESMM).
hxm_status launch_gather_rows64(hxm_dtype dt, const void* src, RowMap map, int64_t d,
                                const int64_t* idx, int n_experts, int64_t bound, void* dst,
                                cudaStream_t st);

// ESTMM operator (bf16): segments re-laid to 64-position multiples (idx64,
// E+1 int32) and both operands gathered into that layout (o1, o2: bound rows)
hxm_status launch_estmm_relayout(const void* x1, int64_t d1, const void* x2, int64_t d2,
                                  const int64_t* v, const int64_t* idx, int E, int64_t bound,
                                  int32_t* idx64, void* o1, void* o2, cudaStream_t st);


// out[e] = sum over e's tiles t (tile_off[e]..tile_off[e+1]) and the
// `parts` partial rows of each tile of partial[(t * parts + r) x d]: the
// deterministic second phase of an ESS fused into a GEMM epilogue.
hxm_status launch_colsum_combine(const float* partial, const int32_t* tile_off, int n_experts,
                                 int parts, int64_t d, float* out, cudaStream_t st,
                                 const char* label, double work_bytes);

// The layer backward's prologue in one cooperative launch: gx = 0, zeroed
// gW1 / gW2 slices of split ESTMM experts (per the ESTMM chunk table), and the
// gb2 ESS of g_y fused with its expert-sorted copy (es.copy_out) + combine.
struct BwdPrologue {
  const char* label;
  double work;
  EssArgs es;
  float* gx;
  int64_t gx_elems;
  const SegTile* ktiles;
  const int32_t* n_ktiles;
  float* gw2;
  int64_t gw2_slice;
  float* gw1;
  int64_t gw1_slice;
  int32_t* done;  // E ESS arrival counters (zero on entry, left zero): the block
                  // that finishes an expert's last ESS item combines its gb2
};
hxm_status launch_bwd_prologue(hxm_dtype dt, BwdPrologue b, cudaStream_t st);

constexpr int kEssRows = 128;
constexpr int kSimtRows = 64;     // SIMT ESMM tile rows
constexpr int kUmmaRows = 128;    // tcgen05 ESMM tile rows (UMMA M)
constexpr int kUmma2Rows = 256;   // CTA-pair (cta_group::2) ESMM tile rows
constexpr int kEstmmChunk = 8192;  // ESTMM: an expert up to this many positions is one
                                   // K chunk; longer (skewed) experts are split into
constexpr int kEstmmSplit = 2048;  // chunks of this many, reduced with fp32 red.add
                                   // into their zeroed gW slices

hxm_status launch_esmm(hxm_dtype dt, const EsmmArgs& a, cudaStream_t st);
hxm_status launch_estmm(hxm_dtype dt, const EstmmArgs& a, cudaStream_t st);
hxm_status launch_ess(hxm_dtype dt, const EssArgs& a, cudaStream_t st);

// fp32 FMA kernels (simt.cu)
hxm_status simt_esmm(hxm_dtype dt, const EsmmArgs& a, cudaStream_t st);
// the dense-operand fp32 ESMM (the one that can fuse gb1 column sums) applies
bool simt_dense_esmm_ok(hxm_dtype dt, const EsmmArgs& a);
hxm_status simt_estmm(hxm_dtype dt, const EstmmArgs& a, cudaStream_t st);
// tcgen05 kernels (umma.cu); return HXM_ERR_UNSUPPORTED for shapes they
// do not cover (d1/d2 not multiples of 64), which the caller reports.
hxm_status umma_esmm(const EsmmArgs& a, cudaStream_t st);
hxm_status umma_estmm(const EstmmArgs& a, cudaStream_t st);
// 256 x 384 whole-tile CTA-pair reduction GEMM (umma_wide.cu): EPI_ATOMIC,
// dense A, 256-row tiles, d2 == 384 (HXM_WIDE=0 disables)
bool umma_wide_ok(const EsmmArgs& a);
hxm_status umma_wide_esmm(const EsmmArgs& a, cudaStream_t st);
// the same whole-tile scheme for ESTMM (umma_wide.cu): out[e] = X1^T X2 with
// d2 == 384 owned whole by a CTA pair per 256 rows of d1 (A read once per
// tile); trans_out writes the tile transposed (gW1 as (g_y1^T x_s)^T)
bool umma_wide_estmm_ok(const EstmmArgs& a);
hxm_status umma_wide_estmm(const EstmmArgs& a, cudaStream_t st);
// Chained layer GEMMs (umma_chain.cu), one persistent CTA-pair kernel over
// 128-column hidden chunks: forward fwd1 -> fwd2 (y1 = x W1 + b1, F / F'
// stash, y += F W2 + b2), backward bwd_act -> gx (g_y1 = (g_y W2^T) F', gb1
// column sums, g_x += g_y1 W1^T).  GEMM2's output width must be 384, GEMM1's
// K a multiple of 192 up to 384; 256-row tiles; no shard-major weights, no
// peer rows.  Opt-in: HXM_CHAIN=1 (forward), HXM_CHAIN_BWD=1 (backward).
struct ChainArgs {
  bool bwd;
  const void* a;   // GEMM1 A rows (bf16): x_s (forward) / g_y_s (backward)
  int64_t rows;    // rows behind a / the stashes
  const void* w1;  // E x d_in x H
  const void* w2;  // E x H x d_out
  const float* b1; // forward: E x H
  const float* b2; // forward: E x d_out or null
  int64_t n_experts, d_in, hidden, d_out;
  const SegTile* tiles;
  const int32_t* n_tiles;
  int max_tiles;
  int act;
  void* dact;       // F'(y1) stash, rows x H: written (forward) / read (backward)
  void* chunk_out;  // F(y1) (forward) / g_y1 (backward) stash, rows x H
  float* out;       // y (forward) / g_x (backward), zeroed; rows via omap
  float* colsum;    // backward: gb1 partials (the BWD_ACT layout), or null
  RowMap omap;
};
bool umma_chain_ok(bool bwd, int64_t d_in, int64_t hidden, int64_t d_out, int tile_rows);
hxm_status umma_chain(const ChainArgs& a, cudaStream_t st);
bool umma_supports_esmm(int64_t d1, int64_t d2);
bool umma_supports_estmm(int64_t d1, int64_t d2);
// CTA-pair ESMM (dense A, 256-row tiles): BN must split into whole B halves
bool umma2_supports_esmm(int64_t d1, int64_t d2, bool w_trans);
// the tile widths the tcgen05 launchers pick for an output width n
// (single CTA / CTA pair with MN-major or K-major B)
int umma_pick_bn(int64_t n);
int umma_pick_bn2(int64_t n, bool b_mn);

// esfk (es_ops.cpp:210-247): grad_x = esmm(g, W^T / w_t), grad_b = ess(g),
// grad_w = estmm(x, g) over the caller's ReIndex.  simt: one launch (fp32);
// umma (esfk.cu, bf16): a gather / ESS prologue + one tcgen05 launch that
// runs the grad-x and grad-W tiles side by side.  w_trans as in EsmmArgs
// for the grad-x GEMM (0: w is E x d2 x d1, 1: w is E x d1 x d2).
hxm_status simt_esfk(hxm_dtype dt, const void* x, const void* g, int64_t n, int64_t d1,
                     int64_t d2, const void* w, int w_trans, const int64_t* v, const int64_t* idx,
                     int64_t E, int64_t np_bound, float* grad_x, float* grad_b, float* grad_w,
                     cudaStream_t st);
hxm_status umma_esfk(const void* x, const void* g, int64_t n, int64_t d1, int64_t d2,
                     const void* w, int w_trans, const int64_t* v, const int64_t* idx,
                     int64_t E, int64_t np_bound, float* grad_x, float* grad_b, float* grad_w,
                     void* ws, size_t ws_bytes, cudaStream_t st);
bool esfk_umma_ok(int64_t d1, int64_t d2);
size_t esfk_ws_bytes(int64_t np_bound, int64_t E, int64_t d1, int64_t d2);

// zero out[e] for experts whose ESTMM is split over several chunks
hxm_status zero_split_experts(const SegTile* tiles, const int32_t* n_tiles,
                              int max_tiles, int64_t slice, float* out,
                              cudaStream_t st);

}  // namespace hxm
