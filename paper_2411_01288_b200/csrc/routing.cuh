// routing.cuh -- internal routing / tiling entry points (see routing.cu).
#pragma once
#include "common.cuh"

namespace hxm {

size_t reindex_ws_bytes(int64_t n, int64_t E, int64_t k = 1);

// Cut every expert segment [idx[e], idx[e+1]) into tiles of <= rows positions.
template <class IdxT>
hxm_status launch_tiles(const IdxT* idx, int64_t E, int rows, bool min_one,
                        SegTile* tiles, int32_t* tile_off, int32_t* n_tiles,
                        cudaStream_t st, int split_rows = 0);

// One tiling of a segment index (rows per tile, see tile_pass).
struct TileSpec {
  int rows;
  int min_one;
  SegTile* tiles;
  int32_t* tile_off;
  int32_t* n_tiles;
  int split_rows = 0;  // > 0: segments longer than `rows` are cut into
                       // split_rows-position tiles instead (ESTMM chunks: one
                       // chunk per expert unless it is heavily skewed)
};
int64_t max_tiles(int64_t n_padded_bound, int64_t E, int rows);

// The layer forward's prologue in one cooperative launch: k-choice slot index
// (v, idx; bit-exact with build_reindex_slots), routing validation into
// `status`, the three tile tables, y = 0 and the expert-sorted copy of x.
struct FwdPrologue {
  const int32_t* a;  // k x N assignments = n_slots slots
  int64_t n_slots, n_tok;
  int k, E;
  int64_t blk;
  int64_t capacity;  // > 0: fixed per-expert segments, overflow dropped
  int32_t* v;
  int32_t* idx;
  TileSpec s0, s1, s2;
  const void* x;  // token-order rows (row_bytes each), or null: no copy
  void* xs;
  int64_t row_bytes;
  int unit;  // copy granule: 16, 4 or 2 bytes
  float* y;
  int64_t y_elems;
  int32_t* status;
  int32_t* zero_i32;  // optional: zeroed in phase 1 (the backward prologue's
  int zero_n;         // per-expert ESS arrival counters)
  void* ws;  // reindex scratch (reindex_ws_bytes)
  size_t ws_bytes;
  // filled by the launcher
  int chunk, nchunks;
  int32_t* cnt;
  int32_t* base;
  int32_t* total;
};
hxm_status launch_fwd_prologue(FwdPrologue a, cudaStream_t st);

}  // namespace hxm
