// routing.cuh -- internal routing / tiling entry points (see routing.cu).
#pragma once
#include <cub/block/block_scan.cuh>

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

// ----------------------------------------------------------- tilers -----
// tiles of at most `rows` positions per expert segment; min_one: experts
// with an empty segment still get one (empty) tile -- used by ESTMM so that
// their zero gradient is written (es_ops.cpp:202 zero-initialised output).
// flags: bit 0 = the expert spans several tiles (split), bit 1 = empty
// segment; with `counts` (real slots per expert) bit 2 is set and bits 8..
// hold how many of the tile's rows are real (the rest are -1 pads).
template <class IdxT, int NT = 1024>
__device__ void tile_pass(const IdxT* __restrict__ idx, int E, int rows, int min_one,
                          SegTile* __restrict__ tiles, int32_t* __restrict__ tile_off,
                          int32_t* __restrict__ n_tiles, const int32_t* counts = nullptr,
                          int split_rows = 0) {
  using Scan = cub::BlockScan<int32_t, NT>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int32_t carry;
  __syncthreads();
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int e0 = 0; e0 < E; e0 += NT) {
    const int e = e0 + threadIdx.x;
    int32_t nt = 0;
    int64_t b = 0, len = 0, re = rows;
    if (e < E) {
      b = idx[e];
      len = static_cast<int64_t>(idx[e + 1]) - b;
      if (split_rows > 0 && len > rows) re = split_rows;
      nt = static_cast<int32_t>((len + re - 1) / re);
      if (nt == 0 && min_one) nt = 1;
    }
    int32_t excl, agg;
    Scan(tmp).ExclusiveSum(nt, excl, agg);
    if (e < E) {
      const int32_t off = carry + excl;
      tile_off[e] = off;
      const int split = nt > 1 ? 1 : 0;
      const int empty = len == 0 ? 2 : 0;
      for (int j = 0; j < nt; ++j) {
        SegTile t;
        t.expert = e;
        t.begin = static_cast<int>(b + static_cast<int64_t>(j) * re);
        const int64_t hi = b + static_cast<int64_t>(j + 1) * re;
        t.end = static_cast<int>(hi < b + len ? hi : b + len);
        if (len == 0) t.end = t.begin;
        t.flags = split | empty;
        if (counts) {
          const int64_t real = b + counts[e] - t.begin;
          const int vr = static_cast<int>(real < 0 ? 0 : (real > t.end - t.begin ? t.end - t.begin : real));
          t.flags |= 4 | (vr << 8);
        }
        tiles[off + j] = t;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tile_off[E] = carry;
    *n_tiles = carry;
  }
}


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
