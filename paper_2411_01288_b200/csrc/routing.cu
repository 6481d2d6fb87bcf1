// routing.cu -- device routing-index build and segment tilers.
//
// Replaces moekit::build_reindex (reference core/src/routing.cpp:42-70):
//   count[e]  -> ceil-to-blk padding -> exclusive scan (idx) -> -1 fill ->
//   stable, in-token-order placement with per-expert cursors.
// The GPU version is bit-exact with it.  Tokens are cut into fixed chunks of
// CHUNK consecutive tokens, one warp per chunk:
//   K1 count_chunks   : per-chunk expert histograms (smem, per warp)
//   K2 scan_experts   : per expert, exclusive scan of its chunk counts
//   K3 scatter        : idx (all blocks recompute it in smem; block 0 stores),
//                       -1 padding, and each warp places its chunk in token
//                       order: __match_any_sync gives the in-warp rank among
//                       equal experts, so the order inside a segment is the
//                       token order exactly as the reference's cursor loop.
// Traffic is read 4 B/token + write 8 B/slot: it is launch/latency bound at
// every BASELINE.json size.
#include <cooperative_groups.h>
#include <cstdlib>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "routing.cuh"

namespace hxm {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// blockIdx.y = routing choice (build_reindex_all: k independent indices in
// one launch; every per-choice array is offset by the choice's stride)
__global__ void count_chunks(const int32_t* __restrict__ a, int64_t n, int E,
                             int chunk, int nchunks, int32_t* __restrict__ cnt,
                             int32_t* status) {
  extern __shared__ int32_t hist[];  // [kWarps][E]
  a += static_cast<int64_t>(blockIdx.y) * n;
  cnt += static_cast<int64_t>(blockIdx.y) * (static_cast<int64_t>(nchunks) * E + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int32_t* h = hist + warp * E;
  for (int e = lane; e < E; e += 32) h[e] = 0;
  __syncwarp();
  const int c = blockIdx.x * kWarps + warp;
  if (c < nchunks) {
    const int64_t t0 = static_cast<int64_t>(c) * chunk;
    const int64_t t1 = min(n, t0 + chunk);
    for (int64_t t = t0 + lane; t < t1; t += 32) {
      const int e = a[t];
      if (e < 0 || e >= E) {
        if (status) atomicExch(status, HXM_ERR_INVALID_ARG);
        continue;
      }
      atomicAdd(&h[e], 1);
    }
    __syncwarp();
    for (int e = lane; e < E; e += 32) cnt[static_cast<int64_t>(c) * E + e] = h[e];
  }
}

// One block per expert: base[c][e] = sum_{c' < c} cnt[c'][e]; total[e].
__global__ void scan_experts(const int32_t* __restrict__ cnt, int E, int nchunks,
                             int32_t* __restrict__ base, int32_t* __restrict__ total) {
  using Scan = cub::BlockScan<int32_t, kThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int32_t carry;
  const int e = blockIdx.x;
  const int64_t cstride = static_cast<int64_t>(nchunks) * E + 1;
  cnt += blockIdx.y * cstride;
  base += blockIdx.y * cstride;
  total += static_cast<int64_t>(blockIdx.y) * (E + 1);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int c0 = 0; c0 < nchunks; c0 += kThreads) {
    const int c = c0 + threadIdx.x;
    int32_t val = c < nchunks ? cnt[static_cast<int64_t>(c) * E + e] : 0;
    int32_t excl, agg;
    Scan(tmp).ExclusiveSum(val, excl, agg);
    if (c < nchunks) base[static_cast<int64_t>(c) * E + e] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) total[e] = carry;
}

// Exclusive scan of padded segment sizes into smem idx[0..E].
template <class IdxT>
__device__ void block_idx(const int32_t* __restrict__ total, int E, int64_t blk,
                          IdxT* sidx, int64_t capacity = 0) {
  using Scan = cub::BlockScan<int64_t, kThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int e0 = 0; e0 < E; e0 += kThreads) {
    const int e = e0 + threadIdx.x;
    int64_t padded = 0;
    if (e < E)
      padded = capacity > 0 ? capacity  // conventional: fixed per-expert buffers
                            : blk * ((static_cast<int64_t>(total[e]) + blk - 1) / blk);
    int64_t excl, agg;
    Scan(tmp).ExclusiveSum(padded, excl, agg);
    if (e < E) sidx[e] = static_cast<IdxT>(carry + excl);
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) sidx[E] = static_cast<IdxT>(carry);
  __syncthreads();
}

// value written into v for token t of the (flattened) assignment:
// reference API -> t itself; combined k-choice index -> slot id t (the
// assignment array is k x N row-major, so the flat position IS the slot).
template <class IdxT, class VT>
__global__ void scatter(const int32_t* __restrict__ a, int64_t n, int E,
                        int64_t blk, int chunk, int nchunks,
                        const int32_t* __restrict__ base,
                        const int32_t* __restrict__ total, VT* __restrict__ v,
                        IdxT* __restrict__ idx_out, int64_t v_stride) {
  extern __shared__ unsigned char smem_raw[];
  {
    const int64_t cstride = static_cast<int64_t>(nchunks) * E + 1;
    a += static_cast<int64_t>(blockIdx.y) * n;
    base += blockIdx.y * cstride;
    total += static_cast<int64_t>(blockIdx.y) * (E + 1);
    v += blockIdx.y * v_stride;
    idx_out += static_cast<int64_t>(blockIdx.y) * (E + 1);
  }
  IdxT* sidx = reinterpret_cast<IdxT*>(smem_raw);                     // E+1
  int64_t* cursor = reinterpret_cast<int64_t*>(
      smem_raw + align_up((E + 1) * sizeof(IdxT), 16));             // [kWarps][E]
  block_idx<IdxT>(total, E, blk, sidx);
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e <= E; e += kThreads) idx_out[e] = sidx[e];
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // -1 padding of segment tails (routing.cpp:62)
  for (int e = blockIdx.x * kWarps + warp; e < E; e += gridDim.x * kWarps) {
    const int64_t s0 = static_cast<int64_t>(sidx[e]) + total[e];
    const int64_t s1 = sidx[e + 1];
    for (int64_t p = s0 + lane; p < s1; p += 32) v[p] = static_cast<VT>(-1);
  }
  const int c = blockIdx.x * kWarps + warp;
  if (c >= nchunks) return;
  int64_t* cur = cursor + static_cast<int64_t>(warp) * E;
  for (int e = lane; e < E; e += 32)
    cur[e] = static_cast<int64_t>(sidx[e]) + base[static_cast<int64_t>(c) * E + e];
  __syncwarp();
  const int64_t t0 = static_cast<int64_t>(c) * chunk;
  const int64_t t1 = min(n, t0 + chunk);
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t tb = t0; tb < t1; tb += 32) {
    const int64_t t = tb + lane;
    const bool live = t < t1;
    int e = live ? a[t] : -1;
    if (e >= E) e = -1;  // out of range: reported by count_chunks, skipped
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    if (e >= 0) {
      const int64_t pos = cur[e] + __popc(peers & lt);
      v[pos] = static_cast<VT>(t);
    }
    __syncwarp();
    if (e >= 0 && (__ffs(peers) - 1) == lane) cur[e] += __popc(peers);
    __syncwarp();
  }
}

int pick_chunk(int64_t n) {
  // >= 64 tokens per warp-chunk (enough warps to fill the GPU at the
  // BASELINE sizes), at most ~2048 chunks so K2's per-expert scan stays short
  int64_t c = 64;
  while (ceil_div(n, c) > 2048) c *= 2;
  return static_cast<int>(c);
}

// k independent indices (k = 1: build_reindex; k > 1: build_reindex_all,
// routing.cpp:72-80) in three launches, choice = blockIdx.y: v of choice i
// at v + i * v_stride, idx at idx + i * (E + 1)
template <class IdxT, class VT>
hxm_status build_impl(const int32_t* a, int64_t n, int64_t E, int64_t blk,
                      VT* v, IdxT* idx, void* ws, size_t ws_bytes,
                      int32_t* status, cudaStream_t st, int k = 1, int64_t v_stride = 0) {
  const int chunk = pick_chunk(n);
  const int nchunks = static_cast<int>(ceil_div(n, chunk));
  Arena ar(ws, ws_bytes);
  int32_t* cnt = ar.take<int32_t>((static_cast<size_t>(nchunks) * E + 1) * k);
  int32_t* base = ar.take<int32_t>((static_cast<size_t>(nchunks) * E + 1) * k);
  int32_t* total = ar.take<int32_t>((E + 1) * k);
  if (ar.overflow) return invalid_arg("build_reindex: workspace too small");
  if (k > 65535) return invalid_arg("build_reindex_all: too many choices");
  const int blocks = static_cast<int>(std::max<int64_t>(1, ceil_div(nchunks, kWarps)));
  const size_t hist_smem = static_cast<size_t>(kWarps) * E * sizeof(int32_t);
  if (nchunks > 0) {
    count_chunks<<<dim3(blocks, k), kThreads, hist_smem, st>>>(a, n, static_cast<int>(E), chunk,
                                                               nchunks, cnt, status);
    HXM_CHECK_LAUNCH();
  }
  scan_experts<<<dim3(static_cast<int>(E), k), kThreads, 0, st>>>(cnt, static_cast<int>(E),
                                                                  nchunks, base, total);
  HXM_CHECK_LAUNCH();
  const size_t sc_smem = align_up((E + 1) * sizeof(IdxT), 16) +
                         static_cast<size_t>(kWarps) * E * sizeof(int64_t);
  if (sc_smem > 48 * 1024) {
    HXM_TRY_CUDA(cudaFuncSetAttribute(scatter<IdxT, VT>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(sc_smem)));
  }
  scatter<IdxT, VT><<<dim3(blocks, k), kThreads, sc_smem, st>>>(
      a, n, static_cast<int>(E), blk, chunk, nchunks, base, total, v, idx, v_stride);
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

template <class IdxT>
__global__ void build_tiles(const IdxT* __restrict__ idx, int E, TileSpec a, TileSpec b,
                            TileSpec c, int count) {
  tile_pass<IdxT>(idx, E, a.rows, a.min_one, a.tiles, a.tile_off, a.n_tiles, nullptr,
                  a.split_rows);
  if (count > 1)
    tile_pass<IdxT>(idx, E, b.rows, b.min_one, b.tiles, b.tile_off, b.n_tiles, nullptr,
                    b.split_rows);
  if (count > 2)
    tile_pass<IdxT>(idx, E, c.rows, c.min_one, c.tiles, c.tile_off, c.n_tiles, nullptr,
                    c.split_rows);
}

// ------------------------------------------------- fused layer prologue --
// The forward's whole index build in ONE cooperative launch (three grid
// barriers instead of seven dependent launches): validation + per-chunk
// counts (+ zeroing y) | per-expert chunk scans | segment offsets, -1 pads,
// in-order placement and the three tile tables | expert-sorted copy of x.
// Same placement rule as count_chunks / scan_experts / scatter above, so v
// and idx are bit-identical to the reference's build_reindex order.
__device__ __forceinline__ void copy_row(const char* src, char* dst, int64_t bytes, int lane,
                                         int unit) {
  if (unit == 16) {
    for (int64_t o = lane * 16; o < bytes; o += 512)
      *reinterpret_cast<uint4*>(dst + o) = __ldg(reinterpret_cast<const uint4*>(src + o));
  } else if (unit == 4) {
    for (int64_t o = lane * 4; o < bytes; o += 128)
      *reinterpret_cast<uint32_t*>(dst + o) = __ldg(reinterpret_cast<const uint32_t*>(src + o));
  } else {
    for (int64_t o = lane * 2; o < bytes; o += 64)
      *reinterpret_cast<uint16_t*>(dst + o) = __ldg(reinterpret_cast<const uint16_t*>(src + o));
  }
}
__device__ __forceinline__ void zero_row(char* dst, int64_t bytes, int lane, int unit) {
  if (unit == 16) {
    for (int64_t o = lane * 16; o < bytes; o += 512)
      *reinterpret_cast<uint4*>(dst + o) = make_uint4(0u, 0u, 0u, 0u);
  } else if (unit == 4) {
    for (int64_t o = lane * 4; o < bytes; o += 128) *reinterpret_cast<uint32_t*>(dst + o) = 0u;
  } else {
    for (int64_t o = lane * 2; o < bytes; o += 64) *reinterpret_cast<uint16_t*>(dst + o) = 0;
  }
}

__device__ unsigned long long g_pro_ts[8];
__device__ __forceinline__ void pro_ts(int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_pro_ts[i] = t;
  }
}
__global__ void __launch_bounds__(kThreads) fwd_prologue(FwdPrologue a) {
  namespace cg = cooperative_groups;
  pro_ts(0);
  cg::grid_group grid = cg::this_grid();
  extern __shared__ unsigned char smem_raw[];
  const int E = a.E;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int gwarp = blockIdx.x * kWarps + warp, nwarps = gridDim.x * kWarps;
  const int64_t gtid = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
  const int64_t gthreads = static_cast<int64_t>(gridDim.x) * kThreads;
  // ---- 1: validation, per-chunk histograms --------------------------------
  if (a.zero_i32 && blockIdx.x == 0)
    for (int i = threadIdx.x; i < a.zero_n; i += kThreads) a.zero_i32[i] = 0;
  {
    int32_t* h = reinterpret_cast<int32_t*>(smem_raw) + warp * E;
    for (int c = gwarp; c < a.nchunks; c += nwarps) {
      for (int e = lane; e < E; e += 32) h[e] = 0;
      __syncwarp();
      const int64_t t0 = static_cast<int64_t>(c) * a.chunk;
      const int64_t t1 = min(a.n_slots, t0 + a.chunk);
      for (int64_t t = t0 + lane; t < t1; t += 32) {
        const int e = a.a[t];
        if (e < 0 || e >= E) {
          if (a.status) atomicExch(a.status, HXM_ERR_INVALID_ARG);
          continue;
        }
        atomicAdd(&h[e], 1);
      }
      __syncwarp();
      for (int e = lane; e < E; e += 32) a.cnt[static_cast<int64_t>(c) * E + e] = h[e];
      __syncwarp();
    }
    // per-token distinctness of the k choices (routing.cpp:30-39)
    if (a.status && a.k > 1) {
      for (int64_t t = gtid; t < a.n_tok; t += gthreads)
        for (int i = 0; i < a.k; ++i) {
          const int ei = a.a[i * a.n_tok + t];
          for (int j = i + 1; j < a.k; ++j)
            if (a.a[j * a.n_tok + t] == ei) atomicExch(a.status, HXM_ERR_INVALID_ARG);
        }
    }
  }
  pro_ts(1);
  grid.sync();
  pro_ts(2);
  // ---- 2: per expert, exclusive scan of its chunk counts; y = 0 ----------
  {
    using Scan = cub::BlockScan<int32_t, kThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int32_t carry;
    for (int e = blockIdx.x; e < E; e += gridDim.x) {
      __syncthreads();
      if (threadIdx.x == 0) carry = 0;
      __syncthreads();
      for (int c0 = 0; c0 < a.nchunks; c0 += kThreads) {
        const int c = c0 + threadIdx.x;
        const int32_t val = c < a.nchunks ? a.cnt[static_cast<int64_t>(c) * E + e] : 0;
        int32_t excl, agg;
        Scan(tmp).ExclusiveSum(val, excl, agg);
        if (c < a.nchunks) a.base[static_cast<int64_t>(c) * E + e] = carry + excl;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
      }
      if (threadIdx.x == 0) a.total[e] = carry;
    }
    // y = 0 by the blocks without a scan (all of them when E >= grid)
    const int zb0 = gridDim.x > static_cast<unsigned>(E) ? E : 0;
    const int64_t zt = static_cast<int64_t>(blockIdx.x - zb0) * kThreads + threadIdx.x;
    const int64_t zn = static_cast<int64_t>(gridDim.x - zb0) * kThreads;
    if (static_cast<int>(blockIdx.x) >= zb0) zero_f32(a.y, a.y_elems, zt, zn);
  }
  pro_ts(3);
  grid.sync();
  pro_ts(4);
  // ---- 3: offsets, -1 pads, stable placement, tile tables ----------------
  int32_t* sidx = reinterpret_cast<int32_t*>(smem_raw);  // E+1
  {
    int32_t* cursor = sidx + align_up(E + 1, 4);  // [kWarps][E]
    block_idx<int32_t>(a.total, E, a.blk, sidx, a.capacity);
    if (blockIdx.x == 0)
      for (int e = threadIdx.x; e <= E; e += kThreads) a.idx[e] = sidx[e];
    for (int e = gwarp; e < E; e += nwarps) {
      const int64_t tot = a.total[e];
      const int64_t kept = (a.capacity > 0 && tot > a.capacity) ? a.capacity : tot;
      const int64_t s0 = static_cast<int64_t>(sidx[e]) + kept;
      for (int64_t p = s0 + lane; p < sidx[e + 1]; p += 32) a.v[p] = -1;
    }
    int32_t* cur = cursor + warp * E;
    const unsigned lt = (1u << lane) - 1u;
    for (int c = gwarp; c < a.nchunks; c += nwarps) {
      for (int e = lane; e < E; e += 32) cur[e] = sidx[e] + a.base[static_cast<int64_t>(c) * E + e];
      __syncwarp();
      const int64_t t0 = static_cast<int64_t>(c) * a.chunk;
      const int64_t t1 = min(a.n_slots, t0 + a.chunk);
      for (int64_t tb = t0; tb < t1; tb += 32) {
        const int64_t t = tb + lane;
        int e = t < t1 ? a.a[t] : -1;
        if (e >= E) e = -1;  // out of range: reported in phase 1, skipped
        const unsigned peers = __match_any_sync(0xffffffffu, e);
        if (e >= 0) {
          const int64_t pos = cur[e] + __popc(peers & lt);
          // conventional baseline: slots past the expert's capacity are
          // dropped (keep-lowest slot ids, gemm_oracle.cpp:91-94)
          if (a.capacity <= 0 || pos - sidx[e] < a.capacity) a.v[pos] = static_cast<int32_t>(t);
        }
        __syncwarp();
        if (e >= 0 && (__ffs(peers) - 1) == lane) cur[e] += __popc(peers);
        __syncwarp();
      }
    }
    // the three tilings on three different blocks (the last ones), so no
    // block carries all of them into the grid barrier
    const int tb = static_cast<int>(gridDim.x) - 1 - static_cast<int>(blockIdx.x);
    const bool one = gridDim.x < 3;  // (tiny grids: the last block does all three)
    if (tb == 0)
      tile_pass<int32_t, kThreads>(sidx, E, a.s0.rows, a.s0.min_one, a.s0.tiles, a.s0.tile_off,
                                   a.s0.n_tiles, a.total, a.s0.split_rows);
    if (one ? tb == 0 : tb == 1)
      tile_pass<int32_t, kThreads>(sidx, E, a.s1.rows, a.s1.min_one, a.s1.tiles, a.s1.tile_off,
                                   a.s1.n_tiles, a.total, a.s1.split_rows);
    if (one ? tb == 0 : tb == 2)
      tile_pass<int32_t, kThreads>(sidx, E, a.s2.rows, a.s2.min_one, a.s2.tiles, a.s2.tile_off,
                                   a.s2.n_tiles, a.total, a.s2.split_rows);
  }
  pro_ts(5);
  if (!a.x) return;
  grid.sync();
  pro_ts(6);
  // ---- 4: expert-sorted copy of x (pads -> zero rows) --------------------
  // a warp moves 4 rows at a time: the 4 index loads, then every 16-byte
  // unit of the 4 rows loaded into registers (8 per lane in flight) before
  // any store, so a warp keeps up to 4 KB of reads outstanding
  {
    const int64_t np = sidx[E];
    const char* X = static_cast<const char*>(a.x);
    char* XS = static_cast<char*>(a.xs);
    const int64_t rb = a.row_bytes;
    if (a.unit == 16) {
      // each warp owns a contiguous run of positions: one coalesced load of
      // its indices, then batches of 8 rows with every load in flight
      // before the stores (8 rows x 1 KB per pass)
      const int upr = static_cast<int>(rb / 16);  // 16-byte units per row
      const int ntok = static_cast<int>(a.n_tok);
      const int64_t per = (ceil_div(np, nwarps) + 7) / 8 * 8;
      const int64_t pb = static_cast<int64_t>(gwarp) * per;
      const int64_t pe = min(np, pb + per);
      for (int64_t q0 = pb; q0 < pe; q0 += 32) {
        const int sv_l = q0 + lane < pe ? a.v[q0 + lane] : -1;
        const int tok_l = sv_l < 0 ? -1 : sv_l % ntok;
        for (int r0 = 0; r0 < 32 && q0 + r0 < pe; r0 += 8) {
          const char* src[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int tk = __shfl_sync(0xffffffffu, tok_l, r0 + u);
            src[u] = tk < 0 ? nullptr : X + static_cast<int64_t>(tk) * rb;
          }
          for (int c0 = 0; c0 < upr; c0 += 64) {
            uint4 buf[8][2];
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
              for (int m = 0; m < 2; ++m) {
                const int o = c0 + m * 32 + lane;
                buf[u][m] = (src[u] && o < upr)
                                ? __ldg(reinterpret_cast<const uint4*>(src[u]) + o)
                                : make_uint4(0u, 0u, 0u, 0u);
              }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (q0 + r0 + u >= pe) break;
              uint4* dst = reinterpret_cast<uint4*>(XS + (q0 + r0 + u) * rb);
#pragma unroll
              for (int m = 0; m < 2; ++m) {
                const int o = c0 + m * 32 + lane;
                if (o < upr) dst[o] = buf[u][m];
              }
            }
          }
        }
      }
    } else {
      for (int64_t p = gwarp; p < np; p += nwarps) {
        const int sv = a.v[p];
        char* dst = XS + p * rb;
        if (sv < 0) zero_row(dst, rb, lane, a.unit);
        else copy_row(X + (sv % a.n_tok) * rb, dst, rb, lane, a.unit);
      }
    }
  }
  __syncthreads();
  pro_ts(7);
}


// ---------------------------------------- one-barrier forward prologue --
// Same outputs as fwd_prologue (bit-identical v / idx / tiles, y = 0, the
// expert-sorted x copy) with ONE grid barrier instead of three:
//   A  block b owns the contiguous slots [b*S, (b+1)*S) as S/32 groups of 32:
//      per group, __match_any_sync gives every slot its rank among equal
//      experts and the group's per-expert counts (smem, no atomics); the
//      group counts are scanned in place, the block's counts published.
//   -- grid.sync --
//   B  every block sums the published counts itself (experts' totals and the
//      counts of the blocks before it: G x E ints from L2), scans the padded
//      totals into idx, places its own slots (position = idx[e] + earlier
//      blocks + earlier groups + rank in group -- the reference's stable
//      token-order placement, routing.cpp:64-68) and copies their x rows to
//      the sorted positions; pads (-1 in v, zero rows in x_s) are spread over
//      the blocks by expert; y is zeroed first so its stores overlap the
//      index arithmetic.  The last three blocks write the three tile tables.
constexpr int kFastMaxE = 256;
constexpr int kFastMaxGroups = 32;
__global__ void __launch_bounds__(kThreads) fwd_prologue_1b(FwdPrologue a) {
  namespace cg = cooperative_groups;
  pro_ts(0);
  pdl_trigger();
  cg::grid_group grid = cg::this_grid();
  const int E = a.E;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int groups = a.chunk / 32;  // S = a.chunk slots per block
  const int64_t s0 = static_cast<int64_t>(blockIdx.x) * a.chunk;
  __shared__ int32_t gh[kFastMaxGroups][kFastMaxE];  // per-group counts -> exclusive scan
  __shared__ int32_t tot[kFastMaxE + 1];
  __shared__ int32_t bef[kFastMaxE];
  __shared__ int32_t sidx[kFastMaxE + 1];
  __shared__ __align__(16) int32_t part4[2 * kThreads * 4];
  extern __shared__ int32_t dyn[];
  int32_t* se = dyn;             // [S] expert of slot i (-1: invalid / past the end)
  int32_t* sr = dyn + a.chunk;   // [S] rank of slot i among its group's equal experts
  // ---- A: group histograms and ranks --------------------------------------
  if (a.zero_i32 && blockIdx.x == 0)
    for (int i = threadIdx.x; i < a.zero_n; i += kThreads) a.zero_i32[i] = 0;
  for (int j = warp; j < groups; j += kWarps) {
    for (int e = lane; e < E; e += 32) gh[j][e] = 0;
    __syncwarp();
    const int64_t s = s0 + 32 * j + lane;
    int e = s < a.n_slots ? a.a[s] : -1;
    if (s < a.n_slots && (e < 0 || e >= E)) {
      if (a.status) atomicExch(a.status, HXM_ERR_INVALID_ARG);
      e = -1;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    se[32 * j + lane] = e;
    sr[32 * j + lane] = __popc(peers & ((1u << lane) - 1u));
    if (e >= 0 && (__ffs(peers) - 1) == lane) gh[j][e] = __popc(peers);
    // per-token distinctness of the k choices (routing.cpp:30-39): a slot
    // checks the later choices of its token
    if (a.status && a.k > 1 && e >= 0) {
      const int ci = static_cast<int>(s / a.n_tok);
      const int64_t t = s - ci * a.n_tok;
      for (int c2 = ci + 1; c2 < a.k; ++c2)
        if (a.a[c2 * a.n_tok + t] == e) atomicExch(a.status, HXM_ERR_INVALID_ARG);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += kThreads) {
    int32_t run = 0;
    for (int j = 0; j < groups; ++j) {
      const int32_t c = gh[j][e];
      gh[j][e] = run;
      run += c;
    }
    a.cnt[static_cast<int64_t>(blockIdx.x) * E + e] = run;
  }
  pro_ts(1);
  grid.sync();
  pro_ts(2);
  // ---- B: totals and the counts of the blocks before this one -------------
  // thread (r, q) reads the int4 column group q (experts 4q..4q+3) of rows
  // r, r + R, ... of the G x E count table, eight rows in flight at a time
  // (one L2 round trip per batch), then the R row groups are added in a
  // fixed order.  E % 4 == 0 and E <= 256 on this path.
  {
    const int Q = E / 4, R = kThreads / Q;
    const int r = threadIdx.x / Q, q = threadIdx.x % Q;
    const int G = gridDim.x, me = blockIdx.x;
    int4 t_all = make_int4(0, 0, 0, 0), t_bef = make_int4(0, 0, 0, 0);
    if (r < R) {
      const int4* cnt4 = reinterpret_cast<const int4*>(a.cnt);
      for (int b0 = r; b0 < G; b0 += 8 * R) {
        int4 c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int b = b0 + u * R;
          c[u] = b < G ? __ldcg(cnt4 + static_cast<int64_t>(b) * Q + q) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int b = b0 + u * R;
          t_all.x += c[u].x; t_all.y += c[u].y; t_all.z += c[u].z; t_all.w += c[u].w;
          if (b < me) { t_bef.x += c[u].x; t_bef.y += c[u].y; t_bef.z += c[u].z; t_bef.w += c[u].w; }
        }
      }
    }
    int4* p4 = reinterpret_cast<int4*>(part4);
    p4[threadIdx.x] = t_all;
    p4[kThreads + threadIdx.x] = t_bef;
    __syncthreads();
    if (threadIdx.x < E) {
      const int qq = threadIdx.x / 4, j = threadIdx.x % 4;
      int32_t s = 0, sb = 0;
      for (int rr = 0; rr < R; ++rr) {
        s += part4[(rr * Q + qq) * 4 + j];
        sb += part4[(kThreads + rr * Q + qq) * 4 + j];
      }
      tot[threadIdx.x] = s;
      bef[threadIdx.x] = sb;
    }
    __syncthreads();
  }
  pro_ts(3);
  block_idx<int32_t>(tot, E, a.blk, sidx, a.capacity);
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e <= E; e += kThreads) a.idx[e] = sidx[e];
  // placement of this block's slots (slot id = flat assignment position)
  const int S = a.chunk;
  for (int i = threadIdx.x; i < S; i += kThreads) {
    const int e = se[i];
    int32_t pos = -1;
    if (e >= 0) {
      const int32_t within = bef[e] + gh[i / 32][e] + sr[i];
      if (a.capacity <= 0 || within < a.capacity) {
        pos = sidx[e] + within;
        a.v[pos] = static_cast<int32_t>(s0 + i);
      }
    }
    sr[i] = pos;  // reused: the sorted position of slot i (-1: none)
  }
  // pads of the experts this block owns: -1 in v, zero rows in x_s
  const char* X = static_cast<const char*>(a.x);
  char* XS = static_cast<char*>(a.xs);
  const int64_t rb = a.row_bytes;
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    const int64_t tt = tot[e];
    const int64_t kept = (a.capacity > 0 && tt > a.capacity) ? a.capacity : tt;
    const int64_t p0 = static_cast<int64_t>(sidx[e]) + kept, p1 = sidx[e + 1];
    for (int64_t p = p0 + threadIdx.x; p < p1; p += kThreads) a.v[p] = -1;
    if (a.x)
      for (int64_t p = p0 + warp; p < p1; p += kWarps) zero_row(XS + p * rb, rb, lane, a.unit);
  }
  pro_ts(4);
  // y = 0: its stores overlap the tile passes and this block's row copies
  {
    const int64_t gtid = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    zero_f32(a.y, a.y_elems, gtid, static_cast<int64_t>(gridDim.x) * kThreads);
  }
  // the three tilings on the last three blocks
  {
    const int tb = static_cast<int>(gridDim.x) - 1 - static_cast<int>(blockIdx.x);
    const bool one = gridDim.x < 3;
    if (tb == 0)
      tile_pass<int32_t, kThreads>(sidx, E, a.s0.rows, a.s0.min_one, a.s0.tiles, a.s0.tile_off,
                                   a.s0.n_tiles, tot, a.s0.split_rows);
    if (one ? tb == 0 : tb == 1)
      tile_pass<int32_t, kThreads>(sidx, E, a.s1.rows, a.s1.min_one, a.s1.tiles, a.s1.tile_off,
                                   a.s1.n_tiles, tot, a.s1.split_rows);
    if (one ? tb == 0 : tb == 2)
      tile_pass<int32_t, kThreads>(sidx, E, a.s2.rows, a.s2.min_one, a.s2.tiles, a.s2.tile_off,
                                   a.s2.n_tiles, tot, a.s2.split_rows);
  }
  pro_ts(5);
  if (!a.x) return;
  __syncthreads();
  // ---- B': x rows of this block's slots to their sorted positions ---------
  // each warp a contiguous run of the block's slots, 8 rows in flight
  const int per = (S + kWarps - 1) / kWarps;
  const int i0 = warp * per, i1 = min(S, i0 + per);
  if (a.unit == 16) {
    const int upr = static_cast<int>(rb / 16);
    for (int r0 = i0; r0 < i1; r0 += 8) {
      const char* src[8];
      int64_t dpos[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = r0 + u;
        const int32_t pos = i < i1 ? sr[i] : -1;
        dpos[u] = pos;
        src[u] = pos < 0 ? nullptr : X + ((s0 + i) % a.n_tok) * rb;
      }
      for (int c0 = 0; c0 < upr; c0 += 64) {
        uint4 buf[8][2];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            const int o = c0 + m * 32 + lane;
            buf[u][m] = (src[u] && o < upr) ? __ldg(reinterpret_cast<const uint4*>(src[u]) + o)
                                            : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (dpos[u] < 0) continue;
          uint4* dst = reinterpret_cast<uint4*>(XS + dpos[u] * rb);
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            const int o = c0 + m * 32 + lane;
            if (o < upr) dst[o] = buf[u][m];
          }
        }
      }
    }
  } else {
    for (int i = i0; i < i1; ++i) {
      const int32_t pos = sr[i];
      if (pos >= 0) copy_row(X + ((s0 + i) % a.n_tok) * rb, XS + pos * rb, rb, lane, a.unit);
    }
  }
  __syncthreads();
  pro_ts(6);
}

}  // namespace

size_t reindex_ws_bytes(int64_t n, int64_t E, int64_t k) {
  const int chunk = pick_chunk(n);
  const int64_t nchunks = ceil_div(n, chunk);
  Arena ar(nullptr, 0);
  ar.take<int32_t>((static_cast<size_t>(nchunks) * E + 1) * k);
  ar.take<int32_t>((static_cast<size_t>(nchunks) * E + 1) * k);
  ar.take<int32_t>((E + 1) * k);
  return ar.used;
}


template <class IdxT>
hxm_status launch_tiles(const IdxT* idx, int64_t E, int rows, bool min_one,
                        SegTile* tiles, int32_t* tile_off, int32_t* n_tiles,
                        cudaStream_t st, int split_rows) {
  const TileSpec s{rows, min_one ? 1 : 0, tiles, tile_off, n_tiles, split_rows};
  build_tiles<IdxT><<<1, 1024, 0, st>>>(idx, static_cast<int>(E), s, s, s, 1);
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}
template hxm_status launch_tiles<int32_t>(const int32_t*, int64_t, int, bool, SegTile*,
                                          int32_t*, int32_t*, cudaStream_t, int);
template hxm_status launch_tiles<int64_t>(const int64_t*, int64_t, int, bool, SegTile*,
                                          int32_t*, int32_t*, cudaStream_t, int);

hxm_status launch_fwd_prologue(FwdPrologue a, cudaStream_t st) {
  static int occ_cache[64] = {0};
  static size_t occ_smem[64] = {0};
  static int occ1_cache[64] = {0};
  static size_t occ1_smem[64] = {0};
  int dev = 0;
  HXM_TRY_CUDA(cudaGetDevice(&dev));
  dev = dev < 64 ? dev : 63;
  const char* ge = std::getenv("HXM_PRO_BLOCKS");
  const int per_sm = ge ? std::max(1, std::atoi(ge)) : 2;
  const char* g1 = std::getenv("HXM_PRO1");  // 0: the three-barrier prologue
  // one-barrier prologue: S = 32 * groups slots per block, every block
  // co-resident, the group counts in static smem
  if (!(g1 && g1[0] == '0') && a.E <= kFastMaxE && a.E % 4 == 0) {
    const int64_t slots_max = static_cast<int64_t>(sm_count()) * per_sm;
    const int groups = static_cast<int>(std::max<int64_t>(1, ceil_div(a.n_slots, 32 * slots_max)));
    if (groups <= kFastMaxGroups) {
      a.chunk = 32 * groups;
      a.nchunks = static_cast<int>(std::max<int64_t>(1, ceil_div(a.n_slots, a.chunk)));
      Arena ar(a.ws, a.ws_bytes);
      a.cnt = ar.take<int32_t>(static_cast<size_t>(a.nchunks) * a.E + 1);
      a.base = nullptr;
      a.total = nullptr;
      if (ar.overflow) return invalid_arg("layer prologue: workspace too small");
      const size_t smem = 2 * static_cast<size_t>(a.chunk) * sizeof(int32_t);
      if (occ1_smem[dev] != smem) {
        HXM_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1_cache[dev],
                                                                   fwd_prologue_1b, kThreads, smem));
        occ1_smem[dev] = smem;
      }
      if (static_cast<int64_t>(occ1_cache[dev]) * sm_count() >= a.nchunks) {
        void* args[] = {&a};
        HXM_TRY_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fwd_prologue_1b),
                                                 dim3(a.nchunks), dim3(kThreads), args, smem, st));
        HXM_CHECK_LAUNCH();
        return HXM_OK;
      }
    }
  }
  a.chunk = pick_chunk(a.n_slots);
  a.nchunks = static_cast<int>(ceil_div(a.n_slots, a.chunk));
  Arena ar(a.ws, a.ws_bytes);
  a.cnt = ar.take<int32_t>(static_cast<size_t>(a.nchunks) * a.E + 1);
  a.base = ar.take<int32_t>(static_cast<size_t>(a.nchunks) * a.E + 1);
  a.total = ar.take<int32_t>(a.E + 1);
  if (ar.overflow) return invalid_arg("layer prologue: workspace too small");
  const size_t smem = std::max(static_cast<size_t>(kWarps) * a.E * sizeof(int32_t),
                               (align_up(a.E + 1, 4) + static_cast<size_t>(kWarps) * a.E) *
                                   sizeof(int32_t));
  // per-device cache of the kernel attribute / occupancy query
  if (occ_smem[dev] != smem) {
    if (smem > 48 * 1024)
      HXM_TRY_CUDA(cudaFuncSetAttribute(fwd_prologue, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    HXM_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_cache[dev], fwd_prologue,
                                                               kThreads, smem));
    occ_smem[dev] = smem;
  }
  const int occ = occ_cache[dev];
  if (occ < 1) return invalid_arg("layer prologue: cannot be resident");
  const int grid = sm_count() * std::min(occ, per_sm);
  void* args[] = {&a};
  HXM_TRY_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fwd_prologue), dim3(grid),
                                           dim3(kThreads), args, smem, st));
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

}  // namespace hxm
extern "C" void hxm_debug_prologue_ts(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, hxm::g_pro_ts, sizeof(unsigned long long) * 8);
}
namespace hxm {
int64_t max_tiles(int64_t n_padded_bound, int64_t E, int rows) {
  return ceil_div(n_padded_bound, rows) + E + 1;
}

}  // namespace hxm

extern "C" {

size_t hxm_reindex_bound(int64_t n, int64_t E, int64_t blk) {
  if (n < 0 || E < 0) return 0;
  return static_cast<size_t>(n + E * (blk > 0 ? blk - 1 : 0));
}

size_t hxm_reindex_workspace_bytes(int64_t n, int64_t E) {
  return hxm::reindex_ws_bytes(n, E, 1);
}

size_t hxm_reindex_all_workspace_bytes(int64_t n, int64_t E, int64_t k) {
  return k < 1 ? 0 : hxm::reindex_ws_bytes(n, E, k);
}

hxm_status hxm_build_reindex_all(const int32_t* assignments, int64_t k, int64_t n, int64_t E,
                                 int64_t blk, int64_t* v, int64_t v_stride, int64_t* idx,
                                 void* ws, size_t ws_bytes, int32_t* status,
                                 hxm_stream_t stream) {
  // routing.cpp:72-80: one build_reindex per choice, same checks first
  if (blk <= 0) return hxm::invalid_arg("build_reindex: blk must be >= 1");
  if (n < 0 || E <= 0 || k < 1) return hxm::invalid_arg("build_reindex_all: need n >= 0, E >= 1, k >= 1");
  if (n > 0x7fffffffLL) return hxm::invalid_arg("build_reindex: n exceeds int32 range");
  if (v_stride < static_cast<int64_t>(hxm_reindex_bound(n, E, blk)))
    return hxm::invalid_arg("build_reindex_all: v_stride below hxm_reindex_bound");
  return hxm::build_impl<int64_t, int64_t>(assignments, n, E, blk, v, idx, ws, ws_bytes, status,
                                           reinterpret_cast<cudaStream_t>(stream),
                                           static_cast<int>(k), v_stride);
}

hxm_status hxm_build_reindex(const int32_t* a, int64_t n, int64_t E, int64_t blk,
                             int64_t* v, int64_t* idx, void* ws, size_t ws_bytes,
                             int32_t* status, hxm_stream_t stream) {
  // routing.cpp:44 -- checked before any device work
  if (blk <= 0) return hxm::invalid_arg("build_reindex: blk must be >= 1");
  if (n < 0 || E <= 0) return hxm::invalid_arg("build_reindex: need n >= 0 and E >= 1");
  if (n > 0x7fffffffLL) return hxm::invalid_arg("build_reindex: n exceeds int32 range");
  return hxm::build_impl<int64_t, int64_t>(a, n, E, blk, v, idx, ws, ws_bytes, status,
                                           reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
