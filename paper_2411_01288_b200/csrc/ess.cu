// ess.cu -- expert-specific segmented sum (ESS), the bias-gradient operator.
//
// Replaces moekit::ess (reference core/src/es_ops.cpp:86-102, 180-191):
// out[e] = sum of the rows routed to expert e.  HBM-bound: every routed row is
// read once (16-byte vector loads, consecutive threads on consecutive
// columns so a gathered row is one coalesced burst) and E x D fp32 is written.
// Two deterministic phases, no float atomics:
//   ess_partial : one CTA per <=128-position segment tile -> partial[tile][D]
//   ess_combine : out[e][d] = sum of e's tile partials in tile order.
#include <cooperative_groups.h>
#include <type_traits>

#include "kernels.cuh"

namespace hxm {
namespace {

constexpr int NT = 256;

template <class T, int VEC>
__device__ __forceinline__ void load_vec(const T* p, float (&v)[VEC]) {
  if constexpr (sizeof(T) * VEC == 16) {
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(p));
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = to_f32(e[i]);
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = to_f32(p[i]);
  }
}

template <class T, int VEC>
__device__ __forceinline__ void store_vec(T* p, const float (&v)[VEC]) {
  if constexpr (sizeof(T) * VEC == 16) {
    uint4 raw;
    T* e = reinterpret_cast<T*>(&raw);
#pragma unroll
    for (int i = 0; i < VEC; ++i) e[i] = from_f32<T>(v[i]);
    *reinterpret_cast<uint4*>(p) = raw;
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) p[i] = from_f32<T>(v[i]);
  }
}

// One (segment tile, column slab) item: the tile's rows summed into
// partial[tile] (and optionally copied to expert-sorted order).  The 8 warps
// split the tile's rows, each keeping U = 4 row loads in flight, and are
// combined in a fixed order through smem (deterministic).
template <class T, int VEC>
__device__ __forceinline__ void ess_item(const EssArgs& a, int ti, int slab) {
  const SegTile tile = a.tiles[ti];
  const T* X = static_cast<const T*>(a.x);
  const int64_t D = a.d;
  const int col_groups = static_cast<int>((D + VEC - 1) / VEC);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int W = NT / 32;
  const int cg = slab * 32 + lane;
  __shared__ int rows[kEssRows];
  __shared__ float red[W][32 * VEC];
  __syncthreads();  // previous item's smem reads are done
  for (int i = threadIdx.x; i < kEssRows; i += NT) {
    const int64_t p = tile.begin + i;
    rows[i] = p < tile.end ? a.map(p) : -1;
  }
  __syncthreads();
  const int nrows = tile.end - tile.begin;
  float acc[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
  if (cg < col_groups) {
    constexpr int U = 4;  // rows in flight per thread
    for (int r0 = warp; r0 < nrows; r0 += W * U) {
      float v[U][VEC];
      int rr[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = r0 + u * W;
        rr[u] = r < nrows ? rows[r] : -2;
        if (rr[u] >= 0) {
          load_vec<T, VEC>(X + static_cast<int64_t>(rr[u]) * D + static_cast<int64_t>(cg) * VEC,
                           v[u]);
        } else {
#pragma unroll
          for (int i = 0; i < VEC; ++i) v[u][i] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int i = 0; i < VEC; ++i) acc[i] += v[u][i];
        if (a.copy_out && rr[u] != -2) {  // padding slots copy as zero rows
          T* dst = static_cast<T*>(a.copy_out) +
                   (static_cast<int64_t>(tile.begin) + r0 + u * W) * D +
                   static_cast<int64_t>(cg) * VEC;
          store_vec<T, VEC>(dst, v[u]);
        }
      }
    }
  }
  if (!a.partial) return;
#pragma unroll
  for (int i = 0; i < VEC; ++i) red[warp][lane * VEC + i] = acc[i];
  __syncthreads();
  // column sums in a fixed warp order (deterministic)
  for (int c = threadIdx.x; c < 32 * VEC; c += NT) {
    const int64_t col = static_cast<int64_t>(slab) * 32 * VEC + c;
    if (col >= D) continue;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) s += red[w][c];
    a.partial[static_cast<int64_t>(ti) * D + col] = s;
  }
}

// Whole-row variant: one item is a full segment tile (every column), the
// lanes loop over GPL column groups, so a bf16 row of up to 32*GPL*VEC
// columns is one item (no half-empty column slabs, one round of items).
template <class T, int VEC, int GPL>
__device__ __forceinline__ void ess_item_rows(const EssArgs& a, int ti) {
  const SegTile tile = a.tiles[ti];
  const T* X = static_cast<const T*>(a.x);
  const int64_t D = a.d;
  const int col_groups = static_cast<int>(D / VEC);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int W = NT / 32;
  __shared__ int rows[kEssRows];
  __shared__ float red[W][32 * VEC * GPL];
  __syncthreads();
  for (int i = threadIdx.x; i < kEssRows; i += NT) {
    const int64_t p = tile.begin + i;
    rows[i] = p < tile.end ? a.map(p) : -1;
  }
  __syncthreads();
  const int nrows = tile.end - tile.begin;
  float acc[GPL][VEC];
#pragma unroll
  for (int g = 0; g < GPL; ++g)
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[g][i] = 0.f;
  // rows in flight per warp (x GPL groups per lane); 16-byte vectors stay
  // raw (4 registers, not VEC floats) until they are summed, so 8 rows fit
  // the register budget of 4 converted ones: a 128-row item is two rounds of
  // loads instead of four.  Each warp still sums rows warp, warp + W, ... in
  // ascending order (the same partials as before).
  constexpr bool kRaw = sizeof(T) * VEC == 16;
  constexpr int U = kRaw ? 8 : 4;
  for (int r0 = warp; r0 < nrows; r0 += W * U) {
    uint4 raw[kRaw ? U : 1][GPL];
    float v[kRaw ? 1 : U][GPL][VEC];
    int rr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * W;
      rr[u] = r < nrows ? rows[r] : -2;
#pragma unroll
      for (int g = 0; g < GPL; ++g) {
        const int cg = lane + 32 * g;
        const bool ok = rr[u] >= 0 && cg < col_groups;
        const T* src = X + static_cast<int64_t>(ok ? rr[u] : 0) * D + static_cast<int64_t>(cg) * VEC;
        if constexpr (kRaw) {
          raw[u][g] = ok ? __ldg(reinterpret_cast<const uint4*>(src)) : make_uint4(0u, 0u, 0u, 0u);
        } else {
          if (ok)
            load_vec<T, VEC>(src, v[u][g]);
          else
#pragma unroll
            for (int i = 0; i < VEC; ++i) v[u][g][i] = 0.f;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (rr[u] == -2) continue;
#pragma unroll
      for (int g = 0; g < GPL; ++g) {
        const int cg = lane + 32 * g;
        if (cg >= col_groups) continue;
        T* dst = a.copy_out ? static_cast<T*>(a.copy_out) +
                                  (static_cast<int64_t>(tile.begin) + r0 + u * W) * D +
                                  static_cast<int64_t>(cg) * VEC
                            : nullptr;
        if constexpr (kRaw) {
          const T* e = reinterpret_cast<const T*>(&raw[u][g]);
#pragma unroll
          for (int i = 0; i < VEC; ++i) acc[g][i] += to_f32(e[i]);
          if (dst) *reinterpret_cast<uint4*>(dst) = raw[u][g];  // padding slots copy as zero rows
        } else {
#pragma unroll
          for (int i = 0; i < VEC; ++i) acc[g][i] += v[u][g][i];
          if (dst) store_vec<T, VEC>(dst, v[u][g]);
        }
      }
    }
  }
  if (!a.partial) return;
#pragma unroll
  for (int g = 0; g < GPL; ++g)
#pragma unroll
    for (int i = 0; i < VEC; ++i) red[warp][(lane + 32 * g) * VEC + i] = acc[g][i];
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += NT) {  // fixed warp order: deterministic
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) s += red[w][c];
    a.partial[static_cast<int64_t>(ti) * D + c] = s;
  }
}

template <class T, int VEC>
__global__ void __launch_bounds__(NT) ess_partial(EssArgs a) {
  // grid: x = segment tile (<= 128 positions), y = column slab of 32 vector
  // groups (one per lane)
  if (static_cast<int>(blockIdx.x) >= *a.n_tiles) return;
  ess_item<T, VEC>(a, blockIdx.x, blockIdx.y);
}

// out_row[c0 .. c0+128) = column sums of partial rows [r0, r1) (row stride d):
// the block's W warps split the rows (4 rows in flight per warp, each lane
// 4 columns), then fixed-order smem combine -> deterministic, and a long
// reduction (a skewed expert's hundreds of tiles) is W-way parallel.
// kFresh: the partial rows were written by other blocks of the running
// kernel -- read them through L2 (ld.global.cg), not the read-only path
template <int W, bool kFresh = false>
__device__ __forceinline__ void combine_block(const float* __restrict__ partial, int64_t r0,
                                              int64_t r1, int64_t d, int64_t c0,
                                              float* __restrict__ out_row) {
  __shared__ float red[W][128];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t c = c0 + lane * 4;
  const bool vec = (d % 4 == 0) && c + 4 <= d;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t r = r0 + warp; r < r1; r += 4 * W) {
    float v[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t rr = r + u * W;
      const float* row = partial + rr * d;
      if (rr < r1 && vec) {
        const float4 q = kFresh ? __ldcg(reinterpret_cast<const float4*>(row + c))
                                : __ldg(reinterpret_cast<const float4*>(row + c));
        v[u][0] = q.x; v[u][1] = q.y; v[u][2] = q.z; v[u][3] = q.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          v[u][j] = (rr < r1 && c + j < d) ? (kFresh ? __ldcg(row + c + j) : __ldg(row + c + j)) : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] += v[u][j];
  }
  __syncthreads();  // red[] reuse across calls
#pragma unroll
  for (int j = 0; j < 4; ++j) red[warp][lane * 4 + j] = acc[j];
  __syncthreads();
  for (int t = threadIdx.x; t < 128; t += W * 32) {
    if (c0 + t >= d) continue;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) s += red[w][t];
    out_row[c0 + t] = s;
  }
}

__global__ void __launch_bounds__(256) ess_combine(EssArgs a) {
  const int e = blockIdx.y;
  combine_block<8>(a.partial, a.tile_off[e], a.tile_off[e + 1], a.d,
                   static_cast<int64_t>(blockIdx.x) * 128, a.out + static_cast<int64_t>(e) * a.d);
}

__global__ void __launch_bounds__(256) colsum_combine(const float* __restrict__ partial,
                                                      const int32_t* __restrict__ tile_off,
                                                      int parts, int64_t d,
                                                      float* __restrict__ out) {
  const int e = blockIdx.y;
  combine_block<8>(partial, static_cast<int64_t>(tile_off[e]) * parts,
                   static_cast<int64_t>(tile_off[e + 1]) * parts, d,
                   static_cast<int64_t>(blockIdx.x) * 128, out + static_cast<int64_t>(e) * d);
}

template <class T>
hxm_status launch_typed(const EssArgs& a, cudaStream_t st) {
  constexpr int V = 16 / sizeof(T);
  if (a.max_tiles > 0) {
    const bool vec_ok = (a.d % V == 0) && (reinterpret_cast<uintptr_t>(a.x) % 16 == 0) &&
                        (reinterpret_cast<uintptr_t>(a.copy_out) % 16 == 0);
    const int64_t groups = vec_ok ? ceil_div(a.d, V) : a.d;
    dim3 grid(static_cast<unsigned>(a.max_tiles), static_cast<unsigned>(ceil_div(groups, 32)));
    if (vec_ok) ess_partial<T, V><<<grid, NT, 0, st>>>(a);
    else ess_partial<T, 1><<<grid, NT, 0, st>>>(a);
    HXM_CHECK_LAUNCH();
  }
  dim3 grid(static_cast<unsigned>(ceil_div(a.d, 128)), static_cast<unsigned>(a.n_experts));
  if (a.d > 0 && a.n_experts > 0 && a.out) {
    ess_combine<<<grid, 256, 0, st>>>(a);
    HXM_CHECK_LAUNCH();
  }
  return HXM_OK;
}

// dst[p] = src[map(p)] (pads -> zero rows) for p < idx[E].  Each warp owns a
// contiguous run of positions: one coalesced load of its indices, then
// batches of 8 rows whose 16-byte units are all loaded before any store.
template <class T, class IdxT>
__global__ void __launch_bounds__(NT) gather_rows(const T* __restrict__ src, RowMap map,
                                                  int64_t d, const IdxT* __restrict__ idx,
                                                  int E, T* __restrict__ dst) {
  const int64_t np = idx[E];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (NT / 32);
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NT / 32) + warp;
  const int64_t rb = d * static_cast<int64_t>(sizeof(T));
  const bool vec = rb % 16 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(dst) % 16 == 0;
  const int64_t per = (ceil_div(np, nwarps) + 7) / 8 * 8;
  const int64_t pb = gw * per, pe = min(np, pb + per);
  const char* S = reinterpret_cast<const char*>(src);
  char* Dst = reinterpret_cast<char*>(dst);
  for (int64_t q0 = pb; q0 < pe; q0 += 32) {
    const int row_l = q0 + lane < pe ? map(q0 + lane) : -1;
    for (int r0 = 0; r0 < 32 && q0 + r0 < pe; r0 += 8) {
      int rows[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) rows[u] = __shfl_sync(0xffffffffu, row_l, r0 + u);
      if (vec) {
        const int64_t upr = rb / 16;
        for (int64_t c0 = 0; c0 < upr; c0 += 64) {
          uint4 buf[8][2];
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int m = 0; m < 2; ++m) {
              const int64_t o = c0 + m * 32 + lane;
              buf[u][m] = (rows[u] >= 0 && o < upr)
                              ? __ldg(reinterpret_cast<const uint4*>(S + rows[u] * rb) + o)
                              : make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (q0 + r0 + u >= pe) break;
            uint4* o4 = reinterpret_cast<uint4*>(Dst + (q0 + r0 + u) * rb);
#pragma unroll
            for (int m = 0; m < 2; ++m) {
              const int64_t o = c0 + m * 32 + lane;
              if (o < upr) o4[o] = buf[u][m];
            }
          }
        }
      } else {
        for (int u = 0; u < 8 && q0 + r0 + u < pe; ++u) {
          T* o = dst + (q0 + r0 + u) * d;
          for (int64_t c = lane; c < d; c += 32)
            o[c] = rows[u] >= 0 ? src[static_cast<int64_t>(rows[u]) * d + c] : from_f32<T>(0.f);
        }
      }
    }
  }
}

template <class T, class IdxT>
hxm_status gather_typed(const void* src, RowMap map, int64_t d, const IdxT* idx, int E,
                        int64_t bound, void* dst, cudaStream_t st) {
  const int blocks = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(bound, 8 * (NT / 32)), static_cast<int64_t>(sm_count()) * 4)));
  gather_rows<T, IdxT><<<blocks, NT, 0, st>>>(static_cast<const T*>(src), map, d, idx, E,
                                              static_cast<T*>(dst));
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

// ------------------------------------------------ fused backward prologue --
// One launch before the backward GEMMs: g_x = 0, zeroed gW slices of the
// experts whose ESTMM is split over chunks (they accumulate with red.add),
// gb2 partials of g_y fused with its expert-sorted copy (ESS,
// es_ops.cpp:86-102), and each expert's gb2 combine by the block that
// finishes its last ESS item.
template <class T, int VEC>
__global__ void __launch_bounds__(NT) bwd_prologue(BwdPrologue b) {
  const EssArgs& a = b.es;
  pdl_trigger();
  const int col_groups = static_cast<int>((a.d + VEC - 1) / VEC);
  const bool rows = VEC > 1 && col_groups <= 32 * 2 && a.d % VEC == 0;
  const int slabs = rows ? 1 : static_cast<int>(ceil_div(col_groups, 32));
  const int chunks = static_cast<int>(ceil_div(a.d, 128));
  // gb2 of an expert without positions is zero
  if (a.out)
    for (int e = blockIdx.x; e < a.n_experts; e += gridDim.x)
      if (a.tile_off[e + 1] == a.tile_off[e])
        for (int64_t c = threadIdx.x; c < a.d; c += NT) a.out[static_cast<int64_t>(e) * a.d + c] = 0.f;
  // after an item: the block that brings an expert's item count to its total
  // combines that expert's partial rows (fixed order: deterministic) -- no
  // grid-wide barrier; the counter is left at zero for the next call.
  // Arrival-counter protocol (a classic threadfence reduction):
  //   release (every arriving block): bar.sync -- all of this block's
  //     partial-row stores precede thread 0's next step in block order;
  //     thread 0 __threadfence() (fence.sc.gpu, cumulative over those
  //     stores); then the counter atomicAdd.
  //   acquire (the last arriver): its atomicAdd observes every other
  //     block's increment, hence (fence cumulativity) their partial rows;
  //     thread 0 __threadfence(); bar.sync publishes `last` to the block;
  //     combine_block then reads the partials with ld.global.cg (L2, never
  //     a stale L1 line).
  __shared__ int last;
  auto arrive = [&](int ti) {
    if (!a.out) return;
    const int e = a.tiles[ti].expert;
    __syncthreads();  // release, step 1: the block's partial stores are issued
    if (threadIdx.x == 0) {
      __threadfence();  // release, step 2 (cumulative over the block's stores)
      const int total = (a.tile_off[e + 1] - a.tile_off[e]) * slabs;
      last = atomicAdd(&b.done[e], 1) == total - 1;
      if (last) {
        b.done[e] = 0;
        __threadfence();
      }
    }
    __syncthreads();
    if (last)
      for (int c = 0; c < chunks; ++c)
        combine_block<NT / 32, true>(a.partial, a.tile_off[e], a.tile_off[e + 1], a.d,
                                     static_cast<int64_t>(c) * 128,
                                     a.out + static_cast<int64_t>(e) * a.d);
  };
  if (rows) {
    // whole rows per item (D <= 64 * VEC): one round of items, no half slabs
    for (int ti = blockIdx.x; ti < *a.n_tiles; ti += gridDim.x) {
      ess_item_rows<T, VEC, 2>(a, ti);
      arrive(ti);
    }
  } else {
    const int items = *a.n_tiles * slabs;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      ess_item<T, VEC>(a, it / slabs, it % slabs);
      arrive(it / slabs);
    }
  }
  // g_x = 0 and the split experts' gW slices = 0 after the (latency-bound)
  // ESS items: on the blocks without an item when at least a quarter of the
  // grid has none (their stores then overlap the items' loads), else on all
  const int items = rows ? *a.n_tiles : *a.n_tiles * slabs;
  const int zb0 = (items < static_cast<int>(gridDim.x) &&
                   static_cast<int>(gridDim.x) - items >= static_cast<int>(gridDim.x) / 4)
                      ? items : 0;
  if (static_cast<int>(blockIdx.x) < zb0) return;
  const int zblk = blockIdx.x - zb0, nzb = gridDim.x - zb0;
  zero_f32(b.gx, b.gx_elems, static_cast<int64_t>(zblk) * NT + threadIdx.x,
           static_cast<int64_t>(nzb) * NT);
  // split experts: kParts (64) block-sized parts of each first chunk's slices
  constexpr int kParts = 64;
  const int nk = *b.n_ktiles;
  for (int it = zblk; it < nk * kParts; it += nzb) {
    const int ti = it / kParts, part = it % kParts;
    const SegTile t = b.ktiles[ti];
    if (!(t.flags & 1) || (ti > 0 && b.ktiles[ti - 1].expert == t.expert)) continue;
    for (int o = 0; o < 2; ++o) {
      float* out = o == 0 ? b.gw2 : b.gw1;
      const int64_t slice = o == 0 ? b.gw2_slice : b.gw1_slice;
      if (!out) continue;
      out += static_cast<int64_t>(t.expert) * slice;
      // float4 granules (slices are multiples of 4 when d1 or d2 is)
      const int64_t per = ceil_div(ceil_div(slice, kParts), 4) * 4;
      const int64_t lo = part * per, hi = min(slice, lo + per);
      const bool v4 = slice % 4 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0;
      if (v4) {
        for (int64_t i = lo + 4 * threadIdx.x; i < hi; i += 4 * NT)
          *reinterpret_cast<float4*>(out + i) = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        for (int64_t i = lo + threadIdx.x; i < hi; i += NT) out[i] = 0.f;
      }
    }
  }
}

template <class T>
hxm_status bwd_prologue_typed(BwdPrologue& b, cudaStream_t st) {
  constexpr int V = 16 / sizeof(T);
  const EssArgs& a = b.es;
  const bool vec_ok = (a.d % V == 0) && (reinterpret_cast<uintptr_t>(a.x) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(a.copy_out) % 16 == 0);
  const void* kern = vec_ok ? reinterpret_cast<const void*>(bwd_prologue<T, V>)
                            : reinterpret_cast<const void*>(bwd_prologue<T, 1>);
  int occ = 0;
  HXM_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, 0));
  if (occ < 1) return invalid_arg("backward prologue: cannot be resident");
  const int grid = sm_count() * std::min(occ, 4);
  void* args[] = {&b};
  HXM_TRY_CUDA(cudaLaunchKernel(kern, dim3(grid), dim3(NT), args, 0, st));
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}


// ---------------------------------------------- ESTMM operator relayout --
// The operator API's ReIndex pads segments to the reference's blk (8); the
// dense tcgen05 ESTMM reads 64-position k-blocks, which must not cross a
// segment.  idx64[e] = sum_{e' < e} roundup64(len_e') (one block scan), then
// both operands are gathered into that layout (pads -> zero rows).
__global__ void relayout_index(const int64_t* __restrict__ idx, int E, int32_t* __restrict__ idx64) {
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int e0 = 0; e0 < E; e0 += blockDim.x) {
    // serial prefix over a block-sized slice (E is at most a few thousand)
    __shared__ int64_t seg[1024];
    const int e = e0 + threadIdx.x;
    seg[threadIdx.x] = e < E ? (idx[e + 1] - idx[e] + 63) / 64 * 64 : 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < static_cast<int>(blockDim.x) && e0 + i < E; ++i) {
        idx64[e0 + i] = static_cast<int32_t>(carry);
        carry += seg[i];
      }
      if (e0 + static_cast<int>(blockDim.x) >= E) idx64[E] = static_cast<int32_t>(carry);
    }
    __syncthreads();
  }
}

// One warp per new position; the expert by binary search over idx64 (its
// first kIdxSmem entries staged in shared memory once per block).  Rows move
// as VEC-element vectors (VEC = 8: 16 B per lane when both row pitches and the
// base pointers are 16 B aligned, else scalar).
template <class T, int VEC>
__global__ void __launch_bounds__(NT) gather_relayout(const T* __restrict__ x1, int64_t d1,
                                                      const T* __restrict__ x2, int64_t d2,
                                                      const int64_t* __restrict__ v,
                                                      const int64_t* __restrict__ idx,
                                                      const int32_t* __restrict__ idx64, int E,
                                                      T* __restrict__ o1, T* __restrict__ o2) {
  constexpr int kIdxSmem = 2048;
  __shared__ int32_t s64[kIdxSmem + 1];
  const bool in_smem = E <= kIdxSmem;
  if (in_smem)
    for (int e = threadIdx.x; e <= E; e += NT) s64[e] = idx64[e];
  __syncthreads();
  const int32_t* i64 = in_smem ? s64 : idx64;
  const int64_t np = i64[E];
  const int lane = threadIdx.x % 32;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (NT / 32);
  using V = typename std::conditional<VEC == 8, uint4, T>::type;
  const V zero = {};
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * (NT / 32) + threadIdx.x / 32; p < np;
       p += nw) {
    int lo = 0, hi = E;  // last e with idx64[e] <= p
    while (hi - lo > 1) {
      const int mid = (lo + hi) / 2;
      if (i64[mid] <= p) lo = mid; else hi = mid;
    }
    const int64_t off = p - i64[lo];
    const int64_t src = off < idx[lo + 1] - idx[lo] ? v[idx[lo] + off] : -1;
    const V* s1 = reinterpret_cast<const V*>(x1 + (src >= 0 ? src : 0) * d1);
    const V* s2 = reinterpret_cast<const V*>(x2 + (src >= 0 ? src : 0) * d2);
    V* t1 = reinterpret_cast<V*>(o1 + p * d1);
    V* t2 = reinterpret_cast<V*>(o2 + p * d2);
    for (int64_t c = lane; c < d1 / VEC; c += 32) t1[c] = src >= 0 ? s1[c] : zero;
    for (int64_t c = lane; c < d2 / VEC; c += 32) t2[c] = src >= 0 ? s2[c] : zero;
  }
}

}  // namespace

hxm_status launch_estmm_relayout(const void* x1, int64_t d1, const void* x2, int64_t d2,
                                  const int64_t* v, const int64_t* idx, int E, int64_t bound,
                                  int32_t* idx64, void* o1, void* o2, cudaStream_t st) {
  ProfScope ps(st, "estmm_relayout", 0.0, WORK_BYTES);
  relayout_index<<<1, 1024, 0, st>>>(idx, E, idx64);
  HXM_CHECK_LAUNCH();
  const int blocks = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(bound, NT / 32), static_cast<int64_t>(sm_count()) * 8)));
  using B = __nv_bfloat16;
  const bool vec = d1 % 8 == 0 && d2 % 8 == 0 &&
                   ((reinterpret_cast<uintptr_t>(x1) | reinterpret_cast<uintptr_t>(x2) |
                     reinterpret_cast<uintptr_t>(o1) | reinterpret_cast<uintptr_t>(o2)) % 16) == 0;
  auto kern = vec ? gather_relayout<B, 8> : gather_relayout<B, 1>;
  kern<<<blocks, NT, 0, st>>>(static_cast<const B*>(x1), d1, static_cast<const B*>(x2), d2, v,
                              idx, idx64, E, static_cast<B*>(o1), static_cast<B*>(o2));
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

hxm_status launch_gather_rows64(hxm_dtype dt, const void* src, RowMap map, int64_t d,
                                const int64_t* idx, int n_experts, int64_t bound, void* dst,
                                cudaStream_t st) {
  ProfScope ps(st, "gather_rows", 0.0, WORK_BYTES);
  return dt == HXM_BF16
             ? gather_typed<__nv_bfloat16, int64_t>(src, map, d, idx, n_experts, bound, dst, st)
             : gather_typed<float, int64_t>(src, map, d, idx, n_experts, bound, dst, st);
}

hxm_status launch_colsum_combine(const float* partial, const int32_t* tile_off, int n_experts,
                                 int parts, int64_t d, float* out, cudaStream_t st,
                                 const char* label, double work_bytes) {
  ProfScope ps(st, label ? label : "colsum_combine", work_bytes, WORK_BYTES);
  if (d <= 0 || n_experts <= 0) return HXM_OK;
  dim3 grid(static_cast<unsigned>(ceil_div(d, 128)), static_cast<unsigned>(n_experts));
  colsum_combine<<<grid, 256, 0, st>>>(partial, tile_off, parts, d, out);
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

hxm_status launch_bwd_prologue(hxm_dtype dt, BwdPrologue b, cudaStream_t st) {
  ProfScope ps(st, b.label ? b.label : "bwd_prologue", b.work, WORK_BYTES);
  return dt == HXM_BF16 ? bwd_prologue_typed<__nv_bfloat16>(b, st)
                        : bwd_prologue_typed<float>(b, st);
}

hxm_status launch_ess(hxm_dtype dt, const EssArgs& a, cudaStream_t st) {
  ProfScope ps(st, a.label ? a.label : "ess", a.work, WORK_BYTES);
  return dt == HXM_BF16 ? launch_typed<__nv_bfloat16>(a, st) : launch_typed<float>(a, st);
}

}  // namespace hxm
