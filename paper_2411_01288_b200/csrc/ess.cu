// ess.cu -- expert-specific segmented sum (ESS), the bias-gradient operator.
//
// Replaces moekit::ess (reference core/src/es_ops.cpp:86-102, 180-191):
// out[e] = sum of the rows routed to expert e.  HBM-bound: every routed row is
// read once (16-byte vector loads, consecutive threads on consecutive
// columns so a gathered row is one coalesced burst) and E x D fp32 is written.
// Two deterministic phases, no float atomics:
//   ess_partial : one CTA per <=128-position segment tile -> partial[tile][D]
//   ess_combine : out[e][d] = sum of e's tile partials in tile order.
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

template <class T, int VEC>
__global__ void __launch_bounds__(NT) ess_partial(EssArgs a) {
  // grid: x = segment tile (<= 128 positions), y = column slab of 32 vector
  // groups (one per lane); the 8 warps split the tile's rows, each keeping
  // U = 4 row loads in flight, and are combined in fixed order through smem.
  const int ti = blockIdx.x;
  if (ti >= *a.n_tiles) return;
  const SegTile tile = a.tiles[ti];
  const T* X = static_cast<const T*>(a.x);
  const int64_t D = a.d;
  const int col_groups = static_cast<int>((D + VEC - 1) / VEC);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int W = NT / 32;
  const int cg = blockIdx.y * 32 + lane;
  __shared__ int rows[kEssRows];
  __shared__ float red[W][32 * VEC];
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
    const int64_t col = static_cast<int64_t>(blockIdx.y) * 32 * VEC + c;
    if (col >= D) continue;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) s += red[w][c];
    a.partial[static_cast<int64_t>(ti) * D + col] = s;
  }
}

__global__ void ess_combine(EssArgs a) {
  const int e = blockIdx.y;
  const int64_t d = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (d >= a.d) return;
  const int t0 = a.tile_off[e], t1 = a.tile_off[e + 1];
  float s = 0.f;
  for (int t = t0; t < t1; ++t) s += a.partial[static_cast<int64_t>(t) * a.d + d];
  a.out[static_cast<int64_t>(e) * a.d + d] = s;
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
  dim3 grid(static_cast<unsigned>(ceil_div(a.d, 256)), static_cast<unsigned>(a.n_experts));
  if (a.d > 0 && a.n_experts > 0 && a.out) {
    ess_combine<<<grid, 256, 0, st>>>(a);
    HXM_CHECK_LAUNCH();
  }
  return HXM_OK;
}

template <class T, int VEC>
__global__ void __launch_bounds__(NT) gather_rows(const T* __restrict__ src, RowMap map,
                                                  int64_t d, const int32_t* __restrict__ idx,
                                                  int E, T* __restrict__ dst) {
  const int64_t np = idx[E];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t groups = d / VEC;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * (NT / 32) + warp; p < np;
       p += static_cast<int64_t>(gridDim.x) * (NT / 32)) {
    const int row = map(p);
    T* o = dst + p * d;
    if (row < 0) {
      float z[VEC];
#pragma unroll
      for (int i = 0; i < VEC; ++i) z[i] = 0.f;
      for (int64_t g = lane; g < groups; g += 32) store_vec<T, VEC>(o + g * VEC, z);
      continue;
    }
    const T* s = src + static_cast<int64_t>(row) * d;
    for (int64_t g = lane; g < groups; g += 32) {
      float v[VEC];
      load_vec<T, VEC>(s + g * VEC, v);
      store_vec<T, VEC>(o + g * VEC, v);
    }
  }
}

template <class T>
hxm_status gather_typed(const void* src, RowMap map, int64_t d, const int32_t* idx, int E,
                        int64_t bound, void* dst, cudaStream_t st) {
  constexpr int V = 16 / sizeof(T);
  const int blocks = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(bound, NT / 32), static_cast<int64_t>(sm_count()) * 8)));
  const bool vec_ok = d % V == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(dst) % 16 == 0;
  if (vec_ok)
    gather_rows<T, V><<<blocks, NT, 0, st>>>(static_cast<const T*>(src), map, d, idx, E,
                                             static_cast<T*>(dst));
  else
    gather_rows<T, 1><<<blocks, NT, 0, st>>>(static_cast<const T*>(src), map, d, idx, E,
                                             static_cast<T*>(dst));
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

}  // namespace

hxm_status launch_gather_rows(hxm_dtype dt, const void* src, RowMap map, int64_t d,
                              const int32_t* idx, int n_experts, int64_t bound, void* dst,
                              cudaStream_t st, double work_bytes) {
  ProfScope ps(st, "gather_rows", work_bytes, WORK_BYTES);
  return dt == HXM_BF16 ? gather_typed<__nv_bfloat16>(src, map, d, idx, n_experts, bound, dst, st)
                        : gather_typed<float>(src, map, d, idx, n_experts, bound, dst, st);
}

hxm_status launch_ess(hxm_dtype dt, const EssArgs& a, cudaStream_t st) {
  ProfScope ps(st, a.label ? a.label : "ess", a.work, WORK_BYTES);
  return dt == HXM_BF16 ? launch_typed<__nv_bfloat16>(a, st) : launch_typed<float>(a, st);
}

}  // namespace hxm
