// simt.cu -- fp32-FMA expert-specific GEMMs.
//
// The fp32 path of the operators (hxm_dtype HXM_F32: BASELINE.json c1 is an
// fp32 layer checked at rtol 1e-4, which TF32 tensor cores cannot meet) and
// bf16 shapes whose row pitch is not a multiple of 16 bytes (TMA cannot
// describe them; only tiny test shapes).  Every bf16 shape of the
// BASELINE.json configs runs on the tcgen05 kernels in umma.cu.
//
// ESMM: 64-row segment tile x 64 columns per CTA, K in steps of 16, 4x4
// outputs per thread; A rows are gathered through the row map (padding slots
// read as zeros), B is W[e] or W[e]^T.  ESTMM: 64x64 output tile per CTA,
// K = the chunk's token positions in steps of 16.
#include "kernels.cuh"

namespace hxm {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <class T>
__device__ __forceinline__ float ld(const T* p, int64_t i) {
  return to_f32(p[i]);
}

template <class T>
__global__ void __launch_bounds__(NT) esmm_simt_kernel(EsmmArgs a) {
  const int ti = blockIdx.y;
  if (ti >= *a.n_tiles) return;
  const SegTile tile = a.tiles[ti];
  const int n0 = blockIdx.x * BN;
  const int64_t K = a.d1, N = a.d2;
  const T* A = static_cast<const T*>(a.a);
  const T* W = static_cast<const T*>(a.w) + static_cast<int64_t>(tile.expert) * K * N;

  __shared__ float As[BK][BM];
  __shared__ float Bs[BK][BN];
  __shared__ int arow[BM];
  const int tid = threadIdx.x;
  if (tid < BM) {
    const int64_t p = tile.begin + tid;
    arow[tid] = p < tile.end ? a.amap(p) : -1;
  }
  __syncthreads();
  const int ty = tid / 16, tx = tid % 16;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
    for (int i = tid; i < BM * BK; i += NT) {
      const int r = i / BK, kk = i % BK;
      const int row = arow[r];
      const int64_t k = k0 + kk;
      As[kk][r] = (row >= 0 && k < K) ? ld(A, static_cast<int64_t>(row) * K + k) : 0.f;
    }
    for (int i = tid; i < BM * BK; i += NT) {
      const int kk = i / BN, c = i % BN;
      const int64_t k = k0 + kk, n = n0 + c;
      float val = 0.f;
      if (k < K && n < N) val = a.w_trans ? ld(W, n * K + k) : ld(W, k * N + n);
      Bs[kk][c] = val;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ty * 4 + i;
    const int64_t p = tile.begin + r;
    if (p >= tile.end) continue;
    const int orow = a.omap(p);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n >= N) continue;
      const float bias = a.bias ? a.bias[static_cast<int64_t>(tile.expert) * N + n] : 0.f;
      const float v = acc[i][j] + bias;
      switch (a.epi) {
        case EPI_WRITE:
          if (orow >= 0) a.out_f32[static_cast<int64_t>(orow) * N + n] = v;
          break;
        case EPI_ACCUM:
          if (orow >= 0) a.out_f32[static_cast<int64_t>(orow) * N + n] += v;
          break;
        case EPI_ATOMIC:
          if (orow >= 0) atomicAdd(a.out_f32 + static_cast<int64_t>(orow) * N + n, v);
          break;
        case EPI_FWD_ACT: {
          T* o1 = static_cast<T*>(a.out1);
          T* o2 = static_cast<T*>(a.out2);
          const bool pad = orow < 0;
          // stash (F'(y1), F(y1)) -- all the backward needs of y1
          o1[p * N + n] = from_f32<T>(pad ? 0.f : act_derivative(a.act, v));
          o2[p * N + n] = from_f32<T>(pad ? 0.f : act_value(a.act, v));
          break;
        }
        default: {  // EPI_BWD_ACT (no bias): g_y1 = g_y2 * F'(y1)
          T* o1 = static_cast<T*>(a.out1);
          const T* dact = static_cast<const T*>(a.y1s);
          const bool pad = orow < 0;
          const float g = acc[i][j] * to_f32(dact[p * N + n]);
          o1[p * N + n] = from_f32<T>(pad ? 0.f : g);
          break;
        }
      }
    }
  }
}

template <class T>
__global__ void __launch_bounds__(NT) estmm_simt_kernel(EstmmArgs a) {
  const int ti = blockIdx.y;
  if (ti >= *a.n_tiles) return;
  const SegTile tile = a.tiles[ti];
  const int64_t D1 = a.d1, D2 = a.d2;
  const int mt = static_cast<int>(ceil_div(D1, BM));
  const int m0 = (blockIdx.x % mt) * BM, n0 = (blockIdx.x / mt) * BN;
  const T* X1 = static_cast<const T*>(a.x1);
  const T* X2 = static_cast<const T*>(a.x2);
  __shared__ float As[BK][BM];
  __shared__ float Bs[BK][BN];
  __shared__ int r1[BK], r2[BK];
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  float acc[4][4] = {};
  for (int64_t p0 = tile.begin; p0 < tile.end; p0 += BK) {
    if (tid < BK) {
      const int64_t p = p0 + tid;
      r1[tid] = p < tile.end ? a.m1(p) : -1;
      r2[tid] = p < tile.end ? a.m2(p) : -1;
    }
    __syncthreads();
    for (int i = tid; i < BK * BM; i += NT) {
      const int kk = i / BM, c = i % BM;
      const int row = r1[kk];
      const int64_t m = m0 + c;
      As[kk][c] = (row >= 0 && m < D1) ? ld(X1, static_cast<int64_t>(row) * D1 + m) : 0.f;
      const int row2 = r2[kk];
      const int64_t n = n0 + c;
      Bs[kk][c] = (row2 >= 0 && n < D2) ? ld(X2, static_cast<int64_t>(row2) * D2 + n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* out = a.out + static_cast<int64_t>(tile.expert) * D1 * D2;
  const bool split = tile.flags & 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= D1) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n >= D2) continue;
      if (split) atomicAdd(out + m * D2 + n, acc[i][j]);
      else out[m * D2 + n] = acc[i][j];
    }
  }
}

__global__ void zero_split_kernel(const SegTile* tiles, const int32_t* n_tiles,
                                  int64_t slice, float* out) {
  const int ti = blockIdx.y;
  if (ti >= *n_tiles) return;
  const SegTile t = tiles[ti];
  // only the first chunk of a split expert zeroes its slice
  if (!(t.flags & 1)) return;
  if (ti > 0 && tiles[ti - 1].expert == t.expert) return;
  float4* o = reinterpret_cast<float4*>(out + static_cast<int64_t>(t.expert) * slice);
  const int64_t n4 = (slice % 4 == 0) ? slice / 4 : 0;
  for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    o[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < slice;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[static_cast<int64_t>(t.expert) * slice + i] = 0.f;
}

}  // namespace

hxm_status simt_esmm(hxm_dtype dt, const EsmmArgs& a, cudaStream_t st) {
  if (a.max_tiles <= 0) return HXM_OK;
  dim3 grid(static_cast<unsigned>(ceil_div(a.d2, BN)), static_cast<unsigned>(a.max_tiles));
  if (dt == HXM_BF16) esmm_simt_kernel<__nv_bfloat16><<<grid, NT, 0, st>>>(a);
  else esmm_simt_kernel<float><<<grid, NT, 0, st>>>(a);
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

hxm_status simt_estmm(hxm_dtype dt, const EstmmArgs& a, cudaStream_t st) {
  if (a.max_tiles <= 0) return HXM_OK;
  dim3 grid(static_cast<unsigned>(ceil_div(a.d1, BM) * ceil_div(a.d2, BN)),
            static_cast<unsigned>(a.max_tiles));
  if (dt == HXM_BF16) estmm_simt_kernel<__nv_bfloat16><<<grid, NT, 0, st>>>(a);
  else estmm_simt_kernel<float><<<grid, NT, 0, st>>>(a);
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

hxm_status zero_split_experts(const SegTile* tiles, const int32_t* n_tiles, int max_tiles,
                              int64_t slice, float* out, cudaStream_t st) {
  if (max_tiles <= 0) return HXM_OK;
  // blocks of non-split tiles exit at once; 16 blocks zero a split expert
  dim3 grid(static_cast<unsigned>(std::min<int64_t>(16, ceil_div(slice, 1024))),
            static_cast<unsigned>(max_tiles));
  zero_split_kernel<<<grid, 256, 0, st>>>(tiles, n_tiles, slice, out);
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

}  // namespace hxm
