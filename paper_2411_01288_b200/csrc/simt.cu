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
// K = the chunk's token positions in steps of 16.  Small grids are split
// along K (blockIdx.z) with fp32 atomic reductions, so the fp32 layer at
// c1's sizes (a few hundred CTAs of long K loops) fills the 148 SMs.
#include "kernels.cuh"
#include "routing.cuh"

namespace hxm {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <class T>
__device__ __forceinline__ float ld(const T* p, int64_t i) {
  return to_f32(p[i]);
}

// Tile loaders.  VEC (fp32 with every extent a multiple of 4 and 16-byte
// aligned bases): one float4 per thread per operand per k-step; otherwise
// scalar loads (tiny / unaligned test shapes, bf16 fallback shapes).
template <class T, bool VEC>
__device__ __forceinline__ void load_rows_kmajor(float (&S)[BK][BM], const T* A, const int* arow,
                                                 int64_t K, int64_t kend, int64_t k0) {
  // S[kk][r] = A[arow[r]][k0 + kk] for k < kend (row stride K)
  const int tid = threadIdx.x;
  if constexpr (VEC) {
    const int r = tid / 4, k4 = (tid % 4) * 4;
    const int row = arow[r];
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row >= 0 && k0 + k4 < kend)
      v = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(A) +
                                                static_cast<int64_t>(row) * K + k0 + k4));
    S[k4][r] = v.x; S[k4 + 1][r] = v.y; S[k4 + 2][r] = v.z; S[k4 + 3][r] = v.w;
  } else {
    for (int i = tid; i < BM * BK; i += NT) {
      const int r = i / BK, kk = i % BK;
      const int row = arow[r];
      const int64_t k = k0 + kk;
      S[kk][r] = (row >= 0 && k < kend) ? ld(A, static_cast<int64_t>(row) * K + k) : 0.f;
    }
  }
}

template <class T, bool VEC>
__device__ __forceinline__ void load_w(float (&S)[BK][BN], const T* W, int w_trans, int64_t K,
                                       int64_t kend, int64_t N, int64_t k0, int n0) {
  // S[kk][c] = B(k0 + kk, n0 + c): W[k][n] (w_trans = 0) or W[n][k] (W^T use)
  const int tid = threadIdx.x;
  if constexpr (VEC) {
    if (!w_trans) {
      const int kk = tid / 16, c4 = (tid % 16) * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k0 + kk < kend && n0 + c4 < N)
        v = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(W) +
                                                  (k0 + kk) * N + n0 + c4));
      S[kk][c4] = v.x; S[kk][c4 + 1] = v.y; S[kk][c4 + 2] = v.z; S[kk][c4 + 3] = v.w;
    } else {
      const int c = tid / 4, k4 = (tid % 4) * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (n0 + c < N && k0 + k4 < kend)
        v = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(W) +
                                                  (n0 + c) * K + k0 + k4));
      S[k4][c] = v.x; S[k4 + 1][c] = v.y; S[k4 + 2][c] = v.z; S[k4 + 3][c] = v.w;
    }
  } else {
    for (int i = tid; i < BM * BK; i += NT) {
      const int kk = i / BN, c = i % BN;
      const int64_t k = k0 + kk, n = n0 + c;
      float val = 0.f;
      if (k < kend && n < N) val = w_trans ? ld(W, n * K + k) : ld(W, k * N + n);
      S[kk][c] = val;
    }
  }
}

__device__ __forceinline__ void mma_tile(const float (&As)[BK][BM], const float (&Bs)[BK][BN],
                                         float (&acc)[4][4], int ty, int tx) {
#pragma unroll
  for (int kk = 0; kk < BK; ++kk) {
    const float4 av = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
    const float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
    const float a4[4] = {av.x, av.y, av.z, av.w}, b4[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a4[i], b4[j], acc[i][j]);
  }
}

// ESMM: 64-row segment tile x 64 columns per CTA (blockIdx.x = column block,
// y = tile); blockIdx.z splits K for the fp32 reduction epilogue (EPI_ATOMIC:
// the partial sums add up in the destination; the bias goes with split 0).
// Double-buffered smem: the next k-step's tiles load while this one computes.
template <class T, bool VEC>
__device__ __forceinline__ void esmm_simt_body(const EsmmArgs& a, const SegTile tile, const int n0,
                                               const int64_t kb, const int64_t ke,
                                               const bool lead) {
  const int64_t K = a.d1, N = a.d2;
  const T* A = static_cast<const T*>(a.a);
  const T* W = static_cast<const T*>(a.w) + static_cast<int64_t>(tile.expert) * K * N;
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  __shared__ int arow[BM];
  const int tid = threadIdx.x;
  if (tid < BM) {
    const int64_t p = tile.begin + tid;
    arow[tid] = p < tile.end ? a.amap(p) : -1;
  }
  __syncthreads();
  const int ty = tid / 16, tx = tid % 16;
  float acc[4][4] = {};
  int buf = 0;
  if (kb < ke) {
    load_rows_kmajor<T, VEC>(As[0], A, arow, K, ke, kb);
    load_w<T, VEC>(Bs[0], W, a.w_trans, K, ke, N, kb, n0);
  }
  __syncthreads();
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    if (k0 + BK < ke) {  // prefetch the next k-step into the other buffer
      load_rows_kmajor<T, VEC>(As[buf ^ 1], A, arow, K, ke, k0 + BK);
      load_w<T, VEC>(Bs[buf ^ 1], W, a.w_trans, K, ke, N, k0 + BK, n0);
    }
    mma_tile(As[buf], Bs[buf], acc, ty, tx);
    __syncthreads();
    buf ^= 1;
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
      const float bias =
          (a.bias && lead) ? a.bias[static_cast<int64_t>(tile.expert) * N + n] : 0.f;
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

// ESMM: 64-row segment tile x 64 columns per CTA (blockIdx.x = column block,
// y = tile); blockIdx.z splits K for the fp32 reduction epilogue (EPI_ATOMIC:
// the partial sums add up in the destination; the bias goes with split 0).
template <class T, bool VEC>
__global__ void __launch_bounds__(NT) esmm_simt_kernel(EsmmArgs a) {
  const int ti = blockIdx.y;
  if (ti >= *a.n_tiles) return;
  const int64_t K = a.d1;
  const int64_t kper = ceil_div(ceil_div(K, BK), gridDim.z) * BK;
  const int64_t kb = blockIdx.z * kper, ke = min(K, kb + kper);
  esmm_simt_body<T, VEC>(a, a.tiles[ti], blockIdx.x * BN, kb, ke, blockIdx.z == 0);
}

// ESTMM: 64 x 64 output tile per CTA over positions [pb, pe) of a chunk;
// `reduce`: atomicAdd into a pre-zeroed output instead of a store.
template <class T, bool VEC>
__device__ __forceinline__ void estmm_simt_body(const EstmmArgs& a, const SegTile tile,
                                                const int m0, const int n0, const int64_t pb,
                                                const int64_t pe, const bool reduce) {
  const int64_t D1 = a.d1, D2 = a.d2;
  const T* X1 = static_cast<const T*>(a.x1);
  const T* X2 = static_cast<const T*>(a.x2);
  __shared__ __align__(16) float As[BK][BM];
  __shared__ __align__(16) float Bs[BK][BN];
  __shared__ int r1[BK], r2[BK];
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  float acc[4][4] = {};
  for (int64_t p0 = pb; p0 < pe; p0 += BK) {
    if (tid < BK) {
      const int64_t p = p0 + tid;
      r1[tid] = p < pe ? a.m1(p) : -1;
      r2[tid] = p < pe ? a.m2(p) : -1;
    }
    __syncthreads();
    if constexpr (VEC) {
      const int kk = tid / 16, c4 = (tid % 16) * 4;
      float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
      const int row = r1[kk], row2 = r2[kk];
      if (row >= 0 && m0 + c4 < D1)
        va = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(X1) +
                                                   static_cast<int64_t>(row) * D1 + m0 + c4));
      if (row2 >= 0 && n0 + c4 < D2)
        vb = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(X2) +
                                                   static_cast<int64_t>(row2) * D2 + n0 + c4));
      *reinterpret_cast<float4*>(&As[kk][c4]) = va;
      *reinterpret_cast<float4*>(&Bs[kk][c4]) = vb;
    } else {
      for (int i = tid; i < BK * BM; i += NT) {
        const int kk = i / BM, c = i % BM;
        const int row = r1[kk];
        const int64_t m = m0 + c;
        As[kk][c] = (row >= 0 && m < D1) ? ld(X1, static_cast<int64_t>(row) * D1 + m) : 0.f;
        const int row2 = r2[kk];
        const int64_t n = n0 + c;
        Bs[kk][c] = (row2 >= 0 && n < D2) ? ld(X2, static_cast<int64_t>(row2) * D2 + n) : 0.f;
      }
    }
    __syncthreads();
    mma_tile(As, Bs, acc, ty, tx);
    __syncthreads();
  }
  float* out = a.out + static_cast<int64_t>(tile.expert) * D1 * D2;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= D1) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n >= D2) continue;
      if (reduce) atomicAdd(out + m * D2 + n, acc[i][j]);
      else out[m * D2 + n] = acc[i][j];
    }
  }
}

// ESTMM: 64 x 64 output tile per CTA, K = the chunk's token positions in
// steps of 16; blockIdx.z splits the positions (the output is then pre-zeroed
// and every split reduces with atomicAdd).
template <class T, bool VEC>
__global__ void __launch_bounds__(NT) estmm_simt_kernel(EstmmArgs a) {
  const int ti = blockIdx.y;
  if (ti >= *a.n_tiles) return;
  const SegTile tile = a.tiles[ti];
  const int mt = static_cast<int>(ceil_div(a.d1, BM));
  const int m0 = (blockIdx.x % mt) * BM, n0 = (blockIdx.x / mt) * BN;
  const int64_t len = tile.end - tile.begin;
  const int64_t per = ceil_div(ceil_div(len, BK), gridDim.z) * BK;
  const int64_t pb = tile.begin + blockIdx.z * per,
                pe = pb + per < tile.end ? pb + per : static_cast<int64_t>(tile.end);
  estmm_simt_body<T, VEC>(a, tile, m0, n0, pb, pe, (tile.flags & 1) || gridDim.z > 1);
}

// ESFK (es_ops.cpp:210-247) in ONE launch on the fp32 path: the 1-D grid is
// the reference's combined work list -- [grad-x ESMM tiles | grad-b ESS
// columns | grad-W ESTMM tiles] -- over the caller's ReIndex directly (tiles
// found by a per-block scan of the segment lengths, rows gathered through v).
// Every output element has exactly one writer (no split-K, no atomics), so
// the launch needs no pre-zeroing and is deterministic.
struct EsfkSimt {
  EsmmArgs gx;   // a = g (K = d2), w = w_t, out = grad_x (EPI_WRITE), maps via v
  EstmmArgs gw;  // x1 = x, x2 = g, out = grad_w
  const void* g;
  int64_t d2;
  float* grad_b;
  const int64_t* idx;
  const int64_t* v;
  int E;
  int r0, r1;  // block ranges: [0, r0) ESMM, [r0, r1) ESS, [r1, grid) ESTMM
  int gx_cb;   // ESMM column blocks (ceil(d1 / 64))
};

template <class T, bool VEC>
__global__ void __launch_bounds__(NT) esfk_simt_kernel(EsfkSimt f) {
  extern __shared__ int32_t toff[];  // E + 1: exclusive scan of 64-row tiles per expert
  const int b = blockIdx.x, E = f.E;
  if (b < f.r0) {
    if (threadIdx.x == 0) {
      int32_t run = 0;
      for (int e = 0; e < E; ++e) {
        toff[e] = run;
        run += static_cast<int32_t>(ceil_div(f.idx[e + 1] - f.idx[e], BM));
      }
      toff[E] = run;
    }
    __syncthreads();
    const int ti = b / f.gx_cb, cb = b % f.gx_cb;
    if (ti >= toff[E]) return;
    int lo = 0, hi = E;  // last e with toff[e] <= ti
    while (hi - lo > 1) {
      const int mid = (lo + hi) / 2;
      if (toff[mid] <= ti) lo = mid; else hi = mid;
    }
    const int64_t begin = f.idx[lo] + static_cast<int64_t>(ti - toff[lo]) * BM;
    const int64_t end = min(f.idx[lo + 1], begin + BM);
    const SegTile t{lo, static_cast<int>(begin), static_cast<int>(end), 0};
    esmm_simt_body<T, VEC>(f.gx, t, cb * BN, 0, f.gx.d1, true);
  } else if (b < f.r1) {
    // grad_b[e][c]: thread per column, the segment's rows in order
    const int cblk = static_cast<int>(ceil_div(f.d2, NT));
    const int e = (b - f.r0) / cblk;
    const int64_t c = static_cast<int64_t>((b - f.r0) % cblk) * NT + threadIdx.x;
    if (c >= f.d2) return;
    const T* G = static_cast<const T*>(f.g);
    float s = 0.f;
    for (int64_t p = f.idx[e]; p < f.idx[e + 1]; ++p) {
      const int64_t t = f.v[p];
      if (t >= 0) s += to_f32(G[t * f.d2 + c]);
    }
    f.grad_b[static_cast<int64_t>(e) * f.d2 + c] = s;
  } else {
    const int mt = static_cast<int>(ceil_div(f.gw.d1, BM)), nt = static_cast<int>(ceil_div(f.gw.d2, BN));
    const int j = b - f.r1;
    const int e = j / (mt * nt), rem = j % (mt * nt);
    const SegTile t{e, static_cast<int>(f.idx[e]), static_cast<int>(f.idx[e + 1]), 0};
    estmm_simt_body<T, VEC>(f.gw, t, (rem % mt) * BM, (rem / mt) * BN, t.begin, t.end, false);
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

// ---------------------------------------------------------------------------
// Dense-operand fp32 kernels: the layer's fp32 path (c1) reads only
// expert-sorted copies (x_s, the stash, g_y_s, g_y1_s), so no row map sits
// between a tile and its operands.  A 3-stage cp.async ring (16-byte copies,
// zero-filled past the ends) replaces the register-staged, transposing loads
// of the mapped kernels above, whose per-k-step map-load -> data-load ->
// store -> barrier chain left these small GEMMs latency-bound (~24 us each at
// c1, IPC 1.5).  Same 64 x 64 tiles, K split and epilogues, same
// summation order per output (k ascending within a split).
constexpr int DS = 3;          // ring stages
constexpr int APAD = BK + 4;   // k-contiguous rows: 80 B (16-B aligned, conflict-free reads)
constexpr int BPAD = BN + 4;   // n-contiguous rows: 272 B

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
               "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ESMM, dense A (rows tile.begin.. of a.a), B = W[e] (BT = 0: K x N rows,
// n-contiguous) or W[e]^T use (BT = 1: W stored N x K, k-contiguous).
// Thread (ty, tx) owns rows ty*4 + i and columns tx*4 + j (BT: tx + 16 j).
template <bool BT>
__global__ void __launch_bounds__(NT) esmm_dense_kernel(EsmmArgs a) {
  const int ti = blockIdx.y;
  if (ti >= *a.n_tiles) return;
  const SegTile tile = a.tiles[ti];
  const int n0 = blockIdx.x * BN;
  const int64_t K = a.d1, N = a.d2;
  const int64_t kper = ceil_div(ceil_div(K, BK), gridDim.z) * BK;
  const int64_t kb = blockIdx.z * kper, ke = min(K, kb + kper);
  const bool lead = blockIdx.z == 0;
  __shared__ __align__(16) float As[DS][BM][APAD];
  __shared__ __align__(16) float Bs[DS][BT ? BN : BK][BT ? APAD : BPAD];
  const float* A = static_cast<const float*>(a.a);
  const float* W = static_cast<const float*>(a.w) + static_cast<int64_t>(tile.expert) * K * N;
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int ar = tid / 4, ak = (tid % 4) * 4;
  const int64_t arow = tile.begin + ar;
  const bool arow_ok = arow < a.a_rows;
  auto load = [&](int stg, int64_t k0) {
    const bool aok = arow_ok && k0 + ak < ke;
    cp_async16(&As[stg][ar][ak], aok ? A + arow * K + k0 + ak : A, aok);
    if constexpr (!BT) {
      const int kk = tid / 16, c4 = (tid % 16) * 4;
      const bool ok = k0 + kk < ke && n0 + c4 < N;
      cp_async16(&Bs[stg][kk][c4], ok ? W + (k0 + kk) * N + n0 + c4 : W, ok);
    } else {
      const int nn = tid / 4, k4 = (tid % 4) * 4;
      const bool ok = n0 + nn < N && k0 + k4 < ke;
      cp_async16(&Bs[stg][nn][k4], ok ? W + (n0 + nn) * K + k0 + k4 : W, ok);
    }
  };
  const int nk = kb < ke ? static_cast<int>(ceil_div(ke - kb, BK)) : 0;
  float acc[4][4] = {};
#pragma unroll
  for (int s = 0; s < DS - 1; ++s) {
    if (s < nk) load(s, kb + s * BK);
    cp_async_commit();
  }
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<DS - 2>();
    __syncthreads();  // stage it complete for everyone; stage it - 1 free
    if (it + DS - 1 < nk) load((it + DS - 1) % DS, kb + (it + DS - 1) * BK);
    cp_async_commit();
    const int stg = it % DS;
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      float4 av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = *reinterpret_cast<const float4*>(&As[stg][ty * 4 + i][kq * 4]);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        bv[j] = BT ? *reinterpret_cast<const float4*>(&Bs[stg][tx + 16 * j][kq * 4])
                   : *reinterpret_cast<const float4*>(&Bs[stg][kq * 4 + j][tx * 4]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a4[4] = {av[i].x, av[i].y, av[i].z, av[i].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if constexpr (BT) {
            acc[i][0] = fmaf(a4[q], (&bv[0].x)[q], acc[i][0]);
            acc[i][1] = fmaf(a4[q], (&bv[1].x)[q], acc[i][1]);
            acc[i][2] = fmaf(a4[q], (&bv[2].x)[q], acc[i][2]);
            acc[i][3] = fmaf(a4[q], (&bv[3].x)[q], acc[i][3]);
          } else {
            acc[i][0] = fmaf(a4[q], bv[q].x, acc[i][0]);
            acc[i][1] = fmaf(a4[q], bv[q].y, acc[i][1]);
            acc[i][2] = fmaf(a4[q], bv[q].z, acc[i][2]);
            acc[i][3] = fmaf(a4[q], bv[q].w, acc[i][3]);
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  // epilogue (as esmm_simt_body); EPI_BWD_ACT with a.colsum also sums this
  // CTA's g_y1 columns over its 64 rows (fused gb1: one deterministic
  // partial row per tile, combined per expert by colsum_combine)
  float colacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ty * 4 + i;
    const int64_t p = tile.begin + r;
    if (p >= tile.end) continue;
    const int orow = a.omap(p);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + (BT ? tx + 16 * j : tx * 4 + j);
      if (n >= N) continue;
      const float bias =
          (a.bias && lead) ? a.bias[static_cast<int64_t>(tile.expert) * N + n] : 0.f;
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
          const bool pad = orow < 0;
          float f, df;
          act_both(a.act, v, f, df);
          static_cast<float*>(a.out1)[p * N + n] = pad ? 0.f : df;
          static_cast<float*>(a.out2)[p * N + n] = pad ? 0.f : f;
          break;
        }
        default: {  // EPI_BWD_ACT: g_y1 = g_y2 * F'(y1)
          const bool pad = orow < 0;
          const float g = acc[i][j] * static_cast<const float*>(a.y1s)[p * N + n];
          static_cast<float*>(a.out1)[p * N + n] = pad ? 0.f : g;
          colacc[j] += pad ? 0.f : g;
          break;
        }
      }
    }
  }
  if (a.epi == EPI_BWD_ACT && a.colsum) {
    __shared__ float red[NT / 16][BN];
    __syncthreads();  // (the operand ring is no longer read)
#pragma unroll
    for (int j = 0; j < 4; ++j) red[ty][BT ? tx + 16 * j : tx * 4 + j] = colacc[j];
    __syncthreads();
    if (tid < BN && n0 + tid < N) {
      float sum = 0.f;
#pragma unroll
      for (int t = 0; t < NT / 16; ++t) sum += red[t][tid];  // fixed order: deterministic
      a.colsum[static_cast<int64_t>(ti) * N + n0 + tid] = sum;
    }
  }
}

// ESTMM, dense X1 / X2 rows (k = positions): 64 x 64 output tile over the
// positions [pb, pe) of a chunk, both operands row-contiguous in m / n.
__global__ void __launch_bounds__(NT) estmm_dense_kernel(EstmmArgs a) {
  const int ti = blockIdx.y;
  if (ti >= *a.n_tiles) return;
  const SegTile tile = a.tiles[ti];
  const int mt = static_cast<int>(ceil_div(a.d1, BM));
  const int m0 = (blockIdx.x % mt) * BM, n0 = (blockIdx.x / mt) * BN;
  const int64_t len = tile.end - tile.begin;
  const int64_t per = ceil_div(ceil_div(len, BK), gridDim.z) * BK;
  const int64_t pb = tile.begin + blockIdx.z * per,
                pe = pb + per < tile.end ? pb + per : static_cast<int64_t>(tile.end);
  const bool reduce = (tile.flags & 1) || gridDim.z > 1;
  const int64_t D1 = a.d1, D2 = a.d2;
  const float* X1 = static_cast<const float*>(a.x1);
  const float* X2 = static_cast<const float*>(a.x2);
  __shared__ __align__(16) float As[DS][BK][BPAD];
  __shared__ __align__(16) float Bs[DS][BK][BPAD];
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int kk = tid / 16, c4 = (tid % 16) * 4;
  auto load = [&](int stg, int64_t p0) {
    const bool rok = p0 + kk < pe;
    const bool okA = rok && m0 + c4 < D1, okB = rok && n0 + c4 < D2;
    cp_async16(&As[stg][kk][c4], okA ? X1 + (p0 + kk) * D1 + m0 + c4 : X1, okA);
    cp_async16(&Bs[stg][kk][c4], okB ? X2 + (p0 + kk) * D2 + n0 + c4 : X2, okB);
  };
  const int nk = pb < pe ? static_cast<int>(ceil_div(pe - pb, BK)) : 0;
  float acc[4][4] = {};
#pragma unroll
  for (int s = 0; s < DS - 1; ++s) {
    if (s < nk) load(s, pb + s * BK);
    cp_async_commit();
  }
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<DS - 2>();
    __syncthreads();
    if (it + DS - 1 < nk) load((it + DS - 1) % DS, pb + (it + DS - 1) * BK);
    cp_async_commit();
    const int stg = it % DS;
#pragma unroll
    for (int k2 = 0; k2 < BK; ++k2) {
      const float4 av = *reinterpret_cast<const float4*>(&As[stg][k2][ty * 4]);
      const float4 bv = *reinterpret_cast<const float4*>(&Bs[stg][k2][tx * 4]);
      const float a4[4] = {av.x, av.y, av.z, av.w}, b4[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a4[i], b4[j], acc[i][j]);
    }
  }
  cp_async_wait<0>();
  float* out = a.out + static_cast<int64_t>(tile.expert) * D1 * D2;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= D1) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n >= D2) continue;
      if (reduce) atomicAdd(out + m * D2 + n, acc[i][j]);
      else out[m * D2 + n] = acc[i][j];
    }
  }
}

}  // namespace

bool vec_ok(const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; }
// HXM_SIMT_DENSE=0: the mapped kernels for dense operands too (A/B)
bool dense_on() {
  static const bool on = [] {
    const char* e = std::getenv("HXM_SIMT_DENSE");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool simt_dense_esmm_ok(hxm_dtype dt, const EsmmArgs& a) {
  return dt == HXM_F32 && a.d1 % 4 == 0 && a.d2 % 4 == 0 && vec_ok(a.a) && vec_ok(a.w) &&
         a.amap.kind == MAP_DENSE && dense_on();
}

hxm_status simt_esmm(hxm_dtype dt, const EsmmArgs& a, cudaStream_t st) {
  if (a.max_tiles <= 0) return HXM_OK;
  // split K for the reduction epilogue when the grid would not fill the GPU
  int kz = 1;
  if (a.epi == EPI_ATOMIC) {
    const int64_t ctas = ceil_div(a.d2, BN) * a.max_tiles;
    while (kz < 8 && ctas * kz < 2LL * sm_count() && ceil_div(a.d1, BK) >= 8 * kz) kz *= 2;
  }
  dim3 grid(static_cast<unsigned>(ceil_div(a.d2, BN)), static_cast<unsigned>(a.max_tiles), kz);
  const bool vec = dt == HXM_F32 && a.d1 % 4 == 0 && a.d2 % 4 == 0 && vec_ok(a.a) && vec_ok(a.w);
  if (a.colsum && !(vec && a.amap.kind == MAP_DENSE && dense_on()))
    return invalid_arg("esmm: fused column sums need the dense fp32 kernel");
  if (vec && a.amap.kind == MAP_DENSE && dense_on()) {
    if (a.w_trans) esmm_dense_kernel<true><<<grid, NT, 0, st>>>(a);
    else esmm_dense_kernel<false><<<grid, NT, 0, st>>>(a);
  } else if (dt == HXM_BF16) esmm_simt_kernel<__nv_bfloat16, false><<<grid, NT, 0, st>>>(a);
  else if (vec) esmm_simt_kernel<float, true><<<grid, NT, 0, st>>>(a);
  else esmm_simt_kernel<float, false><<<grid, NT, 0, st>>>(a);
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

hxm_status simt_estmm(hxm_dtype dt, const EstmmArgs& a, cudaStream_t st) {
  if (a.max_tiles <= 0) return HXM_OK;
  const int64_t ctas = ceil_div(a.d1, BM) * ceil_div(a.d2, BN) * a.max_tiles;
  int kz = 1;
  while (kz < 8 && ctas * kz < 2LL * sm_count()) kz *= 2;
  if (kz > 1)  // every split reduces into a zeroed output
    HXM_TRY_CUDA(cudaMemsetAsync(a.out, 0, sizeof(float) * a.n_experts * a.d1 * a.d2, st));
  dim3 grid(static_cast<unsigned>(ceil_div(a.d1, BM) * ceil_div(a.d2, BN)),
            static_cast<unsigned>(a.max_tiles), kz);
  const bool vec = dt == HXM_F32 && a.d1 % 4 == 0 && a.d2 % 4 == 0 && vec_ok(a.x1) && vec_ok(a.x2);
  if (vec && a.m1.kind == MAP_DENSE && a.m2.kind == MAP_DENSE && dense_on())
    estmm_dense_kernel<<<grid, NT, 0, st>>>(a);
  else if (dt == HXM_BF16) estmm_simt_kernel<__nv_bfloat16, false><<<grid, NT, 0, st>>>(a);
  else if (vec) estmm_simt_kernel<float, true><<<grid, NT, 0, st>>>(a);
  else estmm_simt_kernel<float, false><<<grid, NT, 0, st>>>(a);
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

hxm_status simt_esfk(hxm_dtype dt, const void* x, const void* g, int64_t n, int64_t d1,
                     int64_t d2, const void* w, int w_trans, const int64_t* v, const int64_t* idx,
                     int64_t E, int64_t np_bound, float* grad_x, float* grad_b, float* grad_w,
                     cudaStream_t st) {
  EsfkSimt f{};
  f.gx.a = g;
  f.gx.amap = map_v64(v);
  f.gx.a_rows = n;
  f.gx.n_experts = E;
  f.gx.w = w;
  f.gx.w_trans = w_trans;
  f.gx.d1 = d2;  // K
  f.gx.d2 = d1;  // N
  f.gx.epi = EPI_WRITE;
  f.gx.out_f32 = grad_x;
  f.gx.omap = map_v64(v);
  f.gw.x1 = x;
  f.gw.m1 = map_v64(v);
  f.gw.x2 = g;
  f.gw.m2 = map_v64(v);
  f.gw.d1 = d1;
  f.gw.d2 = d2;
  f.gw.out = grad_w;
  f.g = g;
  f.d2 = d2;
  f.grad_b = grad_b;
  f.idx = idx;
  f.v = v;
  f.E = static_cast<int>(E);
  f.gx_cb = static_cast<int>(ceil_div(d1, BN));
  const int64_t tiles = max_tiles(np_bound, E, BM);
  const int64_t r0 = tiles * f.gx_cb;
  const int64_t r1 = r0 + E * ceil_div(d2, NT);
  const int64_t nb = r1 + E * ceil_div(d1, BM) * ceil_div(d2, BN);
  if (nb > 0x7fffffffLL) return invalid_arg("esfk: grid too large");
  f.r0 = static_cast<int>(r0);
  f.r1 = static_cast<int>(r1);
  const size_t smem = (static_cast<size_t>(E) + 1) * sizeof(int32_t);
  const bool vec = dt == HXM_F32 && d1 % 4 == 0 && d2 % 4 == 0 && vec_ok(x) && vec_ok(g) && vec_ok(w);
  const void* kern = dt == HXM_BF16 ? reinterpret_cast<const void*>(esfk_simt_kernel<__nv_bfloat16, false>)
                     : vec ? reinterpret_cast<const void*>(esfk_simt_kernel<float, true>)
                           : reinterpret_cast<const void*>(esfk_simt_kernel<float, false>);
  if (smem > 48 * 1024)
    HXM_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
  void* args[] = {&f};
  if (nb > 0) {
    HXM_TRY_CUDA(cudaLaunchKernel(kern, dim3(static_cast<unsigned>(nb)), dim3(NT), args, smem, st));
    HXM_CHECK_LAUNCH();
  }
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
