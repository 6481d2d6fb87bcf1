// esfk.cu -- the fused backward of one MLP, moekit::esfk (reference
// core/src/es_ops.cpp:210-247, es_ops.hpp:55-65):
//   grad_x = esmm(g, w_t) (write)   grad_b = ess(g)   grad_w = estmm(x, g)
// The reference runs the three operators' tiles as ONE combined work list.
// Here (bf16, tcgen05) that is two launches:
//   1. esfk_prologue (cooperative, one grid barrier): the caller's ReIndex
//      (segments padded to its blk) re-laid into 64-position segments
//      (idx64); x and g gathered into that expert-sorted layout (pads ->
//      zero rows) with the ESS column sums of g fused into the gather
//      (per 64-row item, fixed-order partials); rv[p] = token of position p;
//      the grad-x tile table and the ESTMM chunk table.  After the barrier:
//      grad_b combined per expert in item order (deterministic) and the gW
//      slices of split experts zeroed.
//   2. esfk_kernel (umma_impl.cuh): one persistent tcgen05 launch whose
//      clusters are split between the grad-x ESMM tiles (W read K-major as
//      W^T, fp32 rows written to token order through rv) and the grad-W
//      ESTMM chunks -- the combined work list, partitioned by cluster in
//      proportion to each side's roofline time.
// The fp32 path (and bf16 shapes TMA cannot describe) runs esfk_simt
// (simt.cu): a single launch whose blocks are partitioned the same way.
#include <cooperative_groups.h>

#include "umma_impl.cuh"
#include "routing.cuh"

namespace hxm {
namespace {

constexpr int kPT = 256;       // prologue threads
constexpr int kItem = 64;      // positions per gather / ESS item (segments are multiples)
constexpr int kColBlk = 256;   // columns per ESS reduction pass

struct EsfkPro {
  const __nv_bfloat16* x;
  const __nv_bfloat16* g;
  int64_t d1, d2;
  const int64_t* v;
  const int64_t* idx;
  int E;
  int32_t* idx64;  // E + 1
  int32_t* rv;     // bound64 positions: token or -1
  __nv_bfloat16* xs;
  __nv_bfloat16* gs;
  float* partial;  // items x d2
  float* grad_b;   // E x d2
  float* grad_w;   // E x d1 x d2: split experts' slices zeroed
  TileSpec s0, s1;
};

// smem idx64[0..E] = exclusive scan of the 64-padded segment lengths
__device__ void scan_idx64(const int64_t* __restrict__ idx, int E, int32_t* sidx) {
  using Scan = cub::BlockScan<int32_t, kPT>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int e0 = 0; e0 < E; e0 += kPT) {
    const int e = e0 + threadIdx.x;
    const int32_t len = e < E ? static_cast<int32_t>((idx[e + 1] - idx[e] + 63) / 64 * 64) : 0;
    int32_t excl, agg;
    Scan(tmp).ExclusiveSum(len, excl, agg);
    if (e < E) sidx[e] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) sidx[E] = carry;
  __syncthreads();
}

__global__ void __launch_bounds__(kPT) esfk_prologue(EsfkPro a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ int32_t sidx[];  // E + 1
  __shared__ float red[kPT / 32][kColBlk];
  __shared__ int64_t srow[kItem];
  const int E = a.E;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int W = kPT / 32;
  scan_idx64(a.idx, E, sidx);
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e <= E; e += kPT) a.idx64[e] = sidx[e];
  {
    const int tb = static_cast<int>(gridDim.x) - 1 - static_cast<int>(blockIdx.x);
    const bool one = gridDim.x < 2;
    if (tb == 0)
      tile_pass<int32_t, kPT>(sidx, E, a.s0.rows, a.s0.min_one, a.s0.tiles, a.s0.tile_off,
                              a.s0.n_tiles, nullptr, a.s0.split_rows);
    if (one ? tb == 0 : tb == 1)
      tile_pass<int32_t, kPT>(sidx, E, a.s1.rows, a.s1.min_one, a.s1.tiles, a.s1.tile_off,
                              a.s1.n_tiles, nullptr, a.s1.split_rows);
  }
  // ---- gather + fused ESS partials, one 64-position item at a time --------
  const int items = sidx[E] / kItem;
  const int u1 = static_cast<int>(a.d1 / 8), u2 = static_cast<int>(a.d2 / 8);  // 16-B units
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int p0 = it * kItem;
    int lo = 0, hi = E;  // expert: last e with sidx[e] <= p0
    while (hi - lo > 1) {
      const int mid = (lo + hi) / 2;
      if (sidx[mid] <= p0) lo = mid; else hi = mid;
    }
    const int e = lo;
    __syncthreads();  // previous item's srow / red reads are done
    if (threadIdx.x < kItem) {
      const int64_t off = p0 + threadIdx.x - sidx[e];
      const int64_t len = a.idx[e + 1] - a.idx[e];
      const int64_t t = off < len ? a.v[a.idx[e] + off] : -1;
      srow[threadIdx.x] = t;
      a.rv[p0 + threadIdx.x] = static_cast<int32_t>(t);
    }
    __syncthreads();
    // x rows: warp w copies rows w, w + 8, ... (8 rows in flight per lane pass)
    for (int c0 = 0; c0 < u1; c0 += 32) {
      const int u = c0 + lane;
      uint4 buf[kItem / W];
#pragma unroll
      for (int r = 0; r < kItem / W; ++r) {
        const int64_t t = srow[warp + r * W];
        buf[r] = (t >= 0 && u < u1)
                     ? __ldg(reinterpret_cast<const uint4*>(a.x + t * a.d1) + u)
                     : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int r = 0; r < kItem / W; ++r)
        if (u < u1)
          reinterpret_cast<uint4*>(a.xs + static_cast<int64_t>(p0 + warp + r * W) * a.d1)[u] =
              buf[r];
    }
    // g rows: copied the same way, their columns summed per warp, then the
    // 8 warps' sums added in a fixed order -> partial[it] (deterministic)
    for (int cb = 0; cb < u2; cb += kColBlk / 8) {
      float acc[kColBlk / 8 / 32][8];
#pragma unroll
      for (int j = 0; j < kColBlk / 8 / 32; ++j)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[j][q] = 0.f;
#pragma unroll
      for (int j = 0; j < kColBlk / 8 / 32; ++j) {
        const int u = cb + j * 32 + lane;
        uint4 buf[kItem / W];
#pragma unroll
        for (int r = 0; r < kItem / W; ++r) {
          const int64_t t = srow[warp + r * W];
          buf[r] = (t >= 0 && u < u2)
                       ? __ldg(reinterpret_cast<const uint4*>(a.g + t * a.d2) + u)
                       : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int r = 0; r < kItem / W; ++r) {
          if (u < u2)
            reinterpret_cast<uint4*>(a.gs + static_cast<int64_t>(p0 + warp + r * W) * a.d2)[u] =
                buf[r];
          const uint32_t w4[4] = {buf[r].x, buf[r].y, buf[r].z, buf[r].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[j][2 * q] += __uint_as_float(w4[q] << 16);
            acc[j][2 * q + 1] += __uint_as_float(w4[q] & 0xffff0000u);
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < kColBlk / 8 / 32; ++j)
#pragma unroll
        for (int q = 0; q < 8; ++q) red[warp][(j * 32 + lane) * 8 + q] = acc[j][q];
      __syncthreads();
      for (int c = threadIdx.x; c < kColBlk; c += kPT) {
        const int64_t col = static_cast<int64_t>(cb) * 8 + c;
        if (col >= a.d2) continue;
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < W; ++w) s += red[w][c];
        a.partial[static_cast<int64_t>(it) * a.d2 + col] = s;
      }
    }
  }
  grid.sync();
  // ---- grad_b[e] = sum of e's item partials in item order -----------------
  const int cblocks = static_cast<int>((a.d2 + kColBlk - 1) / kColBlk);
  for (int job = blockIdx.x; job < E * cblocks; job += gridDim.x) {
    const int e = job / cblocks;
    const int64_t c = static_cast<int64_t>(job % cblocks) * kColBlk + threadIdx.x;
    if (c >= a.d2) continue;
    const int i0 = sidx[e] / kItem, i1 = sidx[e + 1] / kItem;
    float s = 0.f;
    for (int i = i0; i < i1; ++i) s += __ldcg(a.partial + static_cast<int64_t>(i) * a.d2 + c);
    a.grad_b[static_cast<int64_t>(e) * a.d2 + c] = s;
  }
  // ---- split experts (several ESTMM chunks reduce with red.add): zero ------
  const int64_t slice = a.d1 * a.d2;
  constexpr int kParts = 64;
  for (int job = blockIdx.x; job < E * kParts; job += gridDim.x) {
    const int e = job / kParts, part = job % kParts;
    if (sidx[e + 1] - sidx[e] <= a.s1.rows) continue;  // one chunk: written, not reduced
    float* out = a.grad_w + static_cast<int64_t>(e) * slice;
    const int64_t per = ceil_div(ceil_div(slice, kParts), 4) * 4;
    const int64_t lo = part * per, hi = min(slice, lo + per);
    for (int64_t i = lo + 4 * threadIdx.x; i < hi; i += 4 * kPT)
      *reinterpret_cast<float4*>(out + i) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

struct EsfkWs {
  int32_t* idx64;
  int32_t* rv;
  void* xs;
  void* gs;
  float* partial;
  SegTile* tiles;
  int32_t* tile_off;
  int32_t* n_tiles;
  SegTile* ktiles;
  int32_t* ktile_off;
  int32_t* n_ktiles;
  int64_t bound64;
  int max_tiles, max_ktiles;
};

EsfkWs carve_esfk(Arena& ar, int64_t np_bound, int64_t E, int64_t d1, int64_t d2) {
  EsfkWs w{};
  w.bound64 = np_bound + 63 * E;
  w.idx64 = ar.take<int32_t>(E + 1);
  w.rv = ar.take<int32_t>(std::max<int64_t>(w.bound64, 1));
  w.xs = ar.take<char>(static_cast<size_t>(std::max<int64_t>(w.bound64, 1)) * d1 * 2);
  w.gs = ar.take<char>(static_cast<size_t>(std::max<int64_t>(w.bound64, 1)) * d2 * 2);
  w.partial = ar.take<float>(static_cast<size_t>(ceil_div(w.bound64, kItem) + 1) * d2);
  w.max_tiles = static_cast<int>(max_tiles(w.bound64, E, kUmmaRows));
  w.tiles = ar.take<SegTile>(w.max_tiles);
  w.tile_off = ar.take<int32_t>(E + 1);
  w.n_tiles = ar.take<int32_t>(1);
  w.max_ktiles = static_cast<int>(max_tiles(w.bound64, E, kEstmmSplit));
  w.ktiles = ar.take<SegTile>(w.max_ktiles);
  w.ktile_off = ar.take<int32_t>(E + 1);
  w.n_ktiles = ar.take<int32_t>(1);
  return w;
}

// one BN for both sides (the instantiation set stays small): the largest
// width dividing grad-x's N = d1 and grad-W's N = d2 under each side's rules
int esfk_bn(int64_t d1, int64_t d2, int CG, bool gx_b_mn) {
  for (int bn : {256, 192, 128, 64}) {
    if (d1 % bn || d2 % bn) continue;
    if (CG == 2 && (bn < 128)) continue;  // MN-major B halves: whole swizzle atoms
    (void)gx_b_mn;
    return bn;
  }
  return 0;
}

template <int BN, int CG>
hxm_status launch_esfk_bn(const UParams& p0, const UParams& p3, int split, int grid,
                          cudaStream_t st) {
  constexpr int EW = 8;
  auto kern = esfk_kernel<BN, BN, CG, EW>;
  constexpr int kSmem = Cfg<BN, CG, 0, EW>::kSmem > Cfg<BN, CG, 3, EW>::kSmem
                            ? Cfg<BN, CG, 0, EW>::kSmem
                            : Cfg<BN, CG, 3, EW>::kSmem;
  static bool attr_set[64] = {false};
  int dev = 0;
  HXM_TRY_CUDA(cudaGetDevice(&dev));
  dev = dev < 64 ? dev : 63;
  if (!attr_set[dev]) {
    HXM_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(64 + 32 * EW);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_on()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if constexpr (CG == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  HXM_TRY_CUDA(cudaLaunchKernelEx(&cfg, kern, p0, p3, split));
  HXM_CHECK_LAUNCH();
  return HXM_OK;
}

template <int CG>
hxm_status launch_esfk_any(int bn, const UParams& p0, const UParams& p3, int split, int grid,
                           cudaStream_t st) {
  switch (bn) {
    case 256: return launch_esfk_bn<256, CG>(p0, p3, split, grid, st);
    case 192: return launch_esfk_bn<192, CG>(p0, p3, split, grid, st);
    case 128: return launch_esfk_bn<128, CG>(p0, p3, split, grid, st);
    default:
      if constexpr (CG == 1) return launch_esfk_bn<64, 1>(p0, p3, split, grid, st);
      return invalid_arg("esfk: CTA-pair tiles need BN >= 128");
  }
}

}  // namespace

size_t esfk_ws_bytes(int64_t np_bound, int64_t E, int64_t d1, int64_t d2) {
  Arena ar(nullptr, 0);
  carve_esfk(ar, np_bound, E, d1, d2);
  return ar.used;
}

bool esfk_umma_ok(int64_t d1, int64_t d2) {
  return umma_supports_esmm(d1, d2) && esfk_bn(d1, d2, 1, true) > 0;
}

hxm_status umma_esfk(const void* x, const void* g, int64_t n, int64_t d1, int64_t d2,
                     const void* w, int w_trans, const int64_t* v, const int64_t* idx,
                     int64_t E, int64_t np_bound, float* grad_x, float* grad_b, float* grad_w,
                     void* ws, size_t ws_bytes, cudaStream_t st) {
  Arena ar(ws, ws_bytes);
  EsfkWs o = carve_esfk(ar, np_bound, E, d1, d2);
  if (ar.overflow) return invalid_arg("esfk: workspace too small");
  // CTA pairs when both sides tile M = 256: grad-x always (dense sorted A),
  // grad-W when d1 splits into 256-row output blocks
  const bool gx_b_mn = !w_trans;
  int CG = (d1 % 256 == 0 && esfk_bn(d1, d2, 2, gx_b_mn) > 0) ? 2 : 1;
  {
    const char* env = std::getenv("HXM_CTA_PAIR");
    if (env && env[0] == '0') CG = 1;
  }
  const int bn = esfk_bn(d1, d2, CG, gx_b_mn);
  if (bn == 0) return invalid_arg("esfk: no tcgen05 tile width divides d1 and d2");
  const int rows = CG == 2 ? kUmma2Rows : kUmmaRows;
  // (1) prologue
  {
    ProfScope ps(st, "esfk_prologue",
                 static_cast<double>(n) * (d1 + 2.0 * d2) * 2.0 + 4.0 * E * d2, WORK_BYTES);
    EsfkPro p{};
    p.x = static_cast<const __nv_bfloat16*>(x);
    p.g = static_cast<const __nv_bfloat16*>(g);
    p.d1 = d1;
    p.d2 = d2;
    p.v = v;
    p.idx = idx;
    p.E = static_cast<int>(E);
    p.idx64 = o.idx64;
    p.rv = o.rv;
    p.xs = static_cast<__nv_bfloat16*>(o.xs);
    p.gs = static_cast<__nv_bfloat16*>(o.gs);
    p.partial = o.partial;
    p.grad_b = grad_b;
    p.grad_w = grad_w;
    p.s0 = {rows, 0, o.tiles, o.tile_off, o.n_tiles};
    p.s1 = {kEstmmChunk, 1, o.ktiles, o.ktile_off, o.n_ktiles, kEstmmSplit};
    const size_t smem = (static_cast<size_t>(E) + 1) * sizeof(int32_t);
    int occ = 0;
    HXM_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, esfk_prologue, kPT, smem));
    if (occ < 1) return invalid_arg("esfk: prologue cannot be resident");
    const int grid = sm_count() * std::min(occ, 4);
    void* args[] = {&p};
    HXM_TRY_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(esfk_prologue), dim3(grid),
                                             dim3(kPT), args, smem, st));
    HXM_CHECK_LAUNCH();
  }
  // (2) one persistent tcgen05 launch: grad-x tiles | grad-W chunks
  EsmmArgs ax{};
  ax.a = o.gs;
  ax.amap = map_dense();
  ax.a_rows = std::max<int64_t>(o.bound64, 1);
  ax.n_experts = E;
  ax.w = w;
  ax.w_trans = w_trans;
  ax.d1 = d2;  // K
  ax.d2 = d1;  // N
  ax.tiles = o.tiles;
  ax.n_tiles = o.n_tiles;
  ax.max_tiles = static_cast<int>(max_tiles(o.bound64, E, rows));
  ax.tile_rows = rows;
  ax.epi = EPI_WRITE;
  ax.out_f32 = grad_x;
  ax.omap = map_slot(o.rv, std::max<int64_t>(n, 1));
  EstmmArgs aw{};
  aw.x1 = o.xs;
  aw.m1 = map_dense();
  aw.x2 = o.gs;
  aw.m2 = map_dense();
  aw.x1_rows = aw.x2_rows = std::max<int64_t>(o.bound64, 1);
  aw.d1 = d1;
  aw.d2 = d2;
  aw.tiles = o.ktiles;
  aw.n_tiles = o.n_ktiles;
  aw.max_tiles = o.max_ktiles;
  aw.n_experts = static_cast<int>(E);
  aw.out = grad_w;
  UParams p0{}, p3{};
  HXM_RETURN_IF(prep_esmm(ax, CG, bn, p0));
  HXM_RETURN_IF(prep_estmm(aw, CG, bn, p3));
  p0.label = "esfk_gx";
  p3.label = "esfk_gw";
  p0.l2hint = p3.l2hint = 1;
  // clusters split in proportion to each side's roofline time (equal FLOP;
  // grad-W also writes E x d1 x d2 fp32)
  const double flop = 2.0 * static_cast<double>(n) * d1 * d2;
  const double t0 = std::max(flop / 1.6e15, (n * (d2 * 2.0 + d1 * 4.0) + E * d1 * d2 * 2.0) / 6.4e12);
  const double t3 = std::max(flop / 1.6e15, (n * (d1 + d2) * 2.0 + E * d1 * d2 * 4.0) / 6.4e12);
  const int work0 = ax.max_tiles * p0.n_nt, work3 = aw.max_tiles * p3.n_mt * p3.n_nt;
  const int ncl = std::max(2, std::min(sm_count() / CG, work0 + work3));
  int split = static_cast<int>(std::lround(ncl * t0 / (t0 + t3)));
  split = std::max(1, std::min(ncl - 1, split));
  ProfScope ps(st, "esfk_gemm", 2.0 * flop, WORK_FLOP,
               n * (d1 + d2) * 2.0 * 2.0 + E * d1 * d2 * 6.0 + n * d1 * 4.0);
  if (CG == 2) return launch_esfk_any<2>(bn, p0, p3, split, ncl * 2, st);
  return launch_esfk_any<1>(bn, p0, p3, split, ncl, st);
}

}  // namespace hxm
