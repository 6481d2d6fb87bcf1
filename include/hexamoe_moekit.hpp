// hexamoe_moekit.hpp -- header-only C++ shim that re-exposes the reference
// `moekit` hot-path API (core/include/moekit/{routing,es_ops,moe_layer}.hpp)
// on top of the C ABI in hexamoe.h.
//
// Include it AFTER the moekit headers in a translation unit of the reference
// (see INTEGRATION.md).  Every reference signature of SURVEY.md §8(b) has a
// same-named function here taking the reference's own types:
//
//   build_reindex, build_reindex_all             (routing.hpp:42-46)
//   esmm (both forms), ess, estmm, esfk          (es_ops.hpp:37-65)
//   moe_forward, moe_backward                    (moe_layer.hpp:61-73)
//
// Host fp64 containers are rounded to the selected device dtype, copied to the
// device, run through the B200 kernels and copied back; checks run on the host
// first, in the reference's order, and throw the reference's exception types
// (moekit::ShapeError, std::invalid_argument).  EsOptions::stats is honoured
// (OpStats counted exactly as the reference's tiles count them);
// EsOptions::tile_shuffle_seed is accepted and has no effect (the device
// result does not depend on tile order).
//
// Each function takes a trailing `DeviceOptions`: `dtype = HXM_BF16` runs the
// bf16 tcgen05 tensor-core kernels (fp32 accumulation; rtol 2e-2 against the
// fp64 reference), the default HXM_F32 the fp32 path (rtol 1e-4).  The layer
// keeps its forward stash on the device: hexamoe::moe_forward returns a
// hexamoe::ForwardStash holding the device workspace, which
// hexamoe::moe_backward consumes without a round trip (to_moekit() exports
// the reference's ForwardStash type when a caller needs it).  A
// moekit::ForwardStash made by the reference's own moe_forward is accepted
// too: its routing is recovered from stash.reindex and the device forward
// rebuilds the stash from stash.x.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hexamoe.h"

namespace hexamoe {

struct DeviceOptions {
  hxm_dtype dtype = HXM_F32;    // HXM_BF16: tcgen05 tensor cores, fp32 accumulate
  cudaStream_t stream = nullptr;
};

inline void throw_status(hxm_status s, const char* what) {
  if (s == HXM_OK) return;
  std::string msg = std::string(what) + ": " + hxm_last_error();
  if (s == HXM_ERR_SHAPE) throw moekit::ShapeError(msg);
  if (s == HXM_ERR_INVALID_ARG) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  explicit DevBuf(size_t count) : n(count) {
    cuda_check(cudaMalloc(&p, (count ? count : 1) * sizeof(T)), "cudaMalloc");
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// ---------------------------------------------------------------- copies --
// fp64 -> bf16, round to nearest even (through fp32; the same rounding
// callers apply to the values they hand the reference for parity checks)
inline uint16_t bf16_bits(double v) {
  const float f = static_cast<float>(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);  // NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}
inline double bf16_round(double v) {
  const uint32_t u = static_cast<uint32_t>(bf16_bits(v)) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// an input operand on the device in the requested dtype
struct DevOperand {
  DevBuf<char> buf;
  DevOperand(const std::vector<double>& h, hxm_dtype dt, cudaStream_t st)
      : buf(h.size() * (dt == HXM_BF16 ? 2 : 4)) {
    if (dt == HXM_BF16) {
      std::vector<uint16_t> tmp(h.size());
      for (size_t i = 0; i < h.size(); ++i) tmp[i] = bf16_bits(h[i]);
      cuda_check(cudaMemcpyAsync(buf.p, tmp.data(), tmp.size() * 2, cudaMemcpyHostToDevice, st),
                 "H2D");
      cuda_check(cudaStreamSynchronize(st), "H2D");
    } else {
      std::vector<float> tmp(h.begin(), h.end());
      cuda_check(cudaMemcpyAsync(buf.p, tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice, st),
                 "H2D");
      cuda_check(cudaStreamSynchronize(st), "H2D");
    }
  }
  void* get() const { return buf.p; }
};

inline void upload_f32(DevBuf<float>& d, const std::vector<double>& h, cudaStream_t st) {
  std::vector<float> tmp(h.begin(), h.end());
  cuda_check(cudaMemcpyAsync(d.p, tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaStreamSynchronize(st), "H2D");
}
inline void download(std::vector<double>& h, const float* d, cudaStream_t st) {
  std::vector<float> tmp(h.size());
  cuda_check(cudaMemcpyAsync(tmp.data(), d, tmp.size() * 4, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "D2H");
  for (size_t i = 0; i < h.size(); ++i) h[i] = tmp[i];
}

struct DevReIndex {
  DevBuf<int64_t> v, idx;
  DevReIndex(const moekit::ReIndex& rx, cudaStream_t st) : v(rx.v.size()), idx(rx.idx.size()) {
    cuda_check(cudaMemcpyAsync(v.p, rx.v.data(), rx.v.size() * 8, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(idx.p, rx.idx.data(), rx.idx.size() * 8, cudaMemcpyHostToDevice, st),
               "H2D");
    cuda_check(cudaStreamSynchronize(st), "H2D");
  }
};

// check_reindex (es_ops.cpp:12-17): the first check of every operator
inline void check_reindex(const moekit::ReIndex& rx) {
  if (rx.idx.size() < 2 || rx.idx.front() != 0 ||
      rx.idx.back() != static_cast<std::int64_t>(rx.v.size()))
    throw moekit::ShapeError("es-ops: malformed re-index vector");
}

// OpStats exactly as the reference's tiles increment them
inline void count(const moekit::EsOptions& opt, hxm_op_kind op, const moekit::ReIndex& rx,
                  size_t d1, size_t d2) {
  if (!opt.stats) return;
  int64_t pads = 0;
  for (int64_t t : rx.v) pads += t < 0;
  hxm_op_stats s{opt.stats->macs, opt.stats->adds, opt.stats->padding_slots};
  hxm_op_stats_add(op, static_cast<int64_t>(rx.v.size()) - pads, pads, d1, d2, &s);
  opt.stats->macs = s.macs;
  opt.stats->adds = s.adds;
  opt.stats->padding_slots = s.padding_slots;
}

// --------------------------------------------------------------- routing --
// moekit::build_reindex (routing.hpp:42-43) on the device.
inline moekit::ReIndex build_reindex(const std::vector<std::int32_t>& assignment,
                                     std::size_t n_experts, std::size_t blk,
                                     const DeviceOptions& dev = {}) {
  if (blk == 0) throw std::invalid_argument("build_reindex: blk must be >= 1");
  const cudaStream_t st = dev.stream;
  const int64_t n = static_cast<int64_t>(assignment.size());
  const size_t bound = hxm_reindex_bound(n, n_experts, blk);
  DevBuf<int32_t> a(n);
  DevBuf<int64_t> v(bound), idx(n_experts + 1);
  DevBuf<char> ws(hxm_reindex_workspace_bytes(n, n_experts));
  DevBuf<int32_t> status(1);
  cuda_check(cudaMemsetAsync(status.p, 0, sizeof(int32_t), st), "memset");
  cuda_check(cudaMemcpyAsync(a.p, assignment.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, st),
             "H2D");
  throw_status(hxm_build_reindex(a.p, n, n_experts, blk, v.p, idx.p, ws.p, ws.n, status.p,
                                 reinterpret_cast<hxm_stream_t>(st)),
               "build_reindex");
  int32_t bad = 0;
  moekit::ReIndex rx;
  rx.idx.resize(n_experts + 1);
  cuda_check(cudaMemcpyAsync(&bad, status.p, sizeof(bad), cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaMemcpyAsync(rx.idx.data(), idx.p, (n_experts + 1) * 8, cudaMemcpyDeviceToHost, st),
             "D2H");
  cuda_check(cudaStreamSynchronize(st), "D2H");
  if (bad) throw std::invalid_argument("build_reindex: expert id out of range");
  rx.v.resize(static_cast<size_t>(rx.idx.back()));
  cuda_check(cudaMemcpyAsync(rx.v.data(), v.p, rx.v.size() * 8, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "D2H");
  rx.blk = blk;
  rx.n_tokens = assignment.size();
  return rx;
}

// moekit::build_reindex_all (routing.hpp:46): all k choices in one batched call.
inline std::vector<moekit::ReIndex> build_reindex_all(const moekit::RoutingChoice& r,
                                                      std::size_t blk,
                                                      const DeviceOptions& dev = {}) {
  if (blk == 0) throw std::invalid_argument("build_reindex: blk must be >= 1");
  const cudaStream_t st = dev.stream;
  const int64_t k = static_cast<int64_t>(r.assignments.size());
  std::vector<moekit::ReIndex> out;
  if (k == 0) return out;
  const int64_t n = static_cast<int64_t>(r.assignments[0].size());
  for (const auto& a : r.assignments)
    if (static_cast<int64_t>(a.size()) != n)  // ragged choices: one index at a time
      {
        for (const auto& aa : r.assignments) out.push_back(build_reindex(aa, r.n_experts, blk, dev));
        return out;
      }
  const int64_t E = static_cast<int64_t>(r.n_experts);
  const int64_t bound = static_cast<int64_t>(hxm_reindex_bound(n, E, blk));
  std::vector<int32_t> flat(static_cast<size_t>(k * n));
  for (int64_t i = 0; i < k; ++i)
    std::memcpy(flat.data() + i * n, r.assignments[i].data(), n * sizeof(int32_t));
  DevBuf<int32_t> a(flat.size());
  DevBuf<int64_t> v(static_cast<size_t>(k * (bound > 0 ? bound : 1))), idx(k * (E + 1));
  DevBuf<char> ws(hxm_reindex_all_workspace_bytes(n, E, k));
  DevBuf<int32_t> status(1);
  cuda_check(cudaMemsetAsync(status.p, 0, sizeof(int32_t), st), "memset");
  cuda_check(cudaMemcpyAsync(a.p, flat.data(), flat.size() * 4, cudaMemcpyHostToDevice, st), "H2D");
  throw_status(hxm_build_reindex_all(a.p, k, n, E, blk, v.p, bound > 0 ? bound : 1, idx.p, ws.p,
                                     ws.n, status.p, reinterpret_cast<hxm_stream_t>(st)),
               "build_reindex_all");
  int32_t bad = 0;
  std::vector<int64_t> hidx(static_cast<size_t>(k * (E + 1)));
  cuda_check(cudaMemcpyAsync(&bad, status.p, sizeof(bad), cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaMemcpyAsync(hidx.data(), idx.p, hidx.size() * 8, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "D2H");
  if (bad) throw std::invalid_argument("build_reindex: expert id out of range");
  for (int64_t i = 0; i < k; ++i) {
    moekit::ReIndex rx;
    rx.idx.assign(hidx.begin() + i * (E + 1), hidx.begin() + (i + 1) * (E + 1));
    rx.v.resize(static_cast<size_t>(rx.idx.back()));
    cuda_check(cudaMemcpyAsync(rx.v.data(), v.p + i * bound, rx.v.size() * 8, cudaMemcpyDeviceToHost,
                               st),
               "D2H");
    rx.blk = blk;
    rx.n_tokens = static_cast<size_t>(n);
    out.push_back(std::move(rx));
  }
  cuda_check(cudaStreamSynchronize(st), "D2H");
  return out;
}

// ------------------------------------------------------------- operators --
// moekit::esmm, mode-dispatched form (es_ops.hpp:44-46).
inline void esmm(const moekit::Matrix2D& x, const moekit::Tensor3D& w,
                 const moekit::Matrix2D* bias, const moekit::ReIndex& rx,
                 moekit::EsOutputMode mode, moekit::Matrix2D* dest,
                 const moekit::EsOptions& opt = {}, const DeviceOptions& dev = {}) {
  check_reindex(rx);
  if (x.rows() != rx.n_tokens) throw moekit::ShapeError("esmm: token count does not match re-index vector");
  if (w.dim0() != rx.num_experts()) throw moekit::ShapeError("esmm: expert count mismatch between weights and rx");
  if (x.cols() != w.dim1()) throw moekit::ShapeError("esmm: x cols != weights dim1");
  if (bias && (bias->rows() != w.dim0() || bias->cols() != w.dim2()))
    throw moekit::ShapeError("esmm: bias shape must be E x D2");
  if (!dest)
    throw std::invalid_argument(mode == moekit::EsOutputMode::kAccumulate
                                    ? "esmm: Accumulate mode requires a destination"
                                    : "esmm: destination is null");
  if (dest->rows() != x.rows() || dest->cols() != w.dim2())
    throw moekit::ShapeError("esmm: destination shape must be N x D2");
  const cudaStream_t st = dev.stream;
  const int64_t E = w.dim0(), n = x.rows(), d1 = w.dim1(), d2 = w.dim2();
  DevOperand dx(x.data(), dev.dtype, st), dw(w.data(), dev.dtype, st);
  DevBuf<float> db(bias ? bias->size() : 1), dd(dest->size());
  if (bias) upload_f32(db, bias->data(), st);
  if (mode == moekit::EsOutputMode::kAccumulate) upload_f32(dd, dest->data(), st);
  DevReIndex drx(rx, st);
  DevBuf<char> ws(hxm_op_workspace_bytes(n, E, rx.v.size(), d1, d2));
  throw_status(hxm_esmm(dev.dtype, dx.get(), n, d1, dw.get(), E, d2, 0, bias ? db.p : nullptr,
                        drx.v.p, drx.idx.p, static_cast<int64_t>(rx.v.size()),
                        mode == moekit::EsOutputMode::kAccumulate ? HXM_ACCUMULATE : HXM_WRITE,
                        dd.p, ws.p, ws.n, reinterpret_cast<hxm_stream_t>(st)),
               "esmm");
  download(dest->data(), dd.p, st);
  count(opt, HXM_OP_ESMM, rx, d1, d2);
}

// moekit::esmm returning form (es_ops.hpp:39-40).
inline moekit::Matrix2D esmm(const moekit::Matrix2D& x, const moekit::Tensor3D& w,
                             const moekit::Matrix2D* bias, const moekit::ReIndex& rx,
                             const moekit::EsOptions& opt = {}, const DeviceOptions& dev = {}) {
  moekit::Matrix2D out(x.rows(), w.dim2());
  hexamoe::esmm(x, w, bias, rx, moekit::EsOutputMode::kWrite, &out, opt, dev);
  return out;
}

// moekit::ess (es_ops.hpp:49).
inline moekit::Matrix2D ess(const moekit::Matrix2D& x, const moekit::ReIndex& rx,
                            const moekit::EsOptions& opt = {}, const DeviceOptions& dev = {}) {
  check_reindex(rx);
  if (x.rows() != rx.n_tokens) throw moekit::ShapeError("ess: token count does not match re-index vector");
  const cudaStream_t st = dev.stream;
  const int64_t E = rx.num_experts(), n = x.rows(), d = x.cols();
  moekit::Matrix2D out(E, d);
  DevOperand dx(x.data(), dev.dtype, st);
  DevBuf<float> dout(out.size());
  DevReIndex drx(rx, st);
  DevBuf<char> ws(hxm_op_workspace_bytes(n, E, rx.v.size(), d, d));
  throw_status(hxm_ess(dev.dtype, dx.get(), n, d, drx.v.p, drx.idx.p, E, rx.v.size(), dout.p,
                       ws.p, ws.n, reinterpret_cast<hxm_stream_t>(st)),
               "ess");
  download(out.data(), dout.p, st);
  count(opt, HXM_OP_ESS, rx, d, 0);
  return out;
}

// moekit::estmm (es_ops.hpp:52-53).
inline moekit::Tensor3D estmm(const moekit::Matrix2D& x1, const moekit::Matrix2D& x2,
                              const moekit::ReIndex& rx, const moekit::EsOptions& opt = {},
                              const DeviceOptions& dev = {}) {
  check_reindex(rx);
  if (x1.rows() != x2.rows()) throw moekit::ShapeError("estmm: x1 and x2 token counts differ");
  if (x1.rows() != rx.n_tokens) throw moekit::ShapeError("estmm: token count does not match re-index vector");
  const cudaStream_t st = dev.stream;
  const int64_t E = rx.num_experts(), n = x1.rows(), d1 = x1.cols(), d2 = x2.cols();
  moekit::Tensor3D out(E, d1, d2);
  DevOperand a(x1.data(), dev.dtype, st), b(x2.data(), dev.dtype, st);
  DevBuf<float> dout(out.size());
  DevReIndex drx(rx, st);
  DevBuf<char> ws(hxm_op_workspace_bytes(n, E, rx.v.size(), d1, d2));
  throw_status(hxm_estmm(dev.dtype, a.get(), b.get(), n, d1, d2, drx.v.p, drx.idx.p, E,
                         rx.v.size(), dout.p, ws.p, ws.n, reinterpret_cast<hxm_stream_t>(st)),
               "estmm");
  download(out.data(), dout.p, st);
  count(opt, HXM_OP_ESTMM, rx, d1, d2);
  return out;
}

// moekit::esfk (es_ops.hpp:55-65): grad_x = esmm(g, w_t), grad_b = ess(g),
// grad_w = estmm(x, g) in one device call.
inline moekit::EsfkResult esfk(const moekit::Matrix2D& x, const moekit::Matrix2D& g,
                               const moekit::Tensor3D& w_t, const moekit::ReIndex& rx,
                               const moekit::EsOptions& opt = {}, const DeviceOptions& dev = {}) {
  check_reindex(rx);
  if (x.rows() != g.rows()) throw moekit::ShapeError("esfk: x and g token counts differ");
  if (x.rows() != rx.n_tokens) throw moekit::ShapeError("esfk: token count does not match re-index vector");
  if (w_t.dim0() != rx.num_experts() || w_t.dim1() != g.cols())
    throw moekit::ShapeError("esfk: w_t must be E x D2 x D1 for g of width D2");
  const cudaStream_t st = dev.stream;
  const int64_t E = rx.num_experts(), n = x.rows(), d1 = x.cols(), d2 = g.cols();
  if (static_cast<int64_t>(w_t.dim2()) != d1)
    throw moekit::ShapeError("esmm: x cols != weights dim1");
  moekit::EsfkResult r{moekit::Matrix2D(n, d1), moekit::Matrix2D(E, d2), moekit::Tensor3D(E, d1, d2)};
  DevOperand dx(x.data(), dev.dtype, st), dg(g.data(), dev.dtype, st), dw(w_t.data(), dev.dtype, st);
  DevBuf<float> gx(r.grad_x.size()), gb(r.grad_b.size()), gw(r.grad_w.size());
  DevReIndex drx(rx, st);
  DevBuf<char> ws(hxm_op_workspace_bytes(n, E, rx.v.size(), d1, d2));
  throw_status(hxm_esfk(dev.dtype, dx.get(), dg.get(), n, d1, d2, dw.get(), 0, drx.v.p, drx.idx.p,
                        E, rx.v.size(), gx.p, gb.p, gw.p, ws.p, ws.n,
                        reinterpret_cast<hxm_stream_t>(st)),
               "esfk");
  download(r.grad_x.data(), gx.p, st);
  download(r.grad_b.data(), gb.p, st);
  download(r.grad_w.data(), gw.p, st);
  count(opt, HXM_OP_ESFK, rx, d1, d2);
  return r;
}

// ----------------------------------------------------------------- layer --
// Device forward stash: the layer workspace (expert-sorted x, F'(y1), F(y1),
// the k-choice index) plus the device copy of x, alive as long as any copy
// of the stash is.
struct LayerState {
  hxm_layer_desc desc{};
  std::unique_ptr<DevBuf<char>> ws;
  std::unique_ptr<DevOperand> x;
  cudaStream_t stream = nullptr;
};

struct ForwardStash {
  std::shared_ptr<LayerState> dev;
  moekit::Matrix2D x;                     // as moekit::ForwardStash::x
  std::vector<moekit::ReIndex> reindex;   // as moekit::ForwardStash::reindex
  moekit::MoeScheme scheme = moekit::MoeScheme::kMemoryEfficient;
  std::size_t blk = 8;

  // The reference's ForwardStash (moe_layer.hpp:39-46): y2_i = F(y1_i) comes
  // from the device stash; y1_i (which the device does not keep -- it stores
  // F'(y1) instead) is recomputed as esmm(x, W1, b1, R_i) on the device.
  moekit::ForwardStash to_moekit(const moekit::MoeLayerParams& p,
                                 const DeviceOptions& devopt = {}) const;
};

struct MoeForwardResult {
  moekit::Matrix2D y;
  ForwardStash stash;
};

inline hxm_layer_desc layer_desc(const moekit::MoeLayerParams& p, size_t n, size_t k,
                                 hxm_dtype dt) {
  hxm_layer_desc d{};
  d.n_tokens = static_cast<int64_t>(n);
  d.n_experts = static_cast<int64_t>(p.experts());
  d.k = static_cast<int64_t>(k);
  d.d_in = static_cast<int64_t>(p.d_in());
  d.hidden = static_cast<int64_t>(p.hidden());
  d.d_out = static_cast<int64_t>(p.d_out());
  d.activation = static_cast<int32_t>(p.activation);  // same enum order (tensor.hpp:96)
  d.dtype = dt;
  d.add_b2 = 1;
  d.capacity = 0;
  return d;
}

// layer OpStats: the reference passes opt to every operator of the layer
// (moe_layer.cpp:56-62, 98-118)
inline void count_forward(const moekit::EsOptions& opt, const moekit::MoeLayerParams& p,
                          const std::vector<moekit::ReIndex>& rxs) {
  for (const auto& rx : rxs) {
    count(opt, HXM_OP_ESMM, rx, p.d_in(), p.hidden());
    count(opt, HXM_OP_ESMM, rx, p.hidden(), p.d_out());
  }
}
inline void count_backward(const moekit::EsOptions& opt, const moekit::MoeLayerParams& p,
                           const std::vector<moekit::ReIndex>& rxs) {
  for (const auto& rx : rxs) {
    count(opt, HXM_OP_ESFK, rx, p.hidden(), p.d_out());  // esfk(y2, g_y, W2^T)
    count(opt, HXM_OP_ESFK, rx, p.d_in(), p.hidden());   // esfk(x, g_y1, W1^T)
  }
}

// moekit::moe_forward (moe_layer.hpp:64-66, moe_layer.cpp:30-67): all k
// choices in one device forward (one k-merged index, two tcgen05 GEMMs).
inline MoeForwardResult moe_forward(const moekit::Matrix2D& x, const moekit::MoeLayerParams& p,
                                    const moekit::RoutingChoice& r, std::size_t blk,
                                    moekit::MoeScheme scheme, const moekit::EsOptions& opt = {},
                                    const DeviceOptions& dev = {}) {
  p.validate();
  r.validate();
  if (x.rows() != r.n_tokens) throw moekit::ShapeError("moe_forward: x rows != routed token count");
  if (x.cols() != p.d_in()) throw moekit::ShapeError("moe_forward: x cols != layer input size");
  if (r.n_experts != p.experts())
    throw moekit::ShapeError("moe_forward: routing expert count != layer experts");
  if (blk == 0) throw std::invalid_argument("build_reindex: blk must be >= 1");
  const cudaStream_t st = dev.stream;
  const hxm_stream_t hs = reinterpret_cast<hxm_stream_t>(st);
  MoeForwardResult res;
  auto L = std::make_shared<LayerState>();
  L->desc = layer_desc(p, r.n_tokens, r.k, dev.dtype);
  L->stream = st;
  const size_t wsb = hxm_layer_workspace_bytes(&L->desc);
  if (wsb == 0) throw std::invalid_argument("moe_forward: invalid layer descriptor");
  L->ws = std::make_unique<DevBuf<char>>(wsb);
  L->x = std::make_unique<DevOperand>(x.data(), dev.dtype, st);
  DevOperand w1(p.w1.data(), dev.dtype, st), w2(p.w2.data(), dev.dtype, st);
  DevBuf<float> b1(p.b1.size()), b2(p.b2.size()), y(x.rows() * p.d_out());
  upload_f32(b1, p.b1.data(), st);
  upload_f32(b2, p.b2.data(), st);
  std::vector<int32_t> flat;
  flat.reserve(r.k * r.n_tokens);
  for (const auto& a : r.assignments) flat.insert(flat.end(), a.begin(), a.end());
  DevBuf<int32_t> a(flat.size()), status(1);
  cuda_check(cudaMemcpyAsync(a.p, flat.data(), flat.size() * 4, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemsetAsync(status.p, 0, 4, st), "memset");
  throw_status(hxm_moe_forward(&L->desc, L->x->get(), w1.get(), b1.p, w2.get(), b2.p, a.p, y.p,
                               L->ws->p, L->ws->n, status.p, hs),
               "moe_forward");
  res.y = moekit::Matrix2D(x.rows(), p.d_out());
  download(res.y.data(), y.p, st);
  // the reference's per-choice index (ForwardStash::reindex, blk as given)
  res.stash.reindex = build_reindex_all(r, blk, dev);
  res.stash.dev = std::move(L);
  res.stash.x = x;
  res.stash.scheme = scheme;
  res.stash.blk = blk;
  count_forward(opt, p, res.stash.reindex);
  return res;
}

// moekit::moe_backward (moe_layer.hpp:70-73, moe_layer.cpp:69-122) for a
// device stash.  Fused and unfused are the same device schedule (the
// reference proves them bit-identical, test_moe_layer.cpp:169-187).
inline moekit::MoeGrads moe_backward(const ForwardStash& stash, const moekit::MoeLayerParams& p,
                                     const moekit::Matrix2D& g_y, bool use_fused = false,
                                     const moekit::EsOptions& opt = {},
                                     const DeviceOptions& dev = {}) {
  (void)use_fused;
  p.validate();
  const size_t k = stash.reindex.size();
  if (!stash.dev || static_cast<size_t>(stash.dev->desc.k) != k)
    throw moekit::ShapeError("moe_backward: stash is incomplete");
  if (g_y.rows() != stash.x.rows() || g_y.cols() != p.d_out())
    throw moekit::ShapeError("moe_backward: g_y shape must be N x D_o");
  const hxm_layer_desc& d = stash.dev->desc;
  if (stash.x.cols() != p.d_in() || d.hidden != static_cast<int64_t>(p.hidden()) ||
      d.n_experts != static_cast<int64_t>(p.experts()))
    throw moekit::ShapeError("moe_backward: stash does not match params");
  const hxm_dtype dt = static_cast<hxm_dtype>(d.dtype);
  const cudaStream_t st = dev.stream;
  DevOperand w1(p.w1.data(), dt, st), w2(p.w2.data(), dt, st), gy(g_y.data(), dt, st);
  moekit::MoeGrads g{moekit::Tensor3D(p.experts(), p.d_in(), p.hidden()),
                     moekit::Matrix2D(p.experts(), p.hidden()),
                     moekit::Tensor3D(p.experts(), p.hidden(), p.d_out()),
                     moekit::Matrix2D(p.experts(), p.d_out()),
                     moekit::Matrix2D(stash.x.rows(), p.d_in())};
  DevBuf<float> gw1(g.gw1.size()), gb1(g.gb1.size()), gw2(g.gw2.size()), gb2(g.gb2.size()),
      gx(g.gx.size());
  throw_status(hxm_moe_backward(&d, stash.dev->x->get(), w1.get(), w2.get(), gy.get(),
                                stash.dev->ws->p, stash.dev->ws->n, gw1.p, gb1.p, gw2.p, gb2.p,
                                gx.p, reinterpret_cast<hxm_stream_t>(st)),
               "moe_backward");
  download(g.gw1.data(), gw1.p, st);
  download(g.gb1.data(), gb1.p, st);
  download(g.gw2.data(), gw2.p, st);
  download(g.gb2.data(), gb2.p, st);
  download(g.gx.data(), gx.p, st);
  count_backward(opt, p, stash.reindex);
  return g;
}

// The reference's RoutingChoice recovered from a stash's per-choice indices
// (token t in expert e's segment of choice i -> assignments[i][t] = e).
inline moekit::RoutingChoice routing_from_reindex(const std::vector<moekit::ReIndex>& rxs) {
  moekit::RoutingChoice r;
  r.k = rxs.size();
  r.n_tokens = rxs.empty() ? 0 : rxs[0].n_tokens;
  r.n_experts = rxs.empty() ? 0 : rxs[0].num_experts();
  for (const auto& rx : rxs) {
    check_reindex(rx);
    std::vector<std::int32_t> a(r.n_tokens, -1);
    for (size_t e = 0; e + 1 < rx.idx.size(); ++e)
      for (int64_t q = rx.idx[e]; q < rx.idx[e + 1]; ++q)
        if (rx.v[q] >= 0 && static_cast<size_t>(rx.v[q]) < a.size())
          a[rx.v[q]] = static_cast<std::int32_t>(e);
    r.assignments.push_back(std::move(a));
  }
  return r;
}

// moe_backward for a stash made by the reference's own moekit::moe_forward:
// the device forward rebuilds its stash from stash.x and the recovered
// routing (its y1 / y2 equal the reference's up to the device rounding).
inline moekit::MoeGrads moe_backward(const moekit::ForwardStash& stash,
                                     const moekit::MoeLayerParams& p, const moekit::Matrix2D& g_y,
                                     bool use_fused = false, const moekit::EsOptions& opt = {},
                                     const DeviceOptions& dev = {}) {
  p.validate();
  const size_t k = stash.reindex.size();
  if (stash.y1.size() != k || stash.y2.size() != k)
    throw moekit::ShapeError("moe_backward: stash is incomplete");
  if (g_y.rows() != stash.x.rows() || g_y.cols() != p.d_out())
    throw moekit::ShapeError("moe_backward: g_y shape must be N x D_o");
  if (stash.x.cols() != p.d_in() || (k > 0 && stash.y1[0].cols() != p.hidden()))
    throw moekit::ShapeError("moe_backward: stash does not match params");
  const moekit::RoutingChoice r = routing_from_reindex(stash.reindex);
  MoeForwardResult fw = moe_forward(stash.x, p, r, stash.blk, stash.scheme, {}, dev);
  return moe_backward(fw.stash, p, g_y, use_fused, opt, dev);
}

inline moekit::ForwardStash ForwardStash::to_moekit(const moekit::MoeLayerParams& p,
                                                    const DeviceOptions& devopt) const {
  moekit::ForwardStash s;
  s.x = x;
  s.reindex = reindex;
  s.scheme = scheme;
  s.blk = blk;
  const hxm_layer_desc& d = dev->desc;
  const cudaStream_t st = devopt.stream;
  const size_t n = static_cast<size_t>(d.n_tokens), h = static_cast<size_t>(d.hidden);
  DevBuf<float> dact(n * h), y2(n * h);
  DeviceOptions o = devopt;
  o.dtype = static_cast<hxm_dtype>(d.dtype);
  for (size_t i = 0; i < reindex.size(); ++i) {
    throw_status(hxm_moe_stash_export(&d, dev->ws->p, static_cast<int64_t>(i), dact.p, y2.p,
                                      reinterpret_cast<hxm_stream_t>(st)),
                 "stash_export");
    moekit::Matrix2D m(n, h);
    download(m.data(), y2.p, st);
    s.y2.push_back(std::move(m));
    s.y1.push_back(hexamoe::esmm(x, p.w1, &p.b1, reindex[i], {}, o));
  }
  return s;
}

}  // namespace hexamoe
