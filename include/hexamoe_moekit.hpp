// hexamoe_moekit.hpp -- header-only C++ shim that re-exposes the reference
// `moekit` operator signatures (core/include/moekit/{routing,es_ops,
// moe_layer}.hpp) on top of the C ABI in hexamoe.h.
//
// Include it AFTER the moekit headers in a translation unit of the reference
// (see INTEGRATION.md).  Host fp64 containers are rounded to the selected
// device dtype, copied to the device, run through the B200 kernels and copied
// back; exceptions are rethrown with the reference's types.  It is the
// drop-in for code that keeps the reference's host types; device-resident
// callers use hexamoe.h directly.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "hexamoe.h"

namespace hexamoe {

inline void throw_status(hxm_status s, const char* what) {
  if (s == HXM_OK) return;
  std::string msg = std::string(what) + ": " + hxm_last_error();
  if (s == HXM_ERR_SHAPE) throw moekit::ShapeError(msg);
  if (s == HXM_ERR_INVALID_ARG) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  explicit DevBuf(size_t count) : n(count) {
    if (cudaMalloc(&p, (count ? count : 1) * sizeof(T)) != cudaSuccess)
      throw std::runtime_error("cudaMalloc failed");
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// fp64 host -> fp32 device (the fp32 operator path; rtol 1e-4 vs the reference)
inline void upload(DevBuf<float>& d, const std::vector<double>& h) {
  std::vector<float> tmp(h.begin(), h.end());
  cudaMemcpy(d.p, tmp.data(), tmp.size() * sizeof(float), cudaMemcpyHostToDevice);
}
inline void download(std::vector<double>& h, const DevBuf<float>& d) {
  std::vector<float> tmp(h.size());
  cudaMemcpy(tmp.data(), d.p, tmp.size() * sizeof(float), cudaMemcpyDeviceToHost);
  for (size_t i = 0; i < h.size(); ++i) h[i] = tmp[i];
}

// moekit::build_reindex (routing.hpp:42-43) on the device.
inline moekit::ReIndex build_reindex(const std::vector<std::int32_t>& assignment,
                                     std::size_t n_experts, std::size_t blk) {
  if (blk == 0) throw std::invalid_argument("build_reindex: blk must be >= 1");
  const int64_t n = static_cast<int64_t>(assignment.size());
  const size_t bound = hxm_reindex_bound(n, n_experts, blk);
  DevBuf<int32_t> a(n);
  DevBuf<int64_t> v(bound), idx(n_experts + 1);
  DevBuf<char> ws(hxm_reindex_workspace_bytes(n, n_experts));
  DevBuf<int32_t> status(1);
  cudaMemset(status.p, 0, sizeof(int32_t));
  cudaMemcpy(a.p, assignment.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice);
  throw_status(hxm_build_reindex(a.p, n, n_experts, blk, v.p, idx.p, ws.p, ws.n, status.p,
                                 nullptr),
               "build_reindex");
  int32_t st = 0;
  cudaMemcpy(&st, status.p, sizeof(st), cudaMemcpyDeviceToHost);
  if (st) throw std::invalid_argument("build_reindex: expert id out of range");
  moekit::ReIndex rx;
  rx.idx.resize(n_experts + 1);
  cudaMemcpy(rx.idx.data(), idx.p, (n_experts + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost);
  rx.v.resize(static_cast<size_t>(rx.idx.back()));
  cudaMemcpy(rx.v.data(), v.p, rx.v.size() * sizeof(int64_t), cudaMemcpyDeviceToHost);
  rx.blk = blk;
  rx.n_tokens = assignment.size();
  return rx;
}

// moekit::esmm, mode-dispatched form (es_ops.hpp:44-46), fp32 device path.
inline void esmm(const moekit::Matrix2D& x, const moekit::Tensor3D& w,
                 const moekit::Matrix2D* bias, const moekit::ReIndex& rx,
                 moekit::EsOutputMode mode, moekit::Matrix2D* dest) {
  if (x.rows() != rx.n_tokens) throw moekit::ShapeError("esmm: token count does not match re-index vector");
  if (w.dim0() != rx.num_experts()) throw moekit::ShapeError("esmm: expert count mismatch between weights and rx");
  if (x.cols() != w.dim1()) throw moekit::ShapeError("esmm: x cols != weights dim1");
  if (bias && (bias->rows() != w.dim0() || bias->cols() != w.dim2()))
    throw moekit::ShapeError("esmm: bias shape must be E x D2");
  if (!dest) throw std::invalid_argument("esmm: Accumulate mode requires a destination");
  if (dest->rows() != x.rows() || dest->cols() != w.dim2())
    throw moekit::ShapeError("esmm: destination shape must be N x D2");
  const int64_t E = w.dim0(), n = x.rows(), d1 = w.dim1(), d2 = w.dim2();
  DevBuf<float> dx(x.size()), dw(w.size()), db(bias ? bias->size() : 1), dd(dest->size());
  DevBuf<int64_t> v(rx.v.size()), idx(rx.idx.size());
  upload(dx, x.data());
  upload(dw, w.data());
  if (bias) upload(db, bias->data());
  upload(dd, dest->data());
  cudaMemcpy(v.p, rx.v.data(), rx.v.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(idx.p, rx.idx.data(), rx.idx.size() * 8, cudaMemcpyHostToDevice);
  DevBuf<char> ws(hxm_op_workspace_bytes(n, E, rx.v.size(), d1, d2));
  throw_status(hxm_esmm(HXM_F32, dx.p, n, d1, dw.p, E, d2, 0, bias ? db.p : nullptr, v.p,
                        idx.p, static_cast<int64_t>(rx.v.size()),
                        mode == moekit::EsOutputMode::kAccumulate ? HXM_ACCUMULATE : HXM_WRITE,
                        dd.p, ws.p, ws.n, nullptr),
               "esmm");
  download(dest->data(), dd);
}

// moekit::esmm returning form (es_ops.hpp:39-40).
inline moekit::Matrix2D esmm(const moekit::Matrix2D& x, const moekit::Tensor3D& w,
                             const moekit::Matrix2D* bias, const moekit::ReIndex& rx) {
  moekit::Matrix2D out(x.rows(), w.dim2());
  hexamoe::esmm(x, w, bias, rx, moekit::EsOutputMode::kWrite, &out);
  return out;
}

// moekit::ess (es_ops.hpp:49).
inline moekit::Matrix2D ess(const moekit::Matrix2D& x, const moekit::ReIndex& rx) {
  if (x.rows() != rx.n_tokens) throw moekit::ShapeError("ess: token count does not match re-index vector");
  const int64_t E = rx.num_experts(), n = x.rows(), d = x.cols();
  moekit::Matrix2D out(E, d);
  DevBuf<float> dx(x.size()), dout(out.size());
  DevBuf<int64_t> v(rx.v.size()), idx(rx.idx.size());
  upload(dx, x.data());
  cudaMemcpy(v.p, rx.v.data(), rx.v.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(idx.p, rx.idx.data(), rx.idx.size() * 8, cudaMemcpyHostToDevice);
  DevBuf<char> ws(hxm_op_workspace_bytes(n, E, rx.v.size(), d, d));
  throw_status(hxm_ess(HXM_F32, dx.p, n, d, v.p, idx.p, E, rx.v.size(), dout.p, ws.p, ws.n,
                       nullptr),
               "ess");
  download(out.data(), dout);
  return out;
}

// moekit::estmm (es_ops.hpp:52-53).
inline moekit::Tensor3D estmm(const moekit::Matrix2D& x1, const moekit::Matrix2D& x2,
                              const moekit::ReIndex& rx) {
  if (x1.rows() != x2.rows()) throw moekit::ShapeError("estmm: x1 and x2 token counts differ");
  if (x1.rows() != rx.n_tokens) throw moekit::ShapeError("estmm: token count does not match re-index vector");
  const int64_t E = rx.num_experts(), n = x1.rows(), d1 = x1.cols(), d2 = x2.cols();
  moekit::Tensor3D out(E, d1, d2);
  DevBuf<float> a(x1.size()), b(x2.size()), dout(out.size());
  DevBuf<int64_t> v(rx.v.size()), idx(rx.idx.size());
  upload(a, x1.data());
  upload(b, x2.data());
  cudaMemcpy(v.p, rx.v.data(), rx.v.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(idx.p, rx.idx.data(), rx.idx.size() * 8, cudaMemcpyHostToDevice);
  DevBuf<char> ws(hxm_op_workspace_bytes(n, E, rx.v.size(), d1, d2));
  throw_status(hxm_estmm(HXM_F32, a.p, b.p, n, d1, d2, v.p, idx.p, E, rx.v.size(), dout.p,
                         ws.p, ws.n, nullptr),
               "estmm");
  download(out.data(), dout);
  return out;
}

}  // namespace hexamoe
