// dropin_test.cpp -- TEST INFRASTRUCTURE: the reference's own C++ types and
// known-answer tests driven through include/hexamoe_moekit.hpp (the drop-in
// shim over the C ABI), against the reference functions themselves.  Built by
// oracle/Makefile (needs the reference headers), run on the GPU by
// tests/test_gpu_parity.py::test_cpp_dropin.
//
// Covers every signature of SURVEY.md §8(b): build_reindex,
// build_reindex_all, esmm (both forms, write + accumulate), ess, estmm, esfk,
// moe_forward, moe_backward (device stash and reference stash) -- in fp32
// (rtol 1e-4) and on the bf16 tcgen05 path (rtol 2e-2, the reference fed the
// same bf16-rounded operands), OpStats, check_reindex and the exception types.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "moekit/es_ops.hpp"
#include "moekit/moe_layer.hpp"
#include "moekit/random.hpp"
#include "moekit/routing.hpp"
#include "hexamoe_moekit.hpp"

using namespace moekit;

static int fails = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);      \
      ++fails;                                                     \
    }                                                              \
  } while (0)

template <class F>
static bool throws_shape(F f) {
  try {
    f();
  } catch (const ShapeError&) {
    return true;
  } catch (...) {
  }
  return false;
}
template <class F>
static bool throws_invalid(F f) {
  try {
    f();
  } catch (const ShapeError&) {
    return false;
  } catch (const std::invalid_argument&) {
    return true;
  } catch (...) {
  }
  return false;
}

static double err(double d, double m) { return d / (1.0 + m); }
static double serr(const Matrix2D& a, const Matrix2D& b) { return err(max_abs_diff(a, b), max_abs(b)); }
static double serr(const Tensor3D& a, const Tensor3D& b) { return err(max_abs_diff(a, b), max_abs(b)); }

static void round_bf16(std::vector<double>& v) {
  for (double& x : v) x = hexamoe::bf16_round(x);
}

static bool same_stats(const OpStats& a, const OpStats& b) {
  return a.macs == b.macs && a.adds == b.adds && a.padding_slots == b.padding_slots;
}

static void operator_kats() {
  // test_routing.cpp:11-16
  ReIndex rx = hexamoe::build_reindex({0, 1, 0, 0, 1}, 2, 2);
  CHECK((rx.idx == std::vector<int64_t>{0, 4, 6}));
  CHECK((rx.v == std::vector<int64_t>{0, 2, 3, -1, 1, 4}));
  CHECK(throws_invalid([] { hexamoe::build_reindex({0, 3}, 2, 2); }));
  CHECK(throws_invalid([] { hexamoe::build_reindex({0, 1}, 2, 0); }));
  // test_es_ops.cpp:42-50 (fp32 and bf16: small integers are exact)
  for (hxm_dtype dt : {HXM_F32, HXM_BF16}) {
    const hexamoe::DeviceOptions dev{dt};
    Matrix2D x(2, 2, {1, 2, 3, 4});
    Tensor3D w(2, 2, 1, {1, 1, 2, 0});
    Matrix2D b(2, 1, {0, 1});
    Matrix2D y = hexamoe::esmm(x, w, &b, hexamoe::build_reindex({1, 0}, 2, 2), {}, dev);
    CHECK(y.at(0, 0) == 3.0 && y.at(1, 0) == 7.0);
    // test_es_ops.cpp:107-115 and 117-123
    Matrix2D s = hexamoe::ess(Matrix2D(3, 2, {1, 1, 2, 2, 4, 8}),
                              hexamoe::build_reindex({0, 1, 0}, 2, 2), {}, dev);
    CHECK(s.at(0, 0) == 5 && s.at(0, 1) == 9 && s.at(1, 0) == 2 && s.at(1, 1) == 2);
    Tensor3D t = hexamoe::estmm(Matrix2D(2, 1, {2, 3}), Matrix2D(2, 1, {5, 7}),
                                hexamoe::build_reindex({0, 1}, 2, 2), {}, dev);
    CHECK(t.at(0, 0, 0) == 10 && t.at(1, 0, 0) == 21);
  }
  // shape errors keep the reference's exception type (test_es_ops.cpp:289-298)
  CHECK(throws_shape([] {
    hexamoe::esmm(Matrix2D(2, 3), Tensor3D(2, 4, 2), nullptr, hexamoe::build_reindex({0, 1}, 2, 2));
  }));
  // check_reindex comes first (es_ops.cpp:12-17, 143): a malformed index is a
  // ShapeError even when every other argument is also wrong
  ReIndex bad;
  bad.idx = {0, 3};
  bad.v = {0, 1};
  bad.blk = 2;
  bad.n_tokens = 2;
  CHECK(throws_shape([&] { hexamoe::esmm(Matrix2D(5, 3), Tensor3D(7, 4, 2), nullptr, bad); }));
  CHECK(throws_shape([&] { hexamoe::ess(Matrix2D(2, 2), bad); }));
  CHECK(throws_shape([&] { hexamoe::estmm(Matrix2D(2, 2), Matrix2D(2, 2), bad); }));
  CHECK(throws_shape([&] { hexamoe::esfk(Matrix2D(2, 2), Matrix2D(2, 2), Tensor3D(1, 2, 2), bad); }));
  // accumulate without a destination: std::invalid_argument (es_ops.cpp:156-161)
  CHECK(throws_invalid([] {
    hexamoe::esmm(Matrix2D(2, 2), Tensor3D(2, 2, 2), nullptr, hexamoe::build_reindex({0, 1}, 2, 2),
                  EsOutputMode::kAccumulate, nullptr);
  }));
}

static double random_operators(hxm_dtype dt, int iters) {
  Rng rng(11 + dt);
  double worst = 0.0;
  const hexamoe::DeviceOptions dev{dt};
  for (int it = 0; it < iters; ++it) {
    // bf16 iterations use GEMM-friendly widths so the tcgen05 kernels run
    const bool tc = dt == HXM_BF16;
    const size_t n = 1 + rng.below(tc ? 600 : 64), E = 1 + rng.below(8), blk = 2 + rng.below(7);
    const size_t d1 = tc ? 64 * (1 + rng.below(3)) : 1 + rng.below(32);
    const size_t d2 = tc ? 64 * (1 + rng.below(3)) : 1 + rng.below(32);
    std::vector<int32_t> a(n);
    for (auto& e : a) e = static_cast<int32_t>(rng.below(E));
    Matrix2D xx = random_matrix(n, d1, rng), x2 = random_matrix(n, d2, rng);
    Tensor3D ww = random_tensor(E, d1, d2, rng), wt = random_tensor(E, d2, d1, rng);
    Matrix2D bb = random_matrix(E, d2, rng);
    if (tc) {
      round_bf16(xx.data());
      round_bf16(x2.data());
      round_bf16(ww.data());
      round_bf16(wt.data());
    }
    ReIndex want_rx = moekit::build_reindex(a, E, blk);
    ReIndex got_rx = hexamoe::build_reindex(a, E, blk, dev);
    CHECK(want_rx.v == got_rx.v && want_rx.idx == got_rx.idx);
    OpStats ws{}, gs{};
    EsOptions wopt, gopt;
    wopt.stats = &ws;
    gopt.stats = &gs;
    Matrix2D ym = moekit::esmm(xx, ww, &bb, want_rx, wopt);
    worst = std::max(worst, serr(hexamoe::esmm(xx, ww, &bb, got_rx, gopt, dev), ym));
    // accumulate mode into an existing destination (test_es_ops.cpp:60-77)
    Matrix2D acc_w = ym, acc_g = ym;
    moekit::esmm(xx, ww, nullptr, want_rx, EsOutputMode::kAccumulate, &acc_w, wopt);
    hexamoe::esmm(xx, ww, nullptr, got_rx, EsOutputMode::kAccumulate, &acc_g, gopt, dev);
    worst = std::max(worst, serr(acc_g, acc_w));
    Matrix2D ys = moekit::ess(xx, want_rx, wopt);
    worst = std::max(worst, serr(hexamoe::ess(xx, got_rx, gopt, dev), ys));
    Tensor3D yt = moekit::estmm(xx, x2, want_rx, wopt);
    worst = std::max(worst, serr(hexamoe::estmm(xx, x2, got_rx, gopt, dev), yt));
    // esfk (es_ops.cpp:210-247): all three outputs
    EsfkResult fw = moekit::esfk(xx, x2, wt, want_rx, wopt);
    EsfkResult fg = hexamoe::esfk(xx, x2, wt, got_rx, gopt, dev);
    worst = std::max(worst, serr(fg.grad_x, fw.grad_x));
    worst = std::max(worst, serr(fg.grad_b, fw.grad_b));
    worst = std::max(worst, serr(fg.grad_w, fw.grad_w));
    CHECK(same_stats(ws, gs));
  }
  return worst;
}

static void routing_all() {
  for (size_t k : {1, 2, 3}) {
    const RoutingChoice r = synthesize_routing(1000 + 7 * k, 6, k, RoutingDistribution::uniform(), 40 + k);
    for (size_t blk : {1, 3, 8}) {
      auto want = moekit::build_reindex_all(r, blk);
      auto got = hexamoe::build_reindex_all(r, blk);
      CHECK(want.size() == got.size());
      for (size_t i = 0; i < want.size() && i < got.size(); ++i)
        CHECK(want[i].v == got[i].v && want[i].idx == got[i].idx && want[i].blk == got[i].blk &&
              want[i].n_tokens == got[i].n_tokens);
    }
  }
}

static void layer_chain_rule() {
  // test_moe_layer.cpp:120-143, exact in fp32 and bf16
  for (hxm_dtype dt : {HXM_F32, HXM_BF16}) {
    const hexamoe::DeviceOptions dev{dt};
    MoeLayerParams p;
    p.w1 = Tensor3D(1, 1, 1, {3});
    p.b1 = Matrix2D(1, 1, {0});
    p.w2 = Tensor3D(1, 1, 1, {5});
    p.b2 = Matrix2D(1, 1, {0});
    p.activation = ActivationKind::kIdentity;
    const Matrix2D x(1, 1, {2});
    RoutingChoice r;
    r.n_tokens = 1;
    r.n_experts = 1;
    r.k = 1;
    r.assignments = {{0}};
    auto fw = hexamoe::moe_forward(x, p, r, 1, MoeScheme::kMemoryEfficient, {}, dev);
    CHECK(fw.y.at(0, 0) == 30.0);
    const MoeGrads g = hexamoe::moe_backward(fw.stash, p, Matrix2D(1, 1, {1}), false, {}, dev);
    CHECK(g.gx.at(0, 0) == 15.0);
    CHECK(g.gw1.at(0, 0, 0) == 10.0);
    CHECK(g.gw2.at(0, 0, 0) == 6.0);
    CHECK(g.gb1.at(0, 0) == 5.0);
    CHECK(g.gb2.at(0, 0) == 1.0);
  }
  // the layer's validation order and types (test_moe_layer.cpp:207-237)
  Rng rng(3);
  MoeLayerParams p = make_random_params(3, 4, 8, 4, ActivationKind::kGelu, rng);
  RoutingChoice r = synthesize_routing(5, 3, 2, RoutingDistribution::uniform(), 1);
  CHECK(throws_shape([&] { hexamoe::moe_forward(Matrix2D(4, 4), p, r, 8, MoeScheme::kMemoryEfficient); }));
  CHECK(throws_shape([&] { hexamoe::moe_forward(Matrix2D(5, 3), p, r, 8, MoeScheme::kMemoryEfficient); }));
  RoutingChoice big = r;
  big.k = 4;
  CHECK(throws_shape([&] { hexamoe::moe_forward(Matrix2D(5, 4), p, big, 8, MoeScheme::kMemoryEfficient); }));
  RoutingChoice dup = r;
  dup.assignments[1] = dup.assignments[0];
  CHECK(throws_invalid([&] { hexamoe::moe_forward(Matrix2D(5, 4), p, dup, 8, MoeScheme::kMemoryEfficient); }));
}

// random layers against moekit::moe_forward / moe_backward
static double random_layers(hxm_dtype dt) {
  struct Case { size_t E, k, din, hid, dout, n; ActivationKind act; };
  const Case cases[] = {
      {8, 2, 128, 256, 128, 700, ActivationKind::kGelu},
      {4, 1, 64, 128, 192, 300, ActivationKind::kRelu},
      {16, 2, 64, 192, 64, 513, ActivationKind::kIdentity},
  };
  const hexamoe::DeviceOptions dev{dt};
  double worst = 0.0;
  Rng rng(77 + dt);
  for (const Case& c : cases) {
    MoeLayerParams p = make_random_params(c.E, c.din, c.hid, c.dout, c.act, rng);
    Matrix2D x = random_matrix(c.n, c.din, rng), gy = random_matrix(c.n, c.dout, rng);
    if (dt == HXM_BF16) {
      round_bf16(p.w1.data());
      round_bf16(p.w2.data());
      round_bf16(x.data());
      round_bf16(gy.data());
    }
    RoutingChoice r = synthesize_routing(c.n, c.E, c.k, RoutingDistribution::uniform(), c.n);
    OpStats ws{}, gs{};
    EsOptions wopt, gopt;
    wopt.stats = &ws;
    gopt.stats = &gs;
    const MoeForwardResult want = moekit::moe_forward(x, p, r, 8, MoeScheme::kMemoryEfficient, wopt);
    const MoeGrads gw = moekit::moe_backward(want.stash, p, gy, true, wopt);
    auto got = hexamoe::moe_forward(x, p, r, 8, MoeScheme::kMemoryEfficient, gopt, dev);
    worst = std::max(worst, serr(got.y, want.y));
    const MoeGrads gg = hexamoe::moe_backward(got.stash, p, gy, true, gopt, dev);
    worst = std::max({worst, serr(gg.gw1, gw.gw1), serr(gg.gb1, gw.gb1), serr(gg.gw2, gw.gw2),
                      serr(gg.gb2, gw.gb2), serr(gg.gx, gw.gx)});
    CHECK(same_stats(ws, gs));
    // the stash in the reference's type, and a reference-made stash consumed
    // by the device backward
    const ForwardStash ms = got.stash.to_moekit(p, dev);
    CHECK(ms.reindex.size() == c.k && ms.y1.size() == c.k && ms.y2.size() == c.k);
    for (size_t i = 0; i < c.k && i < ms.y1.size(); ++i) {
      worst = std::max(worst, serr(ms.y1[i], want.stash.y1[i]));
      worst = std::max(worst, serr(ms.y2[i], want.stash.y2[i]));
      CHECK(ms.reindex[i].v == want.stash.reindex[i].v);
    }
    const MoeGrads gr = hexamoe::moe_backward(want.stash, p, gy, false, {}, dev);
    worst = std::max({worst, serr(gr.gw1, gw.gw1), serr(gr.gx, gw.gx), serr(gr.gb2, gw.gb2)});
  }
  return worst;
}

int main() {
  operator_kats();
  routing_all();
  const double op32 = random_operators(HXM_F32, 50);
  const double op16 = random_operators(HXM_BF16, 12);
  CHECK(op32 <= 1e-4);
  CHECK(op16 <= 2e-2);
  layer_chain_rule();
  const double l32 = random_layers(HXM_F32);
  const double l16 = random_layers(HXM_BF16);
  CHECK(l32 <= 1e-4);
  CHECK(l16 <= 2e-2);
  // the bf16 layers above ran on the tcgen05 CTA-pair kernels
  hxm_layer_desc d{};
  d.n_tokens = 700; d.n_experts = 8; d.k = 2; d.d_in = 128; d.hidden = 256; d.d_out = 128;
  d.activation = HXM_ACT_GELU; d.dtype = HXM_BF16; d.add_b2 = 1;
  CHECK(hxm_layer_path(&d) >= 1);
  std::printf("dropin: %d failures, worst scaled error fp32 ops %.3e, bf16 ops %.3e, "
              "fp32 layer %.3e, bf16 layer %.3e (tcgen05 path %d)\n",
              fails, op32, op16, l32, l16, hxm_layer_path(&d));
  return fails ? 1 : 0;
}
