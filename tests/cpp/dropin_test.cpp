// dropin_test.cpp -- TEST INFRASTRUCTURE: the reference's own C++ types and
// known-answer tests driven through include/hexamoe_moekit.hpp (the drop-in
// shim over the C ABI).  Built by oracle/Makefile (needs the reference
// headers), run on the GPU by tests/test_gpu_parity.py::test_cpp_dropin.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "moekit/es_ops.hpp"
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

int main() {
  // test_routing.cpp:11-16
  ReIndex rx = hexamoe::build_reindex({0, 1, 0, 0, 1}, 2, 2);
  CHECK((rx.idx == std::vector<int64_t>{0, 4, 6}));
  CHECK((rx.v == std::vector<int64_t>{0, 2, 3, -1, 1, 4}));
  try {
    hexamoe::build_reindex({0, 3}, 2, 2);
    CHECK(false);
  } catch (const std::invalid_argument&) {
  }
  // test_es_ops.cpp:42-50
  Matrix2D x(2, 2, {1, 2, 3, 4});
  Tensor3D w(2, 2, 1, {1, 1, 2, 0});
  Matrix2D b(2, 1, {0, 1});
  Matrix2D y = hexamoe::esmm(x, w, &b, hexamoe::build_reindex({1, 0}, 2, 2));
  CHECK(y.at(0, 0) == 3.0 && y.at(1, 0) == 7.0);
  // test_es_ops.cpp:107-115 and 117-123
  Matrix2D s = hexamoe::ess(Matrix2D(3, 2, {1, 1, 2, 2, 4, 8}), hexamoe::build_reindex({0, 1, 0}, 2, 2));
  CHECK(s.at(0, 0) == 5 && s.at(0, 1) == 9 && s.at(1, 0) == 2 && s.at(1, 1) == 2);
  Tensor3D t = hexamoe::estmm(Matrix2D(2, 1, {2, 3}), Matrix2D(2, 1, {5, 7}),
                              hexamoe::build_reindex({0, 1}, 2, 2));
  CHECK(t.at(0, 0, 0) == 10 && t.at(1, 0, 0) == 21);
  // shape errors keep the reference's exception type (test_es_ops.cpp:289-298)
  try {
    hexamoe::esmm(Matrix2D(2, 3), Tensor3D(2, 4, 2), nullptr, hexamoe::build_reindex({0, 1}, 2, 2));
    CHECK(false);
  } catch (const ShapeError&) {
  }
  // random instances against the reference operators themselves
  Rng rng(11);
  double worst = 0.0;
  for (int it = 0; it < 50; ++it) {
    const size_t n = 1 + rng.below(64), E = 1 + rng.below(8), blk = 2 + rng.below(7);
    const size_t d1 = 1 + rng.below(32), d2 = 1 + rng.below(32);
    std::vector<int32_t> a(n);
    for (auto& e : a) e = static_cast<int32_t>(rng.below(E));
    Matrix2D xx = random_matrix(n, d1, rng), x2 = random_matrix(n, d2, rng);
    Tensor3D ww = random_tensor(E, d1, d2, rng);
    Matrix2D bb = random_matrix(E, d2, rng);
    ReIndex want_rx = moekit::build_reindex(a, E, blk);
    ReIndex got_rx = hexamoe::build_reindex(a, E, blk);
    CHECK(want_rx.v == got_rx.v && want_rx.idx == got_rx.idx);
    auto err = [](double d, double m) { return d / (1.0 + m); };
    Matrix2D ym = moekit::esmm(xx, ww, &bb, want_rx);
    worst = std::max(worst, err(max_abs_diff(hexamoe::esmm(xx, ww, &bb, got_rx), ym), max_abs(ym)));
    Matrix2D ys = moekit::ess(xx, want_rx);
    worst = std::max(worst, err(max_abs_diff(hexamoe::ess(xx, got_rx), ys), max_abs(ys)));
    Tensor3D yt = moekit::estmm(xx, x2, want_rx);
    worst = std::max(worst, err(max_abs_diff(hexamoe::estmm(xx, x2, got_rx), yt), max_abs(yt)));
  }
  CHECK(worst <= 1e-4);
  std::printf("dropin: %d failures, worst scaled error %.3e\n", fails, worst);
  return fails ? 1 : 0;
}
