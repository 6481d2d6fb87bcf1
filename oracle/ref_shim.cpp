// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference moekit sources
// (/root/reference/proj/core/src/{tensor,routing,es_ops,moe_layer}.cpp),
// compiled together by oracle/Makefile into oracle/_ref/libmoekit_ref.so.
// Used (a) to pin the C restatement in oracle/moe_oracle.c bit-for-bit,
// (b) to generate golden fixtures (oracle/make_golden.py), and (c) as the
// CPU baseline / `bench.py --impl reference` arm.  Never linked by the
// product library.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "moekit/es_ops.hpp"
#include "moekit/moe_layer.hpp"
#include "moekit/random.hpp"
#include "moekit/routing.hpp"

using namespace moekit;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ShapeError*>(&e)) return 1;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 2;
  return 3;
}

Matrix2D mat(const double* p, std::size_t r, std::size_t c) {
  return Matrix2D(r, c, std::vector<double>(p, p + r * c));
}
Tensor3D ten(const double* p, std::size_t a, std::size_t b, std::size_t c) {
  return Tensor3D(a, b, c, std::vector<double>(p, p + a * b * c));
}
ReIndex rx_of(const int64_t* v, std::size_t np, const int64_t* idx,
              std::size_t E, std::size_t blk, std::size_t n) {
  ReIndex rx;
  rx.v.assign(v, v + np);
  rx.idx.assign(idx, idx + E + 1);
  rx.blk = blk;
  rx.n_tokens = n;
  return rx;
}
RoutingChoice routing_of(const int32_t* a, std::size_t k, std::size_t n,
                         std::size_t E) {
  RoutingChoice r;
  r.n_tokens = n;
  r.n_experts = E;
  r.k = k;
  for (std::size_t i = 0; i < k; ++i)
    r.assignments.emplace_back(a + i * n, a + (i + 1) * n);
  return r;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Rng stream, random.hpp:13-54
void ref_rng_u64(uint64_t seed, uint64_t* out, std::size_t count) {
  Rng rng(seed);
  for (std::size_t i = 0; i < count; ++i) out[i] = rng.next_u64();
}
void ref_rng_gaussian(uint64_t seed, double* out, std::size_t count) {
  Rng rng(seed);
  for (std::size_t i = 0; i < count; ++i) out[i] = rng.gaussian();
}

// make_random_params + random_matrix(x) from one seeded stream (the bench's
// input generator, tools/commands.cpp:174-176).
void ref_make_inputs(uint64_t seed, std::size_t E, std::size_t din,
                     std::size_t hid, std::size_t dout, std::size_t n,
                     double scale, double* w1, double* b1, double* w2,
                     double* b2, double* x) {
  Rng rng(seed);
  MoeLayerParams p = make_random_params(E, din, hid, dout, ActivationKind::kGelu,
                                        rng, scale);
  Matrix2D xm = random_matrix(n, din, rng);
  std::memcpy(w1, p.w1.data().data(), p.w1.size() * sizeof(double));
  std::memcpy(b1, p.b1.data().data(), p.b1.size() * sizeof(double));
  std::memcpy(w2, p.w2.data().data(), p.w2.size() * sizeof(double));
  std::memcpy(b2, p.b2.data().data(), p.b2.size() * sizeof(double));
  std::memcpy(x, xm.data().data(), xm.size() * sizeof(double));
}

int ref_synthesize_routing(std::size_t n, std::size_t E, std::size_t k,
                           const char* dist, uint64_t seed, int32_t* out) {
  try {
    RoutingChoice r =
        synthesize_routing(n, E, k, RoutingDistribution::parse(dist), seed);
    for (std::size_t i = 0; i < k; ++i)
      std::memcpy(out + i * n, r.assignments[i].data(), n * sizeof(int32_t));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_validate_routing(const int32_t* a, std::size_t k, std::size_t n,
                         std::size_t E) {
  try {
    routing_of(a, k, n, E).validate();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// build_reindex (routing.cpp:42-70).  Returns N' or -(status).
int64_t ref_build_reindex(const int32_t* a, std::size_t n, std::size_t E,
                          std::size_t blk, int64_t* v, int64_t* idx) {
  try {
    ReIndex rx = build_reindex(std::vector<int32_t>(a, a + n), E, blk);
    std::memcpy(v, rx.v.data(), rx.v.size() * sizeof(int64_t));
    std::memcpy(idx, rx.idx.data(), rx.idx.size() * sizeof(int64_t));
    return static_cast<int64_t>(rx.v.size());
  } catch (const std::exception& e) {
    return -fail(e);
  }
}

int ref_esmm(const double* x, std::size_t n, std::size_t d1, const double* w,
             std::size_t E, std::size_t d2, const double* bias,
             const int64_t* v, std::size_t np, const int64_t* idx,
             std::size_t blk, int mode, double* dest) {
  try {
    Matrix2D xm = mat(x, n, d1);
    Tensor3D wm = ten(w, E, d1, d2);
    Matrix2D bm;
    if (bias) bm = mat(bias, E, d2);
    ReIndex rx = rx_of(v, np, idx, E, blk, n);
    Matrix2D out = mat(dest, n, d2);
    esmm(xm, wm, bias ? &bm : nullptr, rx,
         mode ? EsOutputMode::kAccumulate : EsOutputMode::kWrite, &out);
    std::memcpy(dest, out.data().data(), out.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_ess(const double* x, std::size_t n, std::size_t d, const int64_t* v,
            std::size_t np, const int64_t* idx, std::size_t E, std::size_t blk,
            double* out) {
  try {
    Matrix2D r = ess(mat(x, n, d), rx_of(v, np, idx, E, blk, n));
    std::memcpy(out, r.data().data(), r.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_estmm(const double* x1, const double* x2, std::size_t n,
              std::size_t d1, std::size_t d2, const int64_t* v, std::size_t np,
              const int64_t* idx, std::size_t E, std::size_t blk, double* out) {
  try {
    Tensor3D r = estmm(mat(x1, n, d1), mat(x2, n, d2),
                       rx_of(v, np, idx, E, blk, n));
    std::memcpy(out, r.data().data(), r.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Full layer fwd+bwd through moe_forward / moe_backward (moe_layer.cpp:30-122).
int ref_moe_step(const double* x, std::size_t n, std::size_t din,
                 std::size_t hid, std::size_t dout, std::size_t E,
                 const double* w1, const double* b1, const double* w2,
                 const double* b2, int act, const int32_t* a, std::size_t k,
                 std::size_t blk, const double* g_y, int use_fused, double* y,
                 double* y1, double* y2, double* gw1, double* gb1, double* gw2,
                 double* gb2, double* gx) {
  try {
    MoeLayerParams p;
    p.w1 = ten(w1, E, din, hid);
    p.b1 = mat(b1, E, hid);
    p.w2 = ten(w2, E, hid, dout);
    p.b2 = mat(b2, E, dout);
    p.activation = static_cast<ActivationKind>(act);
    RoutingChoice r = routing_of(a, k, n, E);
    MoeForwardResult fw =
        moe_forward(mat(x, n, din), p, r, blk, MoeScheme::kMemoryEfficient);
    std::memcpy(y, fw.y.data().data(), fw.y.size() * sizeof(double));
    for (std::size_t i = 0; i < k; ++i) {
      if (y1) std::memcpy(y1 + i * n * hid, fw.stash.y1[i].data().data(), n * hid * sizeof(double));
      if (y2) std::memcpy(y2 + i * n * hid, fw.stash.y2[i].data().data(), n * hid * sizeof(double));
    }
    if (!g_y) return 0;
    MoeGrads g = moe_backward(fw.stash, p, mat(g_y, n, dout), use_fused != 0);
    std::memcpy(gw1, g.gw1.data().data(), g.gw1.size() * sizeof(double));
    std::memcpy(gb1, g.gb1.data().data(), g.gb1.size() * sizeof(double));
    std::memcpy(gw2, g.gw2.data().data(), g.gw2.size() * sizeof(double));
    std::memcpy(gb2, g.gb2.data().data(), g.gb2.size() * sizeof(double));
    std::memcpy(gx, g.gx.data().data(), g.gx.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// CPU baseline: times the reference's own moe_forward + moe_backward on a
// token sample of n_sample tokens of the (E, k, din, hid, dout) layer, split
// into `threads` disjoint token shards run concurrently (the reference is
// single-threaded; forward is token-parallel and per-shard parameter
// gradients are summed afterwards, as dist_sim's data-centric mode does,
// dist_sim.cpp:373-399).  Inputs come from the reference generators with
// `seed`; g_y = ones (tools/commands.cpp:220-221).  Returns wall seconds of
// the timed fwd+bwd region (input generation excluded).
double ref_time_layer(std::size_t E, std::size_t k, std::size_t din,
                      std::size_t hid, std::size_t dout, std::size_t n_sample,
                      std::size_t blk, int threads, uint64_t seed) {
  if (threads < 1) threads = 1;
  Rng rng(seed);
  MoeLayerParams p =
      make_random_params(E, din, hid, dout, ActivationKind::kGelu, rng, 0.5);
  std::vector<std::size_t> shard_n(threads, n_sample / threads);
  for (std::size_t i = 0; i < n_sample % threads; ++i) ++shard_n[i];
  std::vector<Matrix2D> xs;
  std::vector<RoutingChoice> rs;
  for (int t = 0; t < threads; ++t) {
    xs.push_back(random_matrix(shard_n[t], din, rng));
    rs.push_back(synthesize_routing(shard_n[t], E, k,
                                    RoutingDistribution::uniform(),
                                    rng.next_u64()));
  }
  std::vector<MoeGrads> grads(threads);
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      if (shard_n[t] == 0) return;
      MoeForwardResult fw =
          moe_forward(xs[t], p, rs[t], blk, MoeScheme::kMemoryEfficient);
      Matrix2D gy(shard_n[t], dout);
      for (double& v : gy.data()) v = 1.0;
      grads[t] = moe_backward(fw.stash, p, gy, false);
    });
  }
  for (auto& th : pool) th.join();
  // cross-shard gradient reduction (part of the step)
  for (int t = 1; t < threads; ++t) {
    if (shard_n[t] == 0) continue;
    add_inplace(grads[0].gw1, grads[t].gw1);
    add_inplace(grads[0].gb1, grads[t].gb1);
    add_inplace(grads[0].gw2, grads[t].gw2);
    add_inplace(grads[0].gb2, grads[t].gb2);
  }
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
