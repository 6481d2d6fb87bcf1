// capi.cu -- error state, device queries and the reference's seeded input
// generators (measurement inputs, host memory).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"

namespace hxm {

namespace {
thread_local std::string g_err;
}

void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (dev < 64 && cached[dev] > 0) return cached[dev];
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  if (dev < 64) cached[dev] = n;
  return n;
}

// A non-blocking side stream plus fork/join events per (device, caller
// stream), for independent work that runs beside the caller's stream
// (recorded into CUDA graphs as parallel branches under stream capture).
SideStream side_stream(cudaStream_t caller) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, SideStream> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  SideStream& s = cache[{dev, caller}];
  if (!s.st) {
    cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming);
  }
  return s;
}

bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("HXM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// moekit::Rng (reference core/include/moekit/random.hpp:13-40): the same
// std::mt19937_64 engine and value mappings, so seeds reproduce the
// reference's synthetic inputs bit for bit.
class Rng {
 public:
  explicit Rng(uint64_t seed) : e_(seed) {}
  uint64_t next_u64() { return e_(); }
  double uniform01() { return static_cast<double>(e_() >> 11) * 0x1.0p-53; }
  double gaussian() {
    double u1 = uniform01();
    const double u2 = uniform01();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
  }
  uint64_t below(uint64_t n) { return e_() % n; }

 private:
  std::mt19937_64 e_;
};

}  // namespace hxm

using namespace hxm;

extern "C" {

const char* hxm_last_error(void) { return hxm::last_error(); }
int hxm_version(void) { return 100; }
int hxm_device_sm_count(void) { return hxm::sm_count(); }

// synthesize_routing (reference routing.cpp:121-200)
hxm_status hxm_synthesize_routing(int64_t n, int64_t E, int64_t k, const char* dist,
                                  uint64_t seed, int32_t* out) {
  if (k <= 0 || E <= 0) return invalid_arg("synthesize_routing: k and E must be >= 1");
  if (k > E) return invalid_arg("synthesize_routing: k > n_experts");
  std::string d = dist ? dist : "uniform";
  int kind = 0;
  double zipf_s = 1.0;
  int64_t fixed = 0;
  if (d == "uniform") kind = 0;
  else if (d == "balanced") kind = 3;
  else if (d.rfind("zipf:", 0) == 0) { kind = 1; zipf_s = std::stod(d.substr(5)); }
  else if (d.rfind("fixed:", 0) == 0) { kind = 2; fixed = std::stoll(d.substr(6)); }
  else return invalid_arg("unknown routing distribution: " + d);
  if (kind == 2 && fixed >= E) return invalid_arg("synthesize_routing: fixed expert out of range");
  Rng rng(seed);
  std::vector<double> cdf;
  if (kind == 1) {
    cdf.resize(E);
    double acc = 0.0;
    for (int64_t e = 0; e < E; ++e) {
      acc += 1.0 / std::pow(static_cast<double>(e + 1), zipf_s);
      cdf[e] = acc;
    }
  }
  std::vector<int32_t> pool(E);
  std::vector<int32_t> picked;
  for (int64_t t = 0; t < n; ++t) {
    if (kind == 0) {
      for (int64_t e = 0; e < E; ++e) pool[e] = static_cast<int32_t>(e);
      for (int64_t i = 0; i < k; ++i) {
        const int64_t j = i + static_cast<int64_t>(rng.below(static_cast<uint64_t>(E - i)));
        std::swap(pool[i], pool[j]);
        out[i * n + t] = pool[i];
      }
    } else if (kind == 1) {
      picked.clear();
      while (static_cast<int64_t>(picked.size()) < k) {
        const double u = rng.uniform01() * cdf.back();
        auto it = std::upper_bound(cdf.begin(), cdf.end(), u);
        const int32_t e = static_cast<int32_t>(
            std::min<int64_t>(it - cdf.begin(), E - 1));
        if (std::find(picked.begin(), picked.end(), e) == picked.end()) {
          out[static_cast<int64_t>(picked.size()) * n + t] = e;
          picked.push_back(e);
        }
      }
    } else if (kind == 2) {
      for (int64_t i = 0; i < k; ++i) out[i * n + t] = static_cast<int32_t>((fixed + i) % E);
    } else {
      for (int64_t i = 0; i < k; ++i) out[i * n + t] = static_cast<int32_t>((t + i) % E);
    }
  }
  return HXM_OK;
}

// make_random_params + random_matrix (moe_layer.cpp:136-147, random.hpp:42-54)
void hxm_make_layer_inputs(uint64_t seed, int64_t E, int64_t din, int64_t hid, int64_t dout,
                           int64_t n, double scale, float* w1, float* b1, float* w2,
                           float* b2, float* x) {
  Rng rng(seed);
  auto fill = [&](float* p, int64_t count, double s) {
    for (int64_t i = 0; i < count; ++i) {
      const double v = s * rng.gaussian();
      if (p) p[i] = static_cast<float>(v);
    }
  };
  fill(w1, E * din * hid, scale);
  fill(b1, E * hid, scale);
  fill(w2, E * hid * dout, scale);
  fill(b2, E * dout, scale);
  fill(x, n * din, 1.0);
}

}  // extern "C"

// OpStats (es_ops.hpp:17-24) as the reference increments them: every tile
// visits its blk slots, counting real tokens into macs / adds and -1 pads
// into padding_slots (es_ops.cpp:53-56, 80, 97-101, 124-127); esfk runs the
// three tile lists (es_ops.cpp:226-245).
extern "C" void hxm_op_stats_add(hxm_op_kind op, int64_t real_slots, int64_t padding_slots,
                                 int64_t d1, int64_t d2, hxm_op_stats* s) {
  if (!s || real_slots < 0 || padding_slots < 0 || d1 < 0 || d2 < 0) return;
  const uint64_t r = static_cast<uint64_t>(real_slots), pad = static_cast<uint64_t>(padding_slots);
  const uint64_t a = static_cast<uint64_t>(d1), b = static_cast<uint64_t>(d2);
  switch (op) {
    case HXM_OP_ESMM:
    case HXM_OP_ESTMM:
      s->macs += r * a * b;
      s->padding_slots += pad;
      break;
    case HXM_OP_ESS:  // d1 = row width
      s->adds += r * a;
      s->padding_slots += pad;
      break;
    case HXM_OP_ESFK:  // x: N x d1, g: N x d2 -> esmm(g, w_t) + ess(g) + estmm(x, g)
      s->macs += 2 * r * a * b;
      s->adds += r * b;
      s->padding_slots += 3 * pad;
      break;
  }
}

