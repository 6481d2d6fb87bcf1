// prof.cu -- live kernel timing for bench.py's roofline and launch counting.
//
// When enabled, each kernel region (ProfScope) records a CUDA event pair on
// the stream it launches on, so durations are measured inside the timed
// region of the benchmark, not under a profiler.  Every kernel launch of the
// library bumps a counter (bench.py's gpu_launches).
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "prof.cuh"

namespace hxm {

namespace {
struct Rec {
  std::string name;
  cudaEvent_t a, b;
  double work;
  int kind;
  double bytes;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
std::atomic<uint64_t> g_launches{0};

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Inside a CUDA-graph capture a plain record only adds a dependency; an
// External record becomes an event-record node that timestamps every replay.
static void record(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
  else
    cudaEventRecord(e, st);
}

ProfScope::ProfScope(cudaStream_t st, const char* name, double work, int kind, double bytes)
    : st_(st), name_(name), work_(work), kind_(kind), bytes_(bytes) {
  std::lock_guard<std::mutex> l(g_mu);
  if (!g_on) return;
  active_ = true;
  a_ = get_event();
  b_ = get_event();
  record(static_cast<cudaEvent_t>(a_), st_);
}

ProfScope::~ProfScope() {
  if (!active_) return;
  std::lock_guard<std::mutex> l(g_mu);
  record(static_cast<cudaEvent_t>(b_), st_);
  g_recs.push_back(Rec{name_, static_cast<cudaEvent_t>(a_), static_cast<cudaEvent_t>(b_),
                       work_, kind_, bytes_});
}

}  // namespace hxm

using namespace hxm;

extern "C" {

void hxm_profile_enable(int on) {
  std::lock_guard<std::mutex> l(g_mu);
  g_on = on != 0;
}

void hxm_profile_reset(void) {
  std::lock_guard<std::mutex> l(g_mu);
  for (auto& r : g_recs) {
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
}

int hxm_profile_read(int max, char* names, int name_len, double* total_ms, int64_t* launches,
                     double* work, int32_t* kind) {
  return hxm_profile_read2(max, names, name_len, total_ms, launches, work, kind, nullptr);
}

int hxm_profile_read2(int max, char* names, int name_len, double* total_ms, int64_t* launches,
                      double* work, int32_t* kind, double* bytes) {
  std::lock_guard<std::mutex> l(g_mu);
  struct Agg {
    double ms = 0, work = 0, bytes = 0;
    int64_t n = 0;
    int kind = 0;
  };
  std::map<std::string, Agg> agg;
  std::vector<std::string> order;
  for (auto& r : g_recs) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess ||
        cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) {
      cudaGetLastError();  // an unrecorded region: skip it, keep the rest
      continue;
    }
    if (!agg.count(r.name)) order.push_back(r.name);
    Agg& a = agg[r.name];
    a.ms += ms;
    a.work += r.work;
    a.bytes += r.bytes;
    a.n += 1;
    a.kind = r.kind;
  }
  int i = 0;
  for (auto& nm : order) {
    if (i >= max) break;
    const Agg& a = agg[nm];
    std::snprintf(names + static_cast<size_t>(i) * name_len, name_len, "%s", nm.c_str());
    total_ms[i] = a.ms;
    launches[i] = a.n;
    work[i] = a.work;
    kind[i] = a.kind;
    if (bytes) bytes[i] = a.bytes;
    ++i;
  }
  return i;
}

uint64_t hxm_launch_count(void) { return g_launches.load(); }

}  // extern "C"
