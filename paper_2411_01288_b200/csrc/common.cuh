// common.cuh -- shared host/device plumbing for the hexamoe C ABI.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/hexamoe.h"
#include "prof.cuh"

namespace hxm {

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);
const char* last_error();

struct Err {
  hxm_status code;
  std::string msg;
};

#define HXM_TRY_CUDA(expr)                                                   \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) {                                                 \
      ::hxm::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));  \
      return HXM_ERR_CUDA;                                                   \
    }                                                                        \
  } while (0)

#define HXM_CHECK_LAUNCH()                                                   \
  do {                                                                       \
    cudaError_t _e = cudaGetLastError();                                     \
    if (_e != cudaSuccess) {                                                 \
      ::hxm::set_error(std::string("kernel launch: ") +                      \
                       cudaGetErrorString(_e));                              \
      return HXM_ERR_CUDA;                                                   \
    }                                                                        \
    ::hxm::note_launch();                                                    \
  } while (0)

#define HXM_RETURN_IF(st)                                                    \
  do {                                                                       \
    hxm_status _s = (st);                                                    \
    if (_s != HXM_OK) return _s;                                             \
  } while (0)

inline hxm_status shape_error(const std::string& m) {
  set_error(m);
  return HXM_ERR_SHAPE;
}
inline hxm_status invalid_arg(const std::string& m) {
  set_error(m);
  return HXM_ERR_INVALID_ARG;
}

int sm_count();  // cached per device
bool pdl_on();   // programmatic dependent launch (HXM_PDL=0 disables)
// Programmatic dependent launch, early trigger (build with
// -DHXM_PDL_TRIGGER=1): every layer kernel keeps all its CTAs resident, so it
// could release its dependent at once and let the next kernel's CTAs take SMs
// as this kernel's retire, running their setup under the tail.  Measured
// slower at c2 (0.3303 -> 0.3370 ms/step, profiles/r2_notes.md 11): off, the
// dependent launches at completion.
#ifndef HXM_PDL_TRIGGER
#define HXM_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_trigger() {
#if HXM_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
struct SideStream {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
// A side stream and fork/join events of its own for each (device, caller
// stream): independent callers never share events or serialise through one
// side stream.  Created on first use (thread-safe).
SideStream side_stream(cudaStream_t caller);
// Fork `side` off `main` now; the destructor joins it back (records `join`
// on the side stream and makes `main` wait), also on early error returns,
// so a stream capture never ends with an unjoined branch.
class SideBranch {
 public:
  SideBranch(cudaStream_t main, const SideStream& side) : main_(main), side_(side) {
    ok_ = cudaEventRecord(side_.fork, main_) == cudaSuccess &&
          cudaStreamWaitEvent(side_.st, side_.fork, 0) == cudaSuccess;
  }
  ~SideBranch() { join(); }
  bool ok() const { return ok_; }
  cudaError_t join() {
    if (joined_) return cudaSuccess;
    joined_ = true;
    cudaError_t e = cudaEventRecord(side_.join, side_.st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(main_, side_.join, 0);
    return e;
  }
  SideBranch(const SideBranch&) = delete;
  SideBranch& operator=(const SideBranch&) = delete;

 private:
  cudaStream_t main_;
  SideStream side_;
  bool ok_ = false, joined_ = false;
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) {
  return (a + b - 1) / b;
}
__host__ __device__ inline size_t align_up(size_t a, size_t b) {
  return (a + b - 1) / b * b;
}

// Bump allocator over a caller-provided workspace (256-byte aligned slices).
struct Arena {
  char* base;
  size_t cap;
  size_t used = 0;
  bool overflow = false;
  Arena(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <class T>
  T* take(size_t count) {
    size_t bytes = align_up(count * sizeof(T) + 1, 256);
    if (used + bytes > cap) overflow = true;
    T* p = reinterpret_cast<T*>(base ? base + used : nullptr);
    used += bytes;
    return p;
  }
};

// --------------------------------------------------------------- device --
// out[0:n] = 0 by a grid-stride loop (thread t0 of `stride`): 256-bit stores
// (STG.256) when out is 32-byte aligned, a scalar tail
__device__ __forceinline__ void zero_f32(float* out, int64_t n, int64_t t0, int64_t stride) {
  int64_t done = 0;
  if ((reinterpret_cast<uintptr_t>(out) & 31) == 0) {
    const int64_t n8 = n / 8;
    const float z = 0.f;
    for (int64_t i = t0; i < n8; i += stride)
      asm volatile("st.global.v8.f32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"l"(out + 8 * i), "f"(z)
                   : "memory");
    done = n8 * 8;
  }
  for (int64_t i = done + t0; i < n; i += stride) out[i] = 0.f;
}
__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <class T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// Activations in fp32: GELU tanh approximation and its exact derivative
// (reference core/src/tensor.cpp:39-53), ReLU with ReLU'(0) = 0
// (tensor.cpp:62-72), identity.
__device__ __forceinline__ float act_value(int act, float x) {
  if (act == HXM_ACT_RELU) return x > 0.f ? x : 0.f;
  if (act == HXM_ACT_GELU) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.f + tanhf(u));
  }
  return x;
}
__device__ __forceinline__ float act_derivative(int act, float x) {
  if (act == HXM_ACT_RELU) return x > 0.f ? 1.f : 0.f;
  if (act == HXM_ACT_GELU) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    const float t = tanhf(u);
    const float du = 0.7978845608028654f * (1.f + 3.f * 0.044715f * x * x);
    return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * du;
  }
  return 1.f;
}

// F and F' with one tanh (the same expressions as act_value / act_derivative,
// so the results are identical)
__device__ __forceinline__ void act_both(int act, float x, float& f, float& df) {
  if (act == HXM_ACT_GELU) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    const float t = tanhf(u);
    const float du = 0.7978845608028654f * (1.f + 3.f * 0.044715f * x * x);
    f = 0.5f * x * (1.f + t);
    df = 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * du;
  } else {
    f = act_value(act, x);
    df = act_derivative(act, x);
  }
}

// Row maps: padded-position p -> source row (or -1 for a padding slot).
struct MapV64 {  // reference ReIndex v (int64 token ids, -1 pads)
  const int64_t* v;
  __device__ __forceinline__ int operator()(int64_t p) const {
    return static_cast<int>(v[p]);
  }
};
struct MapSlot {  // combined k-choice index: slot s = choice*N + token
  const int32_t* v;
  int n;
  __device__ __forceinline__ int operator()(int64_t p) const {
    const int s = v[p];
    return s < 0 ? -1 : s % n;
  }
};

// Segment tile descriptor: rows [begin, end) of expert `expert` in the
// padded position space; `flags` bit0 = expert split across several tiles
// (ESTMM split-K), bit1 = expert segment is empty (zero output tile).
struct SegTile {
  int expert;
  int begin;
  int end;
  int flags;
};

}  // namespace hxm
