// prof.cuh -- kernel-region timing scope (see prof.cu).
#pragma once
#include <cuda_runtime.h>

namespace hxm {

enum WorkKind : int { WORK_FLOP = 0, WORK_BYTES = 1 };

void note_launch();

class ProfScope {
 public:
  // bytes: algorithmic HBM bytes of a FLOP-counted region (0 = not stated)
  ProfScope(cudaStream_t st, const char* name, double work, int kind, double bytes = 0.0);
  ~ProfScope();
  ProfScope(const ProfScope&) = delete;
  ProfScope& operator=(const ProfScope&) = delete;

 private:
  cudaStream_t st_;
  const char* name_;
  double work_;
  int kind_;
  double bytes_;
  bool active_ = false;
  void* a_ = nullptr;
  void* b_ = nullptr;
};

}  // namespace hxm
