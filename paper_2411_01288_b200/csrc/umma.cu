// umma.cu -- tcgen05 (5th-gen tensor core) expert-specific GEMMs, bf16 in,
// fp32 accumulate in TMEM.  (placeholder: filled in by the next milestone)
#include "kernels.cuh"

namespace hxm {

bool umma_supports_esmm(int64_t, int64_t) { return false; }
bool umma_supports_estmm(int64_t, int64_t) { return false; }
hxm_status umma_esmm(const EsmmArgs&, cudaStream_t) { return HXM_ERR_UNSUPPORTED; }
hxm_status umma_estmm(const EstmmArgs&, cudaStream_t) { return HXM_ERR_UNSUPPORTED; }

}  // namespace hxm
