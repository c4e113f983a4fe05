// kernels_tc.cu -- tcgen05 / TMEM / TMA kernels (sm_100a) of the LASP path (bf16).
#include "lasp_common.cuh"

namespace lasp {

bool tc_supported(const Plan&) { return false; }

cudaError_t launch_seg_state_tc(const Plan&, Dir, const void*, const void*, float*, cudaStream_t) {
  return cudaErrorNotSupported;
}
cudaError_t launch_core_tc(const Plan&, Dir, const SeqArgs&, cudaStream_t) { return cudaErrorNotSupported; }

}  // namespace lasp
