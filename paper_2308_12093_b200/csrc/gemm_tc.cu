// gemm_tc.cu -- tcgen05 (5th-gen tensor core) GEMM for the float32 dense
// transforms X.Theta and their gradients.  Placeholder until the kernel lands:
// returns false so dense.cu falls back to the SIMT kernel.
#include "common.cuh"
#include "internal.cuh"

namespace sgnn {
bool gemm_tc_f32(sgnn_ctx, const float*, int32_t, int32_t, const float*, int32_t, int32_t, bool,
                 bool, float*, const float*) {
  return false;
}
}  // namespace sgnn
