// hbuild_dense_tc.cu -- tcgen05 tensor-core H builder (placeholder until the
// kernel lands; tc_supported() == false routes every shape to the FMA path).
#include "common.cuh"

namespace elm {

bool tc_supported(const elmrnn*) { return false; }
cudaError_t tc_prepare(elmrnn*) { return cudaErrorNotSupported; }
cudaError_t launch_dense_tc(elmrnn*, const float*, int64_t, int64_t, float*, int64_t) { return cudaErrorNotSupported; }

}  // namespace elm
