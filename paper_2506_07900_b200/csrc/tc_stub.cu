// Placeholder dispatch until the tcgen05 kernels land: nothing is routed to
// the tensor-core path, every call runs the CUDA-core kernels.
#include "tc_dispatch.cuh"

namespace infllm2 {
bool tc_select_supported(const infllm2_geometry&, const CallShape&, bool) { return false; }
size_t tc_select_workspace(const infllm2_geometry&, const CallShape&, int) { return 0; }
cudaError_t launch_select_tc(const infllm2_geometry&, const CallShape&, const void*, int64_t,
                             const float*, const void*, const void*, int64_t, int32_t*, double*,
                             void*, size_t, cudaStream_t) {
  return cudaErrorNotSupported;
}
bool tc_attend_supported(const infllm2_geometry&, const CallShape&) { return false; }
cudaError_t launch_attend_tc(const infllm2_geometry&, const CallShape&, const void*, int64_t,
                             const void*, const void*, int64_t, const int32_t*, void*, int, float*,
                             cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace infllm2
