// small_step_bt12.cu -- instantiation of the K3 small-step kernel for eigen block width <= 12.
#include "small_step.cuh"

namespace wlr {
template cudaError_t launch_ss<12>(const SmallArgs&, int, cudaStream_t);
template int ss_max_clusters<12>(int, size_t);
}  // namespace wlr
