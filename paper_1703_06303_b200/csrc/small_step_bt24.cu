// small_step_bt24.cu -- instantiation of the K3 small-step kernel for eigen block width <= 24.
#include "small_step.cuh"

namespace wlr {
template cudaError_t launch_ss<24>(const SmallArgs&, int, cudaStream_t);
template int ss_max_clusters<24>(int, size_t);
}  // namespace wlr
