// small_step_bt4.cu -- instantiation of the K3 small-step kernel for eigen block width <= 4.
#include "small_step.cuh"

namespace wlr {
template cudaError_t launch_ss<4>(const SmallArgs&, int, cudaStream_t);
template int ss_max_clusters<4>(int, size_t);
}  // namespace wlr
