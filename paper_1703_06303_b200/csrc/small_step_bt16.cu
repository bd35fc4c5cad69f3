// small_step_bt16.cu -- instantiation of the K3 small-step kernel for eigen block width <= 16.
#include "small_step.cuh"

namespace wlr {
template cudaError_t launch_ss<16>(const SmallArgs&, int, cudaStream_t);
template int ss_max_clusters<16>(int, size_t);
}  // namespace wlr
