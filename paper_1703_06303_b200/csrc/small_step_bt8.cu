// small_step_bt8.cu -- instantiation of the K3 small-step kernel for eigen block width <= 8.
#include "small_step.cuh"

namespace wlr {
template cudaError_t launch_ss<8>(const SmallArgs&, int, cudaStream_t);
template int ss_max_clusters<8>(int, size_t);
}  // namespace wlr
