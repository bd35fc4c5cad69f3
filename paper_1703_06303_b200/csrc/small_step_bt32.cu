// small_step_bt32.cu -- instantiation of the K3 small-step kernel for eigen block width <= 32.
#include "small_step.cuh"

namespace wlr {
template cudaError_t launch_ss<32>(const SmallArgs&, int, cudaStream_t);
template int ss_max_clusters<32>(int, size_t);
}  // namespace wlr
