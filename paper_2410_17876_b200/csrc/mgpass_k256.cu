// mgpass_k256.cu — instantiations of the pass kernel with 256 compute threads (a separate
// translation unit so the build compiles them in parallel).
#include "mgpass_impl.cuh"

namespace svi {
template cudaError_t launch_pass_t<256, 1>(const PassParams &, cudaStream_t, const LaunchCfg &);
template cudaError_t launch_pass_t<256, 2>(const PassParams &, cudaStream_t, const LaunchCfg &);
}  // namespace svi
