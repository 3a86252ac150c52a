// mgpass_k384.cu — instantiations of the pass kernel with 384 compute threads (a separate
// translation unit so the build compiles them in parallel).
#include "mgpass_impl.cuh"

namespace svi {
template cudaError_t launch_pass_t<384, 1>(const PassParams &, cudaStream_t, const LaunchCfg &);
template cudaError_t launch_pass_t<384, 2>(const PassParams &, cudaStream_t, const LaunchCfg &);
}  // namespace svi
