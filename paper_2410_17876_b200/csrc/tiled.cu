// tiled.cu — placeholder until the TMA-bulk tiled kernel lands.
#include "sv_internal.h"
namespace svi {
cudaError_t launch_tiled(const GatePlan &, double2 *, cudaStream_t, const LaunchCfg &, uint64_t *,
                         bool *handled) {
    *handled = false;
    return cudaSuccess;
}
}  // namespace svi
