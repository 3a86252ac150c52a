// tiled.cu — dispatch of the TMA-bulk tiled gate kernel (tiled_impl.cuh) by target dimension.
#include "sv_internal.h"

namespace svi {

cudaError_t launch_tiled_dim2(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);
cudaError_t launch_tiled_dim3(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);
cudaError_t launch_tiled_dim4(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);
cudaError_t launch_tiled_dim5(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);
cudaError_t launch_tiled_dim6(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);
cudaError_t launch_tiled_dim8(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);
cudaError_t launch_tiled_dim9(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);
cudaError_t launch_tiled_dim10(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);
cudaError_t launch_tiled_dim12(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);
cudaError_t launch_tiled_dim15(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);
cudaError_t launch_tiled_dim16(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);
cudaError_t launch_tiled_dim0(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled);

cudaError_t launch_tiled(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg,
                         uint64_t *launches, bool *handled) {
    *handled = false;
    cudaError_t e;
    switch (g.d) {
        case 2: e = launch_tiled_dim2(g, psi, st, cfg, handled); break;
        case 3: e = launch_tiled_dim3(g, psi, st, cfg, handled); break;
        case 4: e = launch_tiled_dim4(g, psi, st, cfg, handled); break;
        case 5: e = launch_tiled_dim5(g, psi, st, cfg, handled); break;
        case 6: e = launch_tiled_dim6(g, psi, st, cfg, handled); break;
        case 8: e = launch_tiled_dim8(g, psi, st, cfg, handled); break;
        case 9: e = launch_tiled_dim9(g, psi, st, cfg, handled); break;
        case 10: e = launch_tiled_dim10(g, psi, st, cfg, handled); break;
        case 12: e = launch_tiled_dim12(g, psi, st, cfg, handled); break;
        case 15: e = launch_tiled_dim15(g, psi, st, cfg, handled); break;
        case 16: e = launch_tiled_dim16(g, psi, st, cfg, handled); break;
        default: e = launch_tiled_dim0(g, psi, st, cfg, handled); break;
    }
    if (*handled && e == cudaSuccess && launches) ++*launches;
    return e;
}

}  // namespace svi
