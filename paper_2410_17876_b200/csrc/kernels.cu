// kernels.cu — sm_100a kernels of the block method (§2.1-2.4).
//
// Every kernel visits equivalence classes: the d amplitudes
// base + j*b_k, j < d, that differ only in the target digit.  The class representatives
// `base` are produced by the digit-insertion decomposer from a dense
// class id f in [0, F), so control-unsatisfying classes are never visited (PAPER.md:228
// brute-force filter replaced by direct enumeration).
#include <cuda_runtime.h>

#include "sv_internal.h"
#include "shard.h"

namespace svi {

namespace {

// ------------------------------------------------------------------------------------------
// Direct kernel: one class per thread iteration, grid-stride over the class ids.
// Gather x_j = psi[base + j b_k], y = U x, scatter in place.
// Coalesced when the lowest removed stride is >= 32 amplitudes (consecutive class ids map to
// consecutive addresses within each block).  V = double2 (complex128) or float2 (complex64).
// ------------------------------------------------------------------------------------------
template <int DIM, int MD, int KIND, typename V>
__global__ void __launch_bounds__(256) k_gate_direct(const __grid_constant__ GateParams<MD, V> p) {
    const int d = DIM ? DIM : p.d;
    const uint64_t bk = p.bk;
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t f = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; f < p.F; f += step) {
        V *ptr = p.psi + insert_digits(f, p.nrem, p.rem);
        V x[MD];
        if (KIND == kGeneral) {
#pragma unroll
            for (int j = 0; j < MD; ++j)
                if (DIM || j < d) x[j] = ptr[(uint64_t)j * bk];
#pragma unroll
            for (int i = 0; i < MD; ++i) {
                if (DIM || i < d) {
                    V acc = cz<V>();
#pragma unroll
                    for (int j = 0; j < MD; ++j)
                        if (DIM || j < d) cfma(acc, p.U[i * MD + j], x[j]);
                    ptr[(uint64_t)i * bk] = acc;
                }
            }
        } else {
            // monomial (§2.1 phase / §2.2 permutation): y_{sigma(j)} = c_j x_j, only
            // for the members that move or scale.
#pragma unroll
            for (int j = 0; j < MD; ++j)
                if ((DIM || j < d) && ((p.active >> j) & 1)) x[j] = ptr[(uint64_t)j * bk];
#pragma unroll
            for (int j = 0; j < MD; ++j)
                if ((DIM || j < d) && ((p.active >> j) & 1))
                    ptr[(uint64_t)p.sigma[j] * bk] = cmul(p.U[j], x[j]);
        }
    }
}

template <int MD, typename V>
void fill_params(GateParams<MD, V> &q, const GatePlan &p, V *psi) {
    q.psi = psi;
    q.F = p.F;
    q.bk = p.bk;
    q.d = p.d;
    q.kind = p.kind;
    q.active = p.active;
    q.nrem = p.nrem;
    for (int i = 0; i < MD; ++i) q.sigma[i] = (i < p.d) ? p.sigma[i] : i;
    for (int i = 0; i < p.nrem; ++i) q.rem[i] = p.rem[i];
    for (int i = 0; i < MD * MD; ++i) q.U[i] = to_v<V>(make_double2(0.0, 0.0));
    if (p.kind == kGeneral) {
        for (int i = 0; i < p.d; ++i)
            for (int j = 0; j < p.d; ++j) q.U[i * MD + j] = to_v<V>(p.U[i * p.d + j]);
    } else {
        for (int j = 0; j < p.d; ++j) q.U[j] = to_v<V>(p.U[j]);
    }
}

template <int DIM, int MD, typename V>
cudaError_t launch_direct_v(const GatePlan &p, V *psi, cudaStream_t st, const LaunchCfg &cfg) {
    GateParams<MD, V> q;
    fill_params<MD, V>(q, p, psi);
    const uint64_t want = (p.F + 255) / 256;
    const uint64_t cap = (uint64_t)cfg.num_sms * 16;
    const unsigned blocks = (unsigned)(want < cap ? want : cap);
    if (p.kind == kGeneral)
        k_gate_direct<DIM, MD, kGeneral, V><<<blocks, 256, 0, st>>>(q);
    else
        k_gate_direct<DIM, MD, kMonomial, V><<<blocks, 256, 0, st>>>(q);
    return cudaGetLastError();
}

template <int DIM, int MD>
cudaError_t launch_direct_t(const GatePlan &p, double2 *psi, cudaStream_t st, const LaunchCfg &cfg) {
    if (cfg.c64) return launch_direct_v<DIM, MD, float2>(p, reinterpret_cast<float2 *>(psi), st, cfg);
    return launch_direct_v<DIM, MD, double2>(p, psi, st, cfg);
}

// ------------------------------------------------------------------------------------------
// Norm: deterministic two-level tree (fixed partition, fixed reduction order).
// ------------------------------------------------------------------------------------------
constexpr int kNormParts = 1184;   // 8 per SM on 148 SMs
constexpr int kNormThreads = 256;

template <typename V>
__global__ void __launch_bounds__(kNormThreads) k_norm_partial(const V *__restrict__ psi,
                                                               uint64_t D, double *partial) {
    __shared__ double red[kNormThreads];
    const uint64_t chunk = (D + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = (uint64_t)blockIdx.x * chunk;
    const uint64_t hi = lo + chunk < D ? lo + chunk : D;
    double s = 0.0;                                   // fp64 accumulation for both precisions
    for (uint64_t i = lo + threadIdx.x; i < hi; i += kNormThreads) {
        const V a = psi[i];
        s = fma((double)a.x, (double)a.x, s);
        s = fma((double)a.y, (double)a.y, s);
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = kNormThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(kNormThreads) k_norm_final(const double *partial, int n, double *out) {
    __shared__ double red[kNormThreads];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += kNormThreads) s += partial[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = kNormThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}


// ------------------------------------------------------------------------------------------
// Sharded exchange combine (SURVEY.md §8(e) rule iii): the class of a sharded target qubit
// has one member on this rank and one on the partner, at the same local index.
// psi_loc <- a psi_loc + b psi_partner where the local control digits match.
// ------------------------------------------------------------------------------------------
template <typename V>
__global__ void __launch_bounds__(256) k_combine(V *__restrict__ loc,
                                                 const V *__restrict__ par, uint64_t n,
                                                 uint64_t base, V a, V b,
                                                 const __grid_constant__ CombineCtrl cc) {
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += step) {
        bool ok = true;
        for (int c = 0; c < cc.nctrl; ++c) {
            uint64_t r, r2;
            const uint64_t q = fastdiv64(base + i, cc.b[c], cc.mb[c], r);
            fastdiv64(q, cc.d[c], cc.md[c], r2);
            ok = ok && (r2 == cc.v[c]);
        }
        if (ok) {
            const V x = loc[i], z = par[i];
            V y = cz<V>();
            cfma(y, a, x);
            cfma(y, b, z);
            loc[i] = y;
        }
    }
}

template <typename V>
__global__ void k_set_one(V *psi, uint64_t idx) { psi[idx] = to_v<V>(make_double2(1.0, 0.0)); }

}  // namespace

cudaError_t launch_tiled(const GatePlan &p, double2 *psi, cudaStream_t st, const LaunchCfg &cfg,
                         uint64_t *launches, bool *handled);

cudaError_t launch_gate(const GatePlan &p, double2 *psi, cudaStream_t st, const LaunchCfg &cfg,
                        uint64_t *launches) {
    if (p.F == 0) return cudaSuccess;
    // auto policy (measured, profiles/r01/gatebench): the tiled kernel wins on every stride
    // class, except when a control has stride < 32 amplitudes -- the tiled kernel predicates
    // such controls (moving every amplitude) while the direct kernel visits only the
    // satisfying classes.
    // Fused targets with d >= 10 are FP64-issue heavy; the direct kernel (more warps per SM)
    // hides that better than the tiled kernel's compute phase (profiles/r01: d=12/16 pairs).
    // complex64: cp.async.bulk needs 16-byte aligned addresses and sizes, which 8-byte
    // amplitudes at odd offsets violate, so SV_C64 always runs the direct kernel.
    bool use_tiled = cfg.kernel == 2 && !cfg.c64;
    if (cfg.kernel == 0 && !cfg.c64) {
        use_tiled = p.d <= 9;
        for (int i = 0; i < p.nctrl; ++i)
            if (p.cb[i] < 32) use_tiled = false;
    }
    if (use_tiled) {
        bool handled = false;
        cudaError_t e = launch_tiled(p, psi, st, cfg, launches, &handled);
        if (handled || e != cudaSuccess) return e;
    }
    cudaError_t e;
    switch (p.d) {
        case 2: e = launch_direct_t<2, 2>(p, psi, st, cfg); break;
        case 3: e = launch_direct_t<3, 3>(p, psi, st, cfg); break;
        case 4: e = launch_direct_t<4, 4>(p, psi, st, cfg); break;
        case 5: e = launch_direct_t<5, 5>(p, psi, st, cfg); break;
        case 6: e = launch_direct_t<6, 6>(p, psi, st, cfg); break;
        case 8: e = launch_direct_t<8, 8>(p, psi, st, cfg); break;
        case 9: e = launch_direct_t<9, 9>(p, psi, st, cfg); break;
        case 10: e = launch_direct_t<10, 10>(p, psi, st, cfg); break;
        case 12: e = launch_direct_t<12, 12>(p, psi, st, cfg); break;
        case 15: e = launch_direct_t<15, 15>(p, psi, st, cfg); break;
        case 16: e = launch_direct_t<16, 16>(p, psi, st, cfg); break;
        default: e = launch_direct_t<0, kMaxDim>(p, psi, st, cfg); break;
    }
    if (e == cudaSuccess && launches) ++*launches;
    return e;
}

cudaError_t launch_set_basis(double2 *psi, uint64_t D, uint64_t idx, cudaStream_t st,
                             uint64_t *launches, bool c64) {
    cudaError_t e = cudaMemsetAsync(psi, 0, D * (c64 ? sizeof(float2) : sizeof(double2)), st);
    if (e != cudaSuccess) return e;
    if (c64)
        k_set_one<float2><<<1, 1, 0, st>>>(reinterpret_cast<float2 *>(psi), idx);
    else
        k_set_one<double2><<<1, 1, 0, st>>>(psi, idx);
    if (launches) ++*launches;
    return cudaGetLastError();
}

int norm_parts() { return kNormParts; }

cudaError_t launch_combine(double2 *loc, const double2 *partner, uint64_t n, uint64_t base,
                           double2 a, double2 b, const CombineCtrl &cc, cudaStream_t st,
                           uint64_t *launches, bool c64) {
    if (n == 0) return cudaSuccess;
    const uint64_t want = (n + 255) / 256;
    const unsigned blocks = (unsigned)(want < 148 * 16 ? want : 148 * 16);
    if (c64)       // complex64 slices: the same combine in fp32 (loc / partner point at float2)
        k_combine<float2><<<blocks, 256, 0, st>>>(reinterpret_cast<float2 *>(loc),
                                                  reinterpret_cast<const float2 *>(partner), n, base,
                                                  to_v<float2>(a), to_v<float2>(b), cc);
    else
        k_combine<double2><<<blocks, 256, 0, st>>>(loc, partner, n, base, a, b, cc);
    if (launches) ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_norm2(const double2 *psi, uint64_t D, double *partial, int nparts, double *out,
                         cudaStream_t st, uint64_t *launches, bool c64) {
    if (c64)
        k_norm_partial<float2><<<nparts, kNormThreads, 0, st>>>(reinterpret_cast<const float2 *>(psi), D, partial);
    else
        k_norm_partial<double2><<<nparts, kNormThreads, 0, st>>>(psi, D, partial);
    k_norm_final<<<1, kNormThreads, 0, st>>>(partial, nparts, out);
    if (launches) *launches += 2;
    return cudaGetLastError();
}

}  // namespace svi
