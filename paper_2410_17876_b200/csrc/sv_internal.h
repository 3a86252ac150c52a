// sv_internal.h — types shared by the host planner (plan.cpp, sv_api.cpp) and the sm_100a
// kernels (kernels.cu).  Product code; never includes or links anything from oracle/.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace svi {

constexpr int kMaxDim = 16;     // largest (fused) target dimension a kernel accepts
constexpr int kMaxRem = 32;     // removed-digit runs (target + pinned controls), merged
constexpr int kMaxInner = 8;    // predicated (inner) controls in the tiled kernel

// ---------------------------------------------------------------------------------------
// Invariant-divisor 64-bit division (no hardware div in the inner loop).
// m = floor(2^64 / d) + 1 for d >= 2 gives q_est = umulhi(x, m) in {q, q+1} for every
// x < 2^63; one signed-remainder test fixes it.  d == 1 is encoded as m == 0.
// ---------------------------------------------------------------------------------------
struct FastDiv64 {
    uint64_t d;
    uint64_t m;
};

inline FastDiv64 make_fastdiv64(uint64_t d) {
    FastDiv64 f;
    f.d = d;
    f.m = (d <= 1) ? 0 : (uint64_t)(((unsigned __int128)1 << 64) / d) + 1;
    return f;
}

__host__ __device__ __forceinline__ uint64_t umulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// q = x / f.d, r = x % f.d
__host__ __device__ __forceinline__ uint64_t fastdiv64(uint64_t x, uint64_t d, uint64_t m,
                                                      uint64_t &r) {
    if (m == 0) { r = 0; return x; }
    uint64_t q = umulhi64(x, m);
    uint64_t rr = x - q * d;
    if ((int64_t)rr < 0) { --q; rr += d; }
    r = rr;
    return q;
}

// 32-bit flavour for in-tile arithmetic (x < 2^31).
struct FastDiv32 {
    uint32_t d;
    uint32_t m;
};
inline FastDiv32 make_fastdiv32(uint32_t d) {
    FastDiv32 f;
    f.d = d;
    f.m = (d <= 1) ? 0 : (uint32_t)((((uint64_t)1) << 32) / d) + 1;
    return f;
}
__host__ __device__ __forceinline__ uint32_t fastdiv32(uint32_t x, uint32_t d, uint32_t m,
                                                      uint32_t &r) {
    if (m == 0) { r = 0; return x; }
#ifdef __CUDA_ARCH__
    uint32_t q = __umulhi(x, m);
#else
    uint32_t q = (uint32_t)(((uint64_t)x * m) >> 32);
#endif
    uint32_t rr = x - q * d;
    if ((int32_t)rr < 0) { --q; rr += d; }
    r = rr;
    return q;
}

// ---------------------------------------------------------------------------------------
// One removed-digit run of the fibre decomposer.  Removing the target digit (pin 0) and
// every pinned control digit (pin v) from the index leaves the "compressed" class id
// f in [0, F); re-inserting them in ascending stride order rebuilds the class
// representative:  base <- (base / b) * (b*d) + pin*b + base % b.
// Consecutive removed positions are merged into one run (dims multiply, pins combine).
// ---------------------------------------------------------------------------------------
struct RemovedRun {
    uint64_t b;      // global stride of the run's lowest digit
    uint64_t bd;     // b * (product of the run's dims)
    uint64_t pinb;   // pin * b
    uint64_t m;      // magic for division by b
};

__host__ __device__ __forceinline__ uint64_t insert_digits(uint64_t f, int nrem,
                                                          const RemovedRun *rem) {
    uint64_t base = f;
    for (int i = 0; i < nrem; ++i) {
        uint64_t r;
        uint64_t q = fastdiv64(base, rem[i].b, rem[i].m, r);
        base = q * rem[i].bd + rem[i].pinb + r;
    }
    return base;
}

enum GateKind : int32_t { kGeneral = 0, kMonomial = 1 };

// One-time launch configuration of a kernel (dynamic shared-memory attribute, resident CTAs per
// SM), per device: cudaFuncSetAttribute applies to the current device only.
struct LaunchAttr {
    static constexpr int kDevices = 64;
    size_t configured[kDevices] = {};
    size_t occ_for[kDevices] = {};
    int occ[kDevices] = {};
};
inline int current_device_slot() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
    return dev % LaunchAttr::kDevices;
}

// complex element types: V = double2 (complex128, SV_C128) or float2 (complex64, SV_C64);
// the arithmetic is done in V's precision (the paper fixes none; R11).
template <typename V> struct RealOf;
template <> struct RealOf<double2> { using type = double; };
template <> struct RealOf<float2> { using type = float; };

__host__ __device__ __forceinline__ double2 mkv(double x, double y, const double2 *) { return make_double2(x, y); }
__host__ __device__ __forceinline__ float2 mkv(double x, double y, const float2 *) {
    return make_float2((float)x, (float)y);
}
template <typename V> __host__ __device__ __forceinline__ V to_v(double2 u) { return mkv(u.x, u.y, (const V *)nullptr); }
template <typename V> __host__ __device__ __forceinline__ V cz() { return mkv(0.0, 0.0, (const V *)nullptr); }

#ifdef __CUDACC__
// complex fused multiply-add acc += u * x and product u * x, in V's precision
__device__ __forceinline__ void cfma(double2 &acc, const double2 u, const double2 x) {
    acc.x = fma(u.x, x.x, acc.x);
    acc.x = fma(-u.y, x.y, acc.x);
    acc.y = fma(u.x, x.y, acc.y);
    acc.y = fma(u.y, x.x, acc.y);
}
__device__ __forceinline__ void cfma(float2 &acc, const float2 u, const float2 x) {
    acc.x = fmaf(u.x, x.x, acc.x);
    acc.x = fmaf(-u.y, x.y, acc.x);
    acc.y = fmaf(u.x, x.y, acc.y);
    acc.y = fmaf(u.y, x.x, acc.y);
}
__device__ __forceinline__ double2 cmul(const double2 u, const double2 x) {
    return make_double2(fma(u.x, x.x, -u.y * x.y), fma(u.x, x.y, u.y * x.x));
}
__device__ __forceinline__ float2 cmul(const float2 u, const float2 x) {
    return make_float2(fmaf(u.x, x.x, -u.y * x.y), fmaf(u.x, x.y, u.y * x.x));
}
#endif

// Kernel parameters of one gate launch, passed by value (__grid_constant__).  MD is the
// compile-time capacity of the target dimension.
template <int MD, typename V = double2>
struct GateParams {
    V *psi;
    uint64_t F;          // classes to visit (control-satisfying)
    uint64_t bk;         // target stride b_k
    int32_t d;           // target dimension (<= MD)
    int32_t kind;        // GateKind
    uint32_t active;     // monomial: members that move / scale
    int32_t nrem;
    int32_t sigma[MD];   // monomial: member j -> sigma[j]
    RemovedRun rem[kMaxRem];
    V U[MD * MD];        // general: row-major U; monomial: U[j] = coefficient of member j
};

// Host-side plan of one (possibly fused) gate on a (local) register.
struct GatePlan {
    int32_t kind;
    int32_t d;
    uint64_t bk;
    uint64_t F;
    uint64_t touched;
    uint32_t active;
    int32_t sigma[kMaxDim];
    double2 U[kMaxDim * kMaxDim];   // general: row-major; monomial: coefficients
    double uerr;
    int32_t nrem;
    RemovedRun rem[kMaxRem];
    // what the tiled planner needs: the register size and the raw control list
    uint64_t D;
    int32_t nctrl;
    uint64_t cb[64];      // control strides b_c
    uint32_t cd[64];      // control dims
    uint32_t cv[64];      // control values
};

// Device entry points (kernels.cu).
struct LaunchCfg {
    int kernel;        // 1 = direct, 2 = tiled
    int tile_elems;
    int tile_stages;
    int ctas_per_sm;
    int num_sms;
    int pass_tile;     // amplitudes per smem tile of the multi-gate pass kernel
    int pass_stages;   // smem ring stages of the pass kernel
    int pass_threads;  // threads per CTA of the pass kernel (256 or 512)
    int pass_gates;    // max gates per pass
    int pass_window;   // gates scanned ahead (commuting past skipped ones) when filling a pass
    int pass_merge;    // 1: merge same-target same-control gates across commuting ones first
    int pass_groups;   // consumer warp groups of the pass kernel (ping-pong over tiles)
    int shard_swap;    // 1: sharded mode remaps qubits instead of pairwise exchanges (shard.cpp vi)
    int pass_search;   // 1: pass planner scores in-tile sets (plan.cpp best_in_tile_set)
    int c64;           // 1: the state is complex64 (float2), else complex128 (double2)
    int pass_low;      // SV_BLOCK: qudits with stride below this many amplitudes form the low prefix
    int shard_overlap; // SMs lent to a qubit remap that overlaps the pending local run (0 = off)
    int pass_kernel;   // SV_BLOCK passes: 0 = per-gate kernel (k_gate_pass); 1 = register-blocked
                       // stages (k_gate_stage) when the pass fits them, else per-gate
    int pass_absorb;   // 1: pure permutations on member digits become load / store relabelling
};

// psi points at the state in the handle's element type (cfg.c64 / the c64 flag).
cudaError_t launch_gate(const GatePlan &p, double2 *psi, cudaStream_t st, const LaunchCfg &cfg,
                        uint64_t *launches);
cudaError_t launch_set_basis(double2 *psi, uint64_t D, uint64_t idx, cudaStream_t st,
                             uint64_t *launches, bool c64 = false);
cudaError_t launch_norm2(const double2 *psi, uint64_t D, double *partial, int nparts,
                         double *out, cudaStream_t st, uint64_t *launches, bool c64 = false);
int norm_parts();

}  // namespace svi
