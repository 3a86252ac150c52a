// peer.cu — fused gate + exchange over peer memory for sharded states.
//
// A gate whose target is the sharded qubit j pairs rank r with r ^ 2^j: the class of
// PAPER.md:198-222 has member 0 on the rank whose digit j is 0 ("lo") and member 1 on the
// other ("hi"), at the same local index.  Instead of sending the whole slice to the partner,
// staging it and combining (the NCCL path), each rank of the pair reads and writes BOTH
// slices in place through peer pointers (CUDA IPC mappings over NVLink, or the other slices
// of a loopback handle on one device): rank lo updates the classes of local indices
// [0, L/2), rank hi those of [L/2, L), so every class is updated by exactly one thread —
//     (lo_i, hi_i) <- (u00 lo_i + u01 hi_i, u10 lo_i + u11 hi_i)
// on the local indices whose local control digits match.  No staging buffer,
// no combine pass: HBM traffic per rank is its slice once in, once out; NVLink carries L/2
// amplitudes each way per rank (its remote reads) plus the partner's remote writes.
//
// Qubit remapping (shard.cpp rule vi) is the same pattern without arithmetic: the runs of
// digit k = 1 - beta of rank r trade places with the runs of digit k = beta of the partner,
// element by element, each element pair swapped by one thread of one rank.
//
// Synchronisation is the caller's: both ranks' earlier kernels must be complete before the
// launch and both launches complete before either rank touches its slice again (shard.cpp:
// stream synchronise + host barrier on each side).  The kernels never wait on another rank.
#include <cuda_runtime.h>

#include "shard.h"

namespace svi {

namespace {

constexpr int kPeerThreads = 256;
constexpr int kPeerUnroll = 4;     // independent 16-byte loads in flight per thread (peer latency ~2 us)

template <typename V>
__device__ __forceinline__ bool ctrl_ok(const CombineCtrl &cc, uint64_t i) {
    bool ok = true;
    for (int c = 0; c < cc.nctrl; ++c) {
        uint64_t r, r2;
        const uint64_t q = fastdiv64(i, cc.b[c], cc.mb[c], r);
        fastdiv64(q, cc.d[c], cc.md[c], r2);
        ok = ok && (r2 == cc.v[c]);
    }
    return ok;
}

template <typename V>
__global__ void __launch_bounds__(kPeerThreads) k_pair_update(V *lo, V *hi, uint64_t first, uint64_t n, V u00,
                                                              V u01, V u10, V u11,
                                                              const __grid_constant__ CombineCtrl cc) {
    const uint64_t step = (uint64_t)gridDim.x * kPeerThreads * kPeerUnroll;
    for (uint64_t k0 = (uint64_t)blockIdx.x * kPeerThreads * kPeerUnroll + threadIdx.x; k0 < n; k0 += step) {
        V x0[kPeerUnroll], x1[kPeerUnroll];
        bool ok[kPeerUnroll];
#pragma unroll
        for (int u = 0; u < kPeerUnroll; ++u) {
            const uint64_t k = k0 + (uint64_t)u * kPeerThreads;
            ok[u] = k < n && (cc.nctrl == 0 || ctrl_ok<V>(cc, first + k));
            if (ok[u]) {
                x0[u] = lo[first + k];
                x1[u] = hi[first + k];
            }
        }
#pragma unroll
        for (int u = 0; u < kPeerUnroll; ++u) {
            if (!ok[u]) continue;
            const uint64_t i = first + k0 + (uint64_t)u * kPeerThreads;
            V y0 = cz<V>(), y1 = cz<V>();
            cfma(y0, u00, x0[u]);
            cfma(y0, u01, x1[u]);
            cfma(y1, u10, x0[u]);
            cfma(y1, u11, x1[u]);
            lo[i] = y0;
            hi[i] = y1;
        }
    }
}

// element e of the swap space [first, first + n) of L/2 elements: run m = e / b, offset o = e mod b;
// a and c point at digit value (1 - beta) and beta of the first run pair, runs repeat every 2b.
template <typename V>
__global__ void __launch_bounds__(kPeerThreads) k_pair_swap(V *a, V *c, uint64_t b, uint64_t mb, uint64_t first,
                                                            uint64_t n) {
    const uint64_t step = (uint64_t)gridDim.x * kPeerThreads * kPeerUnroll;
    for (uint64_t k0 = (uint64_t)blockIdx.x * kPeerThreads * kPeerUnroll + threadIdx.x; k0 < n; k0 += step) {
        V xa[kPeerUnroll], xc[kPeerUnroll];
        uint64_t off[kPeerUnroll];
#pragma unroll
        for (int u = 0; u < kPeerUnroll; ++u) {
            const uint64_t k = k0 + (uint64_t)u * kPeerThreads;
            off[u] = 0;
            if (k < n) {
                uint64_t o;
                const uint64_t m = fastdiv64(first + k, b, mb, o);
                off[u] = 2 * b * m + o;
                xa[u] = a[off[u]];
                xc[u] = c[off[u]];
            }
        }
#pragma unroll
        for (int u = 0; u < kPeerUnroll; ++u) {
            if (k0 + (uint64_t)u * kPeerThreads >= n) continue;
            a[off[u]] = xc[u];
            c[off[u]] = xa[u];
        }
    }
}

unsigned peer_grid(uint64_t n, int num_sms) {
    const uint64_t want = (n + kPeerThreads * kPeerUnroll - 1) / (kPeerThreads * kPeerUnroll);
    const uint64_t cap = (uint64_t)num_sms * 8;       // 8 CTAs of 256 threads per SM
    return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

}  // namespace

cudaError_t launch_pair_update(double2 *lo, double2 *hi, uint64_t first, uint64_t n, const double2 u[4],
                               const CombineCtrl &cc, cudaStream_t st, int num_sms, uint64_t *launches, bool c64) {
    if (n == 0) return cudaSuccess;
    const unsigned g = peer_grid(n, num_sms);
    if (c64)
        k_pair_update<float2><<<g, kPeerThreads, 0, st>>>(reinterpret_cast<float2 *>(lo),
                                                          reinterpret_cast<float2 *>(hi), first, n, to_v<float2>(u[0]),
                                                          to_v<float2>(u[1]), to_v<float2>(u[2]), to_v<float2>(u[3]), cc);
    else
        k_pair_update<double2><<<g, kPeerThreads, 0, st>>>(lo, hi, first, n, u[0], u[1], u[2], u[3], cc);
    if (launches) ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_pair_swap(double2 *a, double2 *c, uint64_t b, uint64_t first, uint64_t n, cudaStream_t st,
                             int num_sms, uint64_t *launches, bool c64) {
    if (n == 0) return cudaSuccess;
    const unsigned g = peer_grid(n, num_sms);
    const uint64_t mb = make_fastdiv64(b).m;
    if (c64)
        k_pair_swap<float2><<<g, kPeerThreads, 0, st>>>(reinterpret_cast<float2 *>(a), reinterpret_cast<float2 *>(c),
                                                        b, mb, first, n);
    else
        k_pair_swap<double2><<<g, kPeerThreads, 0, st>>>(a, c, b, mb, first, n);
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace svi
