// sparse.cu — the paper's sparse variant ("Our Method (Sparse)"; SURVEY.md
// §8 f3) on the GPU.  The state is the list of basis indices with non-zero amplitude, sorted.
// A gate visits only the classes that hold a stored index ("identify all basis
// states with non-zero amplitudes in a given class"): every stored amplitude a at index i with
// target digit v contributes U[k][v] a to the class member base + k b_t, base = i - v b_t
// (column v of U, skipping exact zeros), entries whose controls do not hold pass through
// unchanged; the contributions are radix-sorted by index, summed per index
// (the vector addition of PAPER.md:222) and amplitudes below eps are dropped.
// Our kernels do the method's arithmetic; CUB provides the sort / reduce-by-key / select
// primitives (library calls, like cuBLAS for a GEMM).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_select.cuh>

#include <cstring>
#include <string>
#include <vector>

#include "plan.h"
#include "../../include/sv.h"

namespace svi {

std::string *err_slot();
sv_status fail_msg(sv_status s, const std::string &msg);

struct alignas(16) SparseGateP {   // 16-B multiple: copied with 16-B cp.async chunks
    uint64_t bt, mbt;            // target stride (+ magic)
    uint64_t dt, mdt;            // target dim (+ magic)
    int32_t nctrl;
    uint64_t cb[kMaxRem], mcb[kMaxRem], cd[kMaxRem], mcd[kMaxRem], cv[kMaxRem];
    int32_t fan;                 // output slots per stored amplitude
    int32_t nrow[kMaxDim];       // per column v: non-zero rows
    int32_t rows[kMaxDim][kMaxDim];
    double2 coef[kMaxDim][kMaxDim];   // coef[v][r] = U[rows[v][r]][v]
    uint64_t invalid;            // key of unused slots (= D, sorts after every index)
};

namespace {

__global__ void k_sparse_expand(const uint64_t *__restrict__ keys, const double2 *__restrict__ vals, uint64_t nnz,
                                const __grid_constant__ SparseGateP g, uint64_t *okeys, double2 *ovals) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const uint64_t i = keys[e];
    const double2 a = vals[e];
    uint64_t *ok = okeys + e * (uint64_t)g.fan;
    double2 *ov = ovals + e * (uint64_t)g.fan;
    bool fire = true;
    for (int c = 0; c < g.nctrl; ++c) {                       // floor(i/b_c) mod d_c == v_c
        uint64_t r, r2;
        const uint64_t q = fastdiv64(i, g.cb[c], g.mcb[c], r);
        fastdiv64(q, g.cd[c], g.mcd[c], r2);
        fire = fire && (r2 == g.cv[c]);
    }
    if (!fire) {
        ok[0] = i;
        ov[0] = a;
        for (int s = 1; s < g.fan; ++s) { ok[s] = g.invalid; ov[s] = make_double2(0.0, 0.0); }
        return;
    }
    uint64_t r;
    const uint64_t q = fastdiv64(i, g.bt, g.mbt, r);
    uint64_t v;
    fastdiv64(q, g.dt, g.mdt, v);                            // target digit of i
    const uint64_t base = i - v * g.bt;                       // the class's member with digit 0
    for (int s = 0; s < g.fan; ++s) {
        if (s < g.nrow[v]) {
            ok[s] = base + (uint64_t)g.rows[v][s] * g.bt;
            ov[s] = cmul(g.coef[v][s], a);
        } else {
            ok[s] = g.invalid;
            ov[s] = make_double2(0.0, 0.0);
        }
    }
}

__global__ void k_sparse_flags(const uint64_t *keys, const double2 *vals, uint64_t n, uint64_t invalid,
                               double eps2, unsigned char *flags) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const double2 a = vals[e];
    flags[e] = (keys[e] != invalid) && (a.x * a.x + a.y * a.y >= eps2);
}

__global__ void k_sparse_set(uint64_t *keys, double2 *vals, uint64_t idx) {
    keys[0] = idx;
    vals[0] = make_double2(1.0, 0.0);
}

struct CSum {
    __device__ __forceinline__ double2 operator()(const double2 &a, const double2 &b) const {
        return make_double2(a.x + b.x, a.y + b.y);
    }
};

// ---------------------------------------------------------------------------------------
// Small-state path: one CTA keeps the whole sparse state in shared memory and applies a run
// of gates without leaving the kernel (the GHZ circuits of PAPER.md:485-489 hold d entries).
// Per gate: expand the class contributions into a scratch array, bitonic-sort it by index,
// sum each run of equal indices, drop |a| < eps, compact with a block scan.  Stops (and
// reports how many gates it applied) when a gate's contributions would exceed the capacity.
// ---------------------------------------------------------------------------------------
constexpr int kSmallCap = 4096;   // entries of the 1024-thread variant
constexpr int kTinyCap = 256;     // entries of the one-warp variant (GHZ-sized states)
constexpr int kSmallD = 8;        // small-path gate records: d <= 8, at most 8 controls

// compact gate record of the small-state kernel (1.7 KB instead of 6.5 KB)
struct alignas(16) SmallGateP {
    uint64_t bt, mbt, dt, mdt;
    uint64_t cb[kSmallD], mcb[kSmallD], cd[kSmallD], mcd[kSmallD], cv[kSmallD];
    uint64_t invalid;
    int32_t nctrl, fan, ok, pad;
    int32_t nrow[kSmallD];
    int32_t rows[kSmallD][kSmallD];
    double2 coef[kSmallD][kSmallD];
};

template <int NT, int CAP>
__global__ void __launch_bounds__(NT) k_sparse_small(const SmallGateP *__restrict__ gates, int ngates,
                                                                uint64_t *keys_io, double2 *vals_io,
                                                                unsigned long long *io, double eps2) {
    extern __shared__ __align__(16) unsigned char smem[];
    SmallGateP *gbuf = reinterpret_cast<SmallGateP *>(smem);        // 3-slot ring of gate records
    double2 *sv = reinterpret_cast<double2 *>(gbuf + 3);             // state values
    double2 *tv = sv + CAP;                                     // contributions
    uint64_t *sk = reinterpret_cast<uint64_t *>(tv + CAP);      // state keys
    uint64_t *tk = sk + CAP;                                    // contribution keys
    int *scan = reinterpret_cast<int *>(tk + CAP);              // CAP + 1
    __shared__ int s_n;
    const int tid = threadIdx.x;
    // asynchronous copy of gate record k (cp.async, 16 B per thread-instruction) into gbuf[slot];
    // always commits a group (possibly empty) so the wait counts stay aligned
    auto prefetch = [&](int k, int slot) {
        if (k < ngates) {
            const char *src = reinterpret_cast<const char *>(gates + k);
            char *dst = reinterpret_cast<char *>(gbuf + slot);
            for (int o = tid * 16; o < (int)sizeof(SmallGateP); o += NT * 16)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(dst + o)), "l"(src + o) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    prefetch(0, 0);
    prefetch(1, 1);
    if (tid == 0) s_n = (int)io[0];
    __syncthreads();
    int n = s_n;
    for (int i = tid; i < n; i += NT) { sk[i] = keys_io[i]; sv[i] = vals_io[i]; }
    int done = 0;
    for (; done < ngates; ++done) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // record `done` landed (done+1 may be in flight)
        __syncthreads();
        prefetch(done + 2, (done + 2) % 3);                    // two gates ahead
        const SmallGateP &g = gbuf[done % 3];
        if (!g.ok) break;                                      // needs the general path
        const int m = n * g.fan;
        if (m > CAP) break;
        int P = 1;
        while (P < m) P <<= 1;
        // expand (same rule as k_sparse_expand)
        for (int s = tid; s < P; s += NT) { tk[s] = g.invalid; tv[s] = make_double2(0.0, 0.0); }
        __syncthreads();
        for (int e = tid; e < n; e += NT) {
            const uint64_t i = sk[e];
            const double2 a = sv[e];
            uint64_t *ok = tk + e * g.fan;
            double2 *ov = tv + e * g.fan;
            bool fire = true;
            for (int c = 0; c < g.nctrl; ++c) {
                uint64_t r, r2;
                const uint64_t q = fastdiv64(i, g.cb[c], g.mcb[c], r);
                fastdiv64(q, g.cd[c], g.mcd[c], r2);
                fire = fire && (r2 == g.cv[c]);
            }
            if (!fire) { ok[0] = i; ov[0] = a; continue; }
            uint64_t r, v;
            const uint64_t q = fastdiv64(i, g.bt, g.mbt, r);
            fastdiv64(q, g.dt, g.mdt, v);
            const uint64_t base = i - v * g.bt;
            for (int s = 0; s < g.nrow[v]; ++s) {
                ok[s] = base + (uint64_t)g.rows[v][s] * g.bt;
                ov[s] = cmul(g.coef[v][s], a);
            }
        }
        __syncthreads();
        // bitonic sort of the P slots by index (unused slots carry the largest key)
        for (int k = 2; k <= P; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < P; i += NT) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const bool up = (i & k) == 0;
                        const uint64_t a = tk[i], b = tk[ixj];
                        if ((a > b) == up) {
                            tk[i] = b; tk[ixj] = a;
                            const double2 t = tv[i]; tv[i] = tv[ixj]; tv[ixj] = t;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // heads of runs of equal indices: sum the run, keep it if |sum| >= eps
        for (int i = tid; i < P; i += NT) {
            int keep = 0;
            if (tk[i] != g.invalid && (i == 0 || tk[i - 1] != tk[i])) {
                double2 s = tv[i];
                for (int j = i + 1; j < P && tk[j] == tk[i]; ++j) { s.x += tv[j].x; s.y += tv[j].y; }
                tv[i] = s;
                keep = (s.x * s.x + s.y * s.y >= eps2);
            }
            scan[i] = keep;
        }
        __syncthreads();
        // exclusive scan of the keep flags (Hillis-Steele over P <= CAP entries)
        for (int off = 1; off < P; off <<= 1) {
            int add[CAP / NT];
            for (int u = 0, i = tid; i < P; i += NT, ++u) add[u] = i >= off ? scan[i - off] : 0;
            __syncthreads();
            for (int u = 0, i = tid; i < P; i += NT, ++u) scan[i] += add[u];
            __syncthreads();
        }
        // scan now holds inclusive sums; compact the kept heads into the state arrays
        for (int i = tid; i < P; i += NT) {
            const int incl = scan[i];
            const int excl = i ? scan[i - 1] : 0;
            if (incl != excl) { sk[excl] = tk[i]; sv[excl] = tv[i]; }
        }
        __syncthreads();
        n = scan[P - 1];
        __syncthreads();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");       // no copy outlives the CTA
    for (int i = tid; i < n; i += NT) { keys_io[i] = sk[i]; vals_io[i] = sv[i]; }
    if (tid == 0) { io[0] = (unsigned long long)n; io[1] = (unsigned long long)done; }
}

template <int CAP>
size_t small_smem() {
    return 3 * sizeof(SmallGateP) + (size_t)CAP * (2 * sizeof(double2) + 2 * sizeof(uint64_t)) +
           (size_t)(CAP + 1) * sizeof(int);
}

// the compact record of a gate, ok = 0 when it does not fit (d > 8 or more than 8 controls)
void to_small(const SparseGateP &p, SmallGateP &s) {
    std::memset(&s, 0, sizeof(s));
    s.ok = (p.dt <= (uint64_t)kSmallD && p.nctrl <= kSmallD) ? 1 : 0;
    if (!s.ok) return;
    s.bt = p.bt; s.mbt = p.mbt; s.dt = p.dt; s.mdt = p.mdt;
    s.invalid = p.invalid; s.nctrl = p.nctrl; s.fan = p.fan;
    for (int c = 0; c < p.nctrl; ++c) {
        s.cb[c] = p.cb[c]; s.mcb[c] = p.mcb[c]; s.cd[c] = p.cd[c]; s.mcd[c] = p.mcd[c]; s.cv[c] = p.cv[c];
    }
    for (int v = 0; v < (int)p.dt; ++v) {
        s.nrow[v] = p.nrow[v];
        for (int r = 0; r < p.nrow[v]; ++r) { s.rows[v][r] = p.rows[v][r]; s.coef[v][r] = p.coef[v][r]; }
    }
}

}  // namespace
}  // namespace svi

using namespace svi;

struct sv_sparse_s {
    Register reg;
    double eps = 1e-12;
    cudaStream_t stream = nullptr;
    uint64_t nnz = 0, cap = 0;
    uint64_t *keys = nullptr, *keys2 = nullptr;       // state (sorted) / scratch
    double2 *vals = nullptr, *vals2 = nullptr;
    unsigned char *flags = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    uint64_t *d_count = nullptr;
    int nbits = 64;
    SmallGateP *d_gp = nullptr;                      // gate table of the small-state kernel
    size_t gp_cap = 0;
    std::vector<SmallGateP> gp_host;                 // what d_gp holds
    unsigned long long *io_host = nullptr;           // pinned: small-kernel in/out counters
    uint64_t launches = 0;
    bool broken = false;
};

namespace {

sv_status sp_cuda(sv_sparse_handle h, cudaError_t e, const char *where) {
    if (h) h->broken = true;
    return fail_msg(SV_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

template <typename T>
cudaError_t grow(T *&p, uint64_t n) {
    if (p) cudaFree(p);
    p = nullptr;
    return cudaMalloc(&p, n * sizeof(T) + 16);
}

// ensure room for n slots in every buffer
cudaError_t reserve(sv_sparse_handle h, uint64_t n) {
    if (n <= h->cap) return cudaSuccess;
    uint64_t c = h->cap ? h->cap : 1024;
    while (c < n) c *= 2;
    // keep the live state across the resize
    uint64_t *nk = nullptr;
    double2 *nv = nullptr;
    cudaError_t e = cudaMalloc(&nk, c * sizeof(uint64_t));
    if (e == cudaSuccess) e = cudaMalloc(&nv, c * sizeof(double2));
    if (e != cudaSuccess) return e;
    if (h->nnz) {
        e = cudaMemcpyAsync(nk, h->keys, h->nnz * sizeof(uint64_t), cudaMemcpyDeviceToDevice, h->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(nv, h->vals, h->nnz * sizeof(double2), cudaMemcpyDeviceToDevice, h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) return e;
    }
    if (h->keys) cudaFree(h->keys);
    if (h->vals) cudaFree(h->vals);
    h->keys = nk;
    h->vals = nv;
    e = grow(h->keys2, c);
    if (e == cudaSuccess) e = grow(h->vals2, c);
    if (e == cudaSuccess) e = grow(h->flags, c);
    h->cap = c;
    return e;
}

cudaError_t ensure_tmp(sv_sparse_handle h, size_t bytes) {
    if (bytes <= h->tmp_bytes) return cudaSuccess;
    if (h->tmp) cudaFree(h->tmp);
    h->tmp = nullptr;
    h->tmp_bytes = 0;
    cudaError_t e = cudaMalloc(&h->tmp, bytes);
    if (e == cudaSuccess) h->tmp_bytes = bytes;
    return e;
}

sv_status make_sparse_params(const Register &reg, const GateSpec &g, SparseGateP &p) {
    std::memset(&p, 0, sizeof(p));
    const int d = g.d;
    p.bt = reg.b[g.target];
    p.mbt = make_fastdiv64(p.bt).m;
    p.dt = (uint64_t)d;
    p.mdt = make_fastdiv64(p.dt).m;
    p.invalid = reg.D;
    if ((int)g.ctrl.size() > kMaxRem) return fail_msg(SV_ERR_UNSUPPORTED, "too many controls");
    p.nctrl = (int32_t)g.ctrl.size();
    for (size_t c = 0; c < g.ctrl.size(); ++c) {
        p.cb[c] = reg.b[g.ctrl[c].q];
        p.mcb[c] = make_fastdiv64(p.cb[c]).m;
        p.cd[c] = (uint64_t)reg.dims[g.ctrl[c].q];
        p.mcd[c] = make_fastdiv64(p.cd[c]).m;
        p.cv[c] = (uint64_t)g.ctrl[c].v;
    }
    int fan = 1;
    for (int v = 0; v < d; ++v) {                  // column v: the image of |v>
        int nr = 0;
        for (int r = 0; r < d; ++r) {
            const double2 u = g.U[r * d + v];
            if (u.x != 0.0 || u.y != 0.0) {
                p.rows[v][nr] = r;
                p.coef[v][nr] = u;
                ++nr;
            }
        }
        p.nrow[v] = nr;
        fan = nr > fan ? nr : fan;
    }
    p.fan = fan;
    return SV_OK;
}

sv_status sparse_gate(sv_sparse_handle h, const GateSpec &g) {
    SparseGateP p;
    sv_status s0 = make_sparse_params(h->reg, g, p);
    if (s0 != SV_OK) return s0;
    const uint64_t n = h->nnz, N = n * (uint64_t)p.fan;
    if (n == 0) return SV_OK;
    cudaError_t e = reserve(h, N);
    if (e != cudaSuccess) return sp_cuda(h, e, "sparse reserve");
    const unsigned blocks = (unsigned)((n + 255) / 256);
    k_sparse_expand<<<blocks, 256, 0, h->stream>>>(h->keys, h->vals, n, p, h->keys2, h->vals2);
    ++h->launches;
    // sort the contributions by basis index (stable: a fixed, deterministic summation order)
    size_t need = 0, t = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, h->keys2, h->keys, h->vals2, h->vals, (int64_t)N, 0, h->nbits);
    cub::DeviceReduce::ReduceByKey(nullptr, t, h->keys, h->keys2, h->vals, h->vals2, h->d_count, CSum(), (int64_t)N);
    need = need > t ? need : t;
    cub::DeviceSelect::Flagged(nullptr, t, h->keys2, h->flags, h->keys, h->d_count + 1, (int64_t)N);
    need = need > t ? need : t;
    cub::DeviceSelect::Flagged(nullptr, t, h->vals2, h->flags, h->vals, h->d_count + 1, (int64_t)N);
    need = need > t ? need : t;
    e = ensure_tmp(h, need);
    if (e != cudaSuccess) return sp_cuda(h, e, "sparse scratch");
    size_t tb = h->tmp_bytes;
    e = cub::DeviceRadixSort::SortPairs(h->tmp, tb, h->keys2, h->keys, h->vals2, h->vals, (int64_t)N, 0, h->nbits,
                                        h->stream);
    if (e != cudaSuccess) return sp_cuda(h, e, "sparse sort");
    tb = h->tmp_bytes;
    // sum the contributions that land on the same index (the vector addition of PAPER.md:222)
    e = cub::DeviceReduce::ReduceByKey(h->tmp, tb, h->keys, h->keys2, h->vals, h->vals2, h->d_count, CSum(),
                                       (int64_t)N, h->stream);
    if (e != cudaSuccess) return sp_cuda(h, e, "sparse reduce");
    uint64_t runs = 0;
    e = cudaMemcpyAsync(&runs, h->d_count, sizeof(uint64_t), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return sp_cuda(h, e, "sparse count");
    k_sparse_flags<<<(unsigned)((runs + 255) / 256), 256, 0, h->stream>>>(h->keys2, h->vals2, runs, p.invalid,
                                                                           h->eps * h->eps, h->flags);
    ++h->launches;
    tb = h->tmp_bytes;
    e = cub::DeviceSelect::Flagged(h->tmp, tb, h->keys2, h->flags, h->keys, h->d_count + 1, (int64_t)runs, h->stream);
    tb = h->tmp_bytes;
    if (e == cudaSuccess)
        e = cub::DeviceSelect::Flagged(h->tmp, tb, h->vals2, h->flags, h->vals, h->d_count + 1, (int64_t)runs,
                                       h->stream);
    if (e != cudaSuccess) return sp_cuda(h, e, "sparse prune");
    uint64_t kept = 0;
    e = cudaMemcpyAsync(&kept, h->d_count + 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return sp_cuda(h, e, "sparse count");
    h->nnz = kept;
    return SV_OK;
}

// Apply a gate list: runs of gates go through the one-CTA small-state kernel while the
// state's contributions fit its shared-memory capacity; a gate that does not fit goes
// through the general (expand / radix sort / reduce-by-key / select) path.
sv_status sparse_run(sv_sparse_handle h, const std::vector<GateSpec> &specs) {
    std::vector<SparseGateP> ps(specs.size());
    for (size_t i = 0; i < specs.size(); ++i) {
        sv_status s = make_sparse_params(h->reg, specs[i], ps[i]);
        if (s != SV_OK) return s;
    }
    std::vector<SmallGateP> sm(ps.size());
    for (size_t i = 0; i < ps.size(); ++i) to_small(ps[i], sm[i]);
    if (sm.size() > h->gp_cap) {
        if (h->d_gp) cudaFree(h->d_gp);
        h->d_gp = nullptr;
        h->gp_cap = 0;
        h->gp_host.clear();
        cudaError_t e = cudaMalloc(&h->d_gp, sm.size() * sizeof(SmallGateP));
        if (e != cudaSuccess) return sp_cuda(h, e, "sparse gate table");
        h->gp_cap = sm.size();
    }
    // upload the gate table unless the same circuit was submitted last time
    const bool same = sm.size() == h->gp_host.size() &&
                      (sm.empty() || std::memcmp(sm.data(), h->gp_host.data(), sm.size() * sizeof(SmallGateP)) == 0);
    if (!sm.empty() && !same) {
        cudaError_t e = cudaMemcpyAsync(h->d_gp, sm.data(), sm.size() * sizeof(SmallGateP), cudaMemcpyHostToDevice,
                                        h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) return sp_cuda(h, e, "sparse gate table");
        h->gp_host = sm;
    }
    static LaunchAttr attr;                  // per device (cudaFuncSetAttribute is per device)
    const int dv = current_device_slot();
    if (!attr.configured[dv]) {
        cudaError_t e = cudaFuncSetAttribute(k_sparse_small<1024, kSmallCap>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)small_smem<kSmallCap>());
        if (e != cudaSuccess) return sp_cuda(h, e, "sparse small attribute");
        attr.configured[dv] = 1;
    }
    size_t i = 0;
    while (i < ps.size()) {
        const uint64_t m = h->nnz * (uint64_t)ps[i].fan;
        size_t done = 0;
        if (h->nnz > 0 && m <= (uint64_t)kSmallCap && sm[i].ok) {
            h->io_host[0] = (unsigned long long)h->nnz;
            h->io_host[1] = 0ull;
            cudaError_t e = cudaMemcpyAsync(h->d_count, h->io_host, 2 * sizeof(unsigned long long),
                                            cudaMemcpyHostToDevice, h->stream);
            if (e != cudaSuccess) return sp_cuda(h, e, "sparse small setup");
            const int left = (int)(ps.size() - i);
            unsigned long long *io = (unsigned long long *)h->d_count;
            if (m <= (uint64_t)kTinyCap)   // one warp: GHZ-sized states
                k_sparse_small<32, kTinyCap><<<1, 32, small_smem<kTinyCap>(), h->stream>>>(
                    h->d_gp + i, left, h->keys, h->vals, io, h->eps * h->eps);
            else
                k_sparse_small<1024, kSmallCap><<<1, 1024, small_smem<kSmallCap>(), h->stream>>>(
                    h->d_gp + i, left, h->keys, h->vals, io, h->eps * h->eps);
            ++h->launches;
            e = cudaMemcpyAsync(h->io_host, h->d_count, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
            if (e != cudaSuccess) return sp_cuda(h, e, "sparse small path");
            h->nnz = h->io_host[0];
            done = (size_t)h->io_host[1];
            i += done;
        }
        if (done == 0 && i < ps.size()) {                  // the general path for this gate
            sv_status s = sparse_gate(h, specs[i]);
            if (s != SV_OK) return s;
            ++i;
        }
    }
    return SV_OK;
}

sv_status sp_check(sv_sparse_handle h) {
    if (!h) return fail_msg(SV_ERR_INVALID_ARG, "null handle");
    if (h->broken) return fail_msg(SV_ERR_CUDA, "handle is unusable after an earlier CUDA fault");
    return SV_OK;
}

}  // namespace

extern "C" {

sv_status sv_sparse_create(const int32_t *dims, int32_t n, double eps, sv_sparse_handle *out) {
    if (!out) return fail_msg(SV_ERR_INVALID_ARG, "null out");
    *out = nullptr;
    sv_sparse_handle h = new (std::nothrow) sv_sparse_s();
    if (!h) return fail_msg(SV_ERR_NOMEM, "host allocation");
    sv_status s = make_register(dims, n, &h->reg, err_slot());
    if (s != SV_OK) { delete h; return s; }
    if (h->reg.D > (1ull << 63)) { delete h; return fail_msg(SV_ERR_OVERFLOW, "sparse indices need D <= 2^63 (PAPER.md:489)"); }
    h->eps = eps > 0 ? eps : 1e-12;
    int nb = 1;
    while (nb < 64 && (h->reg.D >> nb) != 0) ++nb;      // bits of D (the invalid key) and below
    h->nbits = nb;
    cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&h->d_count, 2 * sizeof(uint64_t));
    if (e == cudaSuccess) e = cudaMallocHost(&h->io_host, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = reserve(h, kSmallCap);      // the small-state kernel writes back up to kSmallCap
    if (e != cudaSuccess) { cudaGetLastError(); sv_sparse_destroy(h); return fail_msg(SV_ERR_CUDA, cudaGetErrorString(e)); }
    s = sv_sparse_reset(h, 0);
    if (s != SV_OK) { sv_sparse_destroy(h); return s; }
    *out = h;
    return SV_OK;
}

sv_status sv_sparse_destroy(sv_sparse_handle h) {
    if (!h) return fail_msg(SV_ERR_INVALID_ARG, "null handle");
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (void *p : {(void *)h->keys, (void *)h->keys2, (void *)h->vals, (void *)h->vals2, (void *)h->flags,
                    h->tmp, (void *)h->d_count, (void *)h->d_gp})
        if (p) cudaFree(p);
    if (h->io_host) cudaFreeHost(h->io_host);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return SV_OK;
}

sv_status sv_sparse_reset(sv_sparse_handle h, uint64_t basis_index) {
    sv_status s = sp_check(h);
    if (s != SV_OK) return s;
    if (basis_index >= h->reg.D) return fail_msg(SV_ERR_INDEX_RANGE, "basis index >= D");
    k_sparse_set<<<1, 1, 0, h->stream>>>(h->keys, h->vals, basis_index);
    ++h->launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return sp_cuda(h, e, "sparse reset");
    h->nnz = 1;
    return SV_OK;
}

sv_status sv_sparse_apply_gate(sv_sparse_handle h, int32_t target, const int32_t *ctrl, const int32_t *ctrl_vals,
                               int32_t nctrl, const double *U) {
    sv_status s = sp_check(h);
    if (s != SV_OK) return s;
    s = validate_gate(h->reg, target, ctrl, ctrl_vals, nctrl, U, err_slot());
    if (s != SV_OK) return s;
    GateSpec g;
    g.target = target;
    g.d = h->reg.dims[target];
    for (int i = 0; i < nctrl; ++i) g.ctrl.push_back({ctrl[i], ctrl_vals[i]});
    g.U.resize((size_t)g.d * g.d);
    for (int i = 0; i < g.d * g.d; ++i) g.U[i] = make_double2(U[2 * i], U[2 * i + 1]);
    if (!(unitarity_error(g.U.data(), g.d) <= 1e-12)) return fail_msg(SV_ERR_NOT_UNITARY, "U is not unitary");
    return sparse_run(h, std::vector<GateSpec>{g});
}

sv_status sv_sparse_apply_circuit(sv_sparse_handle h, const sv_gate *gates, int64_t ngates, uint32_t flags) {
    sv_status s = sp_check(h);
    if (s != SV_OK) return s;
    if (ngates < 0 || (ngates && !gates)) return fail_msg(SV_ERR_INVALID_ARG, "bad gate list");
    std::vector<GateSpec> specs;
    for (int64_t i = 0; i < ngates; ++i) {            // validate everything first
        const sv_gate &x = gates[i];
        s = validate_gate(h->reg, x.target, x.ctrl, x.ctrl_vals, x.nctrl, x.U, err_slot());
        if (s != SV_OK) return s;
        GateSpec g;
        g.target = x.target;
        g.d = h->reg.dims[x.target];
        for (int c = 0; c < x.nctrl; ++c) g.ctrl.push_back({x.ctrl[c], x.ctrl_vals[c]});
        g.U.resize((size_t)g.d * g.d);
        for (int k = 0; k < g.d * g.d; ++k) g.U[k] = make_double2(x.U[2 * k], x.U[2 * k + 1]);
        if (!(flags & SV_NO_CHECK) && !(unitarity_error(g.U.data(), g.d) <= 1e-12))
            return fail_msg(SV_ERR_NOT_UNITARY, "gate " + std::to_string(i) + ": U is not unitary");
        specs.push_back(g);
    }
    return sparse_run(h, specs);
}

sv_status sv_sparse_nnz(sv_sparse_handle h, uint64_t *out) {
    sv_status s = sp_check(h);
    if (s != SV_OK) return s;
    if (!out) return fail_msg(SV_ERR_INVALID_ARG, "null out");
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return sp_cuda(h, e, "sparse sync");
    *out = h->nnz;
    return SV_OK;
}

sv_status sv_sparse_entries(sv_sparse_handle h, uint64_t cap, uint64_t *idx, double *amp, uint64_t *n) {
    sv_status s = sp_check(h);
    if (s != SV_OK) return s;
    if (!n || (cap && (!idx || !amp))) return fail_msg(SV_ERR_INVALID_ARG, "null out");
    const uint64_t k = h->nnz < cap ? h->nnz : cap;
    cudaError_t e = cudaSuccess;
    if (k) {
        e = cudaMemcpyAsync(idx, h->keys, k * sizeof(uint64_t), cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(amp, h->vals, k * sizeof(double2), cudaMemcpyDeviceToHost, h->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return sp_cuda(h, e, "sparse readback");
    *n = h->nnz;
    return SV_OK;
}

sv_status sv_sparse_launches(sv_sparse_handle h, uint64_t *out) {
    if (!h || !out) return fail_msg(SV_ERR_INVALID_ARG, "null handle/out");
    *out = h->launches;
    return SV_OK;
}

}  // extern "C"
