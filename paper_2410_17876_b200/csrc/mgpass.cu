// mgpass.cu — multi-gate cache-blocked pass kernel for sm_100a.
//
// One HBM pass applies a whole list of gates.  A tile holds every digit value of the in-tile
// qudits Q = {q_0..q_{m0-1}} ∪ H (plan_passes) and one value of every other digit, laid out in
// shared memory as [member][run] where a "member" is one combination of the H digits (global
// offset sum_h j_h b_h) and the run is a contiguous stretch of the low space (stride < b_{min H}).
// Loading / storing a tile = one cp.async.bulk per member (TMA bulk copies onto an mbarrier,
// 3-stage ring, persistent grid, as in tiled_impl.cuh).  Between load and store the CTA applies
// the pass's gates one after another in shared memory: each gate visits its equivalence classes
// inside the tile — a target in H has smem stride W_h * LT, a low target has
// stride b_t — and its controls are decided per class (in-tile digits) or once per tile
// (digits outside the tile, constant across it).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "sv_internal.h"
#include "plan.h"

namespace svi {

constexpr int kMaxPassGates = 24;
constexpr int kMaxMembers = 128;
constexpr int kPoolC = 768;
constexpr int kMaxPassCtrl = 4;

struct PassCtrl {
    int32_t cls;          // 0 = H digit (from member index), 1 = low digit (from run position), 2 = per tile
    uint32_t v;
    uint32_t d, md;       // control dimension (+ magic)
    uint32_t w, mw;       // cls 0: member radix weight; cls 1: stride b_c (+ magic)
    uint32_t M, mM;       // cls 1: b_c * d_c (+ magic)
    uint64_t b64, mb64;   // cls 2: global stride (+ magic); cls 1: M and its 64-bit magic
    uint64_t md64;        // cls 2: magic for d
};

struct PassGateP {
    int32_t d, kind, nctrl, uoff;
    int32_t inctl;        // has controls decided inside the tile (cls 0 / 1)
    uint32_t st, mst;     // smem stride of the target (+ magic)
    uint32_t active;
    int8_t sigma[kMaxDim];
    PassCtrl c[kMaxPassCtrl];
};

struct PassParams {
    double2 *psi;
    int32_t nrem;
    RemovedRun rem[kMaxRem];
    uint64_t ntiles, R, tpr, tpr_m;
    uint32_t LT, mLT;     // run elements per member in a tile (+ magic)
    int32_t M;            // members per tile
    int32_t ngates;
    int32_t upool;        // used entries of U (copied to shared memory at kernel start)
    uint64_t moff[kMaxMembers];
    PassGateP g[kMaxPassGates];
    double2 U[kPoolC];    // general: row-major d x d; monomial: coefficient per member
};

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_store(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void cfma(double2 &acc, const double2 u, const double2 x) {
    acc.x = fma(u.x, x.x, acc.x);
    acc.x = fma(-u.y, x.y, acc.x);
    acc.y = fma(u.x, x.y, acc.y);
    acc.y = fma(u.y, x.x, acc.y);
}
__device__ __forceinline__ double2 cmul(const double2 u, const double2 x) {
    return make_double2(fma(u.x, x.x, -u.y * x.y), fma(u.x, x.y, u.y * x.x));
}

struct TileInfo {
    uint64_t gbase;   // global index of member 0, run position 0
    uint64_t s0;      // offset of the tile inside its run
    uint32_t len;     // valid run elements per member
};

__device__ __forceinline__ TileInfo tile_info(const PassParams &p, uint64_t t) {
    TileInfo ti;
    uint64_t sub;
    const uint64_t run = fastdiv64(t, p.tpr, p.tpr_m, sub);
    ti.s0 = sub * p.LT;
    const uint64_t rem = p.R - ti.s0;
    ti.len = (uint32_t)(rem < p.LT ? rem : p.LT);
    ti.gbase = insert_digits(run * p.R + ti.s0, p.nrem, p.rem);
    return ti;
}

// Per-stage record written by warp 0 when it issues a tile's loads (before the mbarrier
// arrive, so the consumers' acquire-wait sees it): the tile geometry, which gates fire on this
// tile (controls outside the tile), and the run offsets of the low controls.
struct StageInfo {
    TileInfo ti;
    uint32_t fire;                                   // bit g: gate g's out-of-tile controls hold
    uint32_t lowoff[kMaxPassGates][kMaxPassCtrl];    // (s0 mod b_c d_c) for low controls
};

__device__ __forceinline__ void issue_loads(const PassParams &p, uint64_t t, double2 *buf, uint64_t *bar,
                                            StageInfo *si, int lane) {
    const TileInfo ti = tile_info(p, t);
    // lane g decides gate g for this tile
    bool fire = true;
    if (lane < p.ngates) {
        const PassGateP &g = p.g[lane];
        for (int k = 0; k < g.nctrl; ++k) {
            const PassCtrl &cc = g.c[k];
            if (cc.cls == 2) {
                uint64_t r;
                const uint64_t q = fastdiv64(ti.gbase, cc.b64, cc.mb64, r);
                fastdiv64(q, cc.d, cc.md64, r);
                fire = fire && (r == cc.v);
            } else if (cc.cls == 1) {
                uint64_t r;
                fastdiv64(ti.s0, cc.M, cc.mb64, r);
                si->lowoff[lane][k] = (uint32_t)r;
            }
        }
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, fire && lane < p.ngates);
    if (lane == 0) {
        si->ti = ti;
        si->fire = bits;
    }
    __syncwarp();
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)p.M * ti.len * (uint32_t)sizeof(double2));
    __syncwarp();
    for (int m = lane; m < p.M; m += 32)
        bulk_load(buf + (size_t)m * p.LT, p.psi + ti.gbase + p.moff[m], ti.len * (uint32_t)sizeof(double2), bar);
}

// y = U x (general) or y_{sigma(j)} = c_j x_j (monomial) on one class at smem e0, stride st
template <int D>
__device__ __forceinline__ void apply_class(double2 *buf, uint32_t e0, uint32_t st, const PassGateP &g,
                                            const double2 *U, int dd) {
    constexpr int MD = D ? D : kMaxDim;
    const int d = D ? D : dd;
    double2 x[MD];
    if (g.kind == kGeneral) {
#pragma unroll
        for (int j = 0; j < MD; ++j)
            if (D || j < d) x[j] = buf[e0 + j * st];
#pragma unroll
        for (int i = 0; i < MD; ++i) {
            if (D || i < d) {
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int j = 0; j < MD; ++j)
                    if (D || j < d) cfma(acc, U[i * d + j], x[j]);
                buf[e0 + i * st] = acc;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < MD; ++j)
            if ((D || j < d) && ((g.active >> j) & 1)) x[j] = buf[e0 + j * st];
#pragma unroll
        for (int j = 0; j < MD; ++j)
            if ((D || j < d) && ((g.active >> j) & 1)) buf[e0 + g.sigma[j] * st] = cmul(U[j], x[j]);
    }
}

// generic dimension: out of line so its 16-wide register arrays do not inflate the kernel
__device__ __noinline__ void apply_class_generic(double2 *buf, uint32_t e0, uint32_t st, const PassGateP &g,
                                                 const double2 *U) {
    const int d = g.d;
    if (g.kind == kGeneral) {
        double2 x[kMaxDim];
        for (int j = 0; j < d; ++j) x[j] = buf[e0 + j * st];
        for (int i = 0; i < d; ++i) {
            double2 acc = make_double2(0.0, 0.0);
            for (int j = 0; j < d; ++j) cfma(acc, U[i * d + j], x[j]);
            buf[e0 + i * st] = acc;
        }
    } else {
        double2 x[kMaxDim];
        for (int j = 0; j < d; ++j)
            if ((g.active >> j) & 1) x[j] = buf[e0 + j * st];
        for (int j = 0; j < d; ++j)
            if ((g.active >> j) & 1) buf[e0 + g.sigma[j] * st] = cmul(U[j], x[j]);
    }
}

// member-0 smem index of class c, and whether the class exists (ragged) and fires (controls)
__device__ __forceinline__ bool class_at(const PassParams &p, const PassGateP &g, uint32_t len, bool needml,
                                         const uint32_t *lowoff, uint32_t c, uint32_t &e0) {
    uint32_t off;
    const uint32_t grp = fastdiv32(c, g.st, g.mst, off);
    e0 = grp * g.st * (uint32_t)g.d + off;
    if (!needml) return true;                            // full tile, no in-tile controls
    uint32_t l;
    const uint32_t m = fastdiv32(e0, p.LT, p.mLT, l);
    if (l >= len) return false;                          // ragged last tile of a run
    bool ok = true;
#pragma unroll
    for (int k = 0; k < kMaxPassCtrl; ++k) {
        if (k >= g.nctrl) break;
        const PassCtrl &cc = g.c[k];
        uint32_t r, r2;
        if (cc.cls == 0) {
            const uint32_t q = fastdiv32(m, cc.w, cc.mw, r);
            fastdiv32(q, cc.d, cc.md, r2);
            ok = ok && (r2 == cc.v);
        } else if (cc.cls == 1) {
            fastdiv32(lowoff[k] + l, cc.M, cc.mM, r);
            const uint32_t q = fastdiv32(r, cc.w, cc.mw, r2);
            fastdiv32(q, cc.d, cc.md, r2);
            ok = ok && (r2 == cc.v);
        }
    }
    return ok;
}

// two classes per iteration: both gathers are issued before either matvec (ILP)
template <int D>
__device__ __forceinline__ void apply_class2(double2 *buf, uint32_t ea, bool oka, uint32_t eb, bool okb,
                                             uint32_t st, const PassGateP &g, const double2 *U) {
    double2 xa[D], xb[D];
    if (g.kind == kGeneral) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if (oka) xa[j] = buf[ea + j * st];
            if (okb) xb[j] = buf[eb + j * st];
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double2 aa = make_double2(0.0, 0.0), ab = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const double2 u = U[i * D + j];
                cfma(aa, u, xa[j]);
                cfma(ab, u, xb[j]);
            }
            if (oka) buf[ea + i * st] = aa;
            if (okb) buf[eb + i * st] = ab;
        }
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j)
            if ((g.active >> j) & 1) {
                if (oka) xa[j] = buf[ea + j * st];
                if (okb) xb[j] = buf[eb + j * st];
            }
#pragma unroll
        for (int j = 0; j < D; ++j)
            if ((g.active >> j) & 1) {
                const double2 u = U[j];
                if (oka) buf[ea + g.sigma[j] * st] = cmul(u, xa[j]);
                if (okb) buf[eb + g.sigma[j] * st] = cmul(u, xb[j]);
            }
    }
}

template <int D, int NT>
__device__ __forceinline__ void apply_gate_tile(const PassParams &p, const PassGateP &g, double2 *buf,
                                                const double2 *Us, uint32_t len, const uint32_t *lowoff,
                                                int tid) {
    const uint32_t nslots = (uint32_t)p.M * p.LT;
    const uint32_t ncls = nslots / (uint32_t)g.d;
    const double2 *U = Us + g.uoff;       // shared-memory copy: not hoisted into registers
    const bool needml = g.inctl || len < p.LT;
    if constexpr (D == 0) {
        for (uint32_t c = tid; c < ncls; c += NT) {
            uint32_t e0;
            if (class_at(p, g, len, needml, lowoff, c, e0)) apply_class_generic(buf, e0, g.st, g, U);
        }
    } else if constexpr (D >= 4) {   // one class per iteration (register pressure)
        for (uint32_t c = tid; c < ncls; c += NT) {
            uint32_t e0;
            if (class_at(p, g, len, needml, lowoff, c, e0)) apply_class<D>(buf, e0, g.st, g, U, g.d);
        }
    } else {                         // two classes per iteration (ILP)
        for (uint32_t c = tid; c < ncls; c += 2 * NT) {
            uint32_t ea = 0, eb = 0;
            const bool oka = class_at(p, g, len, needml, lowoff, c, ea);
            const uint32_t c2 = c + NT;
            const bool okb = c2 < ncls && class_at(p, g, len, needml, lowoff, c2, eb);
            apply_class2<D>(buf, ea, oka, eb, okb, g.st, g, U);
        }
    }
}

}  // namespace

__device__ __forceinline__ void compute_barrier(int nthreads) {   // named barrier 1: compute warps only
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp-specialised: warps 0..NT/32-1 compute, warp NT/32 is the producer (TMA loads, stage
// records, TMA stores).  full[s] completes when a tile's bytes have landed; done[s] when the
// compute warps have finished it (after fence.proxy.async, so the bulk store sees their writes).
template <int NT>
__global__ void __launch_bounds__(NT + 32, 1) k_gate_pass(const __grid_constant__ PassParams p, int S, int TE) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw);
    double2 *Us = bufs + (size_t)S * TE;                       // the pass's matrices
    StageInfo *sinfo = reinterpret_cast<StageInfo *>(Us + p.upool);
    uint64_t *full = reinterpret_cast<uint64_t *>(sinfo + S);
    uint64_t *done = full + S;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&done[s], 1); }
        fence_mbar_init();
    }
    for (int k = tid; k < p.upool; k += NT + 32) Us[k] = p.U[k];
    __syncthreads();
    const uint64_t first = blockIdx.x, step = gridDim.x;
    if (first >= p.ntiles) return;
    const uint64_t my = (p.ntiles - first + step - 1) / step;

    if (warp == NT / 32) {
        // ---------------- producer warp
        for (uint64_t i = 0; i < my + (uint64_t)S; ++i) {
            const int s = (int)(i % (uint64_t)S);
            if (i >= (uint64_t)S) {                   // drain tile i-S from stage s
                const uint64_t j = i - (uint64_t)S;
                if (j >= my) continue;
                mbar_wait(&done[s], (uint32_t)((j / (uint64_t)S) & 1));
                const StageInfo &si = sinfo[s];
                for (int m = lane; m < p.M; m += 32)
                    bulk_store(p.psi + si.ti.gbase + p.moff[m], bufs + (size_t)s * TE + (size_t)m * p.LT,
                               si.ti.len * (uint32_t)sizeof(double2));
                bulk_commit();
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
            }
            if (i < my)
                issue_loads(p, first + i * step, bufs + (size_t)s * TE, &full[s], &sinfo[s], lane);
        }
        bulk_wait_all();
        return;
    }

    // ---------------- compute warps
    for (uint64_t i = 0; i < my; ++i) {
        const int s = (int)(i % (uint64_t)S);
        double2 *buf = bufs + (size_t)s * TE;
        mbar_wait(&full[s], (uint32_t)((i / (uint64_t)S) & 1));
        const StageInfo &si = sinfo[s];
        const uint32_t len = si.ti.len;
        const uint32_t fire = si.fire;
        for (int gi = 0; gi < p.ngates; ++gi) {
            if (!((fire >> gi) & 1)) continue;          // out-of-tile control unmet: uniform skip
            const PassGateP &g = p.g[gi];
            const uint32_t *lo = si.lowoff[gi];
            switch (g.d) {
                case 2: apply_gate_tile<2, NT>(p, g, buf, Us, len, lo, tid); break;
                case 3: apply_gate_tile<3, NT>(p, g, buf, Us, len, lo, tid); break;
                case 4: apply_gate_tile<4, NT>(p, g, buf, Us, len, lo, tid); break;
                case 5: apply_gate_tile<5, NT>(p, g, buf, Us, len, lo, tid); break;
                default: apply_gate_tile<0, NT>(p, g, buf, Us, len, lo, tid); break;
            }
            compute_barrier(NT);
        }
        fence_proxy_async();
        compute_barrier(NT);
        if (tid == 0) mbar_arrive(&done[s]);
    }
}

// ------------------------------------------------------------------------------ host
// Build the pass parameters; returns false if the pass does not fit this kernel.
bool build_pass(const Register &reg, const std::vector<GateSpec> &gates, const PassPlan &pp, double2 *psi,
                int TE, PassParams &p, double *touched) {
    std::memset(&p, 0, sizeof(p));
    if ((int)pp.gates.size() > kMaxPassGates || pp.tile > (uint64_t)TE) return false;
    p.psi = psi;
    const int m0 = pp.m0;
    const uint64_t L = (m0 < reg.n) ? reg.b[m0] : reg.D;
    uint64_t M = 1;
    for (int h : pp.H) M *= (uint64_t)reg.dims[h];
    if (M > (uint64_t)kMaxMembers) return false;
    // member radix weights and global offsets (H ascending)
    std::vector<uint64_t> W(reg.n, 0);
    {
        uint64_t w = 1;
        for (int h : pp.H) { W[h] = w; w *= (uint64_t)reg.dims[h]; }
    }
    for (uint64_t m = 0; m < M; ++m) {
        uint64_t off = 0, rest = m;
        for (int h : pp.H) { off += (rest % (uint64_t)reg.dims[h]) * reg.b[h]; rest /= (uint64_t)reg.dims[h]; }
        p.moff[m] = off;
    }
    p.M = (int32_t)M;
    // H digits removed (pin 0), merged when adjacent
    int nr = 0;
    for (size_t i = 0; i < pp.H.size(); ++i) {
        const int h = pp.H[i];
        if (nr > 0 && p.rem[nr - 1].bd == reg.b[h]) {
            p.rem[nr - 1].bd *= (uint64_t)reg.dims[h];
        } else {
            if (nr >= kMaxRem) return false;
            RemovedRun &r = p.rem[nr++];
            r.b = reg.b[h];
            r.bd = reg.b[h] * (uint64_t)reg.dims[h];
            r.pinb = 0;
            r.m = make_fastdiv64(r.b).m;
        }
    }
    p.nrem = nr;
    // schedule: runs of the low space below min H, split into tiles of LT elements
    // The run per member is widened to fill the tile (a multiple of b_{m0}, so low-prefix
    // classes stay whole, and at most the run R below min H).
    const uint64_t R = pp.H.empty() ? reg.D : reg.b[pp.H[0]];
    uint64_t LT = ((uint64_t)TE / M / L) * L;
    if (LT < L) LT = L;
    if (LT > R) LT = R;
    p.R = R;
    p.LT = (uint32_t)LT;
    p.mLT = make_fastdiv32(p.LT).m;
    p.tpr = (R + LT - 1) / LT;
    p.tpr_m = make_fastdiv64(p.tpr).m;
    const uint64_t nruns = reg.D / (M * R);
    p.ntiles = nruns * p.tpr;
    // gates
    int uoff = 0;
    *touched = 0.0;
    p.ngates = (int32_t)pp.gates.size();
    for (size_t gi = 0; gi < pp.gates.size(); ++gi) {
        const GateSpec &g = gates[pp.gates[gi]];
        GatePlan gp;
        std::string err;
        if (plan_gate(reg, g, false, &gp, &err) != SV_OK) return false;
        *touched += (double)gp.touched;
        PassGateP &q = p.g[gi];
        q.d = gp.d;
        q.kind = gp.kind;
        q.active = gp.active;
        for (int j = 0; j < kMaxDim; ++j) q.sigma[j] = (int8_t)(j < gp.d ? gp.sigma[j] : j);
        const int need = gp.kind == kGeneral ? gp.d * gp.d : gp.d;
        if (uoff + need > kPoolC) return false;
        q.uoff = uoff;
        for (int k = 0; k < need; ++k) p.U[uoff + k] = gp.U[k];
        uoff += need;
        p.upool = uoff;
        const int t = g.target;
        if (g.span != 1 || (t >= m0 && std::find(pp.H.begin(), pp.H.end(), t) == pp.H.end())) return false;
        const uint64_t st = (t < m0) ? reg.b[t] : W[t] * LT;
        q.st = (uint32_t)st;
        q.mst = make_fastdiv32(q.st).m;
        if ((int)g.ctrl.size() > kMaxPassCtrl) return false;
        q.nctrl = (int32_t)g.ctrl.size();
        for (size_t k = 0; k < g.ctrl.size(); ++k) {
            PassCtrl &cc = q.c[k];
            const int c = g.ctrl[k].q;
            cc.v = (uint32_t)g.ctrl[k].v;
            cc.d = (uint32_t)reg.dims[c];
            cc.md = make_fastdiv32(cc.d).m;
            const bool inH = std::find(pp.H.begin(), pp.H.end(), c) != pp.H.end();
            if (inH) {
                cc.cls = 0;
                q.inctl = 1;
                cc.w = (uint32_t)W[c];
                cc.mw = make_fastdiv32(cc.w).m;
            } else if (reg.b[c] < R) {        // below min H: decided by the run position
                cc.cls = 1;
                q.inctl = 1;
                cc.w = (uint32_t)reg.b[c];
                cc.mw = make_fastdiv32(cc.w).m;
                cc.M = cc.w * cc.d;
                cc.mM = make_fastdiv32(cc.M).m;
                cc.mb64 = make_fastdiv64(cc.M).m;
            } else {                          // outside the tile: constant per tile
                cc.cls = 2;
                cc.b64 = reg.b[c];
                cc.mb64 = make_fastdiv64(cc.b64).m;
                cc.md64 = make_fastdiv64(cc.d).m;
            }
        }
    }
    return p.ntiles > 0;
}

template <int NT>
cudaError_t launch_pass_t(const PassParams &p, cudaStream_t st, const LaunchCfg &cfg) {
    const int S = cfg.pass_stages, TE = cfg.pass_tile;
    // size for the largest matrix pool so the attribute and the occupancy are set once per config
    const size_t smem = (size_t)S * TE * sizeof(double2) + (size_t)kPoolC * sizeof(double2) +
                        (size_t)S * sizeof(StageInfo) + (size_t)2 * S * sizeof(uint64_t);
    static size_t configured = 0, occ_for = 0;
    static int occ = 1;
    if (configured < smem) {
        cudaError_t e = cudaFuncSetAttribute(k_gate_pass<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    if (occ_for != smem) {   // resident CTAs per SM at this smem size (persistent grid)
        int o = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_gate_pass<NT>, NT + 32, smem) != cudaSuccess || o < 1) o = 1;
        occ = o;
        occ_for = smem;
    }
    const uint64_t cap = (uint64_t)cfg.num_sms * (uint64_t)occ;
    const unsigned grid = (unsigned)(p.ntiles < cap ? p.ntiles : cap);
    k_gate_pass<NT><<<grid, NT + 32, smem, st>>>(p, S, TE);
    return cudaGetLastError();
}

cudaError_t launch_pass(const PassParams &p, cudaStream_t st, const LaunchCfg &cfg) {
    return cfg.pass_threads >= 512 ? launch_pass_t<512>(p, st, cfg) : launch_pass_t<256>(p, st, cfg);
}

cudaError_t run_pass(const Register &reg, const std::vector<GateSpec> &gates, const PassPlan &pp, double2 *psi,
                     cudaStream_t st, const LaunchCfg &cfg, bool *handled, double *touched) {
    static thread_local PassParams p;   // ~21 KB; parameters are copied at launch
    *handled = build_pass(reg, gates, pp, psi, cfg.pass_tile, p, touched);
    if (!*handled) return cudaSuccess;
    return launch_pass(p, st, cfg);
}

}  // namespace svi
