// mgpass_impl.cuh — multi-gate cache-blocked pass kernel for sm_100a.
// Included by mgpass.cu (host planning, dispatch) and the per-thread-count instantiation
// units mgpass_k256.cu / mgpass_k384.cu (compiled in parallel).
//
// One HBM pass applies a whole list of gates.  A tile holds every digit value of the in-tile
// qudits Q = {q_0..q_{m0-1}} ∪ H (plan_passes) and one value of every other digit, laid out in
// shared memory as [member][run] where a "member" is one combination of the H digits (global
// offset sum_h j_h b_h) and the run is a contiguous stretch of the low space (stride < b_{min H}).
// Loading / storing a tile = one cp.async.bulk per member (TMA bulk copies onto an mbarrier,
// persistent grid, a producer warp and NT compute threads).  Between load and store the CTA
// applies the pass's gates one after another in shared memory: each gate visits its
// equivalence classes inside the tile — a target in H has smem stride
// W_h * LT, a low target has stride b_t — and its controls are decided
//   * per class from static bit masks: controls on H digits (a mask over the M members) and on
//     low-prefix digits (a mask over the position modulo L = b_{m0}, identical in every tile);
//   * per class from the tile's run offset: controls on run digits above the low prefix;
//   * once per tile: controls on digits outside the tile (the producer's fire bits).
#pragma once
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
constexpr int kMaskWords = 4 + 16;   // member mask (128 bits) + low-position mask (L < 512 bits)

// How a gate of a register stage is applied along its axis: dense y = U x (any
// gate, monomials included), or a cyclic shift with coefficients y_{(j+s) mod d} = c_j x_j (the
// §2.1-2.2 phase / permutation structure of X_{+s}, CINC and diagonal gates).  Gates of the
// generic path (d > 5) keep the class-by-class kinds general / monomial.
enum PassForm : int32_t { kFormDense = 0, kFormShift = 1 };

// a control decided at run time (static in-tile controls live in the masks)
struct PassCtrl {
    int32_t cls;          // 1 = run digit above the low prefix (needs the tile's run offset), 2 = outside the tile
    uint32_t v;
    uint32_t d, md;       // control dimension (+ magic)
    uint32_t w, mw;       // cls 1: stride b_c (+ magic)
    uint32_t M, mM;       // cls 1: b_c * d_c (+ magic)
    uint64_t b64, mb64;   // cls 2: global stride (+ magic); cls 1: 64-bit magic of M
    uint64_t md64;        // cls 2: magic for d
};

enum PassFlags : uint32_t { kFMemberMask = 1, kFLowMask = 2, kFRunCtrl = 4 };

struct PassGateP {
    int32_t d, nctrl, uoff;
    int32_t form;         // PassForm (register stages)
    int32_t axis;         // register stage: 0 = the stage's first axis, 1 = its second
    int32_t axctl;        // register stage: -1, or the value of a control on the stage's other axis
    int32_t shift, pure;  // kFormShift: shift s; every coefficient exactly 1
    uint32_t flags;       // PassFlags: in-tile controls checked per class (not on a stage axis)
    // generic path (d > 5): class-by-class application along the target's own stride
    int32_t kind;         // kGeneral / kMonomial
    uint32_t st, mst;
    uint32_t active;
    int8_t sigma[kMaxDim];
    PassCtrl c[kMaxPassCtrl];
};

// A register stage: consecutive gates (after commutation-aware regrouping) whose targets are
// one or two in-tile qudits, the "axes".  Each thread gathers whole 2-D classes (every value of
// both axis digits, the other digits fixed) into registers, applies all the stage's gates
// there and scatters once: one shared-memory round trip per stage instead of per gate.
struct PassStage {
    int32_t g0, g1;         // gates [g0, g1) of PassParams::g
    int32_t da, db;         // axis dimensions (db = 1: one axis); da = 0: generic stage (d > 5)
    uint32_t sta, stb;      // tile strides of axis 0 / axis 1
    uint32_t s1, m1, d1;    // class enumeration: insert the lower-stride axis digit first ...
    uint32_t s2, m2, d2;    // ... then the other (d2 = 1: none)
};

struct PassParams {
    double2 *psi;
    int32_t nrem;
    RemovedRun rem[kMaxRem];
    uint64_t ntiles, R, tpr, tpr_m;
    uint32_t LT, mLT;     // run elements per member in a tile (+ magic)
    uint32_t L, mL;       // low-prefix block b_{m0} (+ magic)
    int32_t M;            // members per tile
    int32_t ngates, nstages;
    int32_t upool;        // used entries of U (copied to shared memory at kernel start)
    uint64_t moff[kMaxMembers];
    PassStage st[kMaxPassGates];
    PassGateP g[kMaxPassGates];
    uint32_t mask[kMaxPassGates][kMaskWords];   // per gate: member mask, low-position mask
    double2 U[kPoolC];    // dense: row-major d x d; shift: coefficient per member
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

// Per-stage record written by the producer when it issues a tile's loads (before the mbarrier
// arrive, so the consumers' acquire-wait sees it): the tile geometry, which gates fire on this
// tile (controls outside the tile), and the run offsets of the run-digit controls.
struct StageInfo {
    TileInfo ti;
    uint32_t fire;                                   // bit g: gate g's out-of-tile controls hold
    uint32_t lowoff[kMaxPassGates][kMaxPassCtrl];    // (s0 mod b_c d_c) for run-digit controls
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

// In-tile division (x < 2^16, d < 2^16): with m = floor(2^32/d) + 1, umulhi(x, m) is exact
// because x * (m d - 2^32) <= x d < 2^32, so no fix-up step is needed (d == 1 <=> m == 0).
__device__ __forceinline__ uint32_t tdiv(uint32_t x, uint32_t d, uint32_t m, uint32_t &r) {
    const uint32_t q = m ? __umulhi(x, m) : x;
    r = x - q * d;
    return q;
}

// member-0 smem index of class c (c < ncls): classes of stride st are grouped d*st apart
__device__ __forceinline__ uint32_t class_e0(uint32_t c, uint32_t st, uint32_t mst, uint32_t d) {
    uint32_t off;
    const uint32_t grp = tdiv(c, st, mst, off);
    return grp * st * d + off;
}

// What one gate needs to decide its classes inside the current tile.
struct TileGate {
    uint32_t LT, mLT, L, mL, len, flags;
    const uint32_t *mask;       // shared memory: member mask words 0..3, low-position mask 4..19
    const uint32_t *lowoff;     // shared memory: run offsets of the run-digit controls
};

// whether class e0 exists (ragged last tile of a run) and its in-tile controls hold
__device__ __forceinline__ bool class_ok(const TileGate &tg, const PassGateP &g, uint32_t e0) {
    uint32_t l;
    const uint32_t m = tdiv(e0, tg.LT, tg.mLT, l);
    // static masks are all ones where a gate has no such control: evaluated without branches
    uint32_t lq;
    tdiv(l, tg.L, tg.mL, lq);
    const uint32_t bits = (tg.mask[m >> 5] >> (m & 31)) & (tg.mask[4 + (lq >> 5)] >> (lq & 31));
    bool ok = (l < tg.len) & (bits & 1u);
    if (tg.flags & kFRunCtrl) {
#pragma unroll 1
        for (int k = 0; k < g.nctrl; ++k) {
            const PassCtrl &cc = g.c[k];
            if (cc.cls != 1) continue;
            uint32_t r, r2;
            fastdiv32(tg.lowoff[k] + l, cc.M, cc.mM, r);
            const uint32_t q = fastdiv32(r, cc.w, cc.mw, r2);
            fastdiv32(q, cc.d, cc.md, r2);
            ok = ok && (r2 == cc.v);
        }
    }
    return ok;
}

// an offset the compiler cannot prove zero: keeps the matrix reads inside the class loop
// (hoisting all d*d entries out of it would cost 4 d^2 registers per thread)
__device__ __forceinline__ uint32_t opaque_zero(uint32_t v) {
    uint32_t z;
    asm("and.b32 %0, %1, 0;" : "=r"(z) : "r"(v));
    return z;
}

// element (line r, position j along axis AX) of a 2-D class held as x[DA][DB]
template <int AX, int DA, int DB>
__device__ __forceinline__ double2 &ax_el(double2 (&x)[DA][DB], int r, int j) {
    return AX == 0 ? x[j][r] : x[r][j];
}

// cyclic shift with coefficients along one line: y_{(j+S) mod D} = c_j x_j (S compile-time)
template <int S, int D, int AX, int DA, int DB, int K>
__device__ __forceinline__ void shift_line(double2 (&x)[K][DA][DB], int r, const double2 (&cj)[D], bool pure,
                                           const bool (&ok)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double2 t[D];
#pragma unroll
        for (int j = 0; j < D; ++j) t[j] = ax_el<AX>(x[k], r, j);
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const double2 y = pure ? t[j] : cmul(cj[j], t[j]);
            if (ok[k]) ax_el<AX>(x[k], r, (j + S) % D) = y;
        }
    }
}

// One gate of a register stage along axis AX of the K classes x (every class
// vector along the target digit is replaced by U x; controls on the stage's other axis select
// the lines, other in-tile controls the classes via ok).
template <int AX, int DA, int DB, int K>
__device__ __forceinline__ void stage_gate(double2 (&x)[K][DA][DB], const PassGateP &g,
                                           const double2 *__restrict__ U, const bool (&ok)[K], uint32_t salt) {
    constexpr int D = AX == 0 ? DA : DB;     // target dimension
    constexpr int NL = AX == 0 ? DB : DA;    // lines along the target
    const int axctl = g.axctl;
    if (g.form == kFormDense) {
        const double2 *__restrict__ Ui = U + opaque_zero(salt);
#pragma unroll
        for (int r = 0; r < NL; ++r) {
            if (axctl >= 0 && r != axctl) continue;
            double2 y[K][D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
#pragma unroll
                for (int k = 0; k < K; ++k) y[k][i] = make_double2(0.0, 0.0);
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    const double2 u = Ui[i * D + j];
#pragma unroll
                    for (int k = 0; k < K; ++k) cfma(y[k][i], u, ax_el<AX>(x[k], r, j));
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int i = 0; i < D; ++i)
                    if (ok[k]) ax_el<AX>(x[k], r, i) = y[k][i];
        }
    } else {
        double2 cj[D];
#pragma unroll
        for (int j = 0; j < D; ++j) cj[j] = U[j];
        const bool pure = g.pure != 0;
#pragma unroll
        for (int r = 0; r < NL; ++r) {
            if (axctl >= 0 && r != axctl) continue;
            switch (g.shift) {
                case 0: shift_line<0, D, AX>(x, r, cj, pure, ok); break;
                case 1: shift_line<1 % D, D, AX>(x, r, cj, pure, ok); break;
                case 2: shift_line<2 % D, D, AX>(x, r, cj, pure, ok); break;
                case 3: shift_line<3 % D, D, AX>(x, r, cj, pure, ok); break;
                default: shift_line<4 % D, D, AX>(x, r, cj, pure, ok); break;
            }
        }
    }
}

// Classes per thread iteration of a stage with axis dimensions DA x DB (registers: 4 K DA DB
// for the gathered classes).
template <int DA, int DB> struct StageK {
    static constexpr int v = 12 / (DA * DB);
    static constexpr int value = v < 1 ? 1 : (v > 4 ? 4 : v);
};

// One register stage on one tile, classes [cbeg, cend) with stride NT (K per iteration).
template <int DA, int DB, int K, int NT>
__device__ __forceinline__ void stage_run(const PassParams &p, const PassStage &S, const TileGate &tg0,
                                          const uint32_t *masks, const uint32_t *lowoff, uint32_t fire,
                                          double2 *__restrict__ buf, const double2 *__restrict__ Us,
                                          uint32_t cbeg, uint32_t cend, uint32_t ncls, int tid) {
    const bool ragged = tg0.len < tg0.LT;
#pragma unroll 1
    for (uint32_t c0 = cbeg + (uint32_t)tid; c0 < cend; c0 += (uint32_t)(NT * K)) {
        uint32_t e[K];
        bool ok[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t c = c0 + (uint32_t)(k * NT);
            ok[k] = c < ncls;
            uint32_t r1, r2;
            uint32_t v = tdiv(ok[k] ? c : 0u, S.s1, S.m1, r1) * S.s1 * S.d1 + r1;   // insert axis digit 1
            v = tdiv(v, S.s2, S.m2, r2) * S.s2 * S.d2 + r2;                           // insert axis digit 2
            e[k] = v;
            if (ragged && ok[k]) {
                uint32_t l;
                tdiv(v, tg0.LT, tg0.mLT, l);
                ok[k] = l < tg0.len;
            }
        }
        double2 x[K][DA][DB];
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int a = 0; a < DA; ++a)
#pragma unroll
                for (int b = 0; b < DB; ++b) x[k][a][b] = buf[e[k] + a * S.sta + b * S.stb];
#pragma unroll 1
        for (int gi = S.g0; gi < S.g1; ++gi) {
            if (!((fire >> gi) & 1)) continue;          // out-of-tile control unmet: uniform skip
            const PassGateP &g = p.g[gi];
            bool okg[K];
#pragma unroll
            for (int k = 0; k < K; ++k) okg[k] = ok[k];
            if (g.flags != 0) {
                TileGate tg = tg0;
                tg.flags = g.flags;
                tg.mask = masks + gi * kMaskWords;
                tg.lowoff = lowoff + gi * kMaxPassCtrl;
#pragma unroll
                for (int k = 0; k < K; ++k) okg[k] = okg[k] && class_ok(tg, g, e[k]);
            }
            if (g.axis == 0) stage_gate<0, DA, DB, K>(x, g, Us + g.uoff, okg, c0);
            else stage_gate<1, DA, DB, K>(x, g, Us + g.uoff, okg, c0);
        }
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int a = 0; a < DA; ++a)
#pragma unroll
                for (int b = 0; b < DB; ++b)
                    if (ok[k]) buf[e[k] + a * S.sta + b * S.stb] = x[k][a][b];
    }
}

template <int DA, int DB, int NT>
__device__ __forceinline__ void stage_tile(const PassParams &p, const PassStage &S, const TileGate &tg0,
                                           const uint32_t *masks, const uint32_t *lowoff, uint32_t fire,
                                           double2 *buf, const double2 *Us, uint32_t slots, int tid) {
    constexpr int K = StageK<DA, DB>::value;
    const uint32_t ncls = slots / (uint32_t)(DA * DB);
    // full batches of K classes per thread, then the remainder one class per thread
    if constexpr (K == 1) {
        stage_run<DA, DB, 1, NT>(p, S, tg0, masks, lowoff, fire, buf, Us, 0, ncls, ncls, tid);
    } else {
        const uint32_t full = ncls / (uint32_t)(NT * K) * (uint32_t)(NT * K);
        stage_run<DA, DB, K, NT>(p, S, tg0, masks, lowoff, fire, buf, Us, 0, full, ncls, tid);
        stage_run<DA, DB, 1, NT>(p, S, tg0, masks, lowoff, fire, buf, Us, full, ncls, ncls, tid);
    }
}

// generic dimension (d > 5): class by class along the target's own stride; out of line so its
// 16-wide register arrays do not inflate the kernel
__device__ __noinline__ void gate_tile_generic(const TileGate tg, const PassGateP &g, double2 *buf,
                                               const double2 *U, uint32_t ncls, int tid, int nt) {
    const int d = g.d;
    const bool needck = tg.flags != 0 || tg.len < tg.LT;
    for (uint32_t c = tid; c < ncls; c += nt) {
        uint32_t off;
        const uint32_t e0 = tdiv(c, g.st, g.mst, off) * g.st * (uint32_t)d + off;
        if (needck && !class_ok(tg, g, e0)) continue;
        double2 x[kMaxDim];
        if (g.kind == kGeneral) {
            for (int j = 0; j < d; ++j) x[j] = buf[e0 + j * g.st];
            for (int i = 0; i < d; ++i) {
                double2 acc = make_double2(0.0, 0.0);
                for (int j = 0; j < d; ++j) cfma(acc, U[i * d + j], x[j]);
                buf[e0 + i * g.st] = acc;
            }
        } else {
            for (int j = 0; j < d; ++j)
                if ((g.active >> j) & 1) x[j] = buf[e0 + j * g.st];
            for (int j = 0; j < d; ++j)
                if ((g.active >> j) & 1) buf[e0 + g.sigma[j] * g.st] = cmul(U[j], x[j]);
        }
    }
}

}  // namespace

// named barrier 1 + group: the compute warps of one consumer group only
__device__ __forceinline__ void compute_barrier(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp-specialised: warps 0..NT/32-1 compute, warp NT/32 is the producer (TMA loads, stage
// records, TMA stores).  full[s] completes when a tile's bytes have landed; done[s] when the
// compute warps have finished it (after fence.proxy.async, so the bulk store sees their writes).
// The compute warps form G consumer groups of NT/G threads; group g takes the CTA's tiles
// g, g+G, ... (ping-pong), so one group's barrier waits overlap the other groups' work.
template <int NT, int G>
__global__ void __launch_bounds__(NT + 32, 1) k_gate_pass(const __grid_constant__ PassParams p, int S, int TE) {
    constexpr int NTG = NT / G;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw);
    double2 *Us = bufs + (size_t)S * TE;                       // the pass's matrices
    uint32_t *masks = reinterpret_cast<uint32_t *>(Us + p.upool);
    StageInfo *sinfo = reinterpret_cast<StageInfo *>(masks + kMaxPassGates * kMaskWords);
    uint64_t *full = reinterpret_cast<uint64_t *>(sinfo + S);
    uint64_t *done = full + S;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&done[s], 1); }
        fence_mbar_init();
    }
    for (int k = tid; k < p.upool; k += NT + 32) Us[k] = p.U[k];
    for (int k = tid; k < p.ngates * kMaskWords; k += NT + 32) masks[k] = (&p.mask[0][0])[k];
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
    const uint32_t slots = (uint32_t)p.M * p.LT;
    const int grp = tid / NTG, gtid = tid % NTG;
    for (uint64_t i = (uint64_t)grp; i < my; i += (uint64_t)G) {
        const int s = (int)(i % (uint64_t)S);
        double2 *buf = bufs + (size_t)s * TE;
        mbar_wait(&full[s], (uint32_t)((i / (uint64_t)S) & 1));
        const StageInfo &si = sinfo[s];
        const uint32_t len = si.ti.len;
        const uint32_t fire = si.fire;
        TileGate tg0;
        tg0.LT = p.LT;
        tg0.mLT = p.mLT;
        tg0.L = p.L;
        tg0.mL = p.mL;
        tg0.len = len;
        tg0.flags = 0;
        tg0.mask = masks;
        tg0.lowoff = &si.lowoff[0][0];
        for (int sg = 0; sg < p.nstages; ++sg) {
            const PassStage &S = p.st[sg];
            if (sg > 0) compute_barrier(1 + grp, NTG);      // stages read what earlier ones wrote
            const uint32_t *lo = &si.lowoff[0][0];
            switch (S.da * 8 + S.db) {
                case 2 * 8 + 1: stage_tile<2, 1, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                case 3 * 8 + 1: stage_tile<3, 1, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                case 4 * 8 + 1: stage_tile<4, 1, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                case 5 * 8 + 1: stage_tile<5, 1, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                case 2 * 8 + 2: stage_tile<2, 2, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                case 2 * 8 + 3: stage_tile<2, 3, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                case 2 * 8 + 4: stage_tile<2, 4, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                case 2 * 8 + 5: stage_tile<2, 5, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                case 3 * 8 + 3: stage_tile<3, 3, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                case 3 * 8 + 4: stage_tile<3, 4, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                case 3 * 8 + 5: stage_tile<3, 5, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                case 4 * 8 + 4: stage_tile<4, 4, NTG>(p, S, tg0, masks, lo, fire, buf, Us, slots, gtid); break;
                default:                                      // generic stage: one gate of d > 5
                    for (int gi = S.g0; gi < S.g1; ++gi) {
                        if (!((fire >> gi) & 1)) continue;
                        const PassGateP &g = p.g[gi];
                        TileGate tg = tg0;
                        tg.flags = g.flags;
                        tg.mask = masks + gi * kMaskWords;
                        tg.lowoff = si.lowoff[gi];
                        if (gi > S.g0) compute_barrier(1 + grp, NTG);
                        gate_tile_generic(tg, g, buf, Us + g.uoff, slots / (uint32_t)g.d, gtid, NTG);
                    }
                    break;
            }
        }
        fence_proxy_async();
        compute_barrier(1 + grp, NTG);
        if (gtid == 0) mbar_arrive(&done[s]);
    }
}

template <int NT, int G>
cudaError_t launch_pass_t(const PassParams &p, cudaStream_t st, const LaunchCfg &cfg) {
    const int S = cfg.pass_stages, TE = cfg.pass_tile;
    // size for the largest matrix pool so the attribute and the occupancy are set once per config
    const size_t smem = (size_t)S * TE * sizeof(double2) + (size_t)kPoolC * sizeof(double2) +
                        (size_t)kMaxPassGates * kMaskWords * sizeof(uint32_t) +
                        (size_t)S * sizeof(StageInfo) + (size_t)2 * S * sizeof(uint64_t);
    static size_t configured = 0, occ_for = 0;
    static int occ = 1;
    if (configured < smem) {
        cudaError_t e = cudaFuncSetAttribute(k_gate_pass<NT, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    if (occ_for != smem) {   // resident CTAs per SM at this smem size (persistent grid)
        int o = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_gate_pass<NT, G>, NT + 32, smem) != cudaSuccess || o < 1) o = 1;
        occ = o;
        occ_for = smem;
    }
    const uint64_t cap = (uint64_t)cfg.num_sms * (uint64_t)occ;
    const unsigned grid = (unsigned)(p.ntiles < cap ? p.ntiles : cap);
    k_gate_pass<NT, G><<<grid, NT + 32, smem, st>>>(p, S, TE);
    return cudaGetLastError();
}

}  // namespace svi
