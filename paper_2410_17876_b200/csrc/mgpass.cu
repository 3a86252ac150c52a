// mgpass.cu — multi-gate cache-blocked pass kernel for sm_100a.
//
// One HBM pass applies a whole list of gates.  A tile holds every digit value of the in-tile
// qudits Q = {q_0..q_{m0-1}} ∪ H (plan_passes) and one value of every other digit, laid out in
// shared memory as [member][run] where a "member" is one combination of the H digits (global
// offset sum_h j_h b_h) and the run is a contiguous stretch of the low space (stride < b_{min H}).
// Loading / storing a tile = one cp.async.bulk per member (TMA bulk copies onto an mbarrier,
// persistent grid, a producer warp and NT compute threads).  Between load and store the CTA
// applies the pass's gates one after another in shared memory: each gate visits its
// equivalence classes inside the tile — a target in H has smem stride
// W_h * LT, a low target has stride b_t — and its controls are handled
//   * by enumeration for controls on H digits and low-prefix digits: their pinned values are
//     inserted into the class index next to the target digit (the §2.4 satisfying set is a
//     Cartesian product), so only firing classes are visited;
//   * per class from the tile's run offset: controls on run digits above the low prefix;
//   * once per tile: controls on digits outside the tile (the producer's fire bits).
// Two commuting qubit gates with the same controls may be applied together as one 4-member
// class (a "pair gate", member offsets from a per-gate table).  The compute threads form G
// consumer groups that ping-pong over the CTA's tiles.  The kernel is templated on the element
// type (complex128, or complex64 when every bulk copy is 16-byte aligned).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "sv_internal.h"
#include "plan.h"

namespace svi {

constexpr int kMaxPassGates = 32;            // fire bits: one 32-bit ballot
constexpr int kMaxMembers = 128;
constexpr int kPoolC = 768;
constexpr int kMaxPassCtrl = 4;
constexpr int kMaxIns = 2 + kMaxPassCtrl;   // inserted in-tile digits: the target(s) + pinned controls
constexpr int kMaxPairDim = 4;             // pair gates: d_a d_b <= 4 (qubit pairs)

// in-pass gate kinds: general y = U x (§2.3), monomial y_{sigma(j)} = c_j x_j (§2.1-2.2),
// and the pure permutation (every moving coefficient exactly 1: no arithmetic at all)
enum PassKind : int32_t { kPGeneral = 0, kPMonomial = 1, kPPerm = 2 };

// a control decided at run time (in-tile controls on H / low-prefix digits are enumerated)
// Run-digit controls (digits below min H and above the low prefix) come in two forms:
//   cls 1: b_c d_c < 2^31 — the digit of run position s0 + l is read from (s0 mod b_c d_c) + l
//          in 32-bit arithmetic (fastdiv32 is exact for divisors <= 2^31);
//   cls 3: b_c d_c >= 2^31 (registers with D > 2^32 whose pass has no H digit, so a run spans
//          the register) — b_c >= 2^27 exceeds any tile, so the digit changes at most once
//          inside a tile; the producer decides, in 64-bit arithmetic, the range of l where it
//          equals the control value.
struct PassCtrl {
    int32_t cls;          // 1, 3 = run digit above the low prefix (see above), 2 = outside the tile
    uint32_t v;
    uint32_t d, md;       // control dimension (+ magic)
    uint32_t w, mw;       // cls 1: stride b_c (+ magic)
    uint32_t M, mM;       // cls 1: b_c * d_c < 2^31 (+ magic)
    uint64_t b64, mb64;   // cls 2, 3: global stride (+ magic); cls 1: 64-bit magic of M
    uint64_t md64;        // cls 2, 3: magic for d
};

// cls 3 per-tile record: the control holds for run positions l < t (mode 1), l >= t (mode 2)
// or none (mode 0); t < 2^30 is clamped (tiles are at most 8192 positions long).
constexpr uint32_t kCls3Mask = (1u << 30) - 1u;

enum PassFlags : uint32_t { kFRunCtrl = 4 };

struct PassGateP {
    int32_t d, kind, nctrl, uoff;
    uint32_t flags;       // PassFlags: which in-tile control checks the gate needs
    uint32_t st, mst;     // smem stride of the target (+ magic)
    uint32_t ncls;        // classes per full tile: M LT / (d prod of the inserted control dims)
    int32_t nins;         // digits inserted into the class index, ascending tile stride:
    uint32_t ins_s[kMaxIns], ins_m[kMaxIns];    //   stride (+ magic)
    uint32_t ins_sd[kMaxIns], ins_ps[kMaxIns];  //   stride * dim, pinned value * stride
    uint32_t active;      // monomial / permutation: members that move or scale
    int8_t sigma[kMaxDim];
    PassCtrl c[kMaxPassCtrl];
};

struct PassParams {
    double2 *psi;
    int32_t nrem;
    RemovedRun rem[kMaxRem];
    uint64_t ntiles, R, tpr, tpr_m;
    uint32_t LT, mLT;     // run elements per member in a tile (+ magic)
    uint32_t L, mL;       // low-prefix block b_{m0} (+ magic)
    int32_t M;            // members per tile
    int32_t ngates;
    int32_t upool;        // used entries of U (copied to shared memory at kernel start)
    uint64_t moff[kMaxMembers];
    PassGateP g[kMaxPassGates];
    uint32_t moff_t[kMaxPassGates][kMaxDim];   // per gate: tile offset of class member j
    uint32_t soff_t[kMaxPassGates][kMaxDim];   // per gate: offset of member sigma(j) (monomial)
    double2 U[kPoolC];    // general: row-major d x d; monomial: coefficient per member
};

static_assert(sizeof(PassParams) <= 32764, "kernel parameter space (32 KB on sm_100)");

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

template <typename V>
__device__ __forceinline__ void issue_loads(const PassParams &p, uint64_t t, V *buf, uint64_t *bar,
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
            } else if (cc.cls == 3) {
                uint64_t r0, dig;
                const uint64_t q = fastdiv64(ti.s0, cc.b64, cc.mb64, r0);
                fastdiv64(q, cc.d, cc.md64, dig);                  // digit of q_c at position s0
                const uint64_t nxt = (dig + 1 == cc.d) ? 0 : dig + 1;   // after the one change
                uint64_t t = cc.b64 - r0;                          // first l where the digit changes
                if (t > kCls3Mask) t = kCls3Mask;
                const uint32_t mode = dig == cc.v ? 1u : (nxt == cc.v ? 2u : 0u);
                si->lowoff[lane][k] = (uint32_t)t | (mode << 30);
            }
        }
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, fire && lane < p.ngates);
    if (lane == 0) {
        si->ti = ti;
        si->fire = bits;
    }
    __syncwarp();
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)p.M * ti.len * (uint32_t)sizeof(V));
    __syncwarp();
    for (int m = lane; m < p.M; m += 32)
        bulk_load(buf + (size_t)m * p.LT, reinterpret_cast<const V *>(p.psi) + ti.gbase + p.moff[m],
                  ti.len * (uint32_t)sizeof(V), bar);
}

// In-tile division (x < 2^16, d < 2^16): with m = floor(2^32/d) + 1, umulhi(x, m) is exact
// because x * (m d - 2^32) <= x d < 2^32, so no fix-up step is needed (d == 1 <=> m == 0).
__device__ __forceinline__ uint32_t tdiv(uint32_t x, uint32_t d, uint32_t m, uint32_t &r) {
    const uint32_t q = m ? __umulhi(x, m) : x;
    r = x - q * d;
    return q;
}

// member-0 tile index of class c (c < ncls): the target digit (value 0) and the pinned in-tile
// control digits inserted into c in ascending stride order, e <- (e / s) s d + pin s + e mod s
// (SURVEY.md §8 a3 inside the tile)
struct Ins1 {            // one insertion, held in registers across a class loop
    uint32_t s, m, sd, ps;
};
__device__ __forceinline__ Ins1 ins_at(const PassGateP &g, int i) {
    return Ins1{g.ins_s[i], g.ins_m[i], g.ins_sd[i], g.ins_ps[i]};
}
__device__ __forceinline__ uint32_t insert1(uint32_t e, const Ins1 &a) {
    uint32_t r;
    const uint32_t q = tdiv(e, a.s, a.m, r);
    return q * a.sd + a.ps + r;
}
// first insertion from registers (the common uncontrolled case has only it), further ones
// (in-tile controls) from the parameter bank
__device__ __forceinline__ uint32_t class_e0(uint32_t c, const PassGateP &g, const Ins1 &first, bool more) {
    uint32_t e = insert1(c, first);
    if (more) {
#pragma unroll 1
        for (int i = 1; i < g.nins; ++i) e = insert1(e, ins_at(g, i));
    }
    return e;
}

// What one gate needs to decide its classes inside the current tile.
struct TileGate {
    uint32_t LT, mLT, len, flags;
    const uint32_t *lowoff;     // shared memory: run offsets of the run-digit controls
    const uint32_t *moff;       // shared memory: tile offset of class member j (j st, or the
                                //   two-digit offset of a pair gate)
    const uint32_t *soff;       // shared memory: offset of member sigma(j) (monomial gates)
};

// whether class e0 exists (ragged last tile of a run) and its in-tile controls hold
__device__ __forceinline__ bool class_ok(const TileGate &tg, const PassGateP &g, uint32_t e0) {
    uint32_t l;
    tdiv(e0, tg.LT, tg.mLT, l);
    bool ok = l < tg.len;
    if (tg.flags & kFRunCtrl) {
#pragma unroll 1
        for (int k = 0; k < g.nctrl; ++k) {
            const PassCtrl &cc = g.c[k];
            if (cc.cls == 3) {
                const uint32_t x = tg.lowoff[k], t = x & kCls3Mask, mode = x >> 30;
                ok = ok && (mode == 1 ? l < t : (mode == 2 && l >= t));
                continue;
            }
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

// The K classes c0, c0+NT, ..., c0+(K-1)NT of one thread iteration (a warp's accesses stay
// contiguous for strides >= 32): member-0 smem index and whether the class exists and fires.
// Classes past ncls read index 0 and do not store.
template <int K, int NT>
__device__ __forceinline__ void class_batch(const TileGate &tg, const PassGateP &g, const Ins1 &first, bool more,
                                            uint32_t c0, uint32_t ncls, bool needck, uint32_t (&e)[K],
                                            bool (&ok)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t c = c0 + (uint32_t)(k * NT);
        ok[k] = c < ncls;
        e[k] = ok[k] ? class_e0(c, g, first, more) : 0u;
        if (needck && ok[k]) ok[k] = class_ok(tg, g, e[k]);
    }
}

// an offset the compiler cannot prove zero: keeps the matrix reads inside the class loop
// (hoisting all d*d entries out of it would cost 4 d^2 registers per thread)
__device__ __forceinline__ uint32_t opaque_zero(uint32_t v) {
    uint32_t z;
    asm("and.b32 %0, %1, 0;" : "=r"(z) : "r"(v));
    return z;
}

// Tile accesses through 32-bit shared-window addresses computed once per gate: with the
// pointer form, ptxas (at 96 registers) re-derived the CTA's shared window base (S2R
// SR_CgaCtaId + LEA) for every store.  volatile keeps their order (class gathers before
// scatters, gates separated by the group barrier).
template <typename V> __device__ __forceinline__ V lds2(uint32_t a);
template <> __device__ __forceinline__ double2 lds2<double2>(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
template <> __device__ __forceinline__ float2 lds2<float2>(uint32_t a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts2(uint32_t a, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void sts2(uint32_t a, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}

// One general gate (y = U x per class) on one tile, K classes per thread
// iteration.  All K*D gathers are issued before the matvecs; buf and U are restrict-qualified
// so the matrix reads may be scheduled across the stores of earlier rows.
template <int D, int K, int NT, typename V>
__device__ __forceinline__ void gate_tile_general(const TileGate &tg, const PassGateP &g, V *__restrict__ buf,
                                                  const V *__restrict__ U, uint32_t cbeg, uint32_t cend,
                                                  uint32_t ncls, bool needck, int tid) {
    // member offsets, read once from shared memory (the stores below may alias that table as
    // far as the compiler knows, so it keeps them in registers)
    uint32_t mo[D];
#pragma unroll
    for (int j = 0; j < D; ++j) mo[j] = tg.moff[j] * (uint32_t)sizeof(V);
    const uint32_t sb = smem_u32(buf);
    const Ins1 first = ins_at(g, 0);
    const bool more = g.nins > 1;
#pragma unroll 1
    for (uint32_t c0 = cbeg + (uint32_t)tid; c0 < cend; c0 += (uint32_t)(NT * K)) {
        uint32_t e[K];
        bool ok[K];
        class_batch<K, NT>(tg, g, first, more, c0, ncls, needck, e, ok);
        const V *__restrict__ Ui = U + opaque_zero(c0);
        V x[K][D];
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int j = 0; j < D; ++j) x[k][j] = lds2<V>(sb + e[k] * (uint32_t)sizeof(V) + mo[j]);
#pragma unroll
        for (int i = 0; i < D; ++i) {
            V acc[K];
#pragma unroll
            for (int k = 0; k < K; ++k) acc[k] = cz<V>();
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const V u = Ui[i * D + j];
#pragma unroll
                for (int k = 0; k < K; ++k) cfma(acc[k], u, x[k][j]);
            }
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (ok[k]) sts2(sb + e[k] * (uint32_t)sizeof(V) + mo[i], acc[k]);
        }
    }
}

// One monomial gate (phase / permutation, y_{sigma(j)} = c_j x_j) on one
// tile; PERM: every moving coefficient is exactly 1, so the gate only moves data.  Only the
// members that move or scale are read and written (select-form predicated gathers: a branch
// per member makes ptxas spill the array).
template <int D, int K, int NT, bool PERM, typename V>
__device__ __forceinline__ void gate_tile_monomial(const TileGate &tg, const PassGateP &g, V *__restrict__ buf,
                                                   const V *__restrict__ U, uint32_t cbeg, uint32_t cend,
                                                   uint32_t ncls, bool needck, int tid) {
    const uint32_t act = g.active;
    const Ins1 first = ins_at(g, 0);
    const bool more = g.nins > 1;
    // destination offsets sigma(j) * st, read once from shared memory: the stores below may
    // alias that table as far as the compiler knows, so it keeps them in registers instead of
    // re-reading the parameter bank inside the loop
    uint32_t so[D], mo[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
        so[j] = tg.soff[j] * (uint32_t)sizeof(V);
        mo[j] = tg.moff[j] * (uint32_t)sizeof(V);
    }
    const uint32_t sb = smem_u32(buf);
#pragma unroll 1
    for (uint32_t c0 = cbeg + (uint32_t)tid; c0 < cend; c0 += (uint32_t)(NT * K)) {
        uint32_t e[K];
        bool ok[K];
        class_batch<K, NT>(tg, g, first, more, c0, ncls, needck, e, ok);
        V x[K][D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const bool aj = (act >> j) & 1;
#pragma unroll
            for (int k = 0; k < K; ++k)
                x[k][j] = aj ? lds2<V>(sb + e[k] * (uint32_t)sizeof(V) + mo[j]) : cz<V>();
        }
#pragma unroll
        for (int j = 0; j < D; ++j)
            if ((act >> j) & 1) {
                if (PERM) {
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        if (ok[k]) sts2(sb + e[k] * (uint32_t)sizeof(V) + so[j], x[k][j]);
                } else {
                    const V u = U[j];
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        if (ok[k]) sts2(sb + e[k] * (uint32_t)sizeof(V) + so[j], cmul(u, x[k][j]));
                }
            }
    }
}

// generic dimension (fused or d > 5): out of line so its 16-wide register arrays do not
// inflate the kernel
template <typename V>
__device__ __noinline__ void gate_tile_generic(const TileGate tg, const PassGateP &g, V *buf,
                                               const V *U, uint32_t ncls, bool needck, int tid, int nt) {
    const int d = g.d;
    for (uint32_t c = tid; c < ncls; c += nt) {
        const uint32_t e0 = class_e0(c, g, ins_at(g, 0), true);
        if (needck && !class_ok(tg, g, e0)) continue;
        V x[kMaxDim];
        if (g.kind == kPGeneral) {
            for (int j = 0; j < d; ++j) x[j] = buf[e0 + tg.moff[j]];
            for (int i = 0; i < d; ++i) {
                V acc = cz<V>();
                for (int j = 0; j < d; ++j) cfma(acc, U[i * d + j], x[j]);
                buf[e0 + tg.moff[i]] = acc;
            }
        } else {
            for (int j = 0; j < d; ++j)
                if ((g.active >> j) & 1) x[j] = buf[e0 + tg.moff[j]];
            for (int j = 0; j < d; ++j)
                if ((g.active >> j) & 1) buf[e0 + tg.soff[j]] = cmul(U[j], x[j]);
        }
    }
}

// classes per thread iteration (registers: 4*K*D for the gathered classes), by thread count:
// 256 threads may use up to ~200 registers, 384 up to 152, 512 up to 120
template <int D, int NT> struct PassK { static constexpr int value = 1; };
template <int NT> struct PassK<2, NT> { static constexpr int value = 4; };
template <int NT> struct PassK<3, NT> { static constexpr int value = NT >= 512 ? 3 : 4; };
template <int NT> struct PassK<4, NT> { static constexpr int value = NT >= 512 ? 2 : 3; };
template <int NT> struct PassK<5, NT> { static constexpr int value = NT >= 384 ? 2 : 3; };

// NT = compute threads of the CTA (sets the register budget), NTG = threads of one consumer
// group (the class stride)
template <int D, int NT, int NTG, typename V>
__device__ __forceinline__ void apply_gate_tile(const TileGate &tg, const PassGateP &g, V *buf,
                                                const V *U, uint32_t ncls, bool needck, int tid) {
    constexpr int K = PassK<D, NT>::value;
    // full batches of K classes per thread, then the remainder one class per thread (no idle
    // batch slots in the tail)
    const uint32_t full = ncls / (uint32_t)(NTG * K) * (uint32_t)(NTG * K);
    if (g.kind == kPGeneral) {
        gate_tile_general<D, K, NTG, V>(tg, g, buf, U, 0, full, ncls, needck, tid);
        gate_tile_general<D, 1, NTG, V>(tg, g, buf, U, full, ncls, ncls, needck, tid);
    } else if (g.kind == kPPerm) {
        gate_tile_monomial<D, K, NTG, true, V>(tg, g, buf, U, 0, full, ncls, needck, tid);
        gate_tile_monomial<D, 1, NTG, true, V>(tg, g, buf, U, full, ncls, ncls, needck, tid);
    } else {
        gate_tile_monomial<D, K, NTG, false, V>(tg, g, buf, U, 0, full, ncls, needck, tid);
        gate_tile_monomial<D, 1, NTG, false, V>(tg, g, buf, U, full, ncls, ncls, needck, tid);
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
template <int NT, int G, typename V>
__global__ void __launch_bounds__(NT + 32, 1) k_gate_pass(const __grid_constant__ PassParams p, int S, int TE) {
    constexpr int NTG = NT / G;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    V *bufs = reinterpret_cast<V *>(smem_raw);
    V *Us = bufs + (size_t)S * TE;                             // the pass's matrices (in V's precision)
    uint32_t *moffs = reinterpret_cast<uint32_t *>(Us + p.upool);   // per gate: member offsets
    uint32_t *soffs = moffs + kMaxPassGates * kMaxDim;               // per gate: sigma-member offsets
    StageInfo *sinfo = reinterpret_cast<StageInfo *>(soffs + kMaxPassGates * kMaxDim);
    uint64_t *full = reinterpret_cast<uint64_t *>(sinfo + S);
    uint64_t *done = full + S;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&done[s], 1); }
        fence_mbar_init();
    }
    for (int k = tid; k < p.upool; k += NT + 32) Us[k] = to_v<V>(p.U[k]);
    for (int k = tid; k < p.ngates * kMaxDim; k += NT + 32) {
        moffs[k] = (&p.moff_t[0][0])[k];
        soffs[k] = (&p.soff_t[0][0])[k];
    }
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
                    bulk_store(reinterpret_cast<V *>(p.psi) + si.ti.gbase + p.moff[m],
                               bufs + (size_t)s * TE + (size_t)m * p.LT, si.ti.len * (uint32_t)sizeof(V));
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
    const int grp = tid / NTG, gtid = tid % NTG;
    for (uint64_t i = (uint64_t)grp; i < my; i += (uint64_t)G) {
        const int s = (int)(i % (uint64_t)S);
        V *buf = bufs + (size_t)s * TE;
        // With several groups, consecutive tiles of a stage belong to different groups, so this
        // group may reach tile i while the stage's previous tile (i - S, another group) is not
        // even loaded: full[s] would still be in the phase before the one awaited, and a parity
        // wait cannot tell a phase two steps back from a completed one.  Waiting first for
        // tile i - S to be consumed (done[s], whose previous phase this group completed itself)
        // puts full[s] exactly one phase before tile i.
        if (G > 1 && i >= (uint64_t)S) mbar_wait(&done[s], (uint32_t)(((i - (uint64_t)S) / (uint64_t)S) & 1));
        mbar_wait(&full[s], (uint32_t)((i / (uint64_t)S) & 1));
        const StageInfo &si = sinfo[s];
        const uint32_t len = si.ti.len;
        const uint32_t fire = si.fire;
        for (int gi = 0; gi < p.ngates; ++gi) {
            if (!((fire >> gi) & 1)) continue;          // out-of-tile control unmet: uniform skip
            const PassGateP &g = p.g[gi];
            TileGate tg;
            tg.LT = p.LT;
            tg.mLT = p.mLT;
            tg.len = len;
            tg.flags = g.flags;
            tg.lowoff = si.lowoff[gi];
            tg.moff = &p.moff_t[gi][0];          // parameter bank (uniform across the CTA)
            tg.soff = &p.soff_t[gi][0];
            const bool needck = g.flags != 0 || len < p.LT;
            const V *U = Us + g.uoff;
            switch (g.d) {
                case 2: apply_gate_tile<2, NT, NTG, V>(tg, g, buf, U, g.ncls, needck, gtid); break;
                case 3: apply_gate_tile<3, NT, NTG, V>(tg, g, buf, U, g.ncls, needck, gtid); break;
                case 4: apply_gate_tile<4, NT, NTG, V>(tg, g, buf, U, g.ncls, needck, gtid); break;
                case 5: apply_gate_tile<5, NT, NTG, V>(tg, g, buf, U, g.ncls, needck, gtid); break;
                default: gate_tile_generic<V>(tg, g, buf, U, g.ncls, needck, gtid, NTG); break;
            }
            compute_barrier(1 + grp, NTG);
        }
        fence_proxy_async();
        compute_barrier(1 + grp, NTG);
        if (gtid == 0) mbar_arrive(&done[s]);
    }
}

// ------------------------------------------------------------------------------ host
// Build the pass parameters; returns false if the pass does not fit this kernel.
bool build_pass(const Register &reg, const std::vector<GateSpec> &gates, const PassPlan &pp, double2 *psi,
                int TE, PassParams &p, PassWork *work) {
    std::memset(&p, 0, sizeof(p));
    if ((int)pp.gates.size() > kMaxPassGates || pp.tile > (uint64_t)TE) return false;
    p.psi = psi;
    const int m0 = pp.m0;
    const uint64_t L = (m0 < reg.n) ? reg.b[m0] : reg.D;
    p.L = (uint32_t)L;
    p.mL = make_fastdiv32(p.L).m;
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
    // The run per member is widened to fill the tile (a multiple of L = b_{m0}, so low-prefix
    // classes stay whole and every tile starts at a multiple of L, and at most the run R below
    // min H).
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
    auto in_tile = [&](int q) {
        return q < m0 || std::find(pp.H.begin(), pp.H.end(), q) != pp.H.end();
    };
    auto tile_stride = [&](int q) -> uint64_t { return q < m0 ? reg.b[q] : W[q] * LT; };
    for (int i : pp.gates) {
        const GateSpec &g = gates[i];
        if (g.span != 1 || !in_tile(g.target) || (int)g.ctrl.size() > kMaxPassCtrl) return false;
    }
    // Pair gates: a gate joins an earlier, still single gate of the pass on another in-tile digit
    // with the same controls (neither target controlling the other) when every gate in between
    // commutes with it; the two then act as one gate on the two digits, U_b (x) U_a, with
    // d_a d_b <= kMaxPairDim classes members: one shared-memory round trip instead of two.
    struct Item { int a, b; };          // gate indices (b = -1: single)
    std::vector<Item> items;
    for (int i : pp.gates) {
        const GateSpec &g = gates[i];
        bool paired = false;
        for (int j = (int)items.size() - 1; j >= 0; --j) {
            Item &it = items[j];
            const GateSpec &h = gates[it.a];
            if (it.b < 0 && h.target != g.target && h.d <= 5 && g.d <= 5 && h.d * g.d <= kMaxPairDim &&
                same_controls(h, g)) {
                bool cross = false;
                for (const auto &c : g.ctrl) cross = cross || c.q == h.target;
                for (const auto &c : h.ctrl) cross = cross || c.q == g.target;
                if (!cross) {
                    it.b = i;
                    paired = true;
                    break;
                }
            }
            if (!commute(gates[it.a], g) || (it.b >= 0 && !commute(gates[it.b], g))) break;
        }
        if (!paired) items.push_back({i, -1});
    }
    // gates
    int uoff = 0;
    *work = PassWork{};
    p.ngates = (int32_t)items.size();
    for (size_t gi = 0; gi < items.size(); ++gi) {
        const GateSpec &g = gates[items[gi].a];
        GatePlan gp;
        std::string err;
        if (plan_gate(reg, g, false, &gp, &err) != SV_OK) return false;
        work->touched += (double)gp.touched;
        PassGateP &q = p.g[gi];
        const int t = g.target;
        const uint64_t st = tile_stride(t);
        q.st = (uint32_t)st;
        q.mst = make_fastdiv32(q.st).m;
        struct Ins { uint64_t s; uint32_t d, pin; };
        std::vector<Ins> ins{{st, (uint32_t)gp.d, 0u}};
        uint64_t cls_div = (uint64_t)gp.d;
        int D = gp.d;
        // member offsets, coefficients / matrix, sigma of this (possibly pair) gate
        std::vector<uint32_t> moff(kMaxDim, 0), sig(kMaxDim, 0);
        std::vector<double2> Ud;                  // dense D x D or coefficients
        int kind = gp.kind;
        if (items[gi].b < 0) {
            for (int j = 0; j < D; ++j) { moff[j] = (uint32_t)(j * st); sig[j] = (uint32_t)gp.sigma[j]; }
            q.active = gp.active;
            const int need = gp.kind == kGeneral ? D * D : D;
            Ud.assign(gp.U, gp.U + need);
        } else {
            const GateSpec &h = gates[items[gi].b];      // h acts on digit b (second), g on a
            GatePlan hp;
            if (plan_gate(reg, h, false, &hp, &err) != SV_OK) return false;
            work->touched += (double)hp.touched;
            const int da = gp.d, db = hp.d;
            D = da * db;
            const uint64_t stb = tile_stride(h.target);
            ins.push_back({stb, (uint32_t)db, 0u});
            cls_div *= (uint64_t)db;
            for (int jb = 0; jb < db; ++jb)
                for (int ja = 0; ja < da; ++ja) moff[ja + da * jb] = (uint32_t)(ja * st + jb * stb);
            if (gp.kind == kMonomial && hp.kind == kMonomial) {
                kind = kMonomial;
                uint32_t act = 0;
                Ud.resize(D);
                for (int jb = 0; jb < db; ++jb)
                    for (int ja = 0; ja < da; ++ja) {
                        const int J = ja + da * jb;
                        sig[J] = (uint32_t)(gp.sigma[ja] + da * hp.sigma[jb]);
                        const double2 ca = gp.U[ja], cb = hp.U[jb];
                        Ud[J] = make_double2(ca.x * cb.x - ca.y * cb.y, ca.x * cb.y + ca.y * cb.x);
                        if (sig[J] != (uint32_t)J || Ud[J].x != 1.0 || Ud[J].y != 0.0) act |= 1u << J;
                    }
                q.active = act;
            } else {
                kind = kGeneral;
                q.active = (1u << D) - 1u;
                Ud.resize((size_t)D * D);
                for (int ib = 0; ib < db; ++ib)
                    for (int ia = 0; ia < da; ++ia)
                        for (int jb = 0; jb < db; ++jb)
                            for (int ja = 0; ja < da; ++ja) {
                                const double2 ua = g.U[ia * da + ja], ub = h.U[ib * db + jb];
                                Ud[(ia + da * ib) * D + (ja + da * jb)] =
                                    make_double2(ua.x * ub.x - ua.y * ub.y, ua.x * ub.y + ua.y * ub.x);
                            }
                for (int J = 0; J < D; ++J) sig[J] = (uint32_t)J;
            }
        }
        q.d = D;
        q.kind = kind == kGeneral ? kPGeneral : kPMonomial;
        {   // executed work of this item: its control-satisfying classes x moving members
            double cprod = 1.0;
            for (const auto &c : g.ctrl) cprod *= (double)reg.dims[c.q];
            const double nact = (double)__builtin_popcount(q.active);
            const double it = (double)reg.D / ((double)D * cprod) * nact;
            work->item_touched += it;
            if (kind == kGeneral) work->flops += 8.0 * D * it;
        }
        if (q.kind == kPMonomial) {            // every moving coefficient exactly 1: pure data movement
            bool perm = true;
            for (int j = 0; j < D; ++j)
                if (((q.active >> j) & 1) && !(Ud[j].x == 1.0 && Ud[j].y == 0.0)) perm = false;
            if (perm) q.kind = kPPerm;
        }
        for (int j = 0; j < kMaxDim; ++j) {
            q.sigma[j] = (int8_t)(j < D ? sig[j] : j);
            p.moff_t[gi][j] = moff[j];
            p.soff_t[gi][j] = j < D ? moff[sig[j]] : 0u;
        }
        const int need = (int)Ud.size();
        if (uoff + need > kPoolC) return false;
        q.uoff = uoff;
        for (int k = 0; k < need; ++k) p.U[uoff + k] = Ud[k];
        uoff += need;
        p.upool = uoff;
        // in-tile controls on H / low-prefix digits are inserted into the class index with
        // their pinned values (only firing classes are visited); the rest are decided at run time
        int nc = 0;
        for (size_t k = 0; k < g.ctrl.size(); ++k) {
            const int c = g.ctrl[k].q;
            const uint32_t v = (uint32_t)g.ctrl[k].v;
            const uint64_t dc = (uint64_t)reg.dims[c];
            const bool inH = std::find(pp.H.begin(), pp.H.end(), c) != pp.H.end();
            if (inH || c < m0) {
                ins.push_back({inH ? W[c] * LT : reg.b[c], (uint32_t)dc, v});
                cls_div *= dc;
                continue;
            }
            PassCtrl &cc = q.c[nc++];
            cc.v = v;
            cc.d = (uint32_t)dc;
            cc.md = make_fastdiv32(cc.d).m;
            if (reg.b[c] < R && reg.b[c] * dc < (1ull << 31)) {   // run digit: tile's run offset
                cc.cls = 1;
                q.flags |= kFRunCtrl;
                cc.w = (uint32_t)reg.b[c];
                cc.mw = make_fastdiv32(cc.w).m;
                cc.M = cc.w * cc.d;
                cc.mM = make_fastdiv32(cc.M).m;
                cc.mb64 = make_fastdiv64(cc.M).m;
            } else if (reg.b[c] < R) {         // run digit with b_c d_c >= 2^31: per-tile threshold
                cc.cls = 3;
                q.flags |= kFRunCtrl;
                cc.b64 = reg.b[c];
                cc.mb64 = make_fastdiv64(cc.b64).m;
                cc.md64 = make_fastdiv64(dc).m;
            } else {                           // outside the tile: constant per tile
                cc.cls = 2;
                cc.b64 = reg.b[c];
                cc.mb64 = make_fastdiv64(cc.b64).m;
                cc.md64 = make_fastdiv64(cc.d).m;
            }
        }
        q.nctrl = nc;
        if ((int)ins.size() > kMaxIns) return false;
        std::sort(ins.begin(), ins.end(), [](const Ins &a, const Ins &b) { return a.s < b.s; });
        q.nins = (int32_t)ins.size();
        for (size_t i = 0; i < ins.size(); ++i) {
            q.ins_s[i] = (uint32_t)ins[i].s;
            q.ins_m[i] = make_fastdiv32(q.ins_s[i]).m;
            q.ins_sd[i] = (uint32_t)(ins[i].s * ins[i].d);
            q.ins_ps[i] = (uint32_t)(ins[i].s * ins[i].pin);
        }
        q.ncls = (uint32_t)((uint64_t)M * LT / cls_div);
    }
    return p.ntiles > 0;
}

template <int NT, int G, typename V>
cudaError_t launch_pass_t(const PassParams &p, cudaStream_t st, const LaunchCfg &cfg) {
    const int S = cfg.pass_stages, TE = cfg.pass_tile;
    // size for the largest matrix pool so the attribute and the occupancy are set once per config
    const size_t smem = (size_t)S * TE * sizeof(V) + (size_t)kPoolC * sizeof(V) +
                        (size_t)2 * kMaxPassGates * kMaxDim * sizeof(uint32_t) +
                        (size_t)S * sizeof(StageInfo) + (size_t)2 * S * sizeof(uint64_t);
    static LaunchAttr attr;
    const int dv = current_device_slot();
    if (attr.configured[dv] < smem) {
        cudaError_t e = cudaFuncSetAttribute(k_gate_pass<NT, G, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr.configured[dv] = smem;
    }
    if (attr.occ_for[dv] != smem) {   // resident CTAs per SM at this smem size (persistent grid)
        int o = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_gate_pass<NT, G, V>, NT + 32, smem) != cudaSuccess || o < 1) o = 1;
        attr.occ[dv] = o;
        attr.occ_for[dv] = smem;
    }
    const uint64_t cap = (uint64_t)cfg.num_sms * (uint64_t)attr.occ[dv];
    const unsigned grid = (unsigned)(p.ntiles < cap ? p.ntiles : cap);
    k_gate_pass<NT, G, V><<<grid, NT + 32, smem, st>>>(p, S, TE);
    return cudaGetLastError();
}

cudaError_t launch_pass(const PassParams &p, cudaStream_t st, const LaunchCfg &cfg) {
    if (cfg.c64) return launch_pass_t<512, 2, float2>(p, st, cfg);   // complex64: one configuration
    int G = cfg.pass_groups;                      // one stage per group at least
    while (G > 1 && cfg.pass_stages < G) G /= 2;
    if (cfg.pass_threads >= 512) {
        if (G >= 4) return launch_pass_t<512, 4, double2>(p, st, cfg);
        if (G == 2) return launch_pass_t<512, 2, double2>(p, st, cfg);
        return launch_pass_t<512, 1, double2>(p, st, cfg);
    }
    if (cfg.pass_threads >= 384) {
        if (G >= 2) return launch_pass_t<384, 2, double2>(p, st, cfg);
        return launch_pass_t<384, 1, double2>(p, st, cfg);
    }
    if (G >= 2) return launch_pass_t<256, 2, double2>(p, st, cfg);
    return launch_pass_t<256, 1, double2>(p, st, cfg);
}

cudaError_t run_pass(const Register &reg, const std::vector<GateSpec> &gates, const PassPlan &pp, double2 *psi,
                     cudaStream_t st, const LaunchCfg &cfg, bool *handled, PassWork *work) {
    static thread_local PassParams p;   // ~23 KB; parameters are copied at launch
    *handled = build_pass(reg, gates, pp, psi, cfg.pass_tile, p, work);
    // complex64 (8-byte elements): every bulk copy must start at a 16-byte aligned address and
    // move a multiple of 16 bytes; tile runs are multiples of L = b_{m0} and start at multiples
    // of L, so an even L suffices (the stage needs the tile plus the fp32 matrix pool)
    if (*handled && cfg.c64 && (p.L % 2 != 0 || p.LT % 2 != 0)) *handled = false;
    if (!*handled) return cudaSuccess;
    return launch_pass(p, st, cfg);
}

}  // namespace svi
