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
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sv_internal.h"
#include "plan.h"

// SV_DEBUG_CHECKS (a debug build, tools/build_variant.py ... -DSV_DEBUG_CHECKS): every
// shared-memory class access is checked against its tile and every mbarrier wait against a spin
// limit; a violation traps (the CUDA error fails the calling test).  Zero cost otherwise.
#ifdef SV_DEBUG_CHECKS
#define SV_DCHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define SV_DCHECK(cond) do { } while (0)
#endif

namespace svi {

constexpr int kMaxPassGates = 32;            // fire bits: one 32-bit ballot
constexpr int kMaxMembers = 128;
constexpr int kPoolC = 768;
constexpr int kMaxPassCtrl = 4;
constexpr int kMaxIns = 2 + kMaxPassCtrl;   // inserted in-tile digits: the target(s) + pinned controls
constexpr int kMaxPairDim = 4;             // dense pair gates (any kinds): d_a d_b <= 4 (qubit pairs)
constexpr int kMaxFactoredPair = 8;        // factored general pairs: d_a <= d_b, d_a d_b <= 8, i.e.
                                           //   (2,2), (2,3), (2,4); (3,3) spilled at 96 registers and
                                           //   slowed every gate (c4 +8%, profiles/r02/ab/r02ae)
constexpr int kGDesc = 16;                 // words of a gate's shared-memory descriptor

// in-pass gate kinds: general y = U x (§2.3), monomial y_{sigma(j)} = c_j x_j (§2.1-2.2),
// and the pure permutation (every moving coefficient exactly 1: no arithmetic at all)
// and the factored pair (two general gates on two in-tile digits, U_b (x) U_a applied to the
// d_a d_b-member class in registers as U_a on each digit-a column, then U_b on each digit-b row)
enum PassKind : int32_t { kPGeneral = 0, kPMonomial = 1, kPPerm = 2, kPPair = 3 };

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

// kFTrans: the gate's classes are enumerated target-run-major (class_idx<true>)
enum PassFlags : uint32_t { kFRunCtrl = 4, kFTrans = 8 };

struct PassGateP {
    int32_t d, kind, nctrl, uoff;
    int32_t da;           // kPPair: dimension of digit a (d = da * db)
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

// A pure permutation gate absorbed into the tile's member addressing (no compute item): its
// target is a member digit (in H) and each control is a member digit or constant over the tile,
// so on every tile it moves whole member runs, member x to member pi(x).  Moved to the front of
// the pass (it commutes with every earlier item) it relabels the load sources — slot y is loaded
// from global member pi^-1(y) — or moved to the back, the store targets — slot x is stored to
// member pi(x).  The data never passes through the compute warps (a monomial
// gate with unit coefficients only relabels amplitudes).
constexpr int kMaxAbs = 8;
constexpr int kMaxAbsOut = 2;       // out-of-tile controls per absorbed gate
struct AbsPerm {
    uint8_t store, d, nmc, noc;     // phase (0 load, 1 store), target dim, member / outside controls
    uint32_t wt;                    // member radix weight of the target digit
    uint8_t mc_w[kMaxPassCtrl], mc_d[kMaxPassCtrl], mc_v[kMaxPassCtrl];   // member controls
    int8_t sig[kMaxDim], inv[kMaxDim];                                      // sigma, sigma^-1
    uint64_t oc_b[kMaxAbsOut], oc_mb[kMaxAbsOut], oc_md[kMaxAbsOut];      // outside: stride, magics
    uint32_t oc_d[kMaxAbsOut], oc_v[kMaxAbsOut];
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
    int32_t nabs;         // absorbed permutations (load phase first, each phase in gate order)
    AbsPerm ab[kMaxAbs];
};

static_assert(sizeof(PassParams) <= 32764, "kernel parameter space (32 KB on sm_100)");

// ---- register-blocked stages (k_gate_stage).  The pass's gates are grouped, in pass order, into
// stages: maximal runs of consecutive gates whose targets lie in one pair of in-tile digits {a, b}
// with d_a d_b <= kStageAmps (a single target is paired with a passive digit).  A thread loads a
// whole d_a x d_b block of the tile into registers (every digit but a and b fixed), applies all
// the stage's gates there — each gate's classes are the block's rows or columns
// — and stores the block once: one shared-memory round trip and one group barrier per stage
// instead of per gate.
constexpr int kStageAmps = 12;
constexpr int kPoolS = 800;                 // 32 gates of d <= 5
enum StageKind : int32_t { kSGeneral = 0, kSDiag = 1, kSShift = 2 };

struct StageGate {
    int32_t nctrl;                          // controls decided per tile (producer): cls 2 out of
    PassCtrl c[kMaxPassCtrl];               //   the tile, cls 1 / 3 run digits
    int32_t axis;                           // target: 0 = the stage's digit a, 1 = digit b
    int32_t kind;                           // StageKind
    int32_t shift;                          // kSShift: y_{(j + shift) mod d} = x_j
    int32_t uoff;                           // kSGeneral: row-major d x d; kSDiag: d entries
    int32_t octrl;                          // control on the stage's other digit: value, or -1
    int32_t nic;                            // controls on in-tile digits outside the stage:
    uint32_t ic_s[kMaxPassCtrl], ic_m[kMaxPassCtrl], ic_d[kMaxPassCtrl], ic_dm[kMaxPassCtrl],
             ic_v[kMaxPassCtrl];            //   digit (e / s) mod d == v (s, d + magics)
    uint32_t runck;                         // 1: c[] holds a run-digit control
};

struct StageRec {
    int32_t da, db;                         // dims of digit a (lower tile stride) and b
    int32_t g0, ng;                         // its gates
    uint32_t sa, sb;                        // tile strides
    uint32_t nblk;                          // blocks per full tile = M LT / (da db)
    uint32_t s0, m0, sd0;                   // block id -> tile offset: insert digit a (stride, magic,
    uint32_t s1, m1, sd1;                   //   stride*dim), then digit b
};

struct StageParams {
    double2 *psi;
    int32_t nrem;
    RemovedRun rem[kMaxRem];
    uint64_t ntiles, R, tpr, tpr_m;
    uint32_t LT, mLT;
    uint32_t L, mL;
    int32_t M;
    int32_t ngates;
    int32_t nstages;
    int32_t upool;
    uint64_t moff[kMaxMembers];
    StageRec st[kMaxPassGates];
    StageGate g[kMaxPassGates];
    double2 U[kPoolS];
};
static_assert(sizeof(StageParams) <= 32764, "kernel parameter space (32 KB on sm_100)");

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds_u128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#ifdef SV_DEBUG_CHECKS
    // bounded spin: a lost arrive (or a phase mix-up) traps instead of hanging the GPU
    for (uint64_t it = 0;; ++it) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (done) break;
        SV_DCHECK(it < (1ull << 26));
    }
#else
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
#endif
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

template <typename PP>
__device__ __forceinline__ TileInfo tile_info(const PP &p, uint64_t t) {
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
    uint32_t afire;                                  // bit a: absorbed permutation a's likewise
    uint32_t lowoff[kMaxPassGates][kMaxPassCtrl];    // (s0 mod b_c d_c) for run-digit controls
};

// member x after absorbed permutation a (forward sigma, or sigma^-1 when inverse): controls
// read the label's member digits; target and controls are distinct digits, so the test holds
// before and after the move
__device__ __forceinline__ uint32_t abs_move(const AbsPerm &a, uint32_t x, bool inverse) {
    for (int k = 0; k < a.nmc; ++k)
        if ((x / a.mc_w[k]) % a.mc_d[k] != a.mc_v[k]) return x;
    const uint32_t dig = (x / a.wt) % a.d;
    const uint32_t to = (uint32_t)(inverse ? a.inv[dig] : a.sig[dig]);
    return x + to * a.wt - dig * a.wt;
}

template <class PP> struct HasAbs { static constexpr bool value = false; };
template <> struct HasAbs<PassParams> { static constexpr bool value = true; };

// PP: PassParams or StageParams (same geometry fields; g[i].nctrl / g[i].c[] = the controls
// decided per tile)
template <typename V, typename PP>
__device__ __forceinline__ void issue_loads(const PP &p, uint64_t t, V *buf, uint64_t *bar,
                                            StageInfo *si, int lane) {
    const TileInfo ti = tile_info(p, t);
    // lane g decides gate g for this tile
    bool fire = true;
    if (lane < p.ngates) {
        const auto &g = p.g[lane];
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
    uint32_t abits = 0;
    if constexpr (HasAbs<PP>::value) {       // lane a decides absorbed permutation a's out-of-tile controls
        bool af = lane < p.nabs;
        if (af) {
            const AbsPerm &a = p.ab[lane];
            for (int k = 0; k < a.noc; ++k) {
                uint64_t r;
                const uint64_t q = fastdiv64(ti.gbase, a.oc_b[k], a.oc_mb[k], r);
                fastdiv64(q, a.oc_d[k], a.oc_md[k], r);
                af = af && (r == a.oc_v[k]);
            }
        }
        abits = __ballot_sync(0xffffffffu, af);
    }
    if (lane == 0) {
        si->ti = ti;
        si->fire = bits;
        si->afire = abits;
    }
    __syncwarp();
    SV_DCHECK(ti.len <= p.LT && ti.len > 0);
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)p.M * ti.len * (uint32_t)sizeof(V));
    __syncwarp();
    for (int m = lane; m < p.M; m += 32) {
        uint32_t src = (uint32_t)m;
        if constexpr (HasAbs<PP>::value) {   // load-phase permutations, last first, inverted
            for (int a = p.nabs - 1; a >= 0; --a)
                if (((abits >> a) & 1) && !p.ab[a].store) src = abs_move(p.ab[a], src, true);
            SV_DCHECK(src < (uint32_t)p.M);
        }
        bulk_load(buf + (size_t)m * p.LT, reinterpret_cast<const V *>(p.psi) + ti.gbase + p.moff[src],
                  ti.len * (uint32_t)sizeof(V), bar);
    }
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
// the first two insertions from registers (an uncontrolled gate has one; a gate with one
// enumerated in-tile control has two), further ones from the parameter bank
struct Ins2 {
    Ins1 a, b;
    uint32_t n;            // insertions in all
};
__device__ __forceinline__ uint32_t class_e0(uint32_t c, const PassGateP &g, const Ins2 &ins, bool more) {
    uint32_t e = insert1(c, ins.a);
    if (more) {
        e = insert1(e, ins.b);
#pragma unroll 1
        for (uint32_t i = 2; i < ins.n; ++i) e = insert1(e, ins_at(g, (int)i));
    }
    return e;
}

// Class index -> member-0 tile index.  TR (kFTrans gates: a lone low-prefix target of stride
// st < 8 with st d odd and d = 3 or 5, no enumerated control): class c = r O + o sits at
// o (st d) + r (o < O = ncls / st, r < st; O in the second insertion slot), so consecutive lanes
// step st d (odd) 16-byte slots and hit distinct banks, where the natural order (r fastest) puts
// runs of st lanes st d apart (st = 5, d = 5: 2-way conflicts).  A template parameter, so the
// other gates' class loops carry no extra instruction.
template <bool TR>
__device__ __forceinline__ uint32_t class_idx(uint32_t c, const PassGateP &g, const Ins2 &ins, bool more) {
    if constexpr (TR) {
        uint32_t o;
        const uint32_t r = tdiv(c, ins.b.s, ins.b.m, o);
        return o * ins.a.sd + r;
    } else {
        return class_e0(c, g, ins, more);
    }
}

// What one gate needs to decide its classes inside the current tile.
struct TileGate {
    uint32_t LT, mLT, len, flags;
    uint32_t tbytes;            // bytes of the tile (debug bound checks)
    uint32_t nins, active;      // hot gate fields, read from the shared-memory descriptor
    Ins2 first;                 // the first two digit insertions of the class index
    const uint32_t *lowoff;     // shared memory: run offsets of the run-digit controls
    const uint32_t *moff;       // shared memory: tile offset of class member j (j st, or the
                                //   two-digit offset of a pair gate)
    const uint32_t *soff;       // shared memory: offset of member sigma(j) (monomial gates)
    uint32_t moff_s, soff_s;    // the same two tables as shared-window addresses (LDS, not generic LD)
    uint32_t lowoff_s;          // lowoff as a shared-window address
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
                const uint32_t x = lds_u32(tg.lowoff_s + 4u * k), t = x & kCls3Mask, mode = x >> 30;
                ok = ok && (mode == 1 ? l < t : (mode == 2 && l >= t));
                continue;
            }
            if (cc.cls != 1) continue;
            uint32_t r, r2;
            fastdiv32(lds_u32(tg.lowoff_s + 4u * k) + l, cc.M, cc.mM, r);
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
template <int K, int NT, bool TR = false>
__device__ __forceinline__ void class_batch(const TileGate &tg, const PassGateP &g, const Ins2 &first, bool more,
                                            uint32_t c0, uint32_t ncls, bool needck, uint32_t (&e)[K],
                                            bool (&ok)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t c = c0 + (uint32_t)(k * NT);
        ok[k] = c < ncls;
        e[k] = ok[k] ? class_idx<TR>(c, g, first, more) : 0u;
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

// matrix-vector order of general gates, by dimension: row-outer (one output row at a time, the
// row's matrix entries read per row) or column-outer (all rows at once, one matrix column at a
// time).  SV_COLOUTER_MASK (bit d): timing A/B builds.
#ifndef SV_COLOUTER_MASK
#define SV_COLOUTER_MASK 0u
#endif
template <int D> struct PassColOuter { static constexpr bool value = (SV_COLOUTER_MASK >> D) & 1u; };

// One general gate (y = U x per class) on one tile, K classes per thread
// iteration.  All K*D gathers are issued before the matvecs; buf and U are restrict-qualified
// so the matrix reads may be scheduled across the stores of earlier rows.  Branch-free: a class
// that does not exist or fire (CHECK) computes on harmless inputs and stores to the lane's trash
// slot, so the K classes' FMA chains stay in one basic block and interleave (with a branch per
// store, ptxas ran the classes' dependent DFMA chains one after another).
template <int D, int K, int NT, bool CHECK, typename V, bool TR = false>
__device__ __forceinline__ void gate_tile_general(const TileGate &tg, const PassGateP &g, V *__restrict__ buf,
                                                  const V *__restrict__ U, uint32_t cbeg, uint32_t cend,
                                                  uint32_t ncls, bool needck, int tid, uint32_t trash) {
    // member offsets, read once from shared memory (the stores below may alias that table as
    // far as the compiler knows, so it keeps them in registers)
    uint32_t mo[D];
#pragma unroll
    for (int j = 0; j < D; ++j) mo[j] = lds_u32(tg.moff_s + 4u * j) * (uint32_t)sizeof(V);
    const uint32_t sb = smem_u32(buf);
    const Ins2 first = tg.first;
    const bool more = tg.nins > 1;
#pragma unroll 1
    for (uint32_t c0 = cbeg + (uint32_t)tid; c0 < cend; c0 += (uint32_t)(NT * K)) {
        uint32_t e[K];
        bool ok[K];
        if (CHECK) {
            class_batch<K, NT, TR>(tg, g, first, more, c0, ncls, needck, e, ok);
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                e[k] = class_idx<TR>(c0 + (uint32_t)(k * NT), g, first, more);
                ok[k] = true;
            }
        }
        const V *__restrict__ Ui = U + opaque_zero(c0);
        uint32_t a[K];
        V x[K][D];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            a[k] = sb + e[k] * (uint32_t)sizeof(V);
#pragma unroll
            for (int j = 0; j < D; ++j) {
                SV_DCHECK(e[k] * (uint32_t)sizeof(V) + mo[j] + (uint32_t)sizeof(V) <= tg.tbytes);
                x[k][j] = lds2<V>(a[k] + mo[j]);
            }
        }
        if constexpr (PassColOuter<D>::value) {
            // column-outer: every output row of every class accumulates at once (2 K D independent
            // FMA chains instead of 2 K), matrix column j read once per iteration; the per-element
            // summation order (j = 0..D-1) is the row-outer one, so results are bit-identical
            V acc[K][D];
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int i = 0; i < D; ++i) acc[k][i] = cz<V>();
#pragma unroll
            for (int j = 0; j < D; ++j) {
                V u[D];
#pragma unroll
                for (int i = 0; i < D; ++i) u[i] = Ui[i * D + j];
#pragma unroll
                for (int i = 0; i < D; ++i)
#pragma unroll
                    for (int k = 0; k < K; ++k) cfma(acc[k][i], u[i], x[k][j]);
            }
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int k = 0; k < K; ++k) sts2(CHECK ? (ok[k] ? a[k] + mo[i] : trash) : a[k] + mo[i], acc[k][i]);
        } else {
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
                for (int k = 0; k < K; ++k) sts2(CHECK ? (ok[k] ? a[k] + mo[i] : trash) : a[k] + mo[i], acc[k]);
            }
        }
    }
}

// One monomial gate (phase / permutation, y_{sigma(j)} = c_j x_j) on one
// tile; PERM: every moving coefficient is exactly 1, so the gate only moves data.  Only the
// members that move or scale are read and written (select-form predicated gathers: a branch
// per member makes ptxas spill the array); skipped classes store to the trash slot.
template <int D, int K, int NT, bool PERM, bool CHECK, typename V, bool TR = false>
__device__ __forceinline__ void gate_tile_monomial(const TileGate &tg, const PassGateP &g, V *__restrict__ buf,
                                                   const V *__restrict__ U, uint32_t cbeg, uint32_t cend,
                                                   uint32_t ncls, bool needck, int tid, uint32_t trash) {
    const uint32_t act = tg.active;
    const Ins2 first = tg.first;
    const bool more = tg.nins > 1;
    // destination offsets sigma(j) * st, read once from shared memory: the stores below may
    // alias that table as far as the compiler knows, so it keeps them in registers instead of
    // re-reading the parameter bank inside the loop
    uint32_t so[D], mo[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
        so[j] = lds_u32(tg.soff_s + 4u * j) * (uint32_t)sizeof(V);
        mo[j] = lds_u32(tg.moff_s + 4u * j) * (uint32_t)sizeof(V);
    }
    const uint32_t sb = smem_u32(buf);
#pragma unroll 1
    for (uint32_t c0 = cbeg + (uint32_t)tid; c0 < cend; c0 += (uint32_t)(NT * K)) {
        uint32_t e[K];
        bool ok[K];
        if (CHECK) {
            class_batch<K, NT, TR>(tg, g, first, more, c0, ncls, needck, e, ok);
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                e[k] = class_idx<TR>(c0 + (uint32_t)(k * NT), g, first, more);
                ok[k] = true;
            }
        }
        uint32_t a[K];
        V x[K][D];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            a[k] = sb + e[k] * (uint32_t)sizeof(V);
#pragma unroll
            for (int j = 0; j < D; ++j)
                SV_DCHECK(!((act >> j) & 1) || (e[k] * (uint32_t)sizeof(V) + (mo[j] > so[j] ? mo[j] : so[j]) +
                                                 (uint32_t)sizeof(V) <= tg.tbytes));
        }
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const bool aj = (act >> j) & 1;
#pragma unroll
            for (int k = 0; k < K; ++k)
                x[k][j] = aj ? lds2<V>(a[k] + mo[j]) : cz<V>();
        }
#pragma unroll
        for (int j = 0; j < D; ++j)
            if ((act >> j) & 1) {
                if (PERM) {
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        sts2(CHECK ? (ok[k] ? a[k] + so[j] : trash) : a[k] + so[j], x[k][j]);
                } else {
                    const V u = U[j];
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        sts2(CHECK ? (ok[k] ? a[k] + so[j] : trash) : a[k] + so[j], cmul(u, x[k][j]));
                }
            }
    }
}

// One factored pair gate on one tile (PAPER.md:222 applied twice): the class's DA*DB members
// x[jb][ja] (member ja + DA jb) are gathered once; U_a (DA x DA, pool offset 0) acts on every
// column jb, then U_b (DB x DB, offset DA*DA) on every row ja, and the results are scattered
// once: one shared-memory round trip for two gates, DA^2 + DB^2 matrix reads per class (a dense
// DA DB x DA DB Kronecker matrix would read (DA DB)^2 and cost DA DB / (DA + DB) times the FLOPs).
template <int DA, int DB, int NT, bool CHECK, typename V>
__device__ __forceinline__ void gate_tile_pair(const TileGate &tg, const PassGateP &g, V *__restrict__ buf,
                                               const V *__restrict__ U, uint32_t cbeg, uint32_t cend,
                                               uint32_t ncls, bool needck, int tid, uint32_t trash) {
    // member (ja, jb) sits at ja sa + jb sb from member 0 (two strides instead of a D-entry
    // offset table: fewer live registers)
    const uint32_t sa = lds_u32(tg.moff_s + 4u) * (uint32_t)sizeof(V);
    const uint32_t sbb = lds_u32(tg.moff_s + 4u * DA) * (uint32_t)sizeof(V);
    const uint32_t sb = smem_u32(buf);
    const Ins2 first = tg.first;
    const bool more = tg.nins > 2;          // the pair's two target digits are always inserted
#pragma unroll 1
    for (uint32_t c0 = cbeg + (uint32_t)tid; c0 < cend; c0 += (uint32_t)NT) {
        uint32_t e[1];
        bool ok[1];
        if (CHECK) {
            class_batch<1, NT>(tg, g, first, more || true, c0, ncls, needck, e, ok);
        } else {
            e[0] = class_e0(c0, g, first, true);
            ok[0] = true;
        }
        const uint32_t a = sb + e[0] * (uint32_t)sizeof(V);
        V x[DB][DA];
#pragma unroll
        for (int jb = 0; jb < DB; ++jb)
#pragma unroll
            for (int ja = 0; ja < DA; ++ja) {
                SV_DCHECK(e[0] * (uint32_t)sizeof(V) + ja * sa + jb * sbb + (uint32_t)sizeof(V) <= tg.tbytes);
                x[jb][ja] = lds2<V>(a + (uint32_t)ja * sa + (uint32_t)jb * sbb);
            }
        // matrix entries re-read (broadcast) per column / row: holding U_a or U_b across the
        // class's columns would cost up to 4 DB^2 registers on top of the 4 D of the class
#pragma unroll
        for (int jb = 0; jb < DB; ++jb) {          // U_a on column jb
            const V *__restrict__ Ua = U + opaque_zero(c0 + (uint32_t)jb);
            V t[DA];
#pragma unroll
            for (int i = 0; i < DA; ++i) {
                V acc = cz<V>();
#pragma unroll
                for (int j = 0; j < DA; ++j) cfma(acc, Ua[i * DA + j], x[jb][j]);
                t[i] = acc;
            }
#pragma unroll
            for (int i = 0; i < DA; ++i) x[jb][i] = t[i];
        }
#pragma unroll
        for (int ja = 0; ja < DA; ++ja) {          // U_b on row ja, scattered
            const V *__restrict__ Ub = U + opaque_zero(c0 + (uint32_t)ja) + DA * DA;
#pragma unroll
            for (int i = 0; i < DB; ++i) {
                V acc = cz<V>();
#pragma unroll
                for (int j = 0; j < DB; ++j) cfma(acc, Ub[i * DB + j], x[j][ja]);
                const uint32_t o = a + (uint32_t)ja * sa + (uint32_t)i * sbb;
                sts2(CHECK ? (ok[0] ? o : trash) : o, acc);
            }
        }
    }
}

template <int DA, int DB, int NTG, typename V>
__device__ __forceinline__ void apply_pair_tile(const TileGate &tg, const PassGateP &g, V *buf, const V *U,
                                                uint32_t ncls, bool needck, int tid, uint32_t trash) {
    if (needck) gate_tile_pair<DA, DB, NTG, true, V>(tg, g, buf, U, 0, ncls, ncls, true, tid, trash);
    else gate_tile_pair<DA, DB, NTG, false, V>(tg, g, buf, U, 0, ncls, ncls, false, tid, trash);
}

// generic dimension (fused or d > 5): out of line so its 16-wide register arrays do not
// inflate the kernel
template <typename V>
__device__ __noinline__ void gate_tile_generic(const TileGate tg, const PassGateP &g, V *buf,
                                               const V *U, uint32_t ncls, bool needck, int tid, int nt) {
    const int d = g.d;
    for (uint32_t c = tid; c < ncls; c += nt) {
        const uint32_t e0 = class_e0(c, g, Ins2{ins_at(g, 0), ins_at(g, g.nins > 1 ? 1 : 0), (uint32_t)g.nins},
                                     g.nins > 1);
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

// classes per thread iteration (registers: 4*K*D for the gathered classes), by thread count.
// With 512+ compute threads (96 registers at 18 warps: the per-SMSP register file holds 5 warps)
// two classes for d <= 3 and one for d = 4, 5 measured best (c4 1816 -> 1628 ms, c3 439 -> 394 ms
// against the earlier 4/3/2/2, same box; profiles/r02/ab/r02m_ksweep, r02n_ksweep2): fewer
// in-flight classes, no spills.  384 threads (128 registers) keep the larger batches.
#ifndef SV_PASSK512               // K for d = 2, 3, 4, 5 at 512+ threads as 4 decimal digits
#define SV_PASSK512 2211          //   (timing builds override; 2221 / 4211 / 2111 / 1111 measured
#endif                            //   slower, profiles/r02/ab/r02ai)
constexpr int kPassK512[4] = {SV_PASSK512 / 1000 % 10, SV_PASSK512 / 100 % 10, SV_PASSK512 / 10 % 10, SV_PASSK512 % 10};
template <int D, int NT> struct PassK { static constexpr int value = 1; };
template <int NT> struct PassK<2, NT> { static constexpr int value = NT >= 512 ? kPassK512[0] : 4; };
template <int NT> struct PassK<3, NT> { static constexpr int value = NT >= 512 ? kPassK512[1] : 4; };
template <int NT> struct PassK<4, NT> { static constexpr int value = NT >= 512 ? kPassK512[2] : 3; };
template <int NT> struct PassK<5, NT> { static constexpr int value = NT >= 512 ? kPassK512[3] : (NT >= 384 ? 2 : 3); };

// NT = compute threads of the CTA (sets the register budget), NTG = threads of one consumer
// group (the class stride)
template <int D, int NT, int NTG, typename V>
__device__ __forceinline__ void apply_gate_tile(const TileGate &tg, const PassGateP &g, int kind, V *buf,
                                                const V *U, uint32_t ncls, bool needck, int tid, uint32_t trash) {
    constexpr int K = PassK<D, NT>::value;
    if constexpr (D == 3 || D == 5) {
        if (tg.flags & kFTrans) {      // general or permutation, see class_idx
            const uint32_t full = needck ? 0u : ncls / (uint32_t)(NTG * K) * (uint32_t)(NTG * K);
            if (kind == kPGeneral) {
                if (full) gate_tile_general<D, K, NTG, false, V, true>(tg, g, buf, U, 0, full, ncls, false, tid, trash);
                gate_tile_general<D, 1, NTG, true, V, true>(tg, g, buf, U, full, ncls, ncls, needck, tid, trash);
            } else {
                if (full) gate_tile_monomial<D, K, NTG, true, false, V, true>(tg, g, buf, U, 0, full, ncls, false, tid, trash);
                gate_tile_monomial<D, 1, NTG, true, true, V, true>(tg, g, buf, U, full, ncls, ncls, needck, tid, trash);
            }
            return;
        }
    }
    // Gates that need per-class checks (ragged tile, run-digit controls) run one class per
    // thread with the checks; the others take full batches of K classes per thread without any
    // predicate, then the remainder one class per thread through the same checked code.  (A
    // checked K-batch variant measured slower: c4 1246 -> 1200 ms, c3 343 -> 331 ms without it,
    // profiles/r02/ab/r02af — one code path fewer per gate kind in the hot instruction stream;
    // a predicated K-batch for the remainder was slower too: its idle slots cost more than the
    // interleaving gains.)
    const uint32_t full = needck ? 0u : ncls / (uint32_t)(NTG * K) * (uint32_t)(NTG * K);
    if (kind == kPGeneral) {
        if (full) gate_tile_general<D, K, NTG, false, V>(tg, g, buf, U, 0, full, ncls, false, tid, trash);
        gate_tile_general<D, 1, NTG, true, V>(tg, g, buf, U, full, ncls, ncls, needck, tid, trash);
    } else if (kind == kPPerm) {
        if (full) gate_tile_monomial<D, K, NTG, true, false, V>(tg, g, buf, U, 0, full, ncls, false, tid, trash);
        gate_tile_monomial<D, 1, NTG, true, true, V>(tg, g, buf, U, full, ncls, ncls, needck, tid, trash);
    } else {
        if (full) gate_tile_monomial<D, K, NTG, false, false, V>(tg, g, buf, U, 0, full, ncls, false, tid, trash);
        gate_tile_monomial<D, 1, NTG, false, true, V>(tg, g, buf, U, full, ncls, ncls, needck, tid, trash);
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

// Warp-specialised: warps 0..NT/32-1 compute, warp NT/32 loads (stage records, TMA loads),
// warp NT/32+1 stores (TMA stores).  full[s] completes when a tile's bytes have landed; done[s]
// when the compute warps have finished it (after fence.proxy.async, so the bulk store sees their
// writes); empty[s] when the store warp's bulk store has read the stage.  With one warp doing
// both, every load waited for the previous store's smem read (wait_group.read covers all of the
// thread's groups), serialising the stages; split, a stage is reloaded as soon as its own store
// has been read.  The compute warps form G consumer groups of NT/G threads; group g takes the
// CTA's tiles g, g+G, ... (ping-pong), so one group's barrier waits overlap the other groups' work.
constexpr int kPassExtra = 64;     // the load warp and the store warp
template <int NT, int G, typename V>
__global__ void __launch_bounds__(NT + kPassExtra, 1) k_gate_pass(const __grid_constant__ PassParams p, int S, int TE) {
    constexpr int NTG = NT / G;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    V *bufs = reinterpret_cast<V *>(smem_raw);
    V *Us = bufs + (size_t)S * TE;                             // the pass's matrices (in V's precision)
    // per gate: member offsets (16-byte aligned: the gate descriptors after them are read as uint4,
    // and a complex64 matrix pool may end at an 8-byte boundary)
    uint32_t *moffs = reinterpret_cast<uint32_t *>((reinterpret_cast<uintptr_t>(Us + p.upool) + 15) & ~(uintptr_t)15);
    uint32_t *soffs = moffs + kMaxPassGates * kMaxDim;               // per gate: sigma-member offsets
    uint32_t *gdesc = soffs + kMaxPassGates * kMaxDim;               // per gate: hot fields (kGDesc words)
    StageInfo *sinfo = reinterpret_cast<StageInfo *>(gdesc + kMaxPassGates * kGDesc);
    uint64_t *full = reinterpret_cast<uint64_t *>(sinfo + S);
    uint64_t *done = full + S;
    uint64_t *empty = done + S;
    // per-lane slots that absorb the stores of classes a thread computes but must not write
    const uint32_t trash_base = (smem_u32(empty + S) + 15u) & ~15u;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t trash = trash_base + (uint32_t)lane * 16u;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&done[s], 1); mbar_init(&empty[s], 1); }
        fence_mbar_init();
    }
    for (int k = tid; k < p.upool; k += NT + kPassExtra) Us[k] = to_v<V>(p.U[k]);
    for (int k = tid; k < p.ngates * kMaxDim; k += NT + kPassExtra) {
        moffs[k] = (&p.moff_t[0][0])[k];
        soffs[k] = (&p.soff_t[0][0])[k];
    }
    if (tid < p.ngates) {      // the fields every gate of every tile needs, one 48-byte record
        const PassGateP &g = p.g[tid];
        uint32_t *d = gdesc + tid * kGDesc;
        d[0] = (uint32_t)g.d; d[1] = (uint32_t)g.kind; d[2] = g.ncls; d[3] = g.flags;
        d[4] = (uint32_t)g.nins; d[5] = (uint32_t)g.uoff; d[6] = g.active; d[7] = g.ins_s[0];
        d[8] = g.ins_m[0]; d[9] = g.ins_sd[0]; d[10] = g.ins_ps[0]; d[11] = (uint32_t)g.da;
        const int i1 = (g.nins > 1 || (g.flags & kFTrans)) ? 1 : 0;   // the second insertion (or O)
        d[12] = g.ins_s[i1]; d[13] = g.ins_m[i1]; d[14] = g.ins_sd[i1]; d[15] = g.ins_ps[i1];
    }
    __syncthreads();
    const uint64_t first = blockIdx.x, step = gridDim.x;
    if (first >= p.ntiles) return;
    // tiles of this CTA (< 2^32: ntiles <= D / b_{m0}); stage i mod S and ring phase (i / S) & 1
    // are tracked incrementally (a 64-bit i % S was a runtime-library call per tile)
    const uint32_t my = (uint32_t)((p.ntiles - first + step - 1) / step);

    if (warp == NT / 32) {
        // ---------------- load warp: tile i into stage i mod S once the store of tile i-S has read it
        int s = 0;
        uint32_t ph = 0;
        for (uint32_t i = 0; i < my; ++i) {
            if (i >= (uint32_t)S) mbar_wait(&empty[s], ph ^ 1u);
            issue_loads(p, first + (uint64_t)i * step, bufs + (size_t)s * TE, &full[s], &sinfo[s], lane);
            if (++s == S) { s = 0; ph ^= 1u; }
        }
        return;
    }
    if (warp == NT / 32 + 1) {
        // ---------------- store warp: tile j back to HBM once computed; frees the stage when read
        int s = 0;
        uint32_t ph = 0;
        for (uint32_t j = 0; j < my; ++j, (++s == S ? (s = 0, ph ^= 1u) : 0u)) {
            mbar_wait(&done[s], ph);
            const StageInfo &si = sinfo[s];
            const uint32_t abits = si.afire;
            for (int m = lane; m < p.M; m += 32) {
                uint32_t dst = (uint32_t)m;             // store-phase permutations, in order
                for (int a = 0; a < p.nabs; ++a)
                    if (((abits >> a) & 1) && p.ab[a].store) dst = abs_move(p.ab[a], dst, false);
                SV_DCHECK(dst < (uint32_t)p.M);
                bulk_store(reinterpret_cast<V *>(p.psi) + si.ti.gbase + p.moff[dst],
                           bufs + (size_t)s * TE + (size_t)m * p.LT, si.ti.len * (uint32_t)sizeof(V));
            }
            bulk_commit();
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
            if (lane == 0 && j + (uint32_t)S < my) mbar_arrive(&empty[s]);
        }
        bulk_wait_all();
        return;
    }

    // ---------------- compute warps
    const int grp = tid / NTG, gtid = tid % NTG;
    int s = grp;                    // G <= S: the group's first stage, phase 0
    uint32_t ph = 0;
    for (uint32_t i = (uint32_t)grp; i < my; i += (uint32_t)G, ((s += G) >= S ? (s -= S, ph ^= 1u) : 0u)) {
        V *buf = bufs + (size_t)s * TE;
        // With several groups, consecutive tiles of a stage belong to different groups, so this
        // group may reach tile i while the stage's previous tile (i - S, another group) is not
        // even loaded: full[s] would still be in the phase before the one awaited, and a parity
        // wait cannot tell a phase two steps back from a completed one.  Waiting first for
        // tile i - S to be consumed (done[s], whose previous phase this group completed itself)
        // puts full[s] exactly one phase before tile i.
        if (G > 1 && i >= (uint32_t)S) mbar_wait(&done[s], ph ^ 1u);
        mbar_wait(&full[s], ph);
        const StageInfo &si = sinfo[s];
        const uint32_t len = si.ti.len;
        const uint32_t fire = si.fire;
        const uint32_t LT = p.LT, mLT = p.mLT;
        const uint32_t gdesc_s = smem_u32(gdesc);
        for (int gi = 0; gi < p.ngates; ++gi) {
            if (!((fire >> gi) & 1)) continue;          // out-of-tile control unmet: uniform skip
            const PassGateP &g = p.g[gi];               // cold fields only (controls, more insertions)
            const uint32_t ga = gdesc_s + (uint32_t)(gi * kGDesc) * 4u;
            const uint4 h0 = lds_u128(ga);         // d, kind, ncls, flags
#ifdef SV_AB_SKIP_KIND   // timing-only A/B builds (wrong results): drop one gate kind's work
            if ((int)h0.y == SV_AB_SKIP_KIND || (SV_AB_SKIP_KIND == 3 && h0.y != 0)) continue;
#endif
            const uint4 h1 = lds_u128(ga + 16u);   // nins, uoff, active, s
            const uint4 h2 = lds_u128(ga + 32u);   // m, sd, ps, da
            const uint4 h3 = lds_u128(ga + 48u);   // second insertion: s, m, sd, ps
            TileGate tg;
            tg.LT = LT;
            tg.mLT = mLT;
            tg.len = len;
            tg.tbytes = (uint32_t)p.M * LT * (uint32_t)sizeof(V);
            tg.flags = h0.w;
            tg.nins = h1.x;
            tg.active = h1.z;
            tg.first = Ins2{Ins1{h1.w, h2.x, h2.y, h2.z}, Ins1{h3.x, h3.y, h3.z, h3.w}, h1.x};
            tg.lowoff = si.lowoff[gi];
            tg.moff = moffs + gi * kMaxDim;
            tg.soff = soffs + gi * kMaxDim;
            tg.moff_s = smem_u32(tg.moff);
            tg.lowoff_s = smem_u32(tg.lowoff);
            tg.soff_s = smem_u32(tg.soff);
            const bool needck = (h0.w & kFRunCtrl) != 0 || len < LT;
            const V *U = Us + h1.y;
            const uint32_t ncls = h0.z;
            if (h0.y == kPPair) {
                switch (h2.w * 8u + h0.x / h2.w) {     // (d_a, d_b), d_a <= d_b
                    case 2 * 8 + 2: apply_pair_tile<2, 2, NTG, V>(tg, g, buf, U, ncls, needck, gtid, trash); break;
                    case 2 * 8 + 3: apply_pair_tile<2, 3, NTG, V>(tg, g, buf, U, ncls, needck, gtid, trash); break;
                    default: apply_pair_tile<2, 4, NTG, V>(tg, g, buf, U, ncls, needck, gtid, trash); break;
                }
            } else switch (h0.x) {
                case 2: apply_gate_tile<2, NT, NTG, V>(tg, g, (int)h0.y, buf, U, ncls, needck, gtid, trash); break;
                case 3: apply_gate_tile<3, NT, NTG, V>(tg, g, (int)h0.y, buf, U, ncls, needck, gtid, trash); break;
                case 4: apply_gate_tile<4, NT, NTG, V>(tg, g, (int)h0.y, buf, U, ncls, needck, gtid, trash); break;
                case 5: apply_gate_tile<5, NT, NTG, V>(tg, g, (int)h0.y, buf, U, ncls, needck, gtid, trash); break;
                default: gate_tile_generic<V>(tg, g, buf, U, ncls, needck, gtid, NTG); break;
            }
            compute_barrier(1 + grp, NTG);
        }
        fence_proxy_async();
        compute_barrier(1 + grp, NTG);
        if (gtid == 0) mbar_arrive(&done[s]);
    }
}

// ------------------------------------------------------------------ register-blocked stages
namespace {

// element (j along the gate's digit, k along the stage's other digit) of a d_a x d_b block
template <int AX, int DA, int DB> struct BlockAx;
template <int DA, int DB> struct BlockAx<0, DA, DB> {
    static constexpr int D = DA, N = DB;
    template <typename V> __device__ __forceinline__ static V &at(V (&x)[DA][DB], int j, int k) { return x[j][k]; }
};
template <int DA, int DB> struct BlockAx<1, DA, DB> {
    static constexpr int D = DB, N = DA;
    template <typename V> __device__ __forceinline__ static V &at(V (&x)[DA][DB], int j, int k) { return x[k][j]; }
};

// One gate of a stage on every class of one block (the block's columns for a gate on digit a,
// its rows for digit b): y = U x, y_j = c_j x_j (§2.1), or a cyclic shift (§2.2).
// A control on the stage's other digit selects one class.  Branch-free over the
// classes (every class is computed, the control selects which results are kept), so the
// classes' FMA chains share one basic block and interleave.
template <int AX, int DA, int DB, typename V>
__device__ __forceinline__ void block_gate(V (&x)[DA][DB], const StageGate &g, const V *__restrict__ Us) {
    using A = BlockAx<AX, DA, DB>;
    constexpr int D = A::D, N = A::N;
    const int oc = g.octrl;
    const V *__restrict__ U = Us + g.uoff;
    bool keep[N];
#pragma unroll
    for (int k = 0; k < N; ++k) keep[k] = oc < 0 || oc == k;
    if (g.kind == kSGeneral) {
        V y[N][D];
        if constexpr (D == 2) {            // 2 x 2: the matrix in registers, reused by every class
            V u[D * D];
#pragma unroll
            for (int t = 0; t < D * D; ++t) u[t] = U[t];
#pragma unroll
            for (int k = 0; k < N; ++k)
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    y[k][i] = cz<V>();
#pragma unroll
                    for (int j = 0; j < D; ++j) cfma(y[k][i], u[i * D + j], A::at(x, j, k));
                }
        } else {                           // matrix entries streamed from shared memory (broadcast)
#pragma unroll
            for (int k = 0; k < N; ++k) {
                // an offset the compiler cannot prove zero: re-read U per class instead of holding
                // all d^2 entries in registers across the block's classes
                const V *__restrict__ Uk = U + opaque_zero((uint32_t)k);
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    y[k][i] = cz<V>();
#pragma unroll
                    for (int j = 0; j < D; ++j) cfma(y[k][i], Uk[i * D + j], A::at(x, j, k));
                }
            }
        }
#pragma unroll
        for (int k = 0; k < N; ++k)
#pragma unroll
            for (int i = 0; i < D; ++i) A::at(x, i, k) = keep[k] ? y[k][i] : A::at(x, i, k);
    } else if (g.kind == kSDiag) {
        V c[D];
#pragma unroll
        for (int j = 0; j < D; ++j) c[j] = U[j];
#pragma unroll
        for (int k = 0; k < N; ++k)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const V t = cmul(c[j], A::at(x, j, k));
                A::at(x, j, k) = keep[k] ? t : A::at(x, j, k);
            }
    } else {                               // kSShift: data movement only (selects)
        const int s = g.shift;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            V t[D];
#pragma unroll
            for (int j = 0; j < D; ++j) t[j] = A::at(x, j, k);
#pragma unroll
            for (int i = 0; i < D; ++i) {  // y_i = x_{(i - s) mod d}
                V v = t[i];
#pragma unroll
                for (int ss = 1; ss < D; ++ss) v = s == ss ? t[(i - ss + D) % D] : v;
                A::at(x, i, k) = keep[k] ? v : t[i];
            }
        }
    }
}

// run-digit controls of a gate (cls 1 / 3) at run position l of the tile
__device__ __forceinline__ bool run_ctrl_ok(const StageGate &g, const uint32_t *lowoff, uint32_t l) {
    bool ok = true;
#pragma unroll 1
    for (int k = 0; k < g.nctrl; ++k) {
        const PassCtrl &cc = g.c[k];
        if (cc.cls == 3) {
            const uint32_t x = lowoff[k], t = x & kCls3Mask, mode = x >> 30;
            ok = ok && (mode == 1 ? l < t : (mode == 2 && l >= t));
        } else if (cc.cls == 1) {
            uint32_t r, r2;
            fastdiv32(lowoff[k] + l, cc.M, cc.mM, r);
            const uint32_t q = fastdiv32(r, cc.w, cc.mw, r2);
            fastdiv32(q, cc.d, cc.md, r2);
            ok = ok && (r2 == cc.v);
        }
    }
    return ok;
}

// One stage on one tile: every block (cb = thread, thread + NTG, ...) loaded once, all the
// stage's gates applied in registers, stored once.
template <int DA, int DB, typename V>
__device__ __forceinline__ void run_stage(const StageParams &p, const StageRec &sr, const StageInfo &si,
                                          V *buf, const V *__restrict__ Us, uint32_t gtid, uint32_t ntg) {
    const uint32_t sbase = smem_u32(buf);
    const Ins1 ia{sr.s0, sr.m0, sr.sd0, 0u}, ib{sr.s1, sr.m1, sr.sd1, 0u};
    const uint32_t oa = sr.sa * (uint32_t)sizeof(V), ob = sr.sb * (uint32_t)sizeof(V);
    const uint32_t len = si.ti.len, LT = p.LT, mLT = p.mLT;
    const bool ragged = len < LT;
    const uint32_t fire = si.fire;
    const int g0 = sr.g0, g1 = sr.g0 + sr.ng;
#pragma unroll 1
    for (uint32_t cb = gtid; cb < sr.nblk; cb += ntg) {
        uint32_t e = insert1(cb, ia);
        if (DB > 1) e = insert1(e, ib);
        uint32_t l;
        tdiv(e, LT, mLT, l);
        if (ragged && l >= len) continue;
        const uint32_t base = sbase + e * (uint32_t)sizeof(V);
        SV_DCHECK(e + (uint32_t)(DA - 1) * sr.sa + (uint32_t)(DB - 1) * sr.sb < (uint32_t)p.M * LT);
        V x[DA][DB];
#pragma unroll
        for (int ja = 0; ja < DA; ++ja)
#pragma unroll
            for (int jb = 0; jb < DB; ++jb) x[ja][jb] = lds2<V>(base + ja * oa + jb * ob);
#pragma unroll 1
        for (int gi = g0; gi < g1; ++gi) {
            if (!((fire >> gi) & 1)) continue;          // out-of-tile control unmet
            const StageGate &g = p.g[gi];
            bool ok = true;
#pragma unroll 1
            for (int k = 0; k < g.nic; ++k) {           // in-tile controls outside the stage
                uint32_t r, r2;
                const uint32_t q = tdiv(e, g.ic_s[k], g.ic_m[k], r);
                tdiv(q, g.ic_d[k], g.ic_dm[k], r2);
                ok = ok && (r2 == g.ic_v[k]);
            }
            if (g.runck) ok = ok && run_ctrl_ok(g, si.lowoff[gi], l);
            if (!ok) continue;
            if (g.axis == 0) block_gate<0, DA, DB, V>(x, g, Us);
            else block_gate<1, DA, DB, V>(x, g, Us);
        }
#pragma unroll
        for (int ja = 0; ja < DA; ++ja)
#pragma unroll
            for (int jb = 0; jb < DB; ++jb) sts2(base + ja * oa + jb * ob, x[ja][jb]);
    }
}

}  // namespace

// The register-blocked pass kernel: the same warp roles, ring and tile geometry as k_gate_pass;
// the compute groups run the pass's stages one after another on each tile, a group barrier
// between stages (a stage's blocks overlap the previous stage's).
template <int NT, int G, typename V>
__global__ void __launch_bounds__(NT + kPassExtra, 1) k_gate_stage(const __grid_constant__ StageParams p, int S, int TE) {
    constexpr int NTG = NT / G;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    V *bufs = reinterpret_cast<V *>(smem_raw);
    V *Us = bufs + (size_t)S * TE;
    StageInfo *sinfo = reinterpret_cast<StageInfo *>(Us + kPoolS);
    uint64_t *full = reinterpret_cast<uint64_t *>(sinfo + S);
    uint64_t *done = full + S;
    uint64_t *empty = done + S;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&done[s], 1); mbar_init(&empty[s], 1); }
        fence_mbar_init();
    }
    for (int k = tid; k < p.upool; k += NT + kPassExtra) Us[k] = to_v<V>(p.U[k]);
    __syncthreads();
    const uint64_t first = blockIdx.x, step = gridDim.x;
    if (first >= p.ntiles) return;
    // tiles of this CTA (< 2^32: ntiles <= D / b_{m0}); stage i mod S and ring phase (i / S) & 1
    // are tracked incrementally (a 64-bit i % S was a runtime-library call per tile)
    const uint32_t my = (uint32_t)((p.ntiles - first + step - 1) / step);

    if (warp == NT / 32) {
        int s = 0;
        uint32_t ph = 0;
        for (uint32_t i = 0; i < my; ++i) {
            if (i >= (uint32_t)S) mbar_wait(&empty[s], ph ^ 1u);
            issue_loads(p, first + (uint64_t)i * step, bufs + (size_t)s * TE, &full[s], &sinfo[s], lane);
            if (++s == S) { s = 0; ph ^= 1u; }
        }
        return;
    }
    if (warp == NT / 32 + 1) {
        int s = 0;
        uint32_t ph = 0;
        for (uint32_t j = 0; j < my; ++j, (++s == S ? (s = 0, ph ^= 1u) : 0u)) {
            mbar_wait(&done[s], ph);
            const StageInfo &si = sinfo[s];
            for (int m = lane; m < p.M; m += 32)
                bulk_store(reinterpret_cast<V *>(p.psi) + si.ti.gbase + p.moff[m],
                           bufs + (size_t)s * TE + (size_t)m * p.LT, si.ti.len * (uint32_t)sizeof(V));
            bulk_commit();
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
            if (lane == 0 && j + (uint32_t)S < my) mbar_arrive(&empty[s]);
        }
        bulk_wait_all();
        return;
    }

    const int grp = tid / NTG, gtid = tid % NTG;
    int s = grp;                    // G <= S: the group's first stage, phase 0
    uint32_t ph = 0;
    for (uint32_t i = (uint32_t)grp; i < my; i += (uint32_t)G, ((s += G) >= S ? (s -= S, ph ^= 1u) : 0u)) {
        V *buf = bufs + (size_t)s * TE;
        if (G > 1 && i >= (uint32_t)S) mbar_wait(&done[s], ph ^ 1u);
        mbar_wait(&full[s], ph);
        const StageInfo &si = sinfo[s];
        for (int st = 0; st < p.nstages; ++st) {
            if (st > 0) compute_barrier(1 + grp, NTG);
            const StageRec &sr = p.st[st];
            const int key = sr.da * 8 + sr.db;
            switch (key) {
                case 2 * 8 + 2: run_stage<2, 2, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 2 * 8 + 3: run_stage<2, 3, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 3 * 8 + 2: run_stage<3, 2, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 2 * 8 + 4: run_stage<2, 4, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 4 * 8 + 2: run_stage<4, 2, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 2 * 8 + 5: run_stage<2, 5, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 5 * 8 + 2: run_stage<5, 2, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 3 * 8 + 3: run_stage<3, 3, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 3 * 8 + 4: run_stage<3, 4, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 4 * 8 + 3: run_stage<4, 3, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 2 * 8 + 1: run_stage<2, 1, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 3 * 8 + 1: run_stage<3, 1, V>(p, sr, si, buf, Us, gtid, NTG); break;
                case 4 * 8 + 1: run_stage<4, 1, V>(p, sr, si, buf, Us, gtid, NTG); break;
                default: run_stage<5, 1, V>(p, sr, si, buf, Us, gtid, NTG); break;
            }
        }
        fence_proxy_async();
        compute_barrier(1 + grp, NTG);
        if (gtid == 0) mbar_arrive(&done[s]);
    }
}

// ------------------------------------------------------------------------------ host
// Tile geometry of a pass (shared by the per-gate and the register-blocked kernels): members
// (combinations of the H digits) with their global offsets, the removed H digits of the tile
// enumeration, the run R below min H and its split into tiles of LT run elements.  W[h] = member
// radix weight of H digit h.  Returns false if the pass does not fit.
template <class PP>
static bool pass_geometry(const Register &reg, const PassPlan &pp, double2 *psi, int TE, PP &p,
                          std::vector<uint64_t> &W, uint64_t &R_out, uint64_t &LT_out) {
    p.psi = psi;
    const int m0 = pp.m0;
    const uint64_t L = (m0 < reg.n) ? reg.b[m0] : reg.D;
    p.L = (uint32_t)L;
    p.mL = make_fastdiv32(p.L).m;
    uint64_t M = 1;
    for (int h : pp.H) M *= (uint64_t)reg.dims[h];
    if (M > (uint64_t)kMaxMembers) return false;
    // member radix weights and global offsets (H ascending)
    W.assign(reg.n, 0);
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
    R_out = R;
    LT_out = LT;
    return true;
}

// A control decided per tile (not on an in-tile digit): a run digit below min H (cls 1, or cls 3
// when b_c d_c >= 2^31) or a digit constant over the tile (cls 2: outside the tile, or a run
// digit whose stride is a multiple of the tile's run length LT — tiles start at multiples of LT,
// so such a digit cannot change inside one; its value is that of the tile's first index and the
// gate is skipped or applied whole, like an out-of-tile control).  Returns true for a run digit
// checked per class.
static bool fill_tile_ctrl(PassCtrl &cc, const Register &reg, int c, uint32_t v, uint64_t R, uint64_t LT) {
    const uint64_t dc = (uint64_t)reg.dims[c];
    cc.v = v;
    cc.d = (uint32_t)dc;
    cc.md = make_fastdiv32(cc.d).m;
    if (reg.b[c] < R && reg.b[c] % LT != 0 && reg.b[c] * dc < (1ull << 31)) {   // run digit: tile's run offset
        cc.cls = 1;
        cc.w = (uint32_t)reg.b[c];
        cc.mw = make_fastdiv32(cc.w).m;
        cc.M = cc.w * cc.d;
        cc.mM = make_fastdiv32(cc.M).m;
        cc.mb64 = make_fastdiv64(cc.M).m;
        return true;
    }
    if (reg.b[c] < R && reg.b[c] % LT != 0) {              // b_c d_c >= 2^31: per-tile threshold
        cc.cls = 3;
        cc.b64 = reg.b[c];
        cc.mb64 = make_fastdiv64(cc.b64).m;
        cc.md64 = make_fastdiv64(dc).m;
        return true;
    }
    cc.cls = 2;                                            // constant over the tile
    cc.b64 = reg.b[c];
    cc.mb64 = make_fastdiv64(cc.b64).m;
    cc.md64 = make_fastdiv64(cc.d).m;
    return false;
}

// Build the pass parameters; returns false if the pass does not fit this kernel.
bool build_pass(const Register &reg, const std::vector<GateSpec> &gates, const PassPlan &pp, double2 *psi,
                int TE, PassParams &p, PassWork *work, bool absorb) {
    std::memset(&p, 0, sizeof(p));
    if ((int)pp.gates.size() > kMaxPassGates || pp.tile > (uint64_t)TE) return false;
    std::vector<uint64_t> W;
    uint64_t R = 0, LT = 0;
    if (!pass_geometry(reg, pp, psi, TE, p, W, R, LT)) return false;
    const int m0 = pp.m0;
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
    // Two general gates may also pair up to d_a d_b <= kMaxFactoredPair: they are then applied
    // factored (kPPair), U_a and U_b one after the other on the class held in registers.
    struct Item { int a, b; };          // gate indices (b = -1: single)
    std::vector<Item> items;
    auto is_general = [&](int i) {
        GatePlan gp;
        std::string err;
        return plan_gate(reg, gates[i], false, &gp, &err) == SV_OK && gp.kind == kGeneral;
    };
    // Absorbed permutations (AbsPerm): a pure permutation on a member digit whose controls are
    // member digits or constant over the tile, moved to the front of the pass past the earlier
    // gates it commutes with (load phase), else to the back past the later ones (store phase).
    std::vector<int> rest;              // the gates left for compute items, in pass order
    *work = PassWork{};
    p.nabs = 0;
    {
        auto member_digit = [&](int q) { return std::find(pp.H.begin(), pp.H.end(), q) != pp.H.end(); };
        auto absorbable = [&](int i) {
            const GateSpec &g = gates[i];
            if (!absorb || !member_digit(g.target) || g.d > kMaxDim) return false;
            int noc = 0;
            for (const auto &c : g.ctrl) {
                if (member_digit(c.q)) continue;
                if (c.q < m0) return false;                                // low prefix: per class
                const uint64_t bc = reg.b[c.q];
                if (bc < R && bc % LT != 0) return false;                  // run digit: per class
                if (++noc > kMaxAbsOut) return false;
            }
            if ((int)g.ctrl.size() - noc > kMaxPassCtrl) return false;
            GatePlan gp;
            std::string err;
            if (plan_gate(reg, g, false, &gp, &err) != SV_OK || gp.kind != kMonomial) return false;
            for (int j = 0; j < gp.d; ++j)
                if (!(gp.U[j].x == 1.0 && gp.U[j].y == 0.0)) return false;
            return true;
        };
        std::vector<int> load, store, mid;
        for (int i : pp.gates) {        // front: commutes with every earlier non-absorbed gate
            bool ok = (int)load.size() < kMaxAbs && absorbable(i);
            for (size_t k = 0; ok && k < mid.size(); ++k) ok = commute(gates[i], gates[mid[k]]);
            (ok ? load : mid).push_back(i);
        }
        std::vector<int> later;         // back: commutes with every later non-absorbed gate
        for (int k = (int)mid.size() - 1; k >= 0; --k) {
            const int i = mid[k];
            bool ok = (int)(load.size() + store.size()) < kMaxAbs && absorbable(i);
            for (size_t j = 0; ok && j < later.size(); ++j) ok = commute(gates[i], gates[later[j]]);
            (ok ? store : later).push_back(i);
        }
        std::reverse(store.begin(), store.end());
        rest.assign(later.rbegin(), later.rend());
        auto put = [&](int i, bool st) {
            const GateSpec &g = gates[i];
            GatePlan gp;
            std::string err;
            plan_gate(reg, g, false, &gp, &err);
            work->touched += (double)gp.touched;
            AbsPerm &a = p.ab[p.nabs++];
            a.store = st ? 1 : 0;
            a.d = (uint8_t)g.d;
            a.wt = (uint32_t)W[g.target];
            for (int j = 0; j < kMaxDim; ++j) { a.sig[j] = (int8_t)j; a.inv[j] = (int8_t)j; }
            for (int j = 0; j < g.d; ++j) {
                a.sig[j] = (int8_t)gp.sigma[j];
                a.inv[gp.sigma[j]] = (int8_t)j;
            }
            for (const auto &c : g.ctrl) {
                if (member_digit(c.q)) {
                    a.mc_w[a.nmc] = (uint8_t)W[c.q];
                    a.mc_d[a.nmc] = (uint8_t)reg.dims[c.q];
                    a.mc_v[a.nmc] = (uint8_t)c.v;
                    ++a.nmc;
                } else {
                    a.oc_b[a.noc] = reg.b[c.q];
                    a.oc_mb[a.noc] = make_fastdiv64(reg.b[c.q]).m;
                    a.oc_d[a.noc] = (uint32_t)reg.dims[c.q];
                    a.oc_md[a.noc] = make_fastdiv64((uint64_t)reg.dims[c.q]).m;
                    a.oc_v[a.noc] = (uint32_t)c.v;
                    ++a.noc;
                }
            }
        };
        for (int i : load) put(i, false);
        for (int i : store) put(i, true);
    }
    for (int i : rest) {
        const GateSpec &g = gates[i];
        bool paired = false;
        for (int j = (int)items.size() - 1; j >= 0; --j) {
            Item &it = items[j];
            const GateSpec &h = gates[it.a];
            const int dd = h.d * g.d;
            if (it.b < 0 && h.target != g.target && h.d <= 5 && g.d <= 5 && same_controls(h, g) &&
                (dd <= kMaxPairDim || (dd <= kMaxFactoredPair && is_general(it.a) && is_general(i)))) {
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
        } else if (is_general(items[gi].a) && is_general(items[gi].b)) {
            // factored general pair: digit a = the smaller dimension (the Kronecker member order
            // is a layout choice; the two gates commute)
            const GateSpec &h = gates[items[gi].b];
            GatePlan hp;
            if (plan_gate(reg, h, false, &hp, &err) != SV_OK || hp.kind != kGeneral) return false;
            work->touched += (double)hp.touched;
            const bool sw = hp.d < gp.d;
            const GateSpec &ga = sw ? h : g, &gb = sw ? g : h;
            const int da = ga.d, db = gb.d;
            D = da * db;
            const uint64_t sta = tile_stride(ga.target), stb = tile_stride(gb.target);
            ins.assign({{sta, (uint32_t)da, 0u}, {stb, (uint32_t)db, 0u}});
            cls_div = (uint64_t)D;
            for (int jb = 0; jb < db; ++jb)
                for (int ja = 0; ja < da; ++ja) moff[ja + da * jb] = (uint32_t)(ja * sta + jb * stb);
            for (int J = 0; J < D; ++J) sig[J] = (uint32_t)J;
            kind = -1;                                   // kPPair (set below)
            q.da = da;
            q.active = (1u << D) - 1u;
            Ud.assign(ga.U.begin(), ga.U.end());
            Ud.insert(Ud.end(), gb.U.begin(), gb.U.end());
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
        q.kind = kind < 0 ? kPPair : kind == kGeneral ? kPGeneral : kPMonomial;
        {   // executed work of this item: its control-satisfying classes x moving members
            double cprod = 1.0;
            for (const auto &c : g.ctrl) cprod *= (double)reg.dims[c.q];
            const double nact = (double)__builtin_popcount(q.active);
            const double it = (double)reg.D / ((double)D * cprod) * nact;
            work->item_touched += it;
            if (kind == kGeneral) work->flops += 8.0 * D * it;
            if (kind < 0) work->flops += 8.0 * (q.da + D / q.da) * it;     // U_a then U_b
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
            if (fill_tile_ctrl(q.c[nc++], reg, c, v, R, LT)) q.flags |= kFRunCtrl;
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
        q.ncls = (uint32_t)((uint64_t)p.M * LT / cls_div);
        if (items[gi].b < 0 && q.nins == 1 && (D == 3 || D == 5) && (q.kind == kPGeneral || q.kind == kPPerm) &&
            st < 8 && ((st * (uint64_t)D) & 1) && q.ncls % st == 0) {
            q.flags |= kFTrans;                  // see class_idx: O = ncls / st in the second slot
            q.ins_s[1] = q.ncls / (uint32_t)st;
            q.ins_m[1] = make_fastdiv32(q.ins_s[1]).m;
        }
    }
    return p.ntiles > 0;
}

template <typename V>
static size_t pass_smem_bytes(int S, int TE) {
    // sized for the largest matrix pool so the attribute is set once per configuration
    return (size_t)S * TE * sizeof(V) + (size_t)kPoolC * sizeof(V) +
           (size_t)2 * kMaxPassGates * kMaxDim * sizeof(uint32_t) +
           (size_t)kMaxPassGates * kGDesc * sizeof(uint32_t) +
           (size_t)S * sizeof(StageInfo) + (size_t)3 * S * sizeof(uint64_t) + 16 + 16 + 32 * 16;
}

// Ring geometry of a pass: stage buffers hold the pass's actual tile (M LT amplitudes, rounded
// to 16 bytes), and the configured capacity (pass_stages x pass_tile) is spent on as many stages
// as fit (at most kMaxRing): a pass whose tile is smaller than pass_tile gets more tiles in flight
// beyond the G being computed, so a group rarely waits for its next tile.
template <typename V>
static void pass_ring(const PassParams &p, const LaunchCfg &cfg, int &S, int &TE) {
    constexpr int kMaxRing = 8;
    TE = (int)((uint64_t)p.M * p.LT);
    if (TE > cfg.pass_tile || TE <= 0) TE = cfg.pass_tile;
    TE = (TE + 1) & ~1;
    S = (int)(((int64_t)cfg.pass_stages * cfg.pass_tile) / TE);
    if (S > kMaxRing) S = kMaxRing;
    if (S < cfg.pass_stages) S = cfg.pass_stages;
    while (S > cfg.pass_stages && pass_smem_bytes<V>(S, TE) > pass_smem_bytes<V>(cfg.pass_stages, cfg.pass_tile)) --S;
}

template <int NT, int G, typename V>
cudaError_t launch_pass_t(const PassParams &p, cudaStream_t st, const LaunchCfg &cfg, int S, int TE) {
    const size_t smem = pass_smem_bytes<V>(S, TE);
    static LaunchAttr attr;
    const int dv = current_device_slot();
    if (attr.configured[dv] < smem) {
        cudaError_t e = cudaFuncSetAttribute(k_gate_pass<NT, G, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr.configured[dv] = smem;
    }
    if (attr.occ_for[dv] != smem) {   // resident CTAs per SM at this smem size (persistent grid)
        int o = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_gate_pass<NT, G, V>, NT + kPassExtra, smem) != cudaSuccess || o < 1) o = 1;
        attr.occ[dv] = o;
        attr.occ_for[dv] = smem;
    }
    const uint64_t cap = (uint64_t)cfg.num_sms * (uint64_t)attr.occ[dv];
    const unsigned grid = (unsigned)(p.ntiles < cap ? p.ntiles : cap);
    k_gate_pass<NT, G, V><<<grid, NT + kPassExtra, smem, st>>>(p, S, TE);
    return cudaGetLastError();
}

cudaError_t launch_pass(const PassParams &p, cudaStream_t st, const LaunchCfg &cfg) {
    int S, TE;
    if (cfg.c64) {                                // complex64: 512 threads, 2 or 4 groups
        pass_ring<float2>(p, cfg, S, TE);
        if (cfg.pass_groups >= 4 && S >= 4) return launch_pass_t<512, 4, float2>(p, st, cfg, S, TE);
        return launch_pass_t<512, 2, float2>(p, st, cfg, S, TE);
    }
    pass_ring<double2>(p, cfg, S, TE);
    int G = cfg.pass_groups;                      // one stage per group at least
    while (G > 1 && S < G) G /= 2;
    if (cfg.pass_threads >= 960) return launch_pass_t<960, 2, double2>(p, st, cfg, S, TE);   // 32 warps, 64 registers
    if (cfg.pass_threads >= 768) return launch_pass_t<768, 2, double2>(p, st, cfg, S, TE);   // 26 warps, 72 registers
    if (cfg.pass_threads == 576) {                // 18 compute warps + 2 = 5 warps per scheduler at 96 registers
        if (cfg.pass_groups == 3 && S >= 3) return launch_pass_t<576, 3, double2>(p, st, cfg, S, TE);
        return launch_pass_t<576, 2, double2>(p, st, cfg, S, TE);
    }
    if (cfg.pass_threads >= 512) {
        if (G >= 8) return launch_pass_t<512, 8, double2>(p, st, cfg, S, TE);
        if (G >= 4) return launch_pass_t<512, 4, double2>(p, st, cfg, S, TE);
        if (G == 2) return launch_pass_t<512, 2, double2>(p, st, cfg, S, TE);
        return launch_pass_t<512, 1, double2>(p, st, cfg, S, TE);
    }
    if (cfg.pass_threads >= 384) {
        if (cfg.pass_groups == 3 && S >= 3) return launch_pass_t<384, 3, double2>(p, st, cfg, S, TE);
        if (G >= 2) return launch_pass_t<384, 2, double2>(p, st, cfg, S, TE);
        return launch_pass_t<384, 1, double2>(p, st, cfg, S, TE);
    }
    if (G >= 2) return launch_pass_t<256, 2, double2>(p, st, cfg, S, TE);
    return launch_pass_t<256, 1, double2>(p, st, cfg, S, TE);
}

// ---- register-blocked stages: host side
// Group the pass's gates (in pass order) into stages and fill the stage kernel's parameters.
// Returns false (the caller then uses k_gate_pass) if a target digit has d > 5, a gate has more
// than kMaxPassCtrl controls, or the matrix pool overflows.
bool build_stage_pass(const Register &reg, const std::vector<GateSpec> &gates, const PassPlan &pp, double2 *psi,
                      int TE, StageParams &p, PassWork *work) {
    std::memset(&p, 0, sizeof(p));
    if ((int)pp.gates.size() > kMaxPassGates || pp.tile > (uint64_t)TE) return false;
    std::vector<uint64_t> W;
    uint64_t R = 0, LT = 0;
    if (!pass_geometry(reg, pp, psi, TE, p, W, R, LT)) return false;
    const int m0 = pp.m0;
    auto in_tile = [&](int q) { return q < m0 || std::find(pp.H.begin(), pp.H.end(), q) != pp.H.end(); };
    auto tile_stride = [&](int q) -> uint64_t { return q < m0 ? reg.b[q] : W[q] * LT; };
    for (int i : pp.gates) {
        const GateSpec &g = gates[i];
        if (g.span != 1 || !in_tile(g.target) || g.d > 5 || (int)g.ctrl.size() > kMaxPassCtrl) return false;
    }
    std::vector<int> tiled;                      // in-tile digits: passive partners for 1-digit stages
    for (int q = 0; q < reg.n; ++q)
        if (in_tile(q)) tiled.push_back(q);
    // stages: maximal runs of consecutive gates whose targets fit one digit pair
    struct St { int a, b; std::vector<int> g; };
    std::vector<St> stages;
    for (int i : pp.gates) {
        const int t = gates[i].target;
        if (!stages.empty()) {
            St &c = stages.back();
            if (t == c.a || t == c.b) { c.g.push_back(i); continue; }
            if (c.b < 0 && reg.dims[c.a] * reg.dims[t] <= kStageAmps) { c.b = t; c.g.push_back(i); continue; }
        }
        stages.push_back({t, -1, {i}});
    }
    if ((int)stages.size() > kMaxPassGates) return false;
    *work = PassWork{};
    int ng = 0, uoff = 0;
    const double Dloc = (double)reg.D;
    for (size_t si = 0; si < stages.size(); ++si) {
        St &S = stages[si];
        if (S.b < 0) {                           // passive partner: the smallest in-tile dim that fits
            int best = -1;
            for (int q : tiled)
                if (q != S.a && reg.dims[S.a] * reg.dims[q] <= kStageAmps &&
                    (best < 0 || reg.dims[q] < reg.dims[best] || (reg.dims[q] == reg.dims[best] && q > best)))
                    best = q;
            S.b = best;                          // may stay -1 (a one-digit tile): d_b = 1
        }
        if (S.b >= 0 && tile_stride(S.b) < tile_stride(S.a)) std::swap(S.a, S.b);   // a = lower stride
        StageRec &r = p.st[si];
        r.da = reg.dims[S.a];
        r.db = S.b >= 0 ? reg.dims[S.b] : 1;
        r.sa = (uint32_t)tile_stride(S.a);
        r.sb = S.b >= 0 ? (uint32_t)tile_stride(S.b) : 0u;
        r.nblk = (uint32_t)((uint64_t)p.M * LT / (uint64_t)(r.da * r.db));
        r.s0 = r.sa;
        r.m0 = make_fastdiv32(r.s0).m;
        r.sd0 = r.sa * (uint32_t)r.da;
        r.s1 = S.b >= 0 ? r.sb : 1u;
        r.m1 = S.b >= 0 ? make_fastdiv32(r.s1).m : 0u;
        r.sd1 = S.b >= 0 ? r.sb * (uint32_t)r.db : 1u;
        r.g0 = ng;
        r.ng = (int32_t)S.g.size();
        work->item_touched += Dloc;              // the stage's one shared-memory round trip
        for (int gi : S.g) {
            const GateSpec &g = gates[gi];
            GatePlan gp;
            std::string err;
            if (plan_gate(reg, g, false, &gp, &err) != SV_OK) return false;
            work->touched += (double)gp.touched;
            StageGate &q = p.g[ng++];
            q.axis = g.target == S.a ? 0 : 1;
            q.octrl = -1;
            const int d = g.d;
            // kind: diagonal (§2.1), pure cyclic shift X_{+s} (§2.2), else the general rule (§2.3)
            bool diag = true, shift = true;
            int sh = -1;
            for (int i = 0; i < d; ++i)
                for (int j = 0; j < d; ++j) {
                    const double2 u = g.U[(size_t)i * d + j];
                    const bool nz = u.x != 0.0 || u.y != 0.0;
                    if (i != j && nz) diag = false;
                    if (nz) {
                        const int k = ((i - j) % d + d) % d;
                        if (!(u.x == 1.0 && u.y == 0.0) || (sh >= 0 && k != sh)) shift = false;
                        sh = k;
                    }
                }
            if (sh <= 0) shift = false;
            double cprod = 1.0;
            for (const auto &c : g.ctrl) cprod *= (double)reg.dims[c.q];
            const int need = shift ? 0 : (diag ? d : d * d);
            if (uoff + need > kPoolS) return false;
            q.uoff = uoff;
            if (shift) {
                q.kind = kSShift;
                q.shift = sh;
            } else if (diag) {
                q.kind = kSDiag;
                for (int j = 0; j < d; ++j) p.U[uoff + j] = g.U[(size_t)j * d + j];
            } else {
                q.kind = kSGeneral;
                for (int k = 0; k < d * d; ++k) p.U[uoff + k] = g.U[k];
                work->flops += 8.0 * d * (Dloc / cprod);
            }
            uoff += need;
            for (const auto &c : g.ctrl) {
                const uint32_t v = (uint32_t)c.v;
                if (c.q == S.a || c.q == S.b) { q.octrl = (int32_t)v; continue; }
                if (in_tile(c.q)) {
                    const int k = q.nic++;
                    q.ic_s[k] = (uint32_t)tile_stride(c.q);
                    q.ic_m[k] = make_fastdiv32(q.ic_s[k]).m;
                    q.ic_d[k] = (uint32_t)reg.dims[c.q];
                    q.ic_dm[k] = make_fastdiv32(q.ic_d[k]).m;
                    q.ic_v[k] = v;
                    continue;
                }
                if (fill_tile_ctrl(q.c[q.nctrl++], reg, c.q, v, R, LT)) q.runck = 1;
            }
        }
    }
    p.nstages = (int32_t)stages.size();
    p.ngates = ng;
    p.upool = uoff;
    return p.ntiles > 0;
}

template <int NT, int G, typename V>
cudaError_t launch_stage_t(const StageParams &p, cudaStream_t st, const LaunchCfg &cfg) {
    const int S = cfg.pass_stages, TE = cfg.pass_tile;
    const size_t smem = (size_t)S * TE * sizeof(V) + (size_t)kPoolS * sizeof(V) + (size_t)S * sizeof(StageInfo) +
                        (size_t)3 * S * sizeof(uint64_t);
    static LaunchAttr attr;
    const int dv = current_device_slot();
    if (attr.configured[dv] < smem) {
        cudaError_t e = cudaFuncSetAttribute(k_gate_stage<NT, G, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr.configured[dv] = smem;
    }
    if (attr.occ_for[dv] != smem) {
        int o = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_gate_stage<NT, G, V>, NT + kPassExtra, smem) != cudaSuccess || o < 1) o = 1;
        attr.occ[dv] = o;
        attr.occ_for[dv] = smem;
    }
    const uint64_t cap = (uint64_t)cfg.num_sms * (uint64_t)attr.occ[dv];
    const unsigned grid = (unsigned)(p.ntiles < cap ? p.ntiles : cap);
    k_gate_stage<NT, G, V><<<grid, NT + kPassExtra, smem, st>>>(p, S, TE);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess && getenv("SV_DEBUG_LAUNCH")) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, k_gate_stage<NT, G, V>);
        fprintf(stderr, "k_gate_stage<%d,%d> launch %s: grid %u block %d smem %zu | regs %d maxThreads %d static smem %zu "
                        "maxDyn %d local %zu\n", NT, G, cudaGetErrorString(e), grid, NT + kPassExtra, smem, fa.numRegs,
                fa.maxThreadsPerBlock, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.localSizeBytes);
    }
    return e;
}

cudaError_t launch_stage(const StageParams &p, cudaStream_t st, const LaunchCfg &cfg) {
    if (cfg.c64) return launch_stage_t<512, 2, float2>(p, st, cfg);
    int G = cfg.pass_groups;
    while (G > 1 && cfg.pass_stages < G) G /= 2;
    if (cfg.pass_threads >= 512) {
        if (G >= 2) return launch_stage_t<512, 2, double2>(p, st, cfg);
        return launch_stage_t<512, 1, double2>(p, st, cfg);
    }
    if (cfg.pass_threads >= 384) {
        if (G >= 2) return launch_stage_t<384, 2, double2>(p, st, cfg);
        return launch_stage_t<384, 1, double2>(p, st, cfg);
    }
    if (G >= 2) return launch_stage_t<256, 2, double2>(p, st, cfg);
    return launch_stage_t<256, 1, double2>(p, st, cfg);
}

cudaError_t run_pass(const Register &reg, const std::vector<GateSpec> &gates, const PassPlan &pp, double2 *psi,
                     cudaStream_t st, const LaunchCfg &cfg, bool *handled, PassWork *work) {
    // register-blocked stages (k_gate_stage) when selected and the pass fits them
    if (cfg.pass_kernel == 1) {
        static thread_local StageParams sp;   // ~27 KB; parameters are copied at launch
        if (build_stage_pass(reg, gates, pp, psi, cfg.pass_tile, sp, work) &&
            !(cfg.c64 && (sp.L % 2 != 0 || sp.LT % 2 != 0))) {
            *handled = true;
            return launch_stage(sp, st, cfg);
        }
    }
    static thread_local PassParams p;   // ~23 KB; parameters are copied at launch
    *handled = build_pass(reg, gates, pp, psi, cfg.pass_tile, p, work, cfg.pass_absorb != 0);
    // complex64 (8-byte elements): every bulk copy must start at a 16-byte aligned address and
    // move a multiple of 16 bytes; tile runs are multiples of L = b_{m0} and start at multiples
    // of L, so an even L suffices (the stage needs the tile plus the fp32 matrix pool)
    if (*handled && cfg.c64 && (p.L % 2 != 0 || p.LT % 2 != 0)) *handled = false;
    if (!*handled) return cudaSuccess;
    return launch_pass(p, st, cfg);
}

}  // namespace svi
