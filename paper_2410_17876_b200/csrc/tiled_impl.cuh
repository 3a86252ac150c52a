// tiled_impl.cuh — the TMA-bulk staged gate kernel for sm_100a (templates; instantiated per
// target dimension in tiled_*.cu so the build parallelises).
//
// Same math as the direct kernel (visit every control-satisfying
// equivalence class, y = U x, store back in place), but the data moves in whole tiles:
//   * one elected warp computes the tile's contiguous global pieces and issues one
//     cp.async.bulk (TMA bulk copy, SASS UBLKCP) per piece into a shared-memory stage, all
//     completing on one mbarrier (complete_tx);
//   * all warps compute the classes of the tile out of shared memory, in place;
//   * the same warp writes the pieces back with cp.async.bulk shared->global (bulk_group).
// A ring of S stages keeps S-1 tiles of loads in flight per CTA while one is computed;
// the grid is persistent (ctas_per_sm x SM count) and strides over the tiles.
//
// Tile geometry (host: plan_tiled):
//   mode W ("member-split", target stride b_k >= 32 or an enumerated control below it):
//     classes are enumerated in runs of B0 consecutive class ids (B0 = stride of the lowest
//     removed digit); within a run every member j is one contiguous piece at
//     insert(f0) + j b_k.  A tile = one sub-run (B0 >= LT) or rpt whole runs (B0 < LT);
//     smem layout [member][class].
//   mode N ("group", target stride b_k < 32): a tile is a contiguous range of whole groups
//     of G = d b_k amplitudes (every class complete inside the tile), possibly several
//     runs when an enumerated control above the target breaks contiguity.
// Controls with stride >= 32 amplitudes are enumerated (digit insertion, never loaded when
// unmet); controls with stride < 32 are predicated per class inside the tile.
#pragma once
#include <cuda_runtime.h>

#include <cstring>

#include "sv_internal.h"

namespace svi {

constexpr int kRunMin = 32;          // controls with stride >= kRunMin are enumerated
constexpr int kTileThreads = 256;
// piece table per stage: TE/32 entries (every piece is >= 32 amplitudes)

enum TileMode : int { kModeW = 0, kModeN = 1 };
enum TileKind : int { kTGeneral = 0, kTMono = 1, kTPerm = 2 };

struct InnerCtrl {
    uint32_t b, mb;     // stride and 32-bit magic
    uint32_t d, md;     // dim and magic
    uint32_t M, mM;     // b*d and magic
    uint64_t mM64;      // 64-bit magic for M
    uint32_t v;
};

template <int MD, typename V = double2>
struct TileParams {
    V *psi;
    int32_t mode, kind, d, nm;
    uint64_t bk;
    int32_t nrem;
    RemovedRun rem[kMaxRem];
    // schedule
    uint64_t ntiles;
    uint64_t nruns;
    uint64_t R;          // run length: classes (W) or elements (N)
    uint32_t per_tile;   // W: classes per member per tile (LT); N: elements per tile
    uint32_t rpt;        // runs per tile (1 when a run spans several tiles)
    uint64_t tpr, tpr_m; // tiles per run (+ magic) when rpt == 1
    uint32_t MS;         // W: smem member stride (elements)
    uint32_t R32, mR32;  // run length + magic when rpt > 1 (for in-tile run index)
    uint32_t G, b32, mb32;   // N: group length, target stride (+ magic)
    int32_t members[MD];     // W: member j of compact slot jj
    int32_t slot_of[MD];     // W: compact slot of member j (or -1)
    int32_t sigma[MD];       // monomial/perm: member j -> sigma[j]
    uint32_t active;
    int32_t ninner;
    InnerCtrl inner[kMaxInner];
    V U[MD * MD];            // general: row-major (stride MD); monomial: U[j] = coef of member j
};

struct Piece {
    uint64_t g;      // global element index of the piece start (load address)
    uint32_t s;      // smem element offset
    uint32_t len;    // elements
};

// ------------------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void *smem_dst, const void *gsrc, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_store(void *gdst, const void *smem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }


// ------------------------------------------------------------------------------ tiles
struct TileDesc {
    uint64_t run0;   // first run of the tile
    uint64_t off;    // offset inside the run (rpt == 1), classes (W) or elements (N)
    uint32_t nr;     // runs in the tile
    uint32_t len;    // classes (W) / elements (N) per run piece
};

template <int MD, typename V>
__device__ __forceinline__ TileDesc tile_desc(const TileParams<MD, V> &p, uint64_t t) {
    TileDesc td;
    if (p.rpt == 1) {
        uint64_t sub;
        const uint64_t run = fastdiv64(t, p.tpr, p.tpr_m, sub);
        td.run0 = run;
        td.off = sub * p.per_tile;
        const uint64_t rem = p.R - td.off;
        td.len = (uint32_t)(rem < p.per_tile ? rem : p.per_tile);
        td.nr = 1;
    } else {
        td.run0 = t * p.rpt;
        td.off = 0;
        const uint64_t left = p.nruns - td.run0;
        td.nr = (uint32_t)(left < p.rpt ? left : p.rpt);
        td.len = (uint32_t)p.R;
    }
    return td;
}

// warp 0: fill the piece table of a stage and issue the bulk loads
template <int MD, typename V>
__device__ __forceinline__ void issue_tile_loads(const TileParams<MD, V> &p, uint64_t t, V *buf,
                                                 Piece *pieces, uint32_t *npieces, uint64_t *bar,
                                                 int lane) {
    const TileDesc td = tile_desc(p, t);
    const int nm = (p.mode == kModeW) ? p.nm : 1;
    const uint32_t np = td.nr * (uint32_t)nm;
    if (lane == 0) {
        *npieces = np;
        mbar_expect_tx(bar, np * td.len * (uint32_t)sizeof(V));
    }
    __syncwarp();
    for (uint32_t q = lane; q < np; q += 32) {
        const uint32_t r = q / (uint32_t)nm;
        const uint32_t jj = q - r * (uint32_t)nm;
        Piece pc;
        if (p.mode == kModeW) {
            const uint64_t f0 = (td.run0 + r) * p.R + td.off;
            const uint64_t base = insert_digits(f0, p.nrem, p.rem);
            pc.g = base + (uint64_t)p.members[jj] * p.bk;
            pc.s = jj * p.MS + r * td.len;
        } else {
            const uint64_t e0 = (td.run0 + r) * p.R + td.off;
            pc.g = insert_digits(e0, p.nrem, p.rem);
            pc.s = r * td.len;
        }
        pc.len = td.len;
        pieces[q] = pc;
        bulk_load(buf + pc.s, p.psi + pc.g, pc.len * (uint32_t)sizeof(V), bar);
    }
}

template <int MD, typename V>
__device__ __forceinline__ bool inner_ok(const TileParams<MD, V> &p, const uint32_t *offmod, uint32_t pos) {
    bool ok = true;
#pragma unroll 1
    for (int c = 0; c < p.ninner; ++c) {
        const InnerCtrl &ic = p.inner[c];
        uint32_t r, r2, r3;
        fastdiv32(offmod[c] + pos, ic.M, ic.mM, r);      // position mod M
        const uint32_t q = fastdiv32(r, ic.b, ic.mb, r2);
        fastdiv32(q, ic.d, ic.md, r3);
        ok = ok && (r3 == ic.v);
    }
    return ok;
}

template <int DIM, int MD, int MODE, int KIND, typename V>
__global__ void __launch_bounds__(kTileThreads) k_gate_tiled(const __grid_constant__ TileParams<MD, V> p,
                                                             int S, int TE) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    V *bufs = reinterpret_cast<V *>(smem_raw);
    const int maxp = TE / 32;
    Piece *ptab = reinterpret_cast<Piece *>(smem_raw + (size_t)S * TE * sizeof(V));
    uint32_t *npc = reinterpret_cast<uint32_t *>(ptab + (size_t)S * maxp);
    uint64_t *bars = reinterpret_cast<uint64_t *>(npc + ((S + 1) & ~1));

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int d = DIM ? DIM : p.d;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint64_t first = blockIdx.x, step = gridDim.x;
    if (first >= p.ntiles) return;
    const uint64_t my = (p.ntiles - first + step - 1) / step;   // tiles of this CTA

    if (warp == 0) {
        for (int i = 0; i < S - 1 && (uint64_t)i < my; ++i)
            issue_tile_loads(p, first + (uint64_t)i * step, bufs + (size_t)i * TE, ptab + (size_t)i * maxp,
                             &npc[i], &bars[i], lane);
    }

    uint32_t offmod[kMaxInner];
    for (uint64_t i = 0; i < my; ++i) {
        const int s = (int)(i % (uint64_t)S);
        const uint64_t t = first + i * step;
        V *buf = bufs + (size_t)s * TE;
        mbar_wait(&bars[s], (uint32_t)((i / (uint64_t)S) & 1));

        if (KIND != kTPerm || MODE == kModeN) {
            const TileDesc td = tile_desc(p, t);
            // per-tile offsets of the inner-control positions (mod M, 64-bit once per tile)
            if (p.ninner) {
                for (int c = 0; c < p.ninner; ++c) {
                    uint64_t r;
                    fastdiv64(td.off, p.inner[c].M, p.inner[c].mM64, r);
                    offmod[c] = (uint32_t)r;
                }
            }
            if (MODE == kModeW) {
                const uint32_t ncls = td.nr * td.len;
                for (uint32_t c = tid; c < ncls; c += kTileThreads) {
                    if (p.ninner) {
                        uint32_t pos = c;
                        if (td.nr > 1) fastdiv32(c, p.R32, p.mR32, pos);
                        if (!inner_ok(p, offmod, pos)) continue;
                    }
                    if (KIND == kTGeneral) {
                        V x[MD];
#pragma unroll
                        for (int j = 0; j < MD; ++j)
                            if (DIM || j < d) x[j] = buf[j * p.MS + c];
#pragma unroll
                        for (int i2 = 0; i2 < MD; ++i2) {
                            if (DIM || i2 < d) {
                                V acc = cz<V>();
#pragma unroll
                                for (int j = 0; j < MD; ++j)
                                    if (DIM || j < d) cfma(acc, p.U[i2 * MD + j], x[j]);
                                buf[i2 * p.MS + c] = acc;
                            }
                        }
                    } else {   // monomial with coefficients: slot jj holds member members[jj]
                        V x[MD];
#pragma unroll
                        for (int jj = 0; jj < MD; ++jj)
                            if (jj < p.nm) x[jj] = buf[jj * p.MS + c];
#pragma unroll
                        for (int jj = 0; jj < MD; ++jj)
                            if (jj < p.nm) {
                                const int j = p.members[jj];
                                buf[p.slot_of[p.sigma[j]] * p.MS + c] = cmul(p.U[j], x[jj]);
                            }
                    }
                }
            } else {   // mode N: whole groups in the tile
                const uint32_t nel = td.nr * td.len;
                const uint32_t ncls = nel / (uint32_t)d;
                for (uint32_t c = tid; c < ncls; c += kTileThreads) {
                    uint32_t off;
                    const uint32_t g = fastdiv32(c, p.b32, p.mb32, off);
                    const uint32_t e = g * p.G + off;            // member-0 element in the tile
                    if (p.ninner) {
                        uint32_t pos = e;
                        if (td.nr > 1) fastdiv32(e, p.R32, p.mR32, pos);
                        if (!inner_ok(p, offmod, pos)) continue;
                    }
                    V *cls = buf + e;
                    V x[MD];
                    if (KIND == kTGeneral) {
#pragma unroll
                        for (int j = 0; j < MD; ++j)
                            if (DIM || j < d) x[j] = cls[j * p.b32];
#pragma unroll
                        for (int i2 = 0; i2 < MD; ++i2) {
                            if (DIM || i2 < d) {
                                V acc = cz<V>();
#pragma unroll
                                for (int j = 0; j < MD; ++j)
                                    if (DIM || j < d) cfma(acc, p.U[i2 * MD + j], x[j]);
                                cls[i2 * p.b32] = acc;
                            }
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < MD; ++j)
                            if ((DIM || j < d) && ((p.active >> j) & 1)) x[j] = cls[j * p.b32];
#pragma unroll
                        for (int j = 0; j < MD; ++j)
                            if ((DIM || j < d) && ((p.active >> j) & 1))
                                cls[p.sigma[j] * p.b32] = (KIND == kTPerm) ? x[j] : cmul(p.U[j], x[j]);
                    }
                }
            }
            fence_proxy_async();
        }
        __syncthreads();

        if (warp == 0) {
            const Piece *pcs = ptab + (size_t)s * maxp;
            const uint32_t np = npc[s];
            for (uint32_t q = lane; q < np; q += 32) {
                const Piece pc = pcs[q];
                uint64_t g = pc.g;
                if (MODE == kModeW && KIND == kTPerm) {     // pure permutation: store to sigma(j)
                    const uint32_t jj = q % (uint32_t)p.nm;
                    const int j = p.members[jj];
                    g = g + ((uint64_t)p.sigma[j] - (uint64_t)j) * p.bk;
                }
                bulk_store(p.psi + g, buf + pc.s, pc.len * (uint32_t)sizeof(V));
            }
            bulk_commit();
            // refill the stage of tile i-1 once its store has finished reading smem
            const uint64_t nxt = i + (uint64_t)(S - 1);
            if (nxt < my) {
                bulk_wait_read_1();
                __syncwarp();
                const int sn = (int)(nxt % (uint64_t)S);
                issue_tile_loads(p, first + nxt * step, bufs + (size_t)sn * TE, ptab + (size_t)sn * maxp,
                                 &npc[sn], &bars[sn], lane);
            }
        }
    }
    if (warp == 0) bulk_wait_all();
}

// ------------------------------------------------------------------------------ host
template <int MD, typename V>
bool plan_tiled(const GatePlan &g, V *psi, const LaunchCfg &cfg, TileParams<MD, V> &p) {
    memset(&p, 0, sizeof(p));
    const int d = g.d;
    const uint64_t bk = g.bk;
    const int TE = cfg.tile_elems;
    p.psi = psi;
    p.d = d;
    p.bk = bk;
    // controls: inner (predicated) vs outer (enumerated)
    struct Rem { uint64_t b; uint64_t dim; uint64_t pin; };
    Rem rems[66];
    int nr = 0;
    uint64_t outer_prod = 1;
    for (int i = 0; i < g.nctrl; ++i) {
        if (g.cb[i] < (uint64_t)kRunMin) {
            if (p.ninner >= kMaxInner) return false;
            InnerCtrl &ic = p.inner[p.ninner++];
            ic.b = (uint32_t)g.cb[i];
            ic.mb = make_fastdiv32(ic.b).m;
            ic.d = g.cd[i];
            ic.md = make_fastdiv32(ic.d).m;
            ic.M = ic.b * ic.d;
            ic.mM = make_fastdiv32(ic.M).m;
            ic.mM64 = make_fastdiv64(ic.M).m;
            ic.v = g.cv[i];
        } else {
            rems[nr++] = {g.cb[i], g.cd[i], g.cv[i]};
            outer_prod *= g.cd[i];
        }
    }
    // kind and the members that are loaded
    if (g.kind == kGeneral) {
        p.kind = kTGeneral;
        p.nm = d;
        for (int j = 0; j < d; ++j) { p.members[j] = j; p.slot_of[j] = j; p.sigma[j] = j; }
        for (int i = 0; i < d; ++i)
            for (int j = 0; j < d; ++j) p.U[i * MD + j] = to_v<V>(g.U[i * d + j]);
    } else {
        bool pure = true;
        int nm = 0;
        for (int j = 0; j < MD; ++j) p.slot_of[j] = -1;
        for (int j = 0; j < d; ++j) {
            p.sigma[j] = g.sigma[j];
            p.U[j] = to_v<V>(g.U[j]);
            if ((g.active >> j) & 1) {
                p.slot_of[j] = nm;
                p.members[nm++] = j;
                if (g.U[j].x != 1.0 || g.U[j].y != 0.0) pure = false;
            }
        }
        p.nm = nm;
        p.active = g.active;
        // a pure permutation moves whole pieces without touching smem -- only valid when every
        // class of the tile fires, i.e. no predicated (inner) control
        p.kind = (pure && p.ninner == 0) ? kTPerm : kTMono;
    }
    const bool modeN = bk < (uint64_t)kRunMin;
    p.mode = modeN ? kModeN : kModeW;
    if (!modeN) rems[nr++] = {bk, (uint64_t)d, 0};    // the target is removed (pin 0)
    // sort removed digits by stride, merge adjacent ones (b_hi == b_lo * dim_lo)
    for (int i = 1; i < nr; ++i)
        for (int j = i; j > 0 && rems[j].b < rems[j - 1].b; --j) { Rem t = rems[j]; rems[j] = rems[j - 1]; rems[j - 1] = t; }
    int nm_ = 0;
    for (int i = 0; i < nr; ++i) {
        if (nm_ > 0 && rems[i].b == p.rem[nm_ - 1].bd) {
            RemovedRun &r = p.rem[nm_ - 1];
            const uint64_t dim_lo = r.bd / r.b;
            r.pinb += rems[i].pin * dim_lo * r.b;
            r.bd *= rems[i].dim;
        } else {
            if (nm_ >= kMaxRem) return false;
            RemovedRun &r = p.rem[nm_++];
            r.b = rems[i].b;
            r.bd = rems[i].b * rems[i].dim;
            r.pinb = rems[i].pin * rems[i].b;
            r.m = make_fastdiv64(r.b).m;
        }
    }
    p.nrem = nm_;
    if (!modeN) {
        const uint64_t F = g.D / ((uint64_t)d * outer_prod);
        const uint64_t B0 = p.rem[0].b;                 // lowest removed stride = run length
        uint32_t LT = (uint32_t)(TE / p.nm);
        if (LT < 1) return false;
        p.R = B0;
        p.nruns = F / B0;
        if (B0 >= LT) {
            p.per_tile = LT;
            p.rpt = 1;
            p.tpr = (B0 + LT - 1) / LT;
            p.ntiles = p.nruns * p.tpr;
            p.MS = LT;
        } else {
            p.per_tile = LT;
            p.rpt = LT / (uint32_t)B0;
            p.ntiles = (p.nruns + p.rpt - 1) / p.rpt;
            p.MS = p.rpt * (uint32_t)B0;
            p.R32 = (uint32_t)B0;
            p.mR32 = make_fastdiv32(p.R32).m;
        }
        if ((uint64_t)p.rpt * p.nm > (uint64_t)(TE / 32)) return false;
    } else {
        const uint64_t G = (uint64_t)d * bk;
        if (G > (uint64_t)TE) return false;
        p.G = (uint32_t)G;
        p.b32 = (uint32_t)bk;
        p.mb32 = make_fastdiv32(p.b32).m;
        const uint64_t E = g.D / outer_prod;           // compressed elements
        const uint64_t R = nm_ ? p.rem[0].b : E;        // contiguous run (elements)
        const uint32_t per = (uint32_t)((TE / G) * G);
        p.R = R;
        p.nruns = E / R;
        p.per_tile = per;
        if (R >= per) {
            p.rpt = 1;
            p.tpr = (R + per - 1) / per;
            p.ntiles = p.nruns * p.tpr;
        } else {
            p.rpt = (uint32_t)(TE / R);
            p.ntiles = (p.nruns + p.rpt - 1) / p.rpt;
            p.R32 = (uint32_t)R;
            p.mR32 = make_fastdiv32(p.R32).m;
        }
        if (p.rpt > (uint32_t)(TE / 32)) return false;
        p.nm = 1;
    }
    p.tpr_m = make_fastdiv64(p.tpr ? p.tpr : 1).m;
    return p.ntiles > 0;
}

template <int DIM, int MD, int MODE, int KIND, typename V>
cudaError_t launch_tiled_k(const TileParams<MD, V> &p, const LaunchCfg &cfg, cudaStream_t st) {
    const int S = cfg.tile_stages, TE = cfg.tile_elems;
    const size_t smem = (size_t)S * TE * sizeof(V) + (size_t)S * (TE / 32) * sizeof(Piece) +
                        (size_t)((S + 1) & ~1) * sizeof(uint32_t) + (size_t)S * sizeof(uint64_t);
    static LaunchAttr attr;
    const int dv = current_device_slot();
    auto kfn = k_gate_tiled<DIM, MD, MODE, KIND, V>;
    if (attr.configured[dv] < smem) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr.configured[dv] = smem;
    }
    if (attr.occ_for[dv] != smem) {   // resident CTAs per SM for this smem size (persistent grid)
        int o = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kfn, kTileThreads, smem) != cudaSuccess || o < 1) o = 1;
        attr.occ[dv] = o;
        attr.occ_for[dv] = smem;
    }
    const int occ = attr.occ[dv];
    const int per_sm = cfg.ctas_per_sm < occ ? cfg.ctas_per_sm : occ;
    const uint64_t cap = (uint64_t)cfg.num_sms * per_sm;
    const unsigned grid = (unsigned)(p.ntiles < cap ? p.ntiles : cap);
    kfn<<<grid, kTileThreads, smem, st>>>(p, S, TE);
    return cudaGetLastError();
}

template <int DIM, int MD, typename V>
cudaError_t launch_tiled_v(const GatePlan &g, V *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled) {
    TileParams<MD, V> p;
    if (!plan_tiled<MD, V>(g, psi, cfg, p)) { *handled = false; return cudaSuccess; }
    *handled = true;
    if (p.mode == kModeW) {
        if (p.kind == kTGeneral) return launch_tiled_k<DIM, MD, kModeW, kTGeneral, V>(p, cfg, st);
        if (p.kind == kTMono) return launch_tiled_k<DIM, MD, kModeW, kTMono, V>(p, cfg, st);
        return launch_tiled_k<DIM, MD, kModeW, kTPerm, V>(p, cfg, st);
    }
    if (p.kind == kTGeneral) return launch_tiled_k<DIM, MD, kModeN, kTGeneral, V>(p, cfg, st);
    if (p.kind == kTMono) return launch_tiled_k<DIM, MD, kModeN, kTMono, V>(p, cfg, st);
    return launch_tiled_k<DIM, MD, kModeN, kTPerm, V>(p, cfg, st);
}

template <int DIM, int MD>
cudaError_t launch_tiled_d(const GatePlan &g, double2 *psi, cudaStream_t st, const LaunchCfg &cfg, bool *handled) {
    if (cfg.c64) return launch_tiled_v<DIM, MD, float2>(g, reinterpret_cast<float2 *>(psi), st, cfg, handled);
    return launch_tiled_v<DIM, MD, double2>(g, psi, st, cfg, handled);
}

}  // namespace svi

#define SV_TILED_DIM(DIM, MD)                                                                      \
    namespace svi {                                                                                \
    cudaError_t launch_tiled_dim##DIM(const GatePlan &g, double2 *psi, cudaStream_t st,           \
                                      const LaunchCfg &cfg, bool *handled) {                       \
        return launch_tiled_d<DIM, MD>(g, psi, st, cfg, handled);                                  \
    }                                                                                              \
    }
