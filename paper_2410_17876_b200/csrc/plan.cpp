// plan.cpp — host-side register model, validation, classification, fibre-decomposer setup,
// fusion and shard planning.  Product code (no oracle dependency).
#include "plan.h"

#include <algorithm>
#include <functional>
#include <cmath>
#include <cstring>

namespace svi {

sv_status make_register(const int32_t *dims, int32_t n, Register *reg, std::string *err) {
    if (!dims || !reg) { *err = "null dims/handle"; return SV_ERR_INVALID_ARG; }
    if (n < 1 || n > 64) { *err = "register must have 1..64 qudits"; return SV_ERR_DIM; }
    uint64_t p = 1;
    for (int k = 0; k < n; ++k) {
        if (dims[k] < 2 || dims[k] > kMaxDim) {
            *err = "qudit " + std::to_string(k) + " has dimension " + std::to_string(dims[k]) +
                   " (need 2..16)";
            return SV_ERR_DIM;
        }
        reg->dims[k] = dims[k];
        reg->b[k] = p;                                   // b_k = prod_{t<k} d_t
        if (p > UINT64_MAX / (uint64_t)dims[k]) { *err = "D overflows uint64"; return SV_ERR_OVERFLOW; }
        p *= (uint64_t)dims[k];
    }
    reg->n = n;
    reg->D = p;
    return SV_OK;
}

sv_status validate_gate(const Register &reg, int target, const int32_t *ctrl, const int32_t *vals,
                        int nctrl, const double *U, std::string *err) {
    if (!U) { *err = "null U"; return SV_ERR_INVALID_ARG; }
    if (target < 0 || target >= reg.n) { *err = "target qudit out of range"; return SV_ERR_QUDIT_RANGE; }
    if (nctrl < 0 || nctrl >= reg.n) { *err = "bad control count"; return SV_ERR_INVALID_ARG; }
    if (nctrl > 0 && (!ctrl || !vals)) { *err = "null control arrays"; return SV_ERR_INVALID_ARG; }
    for (int i = 0; i < nctrl; ++i) {
        const int c = ctrl[i];
        if (c < 0 || c >= reg.n) { *err = "control qudit out of range"; return SV_ERR_QUDIT_RANGE; }
        if (c == target) { *err = "control equals target"; return SV_ERR_CTRL_OVERLAP; }
        for (int j = 0; j < i; ++j)
            if (ctrl[j] == c) { *err = "duplicate control qudit"; return SV_ERR_CTRL_DUP; }
        if (vals[i] < 0 || vals[i] >= reg.dims[c]) { *err = "control value out of range"; return SV_ERR_CTRL_VALUE; }
    }
    return SV_OK;
}

double unitarity_error(const double2 *U, int d) {
    double worst = 0.0;
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            double re = 0.0, im = 0.0;
            for (int k = 0; k < d; ++k) {   // (U^dag U)_{ij} = sum_k conj(U_ki) U_kj
                const double2 a = U[k * d + i], b = U[k * d + j];
                re += a.x * b.x + a.y * b.y;
                im += a.x * b.y - a.y * b.x;
            }
            if (i == j) re -= 1.0;
            const double e = std::sqrt(re * re + im * im);
            if (!(e == e) || std::isinf(e)) return INFINITY;
            worst = std::max(worst, e);
        }
    return worst;
}

sv_status plan_gate(const Register &reg, const GateSpec &g, bool check_unitary, GatePlan *out,
                    std::string *err) {
    GatePlan &p = *out;
    std::memset(&p, 0, sizeof(p));
    const int d = g.d;
    if (d < 2 || d > kMaxDim) { *err = "gate dimension out of range"; return SV_ERR_UNSUPPORTED; }
    p.d = d;
    p.bk = reg.b[g.target];
    p.uerr = unitarity_error(g.U.data(), d);
    if (check_unitary && !(p.uerr <= 1e-12)) {
        *err = "U is not unitary (max |U^dag U - I| = " + std::to_string(p.uerr) + ")";
        return SV_ERR_NOT_UNITARY;
    }
    for (int i = 0; i < d * d; ++i) p.U[i] = g.U[i];

    // ---- classification (§2.1 phase, §2.2 permutation, §2.3 superposition).
    // Monomial = every column has exactly one non-zero entry (exact zeros elsewhere): then
    // y_{sigma(j)} = c_j x_j, which covers both diagonal (phase) gates and X_{+a}-style
    // permutations.  Exact-zero tests keep the specialised result identical to the general
    // formula up to the sign of zero (reading R7).
    bool mono = true;
    int sigma[kMaxDim];
    bool row_used[kMaxDim] = {false};
    for (int j = 0; j < d && mono; ++j) {
        int nz = -1;
        for (int r = 0; r < d; ++r) {
            const double2 u = g.U[r * d + j];
            if (u.x != 0.0 || u.y != 0.0) {
                if (nz >= 0) { mono = false; break; }
                nz = r;
            }
        }
        if (nz < 0 || (mono && row_used[nz])) mono = false;
        if (mono) { sigma[j] = nz; row_used[nz] = true; }
    }
    if (mono) {
        p.kind = kMonomial;
        uint32_t act = 0;
        for (int j = 0; j < d; ++j) {
            const double2 c = g.U[sigma[j] * d + j];
            p.sigma[j] = sigma[j];
            p.U[j] = c;
            if (sigma[j] != j || c.x != 1.0 || c.y != 0.0) act |= 1u << j;
        }
        p.active = act;
    } else {
        p.kind = kGeneral;
        p.active = (d == 32) ? 0xffffffffu : ((1u << d) - 1u);
        for (int j = 0; j < d; ++j) p.sigma[j] = j;
    }

    // ---- fibre decomposer: removed positions (target span pinned to 0, controls pinned
    // to their values), ascending by position = ascending stride; merge adjacent positions.
    struct Pos { int q; int v; };
    std::vector<Pos> pos;
    for (int s = 0; s < g.span; ++s) pos.push_back({g.target + s, 0});
    uint64_t ctrl_prod = 1;
    for (const auto &c : g.ctrl) { pos.push_back({c.q, c.v}); ctrl_prod *= (uint64_t)reg.dims[c.q]; }
    std::sort(pos.begin(), pos.end(), [](const Pos &a, const Pos &b) { return a.q < b.q; });
    int nrem = 0;
    for (size_t i = 0; i < pos.size();) {
        size_t j = i;
        uint64_t dim = 1, pin = 0;
        while (j < pos.size() && (j == i || pos[j].q == pos[j - 1].q + 1)) {
            pin += (uint64_t)pos[j].v * dim;
            dim *= (uint64_t)reg.dims[pos[j].q];
            ++j;
        }
        if (nrem >= kMaxRem) { *err = "too many control runs"; return SV_ERR_UNSUPPORTED; }
        RemovedRun &r = p.rem[nrem++];
        r.b = reg.b[pos[i].q];
        r.bd = r.b * dim;
        r.pinb = pin * r.b;
        r.m = make_fastdiv64(r.b).m;
        i = j;
    }
    p.nrem = nrem;
    p.D = reg.D;
    p.nctrl = (int32_t)g.ctrl.size();
    for (size_t i = 0; i < g.ctrl.size(); ++i) {
        p.cb[i] = reg.b[g.ctrl[i].q];
        p.cd[i] = (uint32_t)reg.dims[g.ctrl[i].q];
        p.cv[i] = (uint32_t)g.ctrl[i].v;
    }
    p.F = reg.D / ((uint64_t)d * ctrl_prod);     // classes satisfying every control
    int nact = 0;
    for (int j = 0; j < d; ++j) nact += (p.active >> j) & 1;
    p.touched = p.F * (uint64_t)nact;
    if (p.active == 0) p.F = 0;                  // identity: nothing to do
    return SV_OK;
}

// ------------------------------------------------------------------------------- fusion
static std::vector<double2> matmul(const std::vector<double2> &A, const std::vector<double2> &B,
                                   int d) {
    std::vector<double2> C(d * d);
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            double re = 0.0, im = 0.0;
            for (int k = 0; k < d; ++k) {
                const double2 a = A[i * d + k], b = B[k * d + j];
                re += a.x * b.x - a.y * b.y;
                im += a.x * b.y + a.y * b.x;
            }
            C[i * d + j] = make_double2(re, im);
        }
    return C;
}

// Embed a d_q×d_q matrix acting on qudit lo+which of the pair (lo, lo+1) into the combined
// (d0*d1)-dim digit J = j0 + d0*j1.
static std::vector<double2> embed_pair(const std::vector<double2> &u, int which, int d0, int d1) {
    const int dd = d0 * d1;
    std::vector<double2> E(dd * dd, make_double2(0.0, 0.0));
    for (int J = 0; J < dd; ++J)
        for (int K = 0; K < dd; ++K) {
            const int j0 = J % d0, j1 = J / d0, k0 = K % d0, k1 = K / d0;
            if (which == 0) {
                if (j1 == k1) E[J * dd + K] = u[j0 * d0 + k0];
            } else {
                if (j0 == k0) E[J * dd + K] = u[j1 * d1 + k1];
            }
        }
    return E;
}

static bool same_ctrl(const std::vector<CtrlSpec> &a, const std::vector<CtrlSpec> &b) {
    if (a.size() != b.size()) return false;
    auto key = [](std::vector<CtrlSpec> v) {
        std::sort(v.begin(), v.end(), [](const CtrlSpec &x, const CtrlSpec &y) { return x.q < y.q; });
        return v;
    };
    auto A = key(a), B = key(b);
    for (size_t i = 0; i < A.size(); ++i)
        if (A[i].q != B[i].q || A[i].v != B[i].v) return false;
    return true;
}

bool same_controls(const GateSpec &a, const GateSpec &b) { return same_ctrl(a.ctrl, b.ctrl); }

std::vector<GateSpec> fuse_gates(const Register &reg, const std::vector<GateSpec> &in) {
    std::vector<GateSpec> out;
    bool have = false;
    GateSpec cur;
    for (const GateSpec &g : in) {
        if (have && g.span == 1 && same_ctrl(cur.ctrl, g.ctrl)) {
            if (g.target >= cur.target && g.target < cur.target + cur.span) {
                std::vector<double2> e = (cur.span == 1)
                    ? g.U
                    : embed_pair(g.U, g.target - cur.target, reg.dims[cur.target],
                                 reg.dims[cur.target + 1]);
                cur.U = matmul(e, cur.U, cur.d);       // later gate on the left
                continue;
            }
            if (cur.span == 1 && (g.target == cur.target + 1 || g.target + 1 == cur.target) &&
                cur.d * g.d <= kMaxDim) {
                const int lo = std::min(cur.target, g.target);
                const int d0 = reg.dims[lo], d1 = reg.dims[lo + 1];
                std::vector<double2> ec = embed_pair(cur.U, cur.target - lo, d0, d1);
                std::vector<double2> eg = embed_pair(g.U, g.target - lo, d0, d1);
                cur.target = lo;
                cur.span = 2;
                cur.d = d0 * d1;
                cur.U = matmul(eg, ec, cur.d);
                continue;
            }
        }
        if (have) out.push_back(cur);
        cur = g;
        have = true;
    }
    if (have) out.push_back(cur);
    return out;
}

std::vector<GateSpec> merge_same_qudit(const std::vector<GateSpec> &in) {
    std::vector<GateSpec> out;
    for (const GateSpec &g : in) {
        if (!out.empty() && out.back().span == 1 && g.span == 1 && out.back().target == g.target &&
            same_ctrl(out.back().ctrl, g.ctrl)) {
            out.back().U = matmul(g.U, out.back().U, g.d);
            continue;
        }
        out.push_back(g);
    }
    return out;
}

// ------------------------------------------------------------------- multi-gate passes

// Commutation-aware merging: a gate joins the latest earlier gate with the same target and the
// same controls when every gate in between commutes with it (it can be moved back next to that
// gate, where the two are one matrix product, later gate on the left).  The window bounds the
// backward scan.
std::vector<GateSpec> merge_commuting(const std::vector<GateSpec> &in, int window) {
    std::vector<GateSpec> out;
    out.reserve(in.size());
    for (const GateSpec &g : in) {
        bool merged = false;
        if (g.span == 1) {
            const int lo = (int)out.size() - window < 0 ? 0 : (int)out.size() - window;
            for (int j = (int)out.size() - 1; j >= lo; --j) {
                GateSpec &h = out[j];
                if (h.span == 1 && h.target == g.target && same_ctrl(h.ctrl, g.ctrl)) {
                    h.U = matmul(g.U, h.U, g.d);
                    merged = true;
                    break;
                }
                if (!commute(h, g)) break;
            }
        }
        if (!merged) out.push_back(g);
    }
    return out;
}

// Whether the gate's matrix is diagonal (§2.1 phase gates): every off-diagonal entry exactly 0.
static bool is_diag(const GateSpec &g) {
    for (int i = 0; i < g.d; ++i)
        for (int j = 0; j < g.d; ++j)
            if (i != j && (g.U[i * g.d + j].x != 0.0 || g.U[i * g.d + j].y != 0.0)) return false;
    return true;
}

// Sufficient commutation test for two (controlled) single-qudit gates, as operators on the
// register: gates on different digits commute unless one's target is a control of the other
// and that target gate is not diagonal (a diagonal gate on a digit commutes with everything
// that is block-diagonal in that digit, i.e. with any gate merely controlled on it); two gates
// on the same digit commute when both are diagonal.
bool commute(const GateSpec &a, const GateSpec &b) {
    if (a.span != 1 || b.span != 1) {            // fused spans: plain disjointness of the digits
        auto in = [](int q, const GateSpec &g) { return q >= g.target && q < g.target + g.span; };
        for (int k = 0; k < a.span; ++k)
            if (in(a.target + k, b)) return false;
        for (const auto &c : b.ctrl)
            if (in(c.q, a)) return false;
        for (const auto &c : a.ctrl)
            if (in(c.q, b)) return false;
        return true;
    }
    if (a.target == b.target) return is_diag(a) && is_diag(b);
    for (const auto &c : b.ctrl)
        if (c.q == a.target && !is_diag(a)) return false;
    for (const auto &c : a.ctrl)
        if (c.q == b.target && !is_diag(b)) return false;
    return true;
}

// In-tile set search for one pass: the window's gates W (not yet applied, in order), the
// distinct targets above the low prefix among them, and every subset S of those targets whose
// tile fits (b_{m0} prod_{q in S} d_q <= tile_cap).  Each S is scored by the gates the pass
// would apply with in-tile set S — a gate qualifies when its target is in the low prefix or
// in S and it commutes with every earlier gate of W left behind — and the best S (first found
// on ties) restricts which targets the pass admits.  Pairwise commutation inside W is computed
// once as bitsets, so scoring one S is O(|W|).
// commute() with the diagonal flags precomputed (span-1 gates; others take commute()).
static bool commute_fast(const GateSpec &a, bool da, const GateSpec &b, bool db) {
    if (a.span != 1 || b.span != 1) return commute(a, b);
    if (a.target == b.target) return da && db;
    if (!da)
        for (const auto &c : b.ctrl)
            if (c.q == a.target) return false;
    if (!db)
        for (const auto &c : a.ctrl)
            if (c.q == b.target) return false;
    return true;
}

static std::vector<char> best_in_tile_set(const Register &reg, const std::vector<GateSpec> &g,
                                          const std::vector<char> &diag,
                                          const std::vector<char> &done, size_t first, int m0,
                                          uint64_t base_tile, uint64_t tile_cap, int max_gates, int window) {
    std::vector<size_t> W;
    for (size_t i = first; i < g.size() && (int)W.size() < window && W.size() < 256; ++i)
        if (!done[i]) W.push_back(i);
    const size_t nw = W.size();
    const size_t nwords = (nw + 63) / 64;
    // blocked[b]: bitset of earlier window gates a with !commute(a, b)
    std::vector<uint64_t> blocked(nw * nwords, 0);
    std::vector<char> eligible(nw, 0);
    std::vector<int> cand;
    for (size_t b = 0; b < nw; ++b) {
        const GateSpec &x = g[W[b]];
        eligible[b] = x.span == 1 && x.ctrl.size() <= 4;
        for (size_t a = 0; a < b; ++a)
            if (!commute_fast(g[W[a]], diag[W[a]], x, diag[W[b]])) blocked[b * nwords + a / 64] |= 1ull << (a % 64);
        if (x.target >= m0 && std::find(cand.begin(), cand.end(), x.target) == cand.end()) cand.push_back(x.target);
    }
    if (cand.size() > 12) cand.resize(12);     // bound the enumeration (first-seen targets kept;
                                               // 12 plans c3/c4 as well as 20: 36 / 22 passes)
    const uint64_t lim = tile_cap / base_tile;
    std::vector<char> inS(reg.n, 0), best(reg.n, 0);
    int best_n = -1;
    std::vector<uint64_t> skipped(nwords);
    auto score = [&]() {
        std::fill(skipped.begin(), skipped.end(), 0);
        int cnt = 0;
        for (size_t b = 0; b < nw && cnt < max_gates; ++b) {
            const GateSpec &x = g[W[b]];
            bool ok = eligible[b] && (x.target < m0 || inS[x.target]);
            for (size_t w = 0; ok && w < nwords; ++w)
                if (skipped[w] & blocked[b * nwords + w]) ok = false;
            if (ok) ++cnt;
            else skipped[b / 64] |= 1ull << (b % 64);
        }
        if (cnt > best_n) { best_n = cnt; best = inS; }
    };
    // Depth-first over subsets in candidate order, pruned by the tile capacity.  The score is
    // monotone in S (a gate admitted with S is admitted with any superset: by induction over
    // the window, the superset leaves behind a subset of the gates), so only subsets that no
    // later candidate extends are scored, and the search stops once a pass is full.
    std::function<void(size_t, uint64_t)> rec = [&](size_t start, uint64_t prod) {
        bool extended = false;
        for (size_t k = start; k < cand.size() && best_n < max_gates; ++k) {
            const uint64_t p = prod * (uint64_t)reg.dims[cand[k]];
            if (p > lim) continue;
            extended = true;
            inS[cand[k]] = 1;
            rec(k + 1, p);
            inS[cand[k]] = 0;
        }
        if (!extended && best_n < max_gates) score();
    };
    rec(0, 1);
    return best;
}

std::vector<PassPlan> plan_passes(const Register &reg, const std::vector<GateSpec> &g, uint64_t tile_cap,
                                  int max_gates, int window, bool search, uint64_t low_stride) {
    std::vector<PassPlan> passes;
    std::vector<char> diag(g.size(), 0);
    if (search)
        for (size_t i = 0; i < g.size(); ++i) diag[i] = is_diag(g[i]);
    // forced low prefix: every qudit whose stride is < 32 amplitudes
    int m0 = 0;
    while (m0 < reg.n && reg.b[m0] < low_stride) ++m0;
    const uint64_t base_tile = (m0 < reg.n) ? reg.b[m0] : reg.D;
    std::vector<char> done(g.size(), 0);
    size_t first = 0;
    while (first < g.size()) {
        while (first < g.size() && done[first]) ++first;
        if (first >= g.size()) break;
        PassPlan pp;
        pp.m0 = m0;
        std::vector<char> inq(reg.n, 0);
        uint64_t tile = base_tile;
        std::vector<size_t> skipped;
        int seen = 0;
        std::vector<char> allowed;
        if (search) allowed = best_in_tile_set(reg, g, diag, done, first, m0, base_tile, tile_cap, max_gates, window);
        for (size_t i = first; i < g.size() && seen < window && (int)pp.gates.size() < max_gates; ++i) {
            if (done[i]) continue;
            ++seen;
            const GateSpec &x = g[i];
            bool ok = x.span == 1 && x.ctrl.size() <= 4;
            for (size_t s : skipped)
                if (ok && !commute(g[s], x)) ok = false;
            uint64_t need = tile;
            if (ok && x.target >= m0 && !inq[x.target]) need = tile * (uint64_t)reg.dims[x.target];
            if (ok && x.target >= m0 && !allowed.empty() && !allowed[x.target]) ok = false;
            if (ok && need > tile_cap) ok = false;
            if (!ok) {
                skipped.push_back(i);
                continue;
            }
            if (x.target >= m0 && !inq[x.target]) {
                inq[x.target] = 1;
                tile = need;
            }
            pp.gates.push_back((int)i);
            done[i] = 1;
        }
        if (pp.gates.empty()) {               // first gate not eligible: single-gate pass
            pp.gates.push_back((int)first);
            done[first] = 1;
        }
        for (int q = m0; q < reg.n; ++q)
            if (inq[q]) pp.H.push_back(q);
        pp.tile = tile;
        passes.push_back(pp);
    }
    return passes;
}

// ------------------------------------------------------------------------- sharding
sv_status shard_plan(const Register &reg, int nranks, int rank, int target,
                     const std::vector<CtrlSpec> &ctrl, ShardAction *out, std::string *err) {
    if (nranks < 1 || (nranks & (nranks - 1))) { *err = "nranks must be a power of two"; return SV_ERR_INVALID_ARG; }
    if (rank < 0 || rank >= nranks) { *err = "rank out of range"; return SV_ERR_INVALID_ARG; }
    int s = 0;
    while ((1 << s) < nranks) ++s;
    if (s >= reg.n) { *err = "too many ranks for this register"; return SV_ERR_UNSUPPORTED; }
    for (int k = reg.n - s; k < reg.n; ++k)
        if (reg.dims[k] != 2) { *err = "sharded digits must be qubits (most significant)"; return SV_ERR_UNSUPPORTED; }
    const int first_sh = reg.n - s;
    out->action = 0;
    out->partner = rank;
    out->beta = 0;
    for (const auto &c : ctrl) {
        if (c.q >= first_sh) {
            const int bit = (rank >> (c.q - first_sh)) & 1;   // rank bit j = digit of q_{n-s+j}
            if (bit != c.v) { out->action = 1; return SV_OK; }
        }
    }
    if (target >= first_sh) {
        const int j = target - first_sh;
        out->action = 2;
        out->partner = rank ^ (1 << j);
        out->beta = (rank >> j) & 1;
    }
    return SV_OK;
}

}  // namespace svi
