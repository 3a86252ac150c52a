// mgpass.cu — host side of the multi-gate pass kernel: pass parameters,
// register-stage planning, launch dispatch.  The kernel is in mgpass_impl.cuh; its
// instantiations live in mgpass_k256.cu / mgpass_k384.cu.
#include "mgpass_impl.cuh"

namespace svi {

// explicit instantiations in mgpass_k256.cu / mgpass_k384.cu
extern template cudaError_t launch_pass_t<256, 1>(const PassParams &, cudaStream_t, const LaunchCfg &);
extern template cudaError_t launch_pass_t<256, 2>(const PassParams &, cudaStream_t, const LaunchCfg &);
extern template cudaError_t launch_pass_t<384, 1>(const PassParams &, cudaStream_t, const LaunchCfg &);
extern template cudaError_t launch_pass_t<384, 2>(const PassParams &, cudaStream_t, const LaunchCfg &);

// ------------------------------------------------------------------------------ host
// Build the pass parameters; returns false if the pass does not fit this kernel.
bool build_pass(const Register &reg, const std::vector<GateSpec> &gates, const PassPlan &pp, double2 *psi,
                int TE, PassParams &p, double *touched) {
    std::memset(&p, 0, sizeof(p));
    if ((int)pp.gates.size() > kMaxPassGates || pp.tile > (uint64_t)TE) return false;
    p.psi = psi;
    const int m0 = pp.m0;
    const uint64_t L = (m0 < reg.n) ? reg.b[m0] : reg.D;
    if (L > 32u * (kMaskWords - 4)) return false;          // low-position mask capacity
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
    // Register stages: regroup the pass's gates, only across gates they
    // commute with, into runs whose targets are one or two in-tile qudits ("axes", product of
    // dimensions <= kMaxPair); gates of dimension > 5 get a generic stage of their own.
    auto generic = [](const GateSpec &g) { return g.span != 1 || g.d < 2 || g.d > 5; };
    auto tile_stride = [&](int t) -> uint64_t { return t < m0 ? reg.b[t] : W[t] * LT; };
    for (int i : pp.gates) {
        const int t = gates[i].target;
        if (gates[i].span != 1 || (t >= m0 && std::find(pp.H.begin(), pp.H.end(), t) == pp.H.end())) return false;
    }
    constexpr int kMaxPair = 16;
    std::vector<int> order, rest(pp.gates.begin(), pp.gates.end());
    std::vector<int> axis_a, axis_b;        // per stage: axis digits (b = -1: one axis)
    p.nstages = 0;
    while (!rest.empty()) {
        std::vector<int> take, skip;
        int a = gates[rest[0]].target, b = -1;
        if (generic(gates[rest[0]])) {
            take.push_back(rest[0]);
            skip.assign(rest.begin() + 1, rest.end());
        } else {
            for (int i : rest) {
                const GateSpec &x = gates[i];
                bool ok = !generic(x);
                for (int j : skip)
                    if (ok && !commute(gates[j], x)) ok = false;
                if (ok && b < 0 && x.target != a && reg.dims[a] * reg.dims[x.target] <= kMaxPair) b = x.target;
                (ok && (x.target == a || x.target == b) ? take : skip).push_back(i);
            }
        }
        PassStage &S = p.st[p.nstages++];
        S.g0 = (int32_t)order.size();
        S.g1 = S.g0 + (int32_t)take.size();
        if (generic(gates[take[0]])) {
            S.da = 0;
            S.db = 0;
            axis_a.push_back(-1);
            axis_b.push_back(-1);
        } else {
            if (b >= 0 && reg.dims[b] < reg.dims[a]) std::swap(a, b);      // axis 0 = smaller dimension
            S.da = reg.dims[a];
            S.db = b >= 0 ? reg.dims[b] : 1;
            S.sta = (uint32_t)tile_stride(a);
            S.stb = b >= 0 ? (uint32_t)tile_stride(b) : 0u;
            // class enumeration: insert the axis digits in ascending stride order
            uint32_t s1 = S.sta, d1 = (uint32_t)S.da, s2 = S.stb, d2 = (uint32_t)S.db;
            if (b < 0) { s2 = 1; d2 = 1; }
            else if (s2 < s1) { std::swap(s1, s2); std::swap(d1, d2); }
            S.s1 = s1; S.m1 = make_fastdiv32(s1).m; S.d1 = d1;
            S.s2 = s2; S.m2 = make_fastdiv32(s2).m; S.d2 = d2;
            axis_a.push_back(a);
            axis_b.push_back(b);
        }
        order.insert(order.end(), take.begin(), take.end());
        rest.swap(skip);
    }
    // gates
    int uoff = 0;
    *touched = 0.0;
    p.ngates = (int32_t)order.size();
    int stage_of[kMaxPassGates];
    for (int k = 0; k < p.nstages; ++k)
        for (int gi = p.st[k].g0; gi < p.st[k].g1; ++gi) stage_of[gi] = k;
    for (size_t gi = 0; gi < order.size(); ++gi) {
        const GateSpec &g = gates[order[gi]];
        GatePlan gp;
        std::string err;
        if (plan_gate(reg, g, false, &gp, &err) != SV_OK) return false;
        *touched += (double)gp.touched;
        PassGateP &q = p.g[gi];
        const int sg = stage_of[gi];
        const int ax_a = axis_a[sg], ax_b = axis_b[sg];
        const bool gen = p.st[sg].da == 0;
        const int t = g.target;
        q.d = gp.d;
        q.kind = gp.kind;
        q.active = gp.active;
        for (int j = 0; j < kMaxDim; ++j) q.sigma[j] = (int8_t)(j < gp.d ? gp.sigma[j] : j);
        q.st = (uint32_t)tile_stride(t);
        q.mst = make_fastdiv32(q.st).m;
        q.axis = (!gen && t == ax_b) ? 1 : 0;
        q.axctl = -1;
        // form: a cyclic shift with coefficients (X_{+s}, CINC, diagonal gates) or dense U
        int shift = -1;
        if (gp.kind == kMonomial) {
            shift = (gp.sigma[0]) % gp.d;
            for (int j = 0; j < gp.d; ++j)
                if (gp.sigma[j] != (j + shift) % gp.d) shift = -1;
        }
        int need;
        if (gen) {
            need = gp.kind == kGeneral ? gp.d * gp.d : gp.d;
            if (uoff + need > kPoolC) return false;
            for (int k = 0; k < need; ++k) p.U[uoff + k] = gp.U[k];
        } else if (shift >= 0) {
            q.form = kFormShift;
            q.shift = shift;
            q.pure = 1;
            need = gp.d;
            if (uoff + need > kPoolC) return false;
            for (int j = 0; j < gp.d; ++j) {
                p.U[uoff + j] = gp.U[j];              // coefficient of member j
                if (!(gp.U[j].x == 1.0 && gp.U[j].y == 0.0)) q.pure = 0;
            }
        } else {
            q.form = kFormDense;
            need = gp.d * gp.d;
            if (uoff + need > kPoolC) return false;
            for (int k = 0; k < need; ++k) p.U[uoff + k] = g.U[k];
        }
        q.uoff = uoff;
        uoff += need;
        p.upool = uoff;
        if ((int)g.ctrl.size() > kMaxPassCtrl) return false;
        // a control on the stage's other axis selects lines; static in-tile controls become
        // bit masks; the rest are decided at run time
        uint32_t *mm = p.mask[gi];
        for (uint64_t m = 0; m < M; ++m) mm[m >> 5] |= 1u << (m & 31);
        for (uint64_t l = 0; l < L; ++l) mm[4 + (l >> 5)] |= 1u << (l & 31);
        int nc = 0;
        for (size_t k = 0; k < g.ctrl.size(); ++k) {
            const int c = g.ctrl[k].q;
            const uint32_t v = (uint32_t)g.ctrl[k].v;
            const uint64_t dc = (uint64_t)reg.dims[c];
            if (!gen && (c == ax_a || c == ax_b)) {
                q.axctl = (int32_t)v;
                continue;
            }
            if (std::find(pp.H.begin(), pp.H.end(), c) != pp.H.end()) {         // H digit: member mask
                for (uint64_t m = 0; m < M; ++m)
                    if ((m / W[c]) % dc != v) mm[m >> 5] &= ~(1u << (m & 31));
                q.flags |= kFMemberMask;
                continue;
            }
            if (c < m0) {                      // low-prefix digit: position mask modulo L
                for (uint64_t l = 0; l < L; ++l)
                    if ((l / reg.b[c]) % dc != v) mm[4 + (l >> 5)] &= ~(1u << (l & 31));
                q.flags |= kFLowMask;
                continue;
            }
            PassCtrl &cc = q.c[nc++];
            cc.v = v;
            cc.d = (uint32_t)dc;
            cc.md = make_fastdiv32(cc.d).m;
            if (reg.b[c] < R) {                // run digit above the low prefix: tile's run offset
                cc.cls = 1;
                q.flags |= kFRunCtrl;
                cc.w = (uint32_t)reg.b[c];
                cc.mw = make_fastdiv32(cc.w).m;
                cc.M = cc.w * cc.d;
                cc.mM = make_fastdiv32(cc.M).m;
                cc.mb64 = make_fastdiv64(cc.M).m;
            } else {                           // outside the tile: constant per tile
                cc.cls = 2;
                cc.b64 = reg.b[c];
                cc.mb64 = make_fastdiv64(cc.b64).m;
                cc.md64 = make_fastdiv64(cc.d).m;
            }
        }
        q.nctrl = nc;
    }
    return p.ntiles > 0;
}

cudaError_t launch_pass(const PassParams &p, cudaStream_t st, const LaunchCfg &cfg) {
    const int G = cfg.pass_groups >= 2 && cfg.pass_stages >= 2 ? 2 : 1;   // one stage per group at least
    if (cfg.pass_threads >= 384) return G == 2 ? launch_pass_t<384, 2>(p, st, cfg) : launch_pass_t<384, 1>(p, st, cfg);
    return G == 2 ? launch_pass_t<256, 2>(p, st, cfg) : launch_pass_t<256, 1>(p, st, cfg);
}

cudaError_t run_pass(const Register &reg, const std::vector<GateSpec> &gates, const PassPlan &pp, double2 *psi,
                     cudaStream_t st, const LaunchCfg &cfg, bool *handled, double *touched) {
    static thread_local PassParams p;   // ~23 KB; parameters are copied at launch
    *handled = build_pass(reg, gates, pp, psi, cfg.pass_tile, p, touched);
    if (!*handled) return cudaSuccess;
    return launch_pass(p, st, cfg);
}

}  // namespace svi
