// sv_api.cpp — the C ABI (include/sv.h): handles, validation, planning, launch driver,
// readback.  Every step of the hot path runs in this library's CUDA kernels; there is no
// CPU fallback.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "plan.h"
#include "shard.h"
#include "state.h"

using namespace svi;

namespace {
thread_local std::string g_err;

sv_status fail(sv_status s, const std::string &msg) {
    g_err = msg;
    return s;
}
}  // namespace



namespace {

sv_status cuda_fail(sv_handle h, cudaError_t e, const char *where) {
    if (h) h->broken = true;
    return fail(SV_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

sv_status check_handle(sv_handle h) {
    if (!h) return fail(SV_ERR_INVALID_ARG, "null handle");
    if (h->broken) return fail(SV_ERR_CUDA, "handle is unusable after an earlier CUDA fault");
    return SV_OK;
}

GateSpec make_spec(const Register &reg, int target, const int32_t *ctrl, const int32_t *vals,
                   int nctrl, const double *U) {
    GateSpec g;
    g.target = target;
    g.span = 1;
    g.d = reg.dims[target];
    for (int i = 0; i < nctrl; ++i) g.ctrl.push_back({ctrl[i], vals[i]});
    g.U.resize((size_t)g.d * g.d);
    for (int i = 0; i < g.d * g.d; ++i) g.U[i] = make_double2(U[2 * i], U[2 * i + 1]);
    return g;
}

void default_cfg(LaunchCfg &c, int device) {
    int sms = 148;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) sms = 148;
    c.kernel = 0;
    c.tile_elems = 2048;
    c.tile_stages = 3;
    c.ctas_per_sm = 2;
    c.num_sms = sms;
    c.pass_tile = 3200;        // planner tile cap; the ring capacity (4 x 3200 amplitudes) is re-cut per pass
    c.pass_stages = 4;         //   into as many stages of the pass's actual tile as fit (mgpass.cu pass_ring):
                               //   c4 1305 -> 1257 ms, c3 369 -> 339 ms against 2560 x 5 (profiles/r02/ab/r02ad)
    c.pass_threads = 512;
    c.pass_gates = 32;         // with the in-tile set search: c3 -1.4%, c4 unchanged (ab/gates_window_*)
    c.pass_window = 256;       // gates scanned ahead when filling a pass (profiles/r01/ab/window_*, ab/gates_window_*)
    c.pass_merge = 1;          // commutation-aware merging before pass planning
    c.pass_groups = 4;         // four consumer groups rotate over the CTA's tiles (one stage in flight)
    c.shard_swap = 1;          // qubit remapping for gates on sharded qubits
    c.pass_search = 1;         // in-tile set chosen by subset search (c4 29 -> 22 passes)
    c.pass_low = 32;           // tile runs of >= 32 amplitudes (512 B bulk copies)
    c.shard_overlap = 16;      // remap overlapped with the pending local run on 132 + 16 SMs
    c.pass_kernel = 0;         // per-gate pass kernel (stages measured slower on c3/c4: profiles/r02)
    c.pass_absorb = 1;         // permutations on member digits relabel the tile's loads / stores
}

}  // namespace

// --------------------------------------------------------------------- shared internals
namespace svi {

sv_status fail_msg(sv_status s, const std::string &msg) { return fail(s, msg); }
sv_status cuda_fail_h(sv_handle h, cudaError_t e, const char *where) { return cuda_fail(h, e, where); }
std::string *err_slot() { return &g_err; }

sv_status state_init_device(sv_handle h, int device, void *cuda_stream, void *ext, size_t ext_bytes) {
    h->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaSetDevice");
    default_cfg(h->cfg, device);
    if (cuda_stream) {
        h->stream = (cudaStream_t)cuda_stream;
    } else {
        e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaStreamCreate");
        h->own_stream = true;
    }
    h->cfg.c64 = h->c64 ? 1 : 0;
    if (h->c64) {                          // 8-byte elements: twice the amplitudes per stage (c4: 1.78 -> 1.25 s);
        h->cfg.pass_tile = 8192;           // ring of 3 x 8192, re-cut per pass; 4 groups where it yields
        h->cfg.pass_stages = 3;            //   4+ stages (c4 765 -> 745 ms against 2 groups, r02/ab/r02ad)
        h->cfg.pass_groups = 4;
    }
    const uint64_t bytes = h->local.D * h->elem;
    if (ext) {
        if (ext_bytes < bytes || ((uintptr_t)ext & 15))
            return fail(SV_ERR_INVALID_ARG, "external buffer too small or misaligned");
        h->psi = (double2 *)ext;
    } else {
        e = cudaMalloc(&h->psi, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(SV_ERR_NOMEM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
        }
        h->own_buf = true;
    }
    e = cudaMalloc(&h->d_partial, (norm_parts() + 1) * sizeof(double));
    if (e != cudaSuccess) { cudaGetLastError(); return fail(SV_ERR_NOMEM, "cudaMalloc (norm scratch)"); }
    return SV_OK;
}

void state_free(sv_handle h) {
    if (!h) return;
    for (auto &r : h->prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
    if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
    if (h->shard) shard_destroy(h->shard);
    if (h->own_buf && h->psi) cudaFree(h->psi);
    if (h->d_partial) cudaFree(h->d_partial);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

// local sum of squares (device -> host), synchronising
sv_status local_norm2(sv_handle h, double *out) {
    cudaError_t e = launch_norm2(h->psi, h->local.D, h->d_partial, norm_parts(),
                                 h->d_partial + norm_parts(), h->stream, &h->launches, h->c64);
    if (e != cudaSuccess) return cuda_fail(h, e, "norm kernel");
    e = cudaMemcpyAsync(out, h->d_partial + norm_parts(), sizeof(double), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "norm readback");
    return SV_OK;
}

static cudaEvent_t pool_event(sv_handle h) {
    if (!h->ev_pool.empty()) {
        cudaEvent_t e = h->ev_pool.back();
        h->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

sv_status launch_on(sv_handle h, const GatePlan &p, double2 *buf) {
    if (p.F == 0) return SV_OK;
    cudaEvent_t a = nullptr, b = nullptr;
    if (h->profile) {
        a = pool_event(h);
        b = pool_event(h);
        cudaEventRecord(a, h->stream);
    }
    cudaError_t e = launch_gate(p, buf, h->stream, h->cfg, &h->launches);
    if (e != cudaSuccess) return cuda_fail(h, e, "gate kernel launch");
    if (h->profile) {
        cudaEventRecord(b, h->stream);
        const double bpu = 2.0 * (double)h->elem;     // one read + one write per touched amplitude
        h->prof.push_back({a, b, bpu * (double)p.touched, (double)p.touched, bpu * (double)p.touched,
                           sv_state_s::kProfGate, (double)p.touched, 0.0, 0.0});
    }
    return SV_OK;
}

sv_status local_apply(sv_handle h, const GatePlan &p) { return launch_on(h, p, h->psi); }

// SV_OPT_PROFILE brackets for the cross-rank kernels (shard.cpp): hbm = bytes this rank's HBM
// moves, nvl = bytes per direction over this rank's NVLink ports.
void prof_begin(sv_handle h, void **tok, cudaStream_t st) {
    *tok = nullptr;
    if (!h->profile) return;
    cudaEvent_t a = pool_event(h);
    cudaEventRecord(a, st ? st : h->stream);
    *tok = a;
}
void prof_end(sv_handle h, void *tok, double hbm, double nvl, double touched, cudaStream_t st) {
    if (!h->profile || !tok) return;
    cudaEvent_t b = pool_event(h);
    cudaEventRecord(b, st ? st : h->stream);
    h->prof.push_back({(cudaEvent_t)tok, b, hbm, touched, hbm, sv_state_s::kProfComm, 0.0, 0.0, nvl});
}

// One multi-gate pass (mgpass.cu); falls back to its gates one by one if the pass kernel
// cannot take it.
static sv_status launch_pass_on(sv_handle h, const std::vector<GateSpec> &specs, const PassPlan &pp,
                                double2 *buf) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (h->profile) {
        a = pool_event(h);
        b = pool_event(h);
        cudaEventRecord(a, h->stream);
    }
    bool handled = false;
    PassWork w;
    cudaError_t e = run_pass(h->local, specs, pp, buf, h->stream, h->cfg, &handled, &w);
    if (e != cudaSuccess) return cuda_fail(h, e, "pass kernel launch");
    if (handled) {
        ++h->launches;
        if (h->profile) {
            cudaEventRecord(b, h->stream);
            // algorithmic bytes per SURVEY.md §8(d): 32 B per touched amplitude of every gate the
            // pass applies; the pass itself moves the local state once (16 B read + 16 B write)
            const double bpu = 2.0 * (double)h->elem;     // one read + one write per amplitude
            h->prof.push_back({a, b, bpu * w.touched, w.touched, bpu * (double)h->local.D, sv_state_s::kProfPass,
                               w.item_touched, w.flops, 0.0});
        }
        return SV_OK;
    }
    if (h->profile) { h->ev_pool.push_back(a); h->ev_pool.push_back(b); }
    for (int gi : pp.gates) {
        GatePlan p;
        sv_status s = plan_gate(h->local, specs[gi], false, &p, &g_err);
        if (s != SV_OK) return s;
        s = launch_on(h, p, buf);
        if (s != SV_OK) return s;
    }
    return SV_OK;
}

// The local circuit driver: plain (gate by gate), SV_FUSE (same-qudit runs + adjacent pairs),
// SV_BLOCK (multi-gate cache-blocked passes), optionally captured into a CUDA graph.
static void append_bytes(std::vector<unsigned char> &k, const void *p, size_t n) {
    const unsigned char *c = static_cast<const unsigned char *>(p);
    k.insert(k.end(), c, c + n);
}

// Everything a captured graph depends on: the gates (targets, controls, matrices), the flags,
// the state buffer and the launch configuration.
static std::vector<unsigned char> graph_key(const sv_handle h, const std::vector<GateSpec> &specs, uint32_t flags,
                                            const double2 *buf) {
    std::vector<unsigned char> k;
    append_bytes(k, &flags, sizeof(flags));
    append_bytes(k, &buf, sizeof(buf));
    append_bytes(k, &h->cfg, sizeof(h->cfg));
    for (const GateSpec &g : specs) {
        const int32_t hdr[4] = {g.target, g.span, g.d, (int32_t)g.ctrl.size()};
        append_bytes(k, hdr, sizeof(hdr));
        for (const auto &c : g.ctrl) append_bytes(k, &c, sizeof(c));
        append_bytes(k, g.U.data(), g.U.size() * sizeof(double2));
    }
    return k;
}

sv_status run_local_circuit(sv_handle h, std::vector<GateSpec> &specs, uint32_t flags, double2 *buf) {
    sv_status s = SV_OK;
    std::vector<unsigned char> key;
    if (flags & SV_GRAPH) {
        key = graph_key(h, specs, flags, buf);
        if (h->graph_exec && key == h->graph_key) {          // same circuit again: replay
            cudaError_t e = cudaGraphLaunch(h->graph_exec, h->stream);
            if (e != cudaSuccess) return cuda_fail(h, e, "graph launch");
            h->launches += h->graph_kernels;
            return SV_OK;
        }
    }
    std::vector<PassPlan> passes;
    if (flags & SV_BLOCK) {
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<unsigned char> pkey;
        if (h->plan_cache) pkey = graph_key(h, specs, flags & (SV_BLOCK | SV_FUSE), nullptr);
        if (h->plan_cache && pkey == h->plan_key) {     // same gates and configuration: same plan
            specs = h->plan_specs;
            passes = h->plan_passes;
        } else {
            if (h->cfg.pass_merge) specs = merge_commuting(specs, 64);
            passes = plan_passes(h->local, specs, (uint64_t)h->cfg.pass_tile, h->cfg.pass_gates,
                                 h->cfg.pass_window, h->cfg.pass_search != 0, (uint64_t)h->cfg.pass_low);
            if (h->plan_cache) {
                h->plan_key.swap(pkey);
                h->plan_specs = specs;
                h->plan_passes = passes;
            }
        }
        h->plan_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    } else {
        if (flags & SV_FUSE) specs = fuse_gates(h->local, specs);
        for (size_t i = 0; i < specs.size(); ++i) {
            PassPlan pp;
            pp.gates.push_back((int)i);
            passes.push_back(pp);
        }
    }
    std::vector<GatePlan> singles(passes.size());
    for (size_t i = 0; i < passes.size(); ++i)
        if (passes[i].gates.size() == 1) {
            s = plan_gate(h->local, specs[passes[i].gates[0]], false, &singles[i], &g_err);
            if (s != SV_OK) return s;
        }
    const bool graph = (flags & SV_GRAPH) != 0;
    const bool keep_profile = h->profile;
    const uint64_t launches0 = h->launches;
    if (graph) {
        h->profile = false;       // events cannot be recorded inside a capture for later reads
        cudaError_t e = cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) { h->profile = keep_profile; return cuda_fail(h, e, "graph capture begin"); }
    }
    for (size_t i = 0; i < passes.size() && s == SV_OK; ++i)
        s = (passes[i].gates.size() == 1) ? launch_on(h, singles[i], buf) : launch_pass_on(h, specs, passes[i], buf);
    if (graph) {
        h->profile = keep_profile;
        cudaGraph_t g;
        cudaError_t e2 = cudaStreamEndCapture(h->stream, &g);
        if (s != SV_OK) return s;
        if (e2 != cudaSuccess) return cuda_fail(h, e2, "graph capture end");
        cudaGraphExec_t exec;
        cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return cuda_fail(h, e, "graph instantiate");
        if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
        h->graph_exec = exec;
        h->graph_key.swap(key);
        h->graph_kernels = h->launches - launches0;
        e = cudaGraphLaunch(exec, h->stream);
        if (e != cudaSuccess) return cuda_fail(h, e, "graph launch");
    }
    return s;
}

}  // namespace svi

// ------------------------------------------------------------------------------ ABI
extern "C" {

const char *sv_last_error(void) { return g_err.c_str(); }

const char *sv_version(void) { return "paper_2410_17876_b200 sv 0.1 (sm_100a)"; }

sv_status sv_create_ex(const int32_t *dims, int32_t n, sv_dtype dt, int device, void *cuda_stream,
                       void *ext_device_buf, size_t ext_bytes, sv_handle *out) {
    if (!out) return fail(SV_ERR_INVALID_ARG, "null out");
    *out = nullptr;
    if (dt != SV_C128 && dt != SV_C64) return fail(SV_ERR_INVALID_ARG, "unknown dtype");
    sv_handle h = new (std::nothrow) sv_state_s();
    if (!h) return fail(SV_ERR_NOMEM, "host allocation");
    sv_status s = make_register(dims, n, &h->reg, &g_err);
    if (s != SV_OK) { delete h; return s; }
    h->local = h->reg;
    h->c64 = dt == SV_C64;
    h->elem = h->c64 ? sizeof(float2) : sizeof(double2);
    if (h->reg.D > (UINT64_MAX >> 5)) { delete h; return fail(SV_ERR_NOMEM, "state too large"); }
    s = state_init_device(h, device, cuda_stream, ext_device_buf, ext_bytes);
    if (s != SV_OK) { state_free(h); return s; }
    s = sv_reset(h, 0);
    if (s != SV_OK) { state_free(h); return s; }
    *out = h;
    return SV_OK;
}

sv_status sv_create(const int32_t *dims, int32_t n, sv_dtype dt, sv_handle *out) {
    Register probe;                       // validate before touching the device
    sv_status s = make_register(dims, n, &probe, &g_err);
    if (s != SV_OK) return s;
    if (!out) return fail(SV_ERR_INVALID_ARG, "null out");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) { cudaGetLastError(); return fail(SV_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e)); }
    return sv_create_ex(dims, n, dt, dev, nullptr, nullptr, 0, out);
}

sv_status sv_destroy(sv_handle h) {
    if (!h) return fail(SV_ERR_INVALID_ARG, "null handle");
    if (h->stream && !h->broken) cudaStreamSynchronize(h->stream);
    state_free(h);
    return SV_OK;
}

sv_status sv_reset(sv_handle h, uint64_t basis_index) {
    sv_status s = check_handle(h);
    if (s != SV_OK) return s;
    if (basis_index >= h->reg.D) return fail(SV_ERR_INDEX_RANGE, "basis index >= D");
    if (h->shard) return shard_reset(h, basis_index);
    cudaError_t e = launch_set_basis(h->psi, h->local.D, basis_index, h->stream, &h->launches, h->c64);
    if (e != cudaSuccess) return cuda_fail(h, e, "reset");
    return SV_OK;
}

sv_status sv_apply_gate(sv_handle h, int32_t target, const int32_t *ctrl, const int32_t *ctrl_vals,
                        int32_t nctrl, const double *U) {
    sv_status s = check_handle(h);
    if (s != SV_OK) return s;
    s = validate_gate(h->reg, target, ctrl, ctrl_vals, nctrl, U, &g_err);
    if (s != SV_OK) return s;
    GateSpec g = make_spec(h->reg, target, ctrl, ctrl_vals, nctrl, U);
    if (h->shard) return shard_apply(h, g, true);
    GatePlan p;
    s = plan_gate(h->local, g, true, &p, &g_err);
    if (s != SV_OK) return s;
    return local_apply(h, p);
}

sv_status sv_apply_circuit(sv_handle h, const sv_gate *gates, int64_t ngates, uint32_t flags) {
    sv_status s = check_handle(h);
    if (s != SV_OK) return s;
    if (ngates < 0 || (ngates > 0 && !gates)) return fail(SV_ERR_INVALID_ARG, "bad gate list");
    std::vector<GateSpec> specs;
    specs.reserve((size_t)ngates);
    for (int64_t i = 0; i < ngates; ++i) {
        const sv_gate &g = gates[i];
        s = validate_gate(h->reg, g.target, g.ctrl, g.ctrl_vals, g.nctrl, g.U, &g_err);
        if (s != SV_OK) { g_err = "gate " + std::to_string(i) + ": " + g_err; return s; }
        specs.push_back(make_spec(h->reg, g.target, g.ctrl, g.ctrl_vals, g.nctrl, g.U));
        if (!(flags & SV_NO_CHECK)) {
            const double err = unitarity_error(specs.back().U.data(), specs.back().d);
            if (!(err <= 1e-12))
                return fail(SV_ERR_NOT_UNITARY, "gate " + std::to_string(i) + ": U is not unitary");
        }
    }
    if (h->shard) return shard_apply_circuit(h, specs, flags);
    return run_local_circuit(h, specs, flags, h->psi);
}

sv_status sv_amplitudes(sv_handle h, uint64_t first, uint64_t count, double *out) {
    sv_status s = check_handle(h);
    if (s != SV_OK) return s;
    if (count == 0) return SV_OK;
    if (!out) return fail(SV_ERR_INVALID_ARG, "null out");
    if (first >= h->reg.D || count > h->reg.D - first) return fail(SV_ERR_INDEX_RANGE, "range outside [0, D)");
    if (h->shard) return shard_amplitudes(h, first, count, out);
    if (h->c64) {                           // complex64: widen to the ABI's doubles on the host
        const uint64_t chunk = 1ull << 24;
        std::vector<float2> tmp((size_t)(count < chunk ? count : chunk));
        const float2 *src = reinterpret_cast<const float2 *>(h->psi) + first;
        for (uint64_t o = 0; o < count; o += chunk) {
            const uint64_t n = count - o < chunk ? count - o : chunk;
            cudaError_t e = cudaMemcpyAsync(tmp.data(), src + o, n * sizeof(float2), cudaMemcpyDeviceToHost, h->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
            if (e != cudaSuccess) return cuda_fail(h, e, "amplitude readback");
            for (uint64_t i = 0; i < n; ++i) {
                out[2 * (o + i)] = tmp[i].x;
                out[2 * (o + i) + 1] = tmp[i].y;
            }
        }
        return SV_OK;
    }
    cudaError_t e = cudaMemcpyAsync(out, h->psi + first, count * sizeof(double2), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "amplitude readback");
    return SV_OK;
}

sv_status sv_set_amplitudes(sv_handle h, uint64_t first, uint64_t count, const double *in) {
    sv_status s = check_handle(h);
    if (s != SV_OK) return s;
    if (count == 0) return SV_OK;
    if (!in) return fail(SV_ERR_INVALID_ARG, "null in");
    if (first >= h->reg.D || count > h->reg.D - first) return fail(SV_ERR_INDEX_RANGE, "range outside [0, D)");
    if (h->shard) return shard_set_amplitudes(h, first, count, in);
    if (h->c64) {                           // complex64: round the ABI's doubles on the host
        const uint64_t chunk = 1ull << 24;
        std::vector<float2> tmp((size_t)(count < chunk ? count : chunk));
        float2 *dst = reinterpret_cast<float2 *>(h->psi) + first;
        for (uint64_t o = 0; o < count; o += chunk) {
            const uint64_t n = count - o < chunk ? count - o : chunk;
            for (uint64_t i = 0; i < n; ++i)
                tmp[i] = make_float2((float)in[2 * (o + i)], (float)in[2 * (o + i) + 1]);
            cudaError_t e = cudaMemcpyAsync(dst + o, tmp.data(), n * sizeof(float2), cudaMemcpyHostToDevice, h->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
            if (e != cudaSuccess) return cuda_fail(h, e, "amplitude upload");
        }
        return SV_OK;
    }
    cudaError_t e = cudaMemcpyAsync(h->psi + first, in, count * sizeof(double2), cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "amplitude upload");
    return SV_OK;
}

sv_status sv_norm(sv_handle h, double *out) {
    sv_status s = check_handle(h);
    if (s != SV_OK) return s;
    if (!out) return fail(SV_ERR_INVALID_ARG, "null out");
    double s2 = 0.0;
    s = local_norm2(h, &s2);
    if (s != SV_OK) return s;
    if (h->shard) {
        s = shard_allreduce_sum(h, &s2);
        if (s != SV_OK) return s;
    }
    *out = std::sqrt(s2);
    return SV_OK;
}

sv_status sv_sync(sv_handle h) {
    sv_status s = check_handle(h);
    if (s != SV_OK) return s;
    if (h->shard) return shard_sync(h);      // watches NCCL / IPC faults while waiting
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "sync");
    return SV_OK;
}

sv_status sv_get_info(sv_handle h, sv_info *out) {
    if (!h || !out) return fail(SV_ERR_INVALID_ARG, "null handle/out");
    out->D = h->reg.D;
    out->local_D = h->local.D;
    out->n = h->reg.n;
    out->rank = h->shard ? shard_rank(h->shard) : 0;
    out->nranks = h->shard ? shard_nranks(h->shard) : 1;
    out->device_ptr = h->psi;
    out->cuda_stream = h->stream;
    out->kernel_launches = h->launches;
    out->exchanges = h->exchanges;
    out->overlapped = h->shard ? shard_overlapped(h->shard) : 0;
    return SV_OK;
}

sv_status sv_set_option(sv_handle h, int32_t option, int64_t value) {
    if (!h) return fail(SV_ERR_INVALID_ARG, "null handle");
    switch (option) {
        case SV_OPT_KERNEL:
            if (value < 0 || value > 2) return fail(SV_ERR_INVALID_ARG, "kernel must be 0..2");
            h->cfg.kernel = (int)value;
            return SV_OK;
        case SV_OPT_TILE_ELEMS:
            if (value < 256 || value > 8192 || (value & 63)) return fail(SV_ERR_INVALID_ARG, "tile elems 256..8192, multiple of 64");
            h->cfg.tile_elems = (int)value;
            return SV_OK;
        case SV_OPT_TILE_STAGES:
            if (value < 2 || value > 8) return fail(SV_ERR_INVALID_ARG, "stages 2..8");
            h->cfg.tile_stages = (int)value;
            return SV_OK;
        case SV_OPT_PROFILE:
            h->profile = value != 0;
            return SV_OK;
        case SV_OPT_PASS_TILE:
            if (value < 256 || value > 8192) return fail(SV_ERR_INVALID_ARG, "pass tile 256..8192");
            h->cfg.pass_tile = (int)value;
            return SV_OK;
        case SV_OPT_PASS_STAGES:
            if (value < 2 || value > 12) return fail(SV_ERR_INVALID_ARG, "pass stages 2..12");
            h->cfg.pass_stages = (int)value;
            return SV_OK;
        case SV_OPT_PASS_THREADS:
            if (value != 256 && value != 384 && value != 512 && value != 576 && value != 768 && value != 960)
                return fail(SV_ERR_INVALID_ARG, "pass threads 256, 384, 512, 576, 768 or 960");
            h->cfg.pass_threads = (int)value;
            return SV_OK;
        case SV_OPT_PASS_GROUPS:
            if (value != 1 && value != 2 && value != 3 && value != 4 && value != 8)
                return fail(SV_ERR_INVALID_ARG, "pass groups 1, 2, 3 (384 or 576 threads), 4 or 8");
            h->cfg.pass_groups = (int)value;
            return SV_OK;
        case SV_OPT_PASS_MERGE:
            h->cfg.pass_merge = value != 0;
            return SV_OK;
        case SV_OPT_SHARD_SWAP:
            h->cfg.shard_swap = value != 0;
            return SV_OK;
        case SV_OPT_PASS_SEARCH:
            h->cfg.pass_search = value != 0;
            return SV_OK;
        case SV_OPT_PASS_LOW:
            if (value < 1 || value > 4096) return fail(SV_ERR_INVALID_ARG, "pass low-prefix stride 1..4096");
            h->cfg.pass_low = (int)value;
            return SV_OK;
        case SV_OPT_SHARD_OVERLAP:
            if (value < 0 || value > 64) return fail(SV_ERR_INVALID_ARG, "shard overlap SMs 0..64");
            h->cfg.shard_overlap = (int)value;
            return SV_OK;
        case SV_OPT_PASS_ABSORB:
            h->cfg.pass_absorb = value != 0;
            return SV_OK;
        case SV_OPT_PASS_KERNEL:
            if (value < 0 || value > 1) return fail(SV_ERR_INVALID_ARG, "pass kernel 0 or 1");
            h->cfg.pass_kernel = (int)value;
            return SV_OK;
        case SV_OPT_PLAN_CACHE:
            h->plan_cache = value != 0;
            if (!h->plan_cache) { h->plan_key.clear(); h->plan_specs.clear(); h->plan_passes.clear(); }
            return SV_OK;
        case SV_OPT_PASS_WINDOW:
            if (value < 1 || value > 4096) return fail(SV_ERR_INVALID_ARG, "pass window 1..4096");
            h->cfg.pass_window = (int)value;
            return SV_OK;
        case SV_OPT_PASS_GATES:
            if (value < 1 || value > 32) return fail(SV_ERR_INVALID_ARG, "pass gates 1..32");
            h->cfg.pass_gates = (int)value;
            return SV_OK;
        case SV_OPT_CTAS_PER_SM:
            if (value < 1 || value > 8) return fail(SV_ERR_INVALID_ARG, "ctas per SM 1..8");
            h->cfg.ctas_per_sm = (int)value;
            return SV_OK;
        default:
            return fail(SV_ERR_INVALID_ARG, "unknown option");
    }
}

sv_status sv_profile_read(sv_handle h, int32_t reset, sv_profile *out) {
    sv_status s = check_handle(h);
    if (s != SV_OK) return s;
    if (!out) return fail(SV_ERR_INVALID_ARG, "null out");
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "profile sync");
    std::memset(out, 0, sizeof(*out));
    out->launches = h->prof.size();
    for (auto &r : h->prof) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) out->kernel_ms += ms;
        out->algorithmic_bytes += r.bytes;
        out->touched += r.touched;
        out->state_bytes += r.state_bytes;
        if (r.kind == sv_state_s::kProfComm) {
            ++out->comm_launches;
            out->comm_ms += ms;
            out->comm_hbm_bytes += r.bytes;
            out->comm_nvlink_bytes += r.nvl_bytes;
        }
        if (r.kind == sv_state_s::kProfPass) {
            ++out->pass_launches;
            out->pass_ms += ms;
            out->pass_touched += r.touched;
            out->pass_item_touched += r.item_touched;
            out->pass_flops += r.flops;
            out->pass_state_bytes += r.state_bytes;
        }
    }
    out->plan_ms = h->plan_ms;
    if (reset) {
        for (auto &r : h->prof) { h->ev_pool.push_back(r.a); h->ev_pool.push_back(r.b); }
        h->prof.clear();
        h->plan_ms = 0.0;
    }
    return SV_OK;
}

// ------------------------------------------------------------------ host-only planning
sv_status sv_plan_gate(const int32_t *dims, int32_t n, int32_t target, const int32_t *ctrl,
                       const int32_t *ctrl_vals, int32_t nctrl, const double *U, sv_gate_plan *out) {
    if (!out) return fail(SV_ERR_INVALID_ARG, "null out");
    Register reg;
    sv_status s = make_register(dims, n, &reg, &g_err);
    if (s != SV_OK) return s;
    s = validate_gate(reg, target, ctrl, ctrl_vals, nctrl, U, &g_err);
    if (s != SV_OK) return s;
    GateSpec g = make_spec(reg, target, ctrl, ctrl_vals, nctrl, U);
    GatePlan p;
    s = plan_gate(reg, g, false, &p, &g_err);
    if (s != SV_OK) return s;
    out->kind = p.kind;
    out->d = p.d;
    out->b = p.bk;
    out->fibres = p.F;
    out->touched = p.touched;
    out->active_mask = p.active;
    for (int j = 0; j < 16; ++j) out->sigma[j] = j < p.d ? p.sigma[j] : j;
    out->unitarity_err = p.uerr;
    return SV_OK;
}

sv_status sv_enumerate_fibres(const int32_t *dims, int32_t n, int32_t target, const int32_t *ctrl,
                              const int32_t *ctrl_vals, int32_t nctrl, uint64_t first,
                              uint64_t count, uint64_t *out) {
    Register reg;
    sv_status s = make_register(dims, n, &reg, &g_err);
    if (s != SV_OK) return s;
    if (reg.D >= (1ull << 62)) return fail(SV_ERR_UNSUPPORTED, "enumeration needs D < 2^62");
    std::vector<double> I(2 * 16 * 16, 0.0);
    for (int j = 0; j < reg.dims[target < 0 || target >= n ? 0 : target]; ++j) I[2 * (j * reg.dims[target] + j)] = 1.0;
    s = validate_gate(reg, target, ctrl, ctrl_vals, nctrl, I.data(), &g_err);
    if (s != SV_OK) return s;
    GateSpec g = make_spec(reg, target, ctrl, ctrl_vals, nctrl, I.data());
    g.U[0] = make_double2(0.0, 0.0);    // make it "general" so F counts all classes
    g.U[1] = make_double2(1.0, 0.0);
    GatePlan p;
    s = plan_gate(reg, g, false, &p, &g_err);
    if (s != SV_OK) return s;
    if (first > p.F || count > p.F - first) return fail(SV_ERR_INDEX_RANGE, "class ids outside [0, F)");
    if (count && !out) return fail(SV_ERR_INVALID_ARG, "null out");
    for (uint64_t i = 0; i < count; ++i) out[i] = insert_digits(first + i, p.nrem, p.rem);
    return SV_OK;
}

}  // extern "C"

template <class Planner>
static sv_status host_gate_plan(const int32_t *dims, int32_t n, const sv_gate *gates, int64_t ngates,
                                int32_t *out_target, int32_t *out_span, int32_t *out_dim, int32_t *out_nctrl,
                                int32_t *out_ctrl, int32_t *out_vals, double *out_U, int64_t *out_n,
                                Planner plan) {
    Register reg;
    sv_status s = make_register(dims, n, &reg, &g_err);
    if (s != SV_OK) return s;
    if (ngates < 0 || (ngates && !gates) || !out_n) return fail(SV_ERR_INVALID_ARG, "bad arguments");
    std::vector<GateSpec> specs;
    for (int64_t i = 0; i < ngates; ++i) {
        const sv_gate &g = gates[i];
        s = validate_gate(reg, g.target, g.ctrl, g.ctrl_vals, g.nctrl, g.U, &g_err);
        if (s != SV_OK) return s;
        specs.push_back(make_spec(reg, g.target, g.ctrl, g.ctrl_vals, g.nctrl, g.U));
    }
    std::vector<GateSpec> f = plan(reg, specs);
    int64_t co = 0;
    for (size_t i = 0; i < f.size(); ++i) {
        out_target[i] = f[i].target;
        out_span[i] = f[i].span;
        out_dim[i] = f[i].d;
        out_nctrl[i] = (int32_t)f[i].ctrl.size();
        for (const auto &c : f[i].ctrl) { out_ctrl[co] = c.q; out_vals[co] = c.v; ++co; }
        for (int k = 0; k < f[i].d * f[i].d; ++k) {
            out_U[i * 512 + 2 * k] = f[i].U[k].x;
            out_U[i * 512 + 2 * k + 1] = f[i].U[k].y;
        }
    }
    *out_n = (int64_t)f.size();
    return SV_OK;
}

extern "C" {

sv_status sv_fuse_plan(const int32_t *dims, int32_t n, const sv_gate *gates, int64_t ngates,
                       int32_t *out_target, int32_t *out_span, int32_t *out_dim, int32_t *out_nctrl,
                       int32_t *out_ctrl, int32_t *out_vals, double *out_U, int64_t *out_n) {
    return host_gate_plan(dims, n, gates, ngates, out_target, out_span, out_dim, out_nctrl, out_ctrl, out_vals,
                          out_U, out_n, [](const Register &r, const std::vector<GateSpec> &g) { return fuse_gates(r, g); });
}

sv_status sv_merge_plan(const int32_t *dims, int32_t n, const sv_gate *gates, int64_t ngates, int32_t window,
                        int32_t *out_target, int32_t *out_span, int32_t *out_dim, int32_t *out_nctrl,
                        int32_t *out_ctrl, int32_t *out_vals, double *out_U, int64_t *out_n) {
    if (window < 1) return fail(SV_ERR_INVALID_ARG, "window >= 1");
    return host_gate_plan(dims, n, gates, ngates, out_target, out_span, out_dim, out_nctrl, out_ctrl, out_vals,
                          out_U, out_n,
                          [window](const Register &, const std::vector<GateSpec> &g) { return merge_commuting(g, window); });
}

sv_status sv_block_plan(const int32_t *dims, int32_t n, const sv_gate *gates, int64_t ngates,
                        int64_t tile_cap, int64_t *out_order, int64_t *out_pass, int64_t *out_tile,
                        int64_t *out_npasses) {
    return sv_block_plan_ex(dims, n, gates, ngates, tile_cap, 24, 64, 1, out_order, out_pass, out_tile,
                            out_npasses);
}

sv_status sv_block_plan_ex(const int32_t *dims, int32_t n, const sv_gate *gates, int64_t ngates,
                           int64_t tile_cap, int32_t max_gates, int32_t window, int32_t search,
                           int64_t *out_order, int64_t *out_pass, int64_t *out_tile, int64_t *out_npasses) {
    if (max_gates < 1 || max_gates > 32 || window < 1) return fail(SV_ERR_INVALID_ARG, "max_gates 1..32, window >= 1");
    Register reg;
    sv_status s = make_register(dims, n, &reg, &g_err);
    if (s != SV_OK) return s;
    if (ngates < 0 || (ngates && (!gates || !out_order || !out_pass || !out_tile)) || !out_npasses)
        return fail(SV_ERR_INVALID_ARG, "bad arguments");
    std::vector<GateSpec> specs;
    for (int64_t i = 0; i < ngates; ++i) {
        const sv_gate &g = gates[i];
        s = validate_gate(reg, g.target, g.ctrl, g.ctrl_vals, g.nctrl, g.U, &g_err);
        if (s != SV_OK) return s;
        specs.push_back(make_spec(reg, g.target, g.ctrl, g.ctrl_vals, g.nctrl, g.U));
    }
    std::vector<PassPlan> passes = plan_passes(reg, specs, (uint64_t)tile_cap, max_gates, window, search != 0);
    int64_t k = 0;
    for (size_t p = 0; p < passes.size(); ++p) {
        out_tile[p] = (int64_t)passes[p].tile;
        for (int gi : passes[p].gates) {
            out_order[k] = gi;
            out_pass[k] = (int64_t)p;
            ++k;
        }
    }
    *out_npasses = (int64_t)passes.size();
    return SV_OK;
}

sv_status sv_shard_plan(const int32_t *dims, int32_t n, int32_t nranks, int32_t rank, int32_t target,
                        const int32_t *ctrl, const int32_t *ctrl_vals, int32_t nctrl,
                        int32_t *action, int32_t *partner, int32_t *beta) {
    Register reg;
    sv_status s = make_register(dims, n, &reg, &g_err);
    if (s != SV_OK) return s;
    std::vector<double> I(2 * 256, 0.0);
    s = validate_gate(reg, target, ctrl, ctrl_vals, nctrl, I.data(), &g_err);
    if (s != SV_OK) return s;
    std::vector<CtrlSpec> cs;
    for (int i = 0; i < nctrl; ++i) cs.push_back({ctrl[i], ctrl_vals[i]});
    ShardAction a;
    s = shard_plan(reg, nranks, rank, target, cs, &a, &g_err);
    if (s != SV_OK) return s;
    *action = a.action;
    *partner = a.partner;
    *beta = a.beta;
    return SV_OK;
}

}  // extern "C"
