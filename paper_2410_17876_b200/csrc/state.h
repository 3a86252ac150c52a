// state.h — the handle behind sv_handle (shared by sv_api.cpp and shard.cpp).
#pragma once

#include "plan.h"
#include "shard.h"

#include <vector>

using svi::Register;
using svi::LaunchCfg;
using svi::ShardCtx;

struct sv_state_s {
    Register reg;          // global register
    Register local;        // register of the local slice (sharded: top s digits removed)
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    double2 *psi = nullptr;
    bool own_buf = false;
    bool c64 = false;              // SV_C64: the state is float2 (8 B per amplitude)
    size_t elem = 16;              // bytes per amplitude
    double *d_partial = nullptr;   // norm partials + 1 result slot
    uint64_t launches = 0;
    uint64_t exchanges = 0;
    bool broken = false;
    LaunchCfg cfg{};
    ShardCtx *shard = nullptr;     // non-null for sharded handles
    // SV_OPT_PROFILE: events bracketing each gate launch
    bool profile = false;
    enum ProfKind { kProfGate = 0, kProfPass = 1, kProfComm = 2 };
    struct ProfRec {
        cudaEvent_t a, b;
        double bytes, touched, state_bytes;
        int kind;                        // ProfKind: single-gate kernel, multi-gate pass, cross-rank kernel
        double item_touched, flops;      // passes: executed shared-memory round trips, FP64 flops
        double nvl_bytes;                // cross-rank kernels: bytes per direction over NVLink
    };
    std::vector<ProfRec> prof;
    double plan_ms = 0.0;              // host planning time (SV_BLOCK merge + passes), accumulated
    bool plan_cache = true;            // SV_OPT_PLAN_CACHE
    std::vector<cudaEvent_t> ev_pool;
    // SV_GRAPH: the last captured circuit, replayed while the same circuit is submitted again
    std::vector<unsigned char> graph_key;
    cudaGraphExec_t graph_exec = nullptr;
    uint64_t graph_kernels = 0;
    // SV_BLOCK: the last host plan (merged gates + passes), reused while the same gate list and
    // configuration are submitted again (host memoisation only: every pass still launches)
    std::vector<unsigned char> plan_key;
    std::vector<svi::GateSpec> plan_specs;
    std::vector<svi::PassPlan> plan_passes;
    // gate-time errors are reported through the thread-local message in sv_api.cpp
};

namespace svi {
sv_status fail_msg(sv_status s, const std::string &msg);
sv_status cuda_fail_h(sv_handle h, cudaError_t e, const char *where);
std::string *err_slot();
}
