// shard.cpp — sharded mode over P = 2^s GPUs.
//
// The state is split on its s most-significant digits, which must be qubits: rank r owns
// the contiguous slice [r L, (r+1) L), L = D/P, and bit j of r is the digit of q_{n-s+j}.
// Local strides are unchanged because the sharded digits sit above every local one.
//   (i)   target and controls local        -> the ordinary local kernel on the slice;
//   (ii)  a control on a sharded digit     -> rank predicate (skip when unmet);
//   (iii) target on sharded qubit j        -> pairwise exchange with r ^ 2^j and the combine
//         psi_loc <- U[beta][beta] psi_loc + U[beta][1-beta] psi_partner on the local indices
//         whose local control digits match (beta = this rank's digit of q_target): the class
//         of PAPER.md:198-222 now spans two ranks and the partner holds the other member.
//   (iv)  diagonal gate on sharded qubit j -> no exchange: each rank applies the phase
//         U[beta][beta] to its local amplitudes whose local controls match (a local gate);
//   (v)   anti-diagonal (X-like) gate on sharded qubit j with no local controls -> no data
//         moves: the slices swap their logical labels (rank relabelling) and a
//         slice is scaled when its entry of U is not exactly 1.
//   (vi)  any other gate on sharded qubit j (default, SV_OPT_SHARD_SWAP) -> qubit remapping:
//         the qubit at sharded position j swaps places with a local qubit k whose digit
//         runs are long (b_k >= L/16; chosen by furthest next use, see pick_local).  Each rank
//         sends the half of its slice whose digit k differs from its own digit j and
//         receives the partner's matching half in its place (half the bytes of a pairwise
//         exchange, no combine pass); the gate is then local and joins the multi-gate passes.
// Rank relabelling: physical rank r holds the slice of logical index lrank[r] (bit j of the
// logical index = digit at sharded position n-s+j); every rank keeps the same maps because
// every rank plans the same gate list.  Qubit remapping: logical qudit q sits at digit
// position pos_of[q] (disjoint local <-> sharded qubit pairs); gates are
// translated to positions before planning, and readback / uploads first swap the qubits
// back home.  sv_reset restores both identity maps.
// Transports (one schedule, three ways to move the data):
//   * IPC (sv_create_sharded_ipc): one process per rank on one node (one GPU each, or several
//     ranks on one GPU for testing); every rank maps every other rank's slice through CUDA IPC
//     and the fused peer kernels (peer.cu) read and write the partner's slice in place over
//     NVLink — gate + exchange in one kernel, qubit swaps element by element, no staging.
//     Ranks order their accesses with host barriers in POSIX shared memory (stream
//     synchronise, then barrier, before and after every cross-rank kernel); the kernels never
//     wait on another rank.  Norms reduce through the same shared memory in rank order.
//   * NCCL send/recv over NVLink (one process per GPU; NCCL is dlopen'ed so the core library
//     loads without it), chunked and double-buffered on a comm stream so the transfer of chunk
//     c+1 overlaps the combine of chunk c (the baseline the fused path replaces).
//   * Loopback: all P slices in one process on one device; the fused peer kernels run over
//     the slice pairs (one kernel over both ranks' data), exercising the same planner, maps
//     and rank predicates on a single GPU.
#include <dlfcn.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "nccl.h"
#include "shard.h"
#include "state.h"

namespace svi {

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t);
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t);
    const char *(*GetErrorString)(ncclResult_t);
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;   // optional
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;                           // optional
};

NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void *lib = nullptr;
    const char *env = getenv("SV_NCCL_LIB");
    const char *cands[] = {env, "libnccl.so.2", SV_NCCL_WHEEL_LIB};
    for (const char *c : cands)
        if (c && !lib) lib = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (!lib) { api.why = "libnccl.so.2 not found"; return api; }
#define SV_SYM(f, name)                                              \
    api.f = reinterpret_cast<decltype(api.f)>(dlsym(lib, name));     \
    if (!api.f) { api.why = std::string("missing ") + name; return api; }
    SV_SYM(GetUniqueId, "ncclGetUniqueId");
    SV_SYM(CommInitRank, "ncclCommInitRank");
    SV_SYM(CommDestroy, "ncclCommDestroy");
    SV_SYM(Send, "ncclSend");
    SV_SYM(Recv, "ncclRecv");
    SV_SYM(GroupStart, "ncclGroupStart");
    SV_SYM(GroupEnd, "ncclGroupEnd");
    SV_SYM(AllReduce, "ncclAllReduce");
    SV_SYM(Broadcast, "ncclBroadcast");
    SV_SYM(GetErrorString, "ncclGetErrorString");
#undef SV_SYM
    api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(dlsym(lib, "ncclCommGetAsyncError"));
    api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(dlsym(lib, "ncclCommAbort"));
    api.ok = true;
    return api;
}

sv_status nccl_fail(sv_handle h, ncclResult_t r, const char *where) {
    if (h) h->broken = true;
    return fail_msg(SV_ERR_NCCL, std::string(where) + ": " + nccl().GetErrorString(r));
}

}  // namespace

// The IPC transport's control block, in POSIX shared memory (one per sharded state; all ranks
// of one node map it).  Zero-filled on creation.
constexpr int kMaxIpcRanks = 64;
struct IpcShm {
    std::atomic<uint32_t> arrived;          // barrier: ranks arrived in this generation
    std::atomic<uint32_t> generation;       // barrier: completed barriers
    std::atomic<uint32_t> failed;           // a rank gave up (timeout / fault): everyone stops
    uint32_t pad;
    cudaIpcMemHandle_t mem[kMaxIpcRanks];   // each rank's slice
    int device[kMaxIpcRanks];
    double red[2][kMaxIpcRanks];            // norm partials, double-buffered by parity
};
static_assert(std::atomic<uint32_t>::is_always_lock_free, "process-shared atomics");

enum Transport { kLoopback = 0, kNccl = 1, kIpc = 2, kDryRun = 3 };

// Dry run (sv_shard_schedule, host only): the schedule of one rank recorded instead of executed —
// the local gate lists its slice runs, and the cross-rank steps with their partners — so a CPU
// test can replay it on numpy slices over gloo (tests/test_shard_gloo.py).
struct DryOp {
    int kind;                    // 0 local gates, 1 qubit swap (rule vi), 2 exchange (rule iii)
    int partner, beta, k, j;     // swap: local position k <-> sharded position j; exchange: partner, beta
    std::vector<GateSpec> gates; // local: the gates (local positions); exchange: the gate
};

double comm_timeout_s() {
    const char *e = getenv("SV_COMM_TIMEOUT_S");
    const double t = e ? atof(e) : 600.0;
    return t > 0 ? t : 600.0;
}

struct ShardCtx {
    int P = 1;
    int s = 0;
    int rank = 0;                  // -1: loopback (all ranks in this handle)
    int transport = kLoopback;
    ncclComm_t comm = nullptr;
    // IPC transport: every rank's slice mapped into this process (peer[rank] = own slice)
    std::vector<double2 *> peer;
    IpcShm *shm = nullptr;
    char shm_name[129] = {0};      // unlinked once every rank has attached (or on failure)
    std::vector<DryOp> dry;        // kDryRun: the recorded schedule
    cudaEvent_t ev_join = nullptr; // overlapped remap: the comm stream's swap done
    uint64_t overlapped = 0;       // remaps that overlapped a local run
    int red_parity = 0;
    std::vector<double2 *> slices; // loopback: P slices (slices[0] is h->psi); NCCL: {h->psi}
    double2 *stage[2] = {nullptr, nullptr};
    uint64_t chunk = 0;            // amplitudes per exchange chunk
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_recv[2] = {nullptr, nullptr};
    cudaEvent_t ev_done[2] = {nullptr, nullptr};
    cudaEvent_t ev_start = nullptr;
    double *d_scalar = nullptr;
    std::vector<int> lrank, prank; // physical rank -> logical slice index, and its inverse
    std::vector<int> pos_of, log_at; // logical qudit -> digit position, and its inverse
    bool loopback() const { return rank < 0; }
    bool dryrun() const { return transport == kDryRun; }
    void identity_map(int n) {
        lrank.resize(P);
        prank.resize(P);
        for (int r = 0; r < P; ++r) lrank[r] = prank[r] = r;
        pos_of.resize(n);
        log_at.resize(n);
        for (int q = 0; q < n; ++q) pos_of[q] = log_at[q] = q;
    }
};

sv_status ipc_barrier_raw(ShardCtx *c);

void shard_destroy(ShardCtx *c) {
    if (!c) return;
    if (c->transport == kIpc && c->shm) {
        // peers may still read this slice until every rank has arrived here
        cudaDeviceSynchronize();
        ipc_barrier_raw(c);
        for (int r = 0; r < (int)c->peer.size(); ++r)
            if (r != c->rank && c->peer[r]) cudaIpcCloseMemHandle(c->peer[r]);
        munmap(c->shm, sizeof(IpcShm));
        if (c->shm_name[0]) shm_unlink(c->shm_name);     // no-op once unlinked
    }
    if (c->comm) nccl().CommDestroy(c->comm);
    for (size_t i = 1; i < c->slices.size(); ++i) cudaFree(c->slices[i]);
    for (double2 *p : c->stage) if (p) cudaFree(p);
    for (cudaEvent_t e : c->ev_recv) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_done) if (e) cudaEventDestroy(e);
    if (c->ev_start) cudaEventDestroy(c->ev_start);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->d_scalar) cudaFree(c->d_scalar);
    delete c;
}

// Sense-reversing barrier over the ranks of an IPC state (host side only).  Spins with
// sched_yield, then short sleeps; gives up after SV_COMM_TIMEOUT_S and marks the state failed
// so that the other ranks stop too.
sv_status ipc_barrier_raw(ShardCtx *c) {
    IpcShm *m = c->shm;
    const uint32_t g = m->generation.load(std::memory_order_acquire);
    if (m->arrived.fetch_add(1, std::memory_order_acq_rel) == (uint32_t)c->P - 1) {
        m->arrived.store(0, std::memory_order_relaxed);
        m->generation.store(g + 1, std::memory_order_release);
        return SV_OK;
    }
    const auto t0 = std::chrono::steady_clock::now();
    const double limit = comm_timeout_s();
    for (uint64_t it = 0; m->generation.load(std::memory_order_acquire) == g; ++it) {
        if (m->failed.load(std::memory_order_relaxed))
            return fail_msg(SV_ERR_NCCL, "IPC transport: another rank failed");
        if (it < 2048) {
            sched_yield();
            continue;
        }
        struct timespec ts = {0, 20000};
        nanosleep(&ts, nullptr);
        if ((it & 1023) == 0 &&
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
            m->failed.store(1, std::memory_order_relaxed);
            return fail_msg(SV_ERR_NCCL, "IPC transport: barrier timeout (a peer process is gone or stuck)");
        }
    }
    return SV_OK;
}

int shard_rank(const ShardCtx *c) { return c->rank; }
uint64_t shard_overlapped(const ShardCtx *c) { return c->overlapped; }
int shard_nranks(const ShardCtx *c) { return c->P; }

namespace {

std::vector<int> ranks_of(const ShardCtx *c) {
    std::vector<int> r;
    if (c->loopback())
        for (int i = 0; i < c->P; ++i) r.push_back(i);
    else
        r.push_back(c->rank);
    return r;
}

double2 *slice_of(const ShardCtx *c, int r) { return c->loopback() ? c->slices[r] : c->slices[0]; }

// element `off` of a state buffer whose elements are `elem` bytes (complex128 or complex64)
inline double2 *at(double2 *p, uint64_t off, size_t elem) {
    return reinterpret_cast<double2 *>(reinterpret_cast<char *>(p) + off * elem);
}

CombineCtrl local_ctrl(const Register &local, const std::vector<CtrlSpec> &ctrl) {
    CombineCtrl cc;
    std::memset(&cc, 0, sizeof(cc));
    for (const auto &c : ctrl) {
        if (c.q >= local.n) continue;                 // sharded controls: rank predicate
        const int i = cc.nctrl++;
        cc.b[i] = local.b[c.q];
        cc.mb[i] = make_fastdiv64(cc.b[i]).m;
        cc.d[i] = (uint64_t)local.dims[c.q];
        cc.md[i] = make_fastdiv64(cc.d[i]).m;
        cc.v[i] = (uint64_t)c.v;
    }
    return cc;
}

enum ShardKind { SK_LOCAL, SK_PHASE, SK_RELABEL, SK_EXCHANGE };

inline bool is_zero(double2 z) { return z.x == 0.0 && z.y == 0.0; }
inline bool is_one(double2 z) { return z.x == 1.0 && z.y == 0.0; }

// How a gate is applied under sharding (rules i, iii, iv, v above).
ShardKind classify(const Register &local, const GateSpec &g) {
    if (g.target < local.n) return SK_LOCAL;
    if (is_zero(g.U[1]) && is_zero(g.U[2])) return SK_PHASE;
    bool local_ctrl = false;
    for (const auto &c : g.ctrl) local_ctrl = local_ctrl || c.q < local.n;
    if (is_zero(g.U[0]) && is_zero(g.U[3]) && !local_ctrl) return SK_RELABEL;
    return SK_EXCHANGE;
}

// Rule ii on logical slice index l: do the gate's sharded controls hold there?
bool fires_on(const std::vector<CtrlSpec> &ctrl, int first_sh, int l) {
    for (const auto &c : ctrl)
        if (c.q >= first_sh && ((l >> (c.q - first_sh)) & 1) != c.v) return false;
    return true;
}

// The gate u * I on q_0: a uniform scale of a slice.
GateSpec scale_gate(const Register &local, double2 u) {
    GateSpec s;
    s.target = 0;
    s.d = local.dims[0];
    s.U.assign((size_t)s.d * s.d, make_double2(0.0, 0.0));
    for (int i = 0; i < s.d; ++i) s.U[(size_t)i * s.d + i] = u;
    return s;
}

// Rule iv: the local form, on logical slice l, of a diagonal gate on a sharded qubit.  The
// phase u = U[beta][beta] multiplies the amplitudes whose local control digits match: with
// local controls, a diagonal gate on the first one (entry u at its control value, 1
// elsewhere) controlled on the rest; without, u * I on q_0.  False when u is exactly 1.
bool phase_local(const Register &local, const GateSpec &g, int l, GateSpec *out) {
    const int first_sh = local.n;
    const int beta = (l >> (g.target - first_sh)) & 1;
    const double2 u = g.U[beta * 2 + beta];
    if (is_one(u)) return false;
    std::vector<CtrlSpec> lc;
    for (const auto &c : g.ctrl)
        if (c.q < first_sh) lc.push_back(c);
    if (lc.empty()) { *out = scale_gate(local, u); return true; }
    GateSpec p;
    p.target = lc[0].q;
    p.d = local.dims[p.target];
    p.U.assign((size_t)p.d * p.d, make_double2(0.0, 0.0));
    for (int i = 0; i < p.d; ++i) p.U[(size_t)i * p.d + i] = (i == lc[0].v) ? u : make_double2(1.0, 0.0);
    p.ctrl.assign(lc.begin() + 1, lc.end());
    *out = std::move(p);
    return true;
}

// Rule v: y_{b'} = U[b'][1-b'] x_{1-b'} on sharded qubit j.  On every logical slice l whose
// sharded controls hold, the slice holding x_beta becomes logical l ^ 2^j, scaled by
// U[1-beta][beta].  Updates the map; returns (physical rank, factor) for factors != 1.
std::vector<std::pair<int, double2>> relabel(ShardCtx *c, const GateSpec &g, int first_sh) {
    const int j = g.target - first_sh;
    std::vector<std::pair<int, double2>> scales;
    std::vector<int> nl = c->lrank;
    for (int r = 0; r < c->P; ++r) {
        const int l = c->lrank[r];
        if (!fires_on(g.ctrl, first_sh, l)) continue;
        const int beta = (l >> j) & 1;
        nl[r] = l ^ (1 << j);
        const double2 u = g.U[(1 - beta) * 2 + beta];
        if (!is_one(u)) scales.push_back({r, u});
    }
    c->lrank = nl;
    for (int r = 0; r < c->P; ++r) c->prank[nl[r]] = r;
    return scales;
}

bool owns(const ShardCtx *c, int r) { return c->loopback() || r == c->rank; }

// IPC: this rank's queued work is complete and so is every other rank's (before a kernel
// touches a peer's slice, and after, before anyone touches its own slice again).
sv_status ipc_fence(sv_handle h) {
    if (h->shard->transport != kIpc) return SV_OK;
    sv_status s = shard_sync(h);
    if (s != SV_OK) {
        h->shard->shm->failed.store(1, std::memory_order_relaxed);
        return s;
    }
    s = ipc_barrier_raw(h->shard);
    if (s != SV_OK) h->broken = true;
    return s;
}

// A logical gate at the current digit positions (rule vi).
GateSpec to_phys(const ShardCtx *c, const GateSpec &g) {
    GateSpec p = g;
    p.target = c->pos_of[g.target];
    for (auto &cs : p.ctrl) cs.q = c->pos_of[cs.q];
    return p;
}

// Rule vi candidates: local qubit positions whose digit blocks are at least L/16 amplitudes
// long (a half slice is at most 8 contiguous runs).
bool swappable(sv_handle h, int k) {
    return h->local.dims[k] == 2 && h->local.b[k] * 16 >= h->local.D;
}

bool diag_gate(const GateSpec &g) {
    for (int a = 0; a < g.d; ++a)
        for (int b = 0; b < g.d; ++b)
            if (a != b && !is_zero(g.U[(size_t)a * g.d + b])) return false;
    return true;
}

// Rule vi policy.  Remapped qubits always form disjoint pairs (local position k <-> sharded
// position j), so the layout is a product of disjoint transpositions:
//   * the qudit at sharded position j belongs at local position k (swapped out earlier):
//     swap it home, undoing that pair;
//   * otherwise pair j with a local qubit still at home: the one whose next non-diagonal gate
//     (in specs after index i; none when specs is null) is furthest ahead, top first on ties.
// Returns -1 when no local qubit qualifies (the gate then exchanges).
int pick_local(sv_handle h, int j, const std::vector<GateSpec> *specs, size_t i) {
    ShardCtx *c = h->shard;
    const int q = c->log_at[h->local.n + j];
    if (q < h->local.n) return q;
    int best = -1;
    size_t best_next = 0;
    for (int k = h->local.n - 1; k >= 0; --k) {
        if (!swappable(h, k) || c->log_at[k] != k) continue;
        size_t next = specs ? specs->size() : 0;
        if (specs)
            for (size_t t = i + 1; t < specs->size(); ++t)
                if ((*specs)[t].target == k && !diag_gate((*specs)[t])) { next = t; break; }
        if (best < 0 || next > best_next) { best = k; best_next = next; }
    }
    return best;
}

// Rule vi: swap the qubits at local position k (stride b) and sharded position n-s+j.  A
// rank whose digit j is beta keeps the amplitudes with digit k = beta and trades those with
// digit k = 1-beta (runs of b amplitudes at m 2b + (1-beta) b) for the partner's amplitudes
// with digit k = beta, which land in the same places.
sv_status swap_qubits(sv_handle h, int k, int j) {
    ShardCtx *c = h->shard;
    const uint64_t L = h->local.D, b = h->local.b[k];
    // (run offset, length) pieces of at most one chunk over the runs of digit k = v
    auto pieces = [&](int v) {
        std::vector<std::pair<uint64_t, uint64_t>> out;
        for (uint64_t m = 0; m < L; m += 2 * b)
            for (uint64_t o = 0; o < b; o += c->chunk)
                out.push_back({m + (uint64_t)v * b + o, (b - o < c->chunk) ? b - o : c->chunk});
        return out;
    };
    if (c->dryrun()) {
        const int l = c->lrank[c->rank], beta = (l >> j) & 1;
        c->dry.push_back({1, c->prank[l ^ (1 << j)], beta, k, j, {}});
        ++h->exchanges;
    }
    if (c->transport == kIpc) {                  // fused: half of the pair's swap space per rank
        sv_status s = ipc_fence(h);
        if (s != SV_OK) return s;
        const int r = c->rank, l = c->lrank[r], beta = (l >> j) & 1;
        const int p = c->prank[l ^ (1 << j)];
        const uint64_t half = L / 2, q0 = half / 2;  // swap space [0, L/2): lo rank [0, q0), hi rank the rest
        const uint64_t n = beta ? half - q0 : q0;
        void *tok;
        prof_begin(h, &tok);
        cudaError_t e = launch_pair_swap(at(c->peer[r], (uint64_t)(1 - beta) * b, h->elem),
                                         at(c->peer[p], (uint64_t)beta * b, h->elem), b, beta ? q0 : 0,
                                         n, h->stream, h->cfg.num_sms, &h->launches, h->c64);
        if (e != cudaSuccess) return cuda_fail_h(h, e, "peer qubit swap");
        // this rank's half slice in and out of HBM; n elements cross each way twice (own + partner's)
        prof_end(h, tok, (double)h->elem * (double)L, 2.0 * (double)h->elem * (double)n, 0.0);
        ++h->exchanges;
        s = ipc_fence(h);
        if (s != SV_OK) return s;
    }
    for (int r : (c->transport == kIpc || c->dryrun() ? std::vector<int>{} : ranks_of(c))) {
        const int l = c->lrank[r];
        const int beta = (l >> j) & 1;
        const int p = c->prank[l ^ (1 << j)];
        const auto mine = pieces(1 - beta);          // what this rank gives away
        if (c->loopback()) {
            if (p < r) continue;                      // each pair once: one kernel over both slices
            void *tok;
            prof_begin(h, &tok);
            cudaError_t e = launch_pair_swap(at(c->slices[r], (uint64_t)(1 - beta) * b, h->elem),
                                             at(c->slices[p], (uint64_t)beta * b, h->elem), b, 0, L / 2, h->stream,
                                             h->cfg.num_sms, &h->launches, h->c64);
            if (e != cudaSuccess) return cuda_fail_h(h, e, "loopback qubit swap");
            prof_end(h, tok, 2.0 * (double)h->elem * (double)L, 0.0, 0.0);
            ++h->exchanges;
            continue;
        }
        cudaError_t e = cudaEventRecord(c->ev_start, h->stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(c->comm_stream, c->ev_start, 0);
        if (e != cudaSuccess) return cuda_fail_h(h, e, "qubit swap setup");
        const ncclDataType_t ty = h->c64 ? ncclFloat32 : ncclFloat64;     // 2 reals per amplitude
        for (size_t x = 0; x < mine.size(); ++x) {
            const uint64_t len = mine[x].second;
            const int sb = (int)(x & 1);
            if (x >= 2) {                                                   // stage free again
                e = cudaStreamWaitEvent(c->comm_stream, c->ev_done[sb], 0);
                if (e != cudaSuccess) return cuda_fail_h(h, e, "qubit swap stage wait");
            }
            double2 *a = at(c->slices[0], mine[x].first, h->elem);
            ncclResult_t rr = nccl().GroupStart();
            if (rr == ncclSuccess) rr = nccl().Send(a, 2 * len, ty, p, c->comm, c->comm_stream);
            if (rr == ncclSuccess) rr = nccl().Recv(c->stage[sb], 2 * len, ty, p, c->comm, c->comm_stream);
            ncclResult_t r2 = nccl().GroupEnd();
            if (rr != ncclSuccess) return nccl_fail(h, rr, "ncclSend/Recv");
            if (r2 != ncclSuccess) return nccl_fail(h, r2, "ncclGroupEnd");
            e = cudaEventRecord(c->ev_recv[sb], c->comm_stream);    // piece sent and received
            if (e == cudaSuccess) e = cudaStreamWaitEvent(h->stream, c->ev_recv[sb], 0);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(a, c->stage[sb], len * h->elem, cudaMemcpyDeviceToDevice, h->stream);
            if (e == cudaSuccess) e = cudaEventRecord(c->ev_done[sb], h->stream);
            if (e != cudaSuccess) return cuda_fail_h(h, e, "qubit swap chunk");
        }
        ++h->exchanges;
    }
    const int q = h->local.n + j;
    std::swap(c->log_at[k], c->log_at[q]);
    c->pos_of[c->log_at[k]] = k;
    c->pos_of[c->log_at[q]] = q;
    return SV_OK;
}

// Rule vi for a gate on sharded position j: remap if a local qubit qualifies.
sv_status try_swap(sv_handle h, int j, const std::vector<GateSpec> *specs, size_t i, bool *swapped) {
    *swapped = false;
    if (!h->cfg.shard_swap) return SV_OK;
    const int k = pick_local(h, j, specs, i);
    if (k < 0) return SV_OK;
    *swapped = true;
    return swap_qubits(h, k, j);
}

// Swap every remapped pair back (before readback and uploads).
sv_status restore_layout(sv_handle h) {
    ShardCtx *c = h->shard;
    for (int k = 0; k < h->local.n; ++k)
        if (c->log_at[k] != k) {
            sv_status s = swap_qubits(h, k, c->log_at[k] - h->local.n);
            if (s != SV_OK) return s;
        }
    return SV_OK;
}

sv_status exchange_nccl(sv_handle h, const GateSpec &g, const ShardAction &a) {
    ShardCtx *c = h->shard;
    const double2 A = g.U[a.beta * 2 + a.beta], B = g.U[a.beta * 2 + (1 - a.beta)];
    const CombineCtrl cc = local_ctrl(h->local, g.ctrl);
    const uint64_t L = h->local.D;
    cudaError_t e = cudaEventRecord(c->ev_start, h->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->comm_stream, c->ev_start, 0);
    if (e != cudaSuccess) return cuda_fail_h(h, e, "exchange setup");
    uint64_t k = 0;
    for (uint64_t off = 0; off < L; off += c->chunk, ++k) {
        const uint64_t len = (L - off < c->chunk) ? L - off : c->chunk;
        const int sb = (int)(k & 1);
        if (k >= 2) {                                                       // stage free again
            e = cudaStreamWaitEvent(c->comm_stream, c->ev_done[sb], 0);
            if (e != cudaSuccess) return cuda_fail_h(h, e, "exchange stage wait");
        }
        ncclResult_t r = nccl().GroupStart();
        const ncclDataType_t ty = h->c64 ? ncclFloat32 : ncclFloat64;     // 2 reals per amplitude
        if (r == ncclSuccess) r = nccl().Send(at(c->slices[0], off, h->elem), 2 * len, ty, a.partner, c->comm, c->comm_stream);
        if (r == ncclSuccess) r = nccl().Recv(c->stage[sb], 2 * len, ty, a.partner, c->comm, c->comm_stream);
        ncclResult_t r2 = nccl().GroupEnd();
        if (r != ncclSuccess) return nccl_fail(h, r, "ncclSend/Recv");
        if (r2 != ncclSuccess) return nccl_fail(h, r2, "ncclGroupEnd");
        e = cudaEventRecord(c->ev_recv[sb], c->comm_stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(h->stream, c->ev_recv[sb], 0);
        if (e == cudaSuccess)
            e = launch_combine(at(c->slices[0], off, h->elem), c->stage[sb], len, off, A, B, cc, h->stream,
                               &h->launches, h->c64);
        if (e == cudaSuccess) e = cudaEventRecord(c->ev_done[sb], h->stream);
        if (e != cudaSuccess) return cuda_fail_h(h, e, "exchange chunk");
    }
    ++h->exchanges;
    return SV_OK;
}

// Rule iii through peer memory (loopback: one kernel over both slices; IPC: each rank of the
// pair updates half of the local indices, reading and writing the partner's slice in place).
// lo = the slice whose digit of the target is 0.
sv_status exchange_fused(sv_handle h, const GateSpec &g, double2 *lo, double2 *hi, uint64_t first, uint64_t n) {
    const double2 u[4] = {g.U[0], g.U[1], g.U[2], g.U[3]};
    const CombineCtrl cc = local_ctrl(h->local, g.ctrl);
    void *tok;
    prof_begin(h, &tok);
    cudaError_t e = launch_pair_update(lo, hi, first, n, u, cc, h->stream, h->cfg.num_sms, &h->launches, h->c64);
    if (e != cudaSuccess) return cuda_fail_h(h, e, "fused exchange");
    // IPC: this rank's slice is read and written once (half by each rank of the pair); n index
    // pairs cross NVLink both ways.  Loopback: both slices on this device, nothing crosses.
    const double el = (double)h->elem, L = (double)h->local.D;
    if (h->shard->transport == kIpc) prof_end(h, tok, 2.0 * el * L, 2.0 * el * (double)n, 2.0 * (double)n);
    else prof_end(h, tok, 4.0 * el * (double)n, 0.0, 2.0 * (double)n);
    ++h->exchanges;
    return SV_OK;
}

// One gate at digit positions (already translated), by rules i-v.
sv_status apply_phys(sv_handle h, const GateSpec &g) {
    ShardCtx *c = h->shard;
    std::string *err = err_slot();
    const ShardKind kind = classify(h->local, g);
    if (kind == SK_PHASE) {
        for (int r : ranks_of(c)) {
            GateSpec pl;
            if (!fires_on(g.ctrl, h->local.n, c->lrank[r]) || !phase_local(h->local, g, c->lrank[r], &pl))
                continue;
            if (c->dryrun()) { c->dry.push_back({0, r, 0, 0, 0, {pl}}); continue; }
            GatePlan p;
            sv_status s = plan_gate(h->local, pl, false, &p, err);
            if (s == SV_OK) s = launch_on(h, p, slice_of(c, r));
            if (s != SV_OK) return s;
        }
        return SV_OK;
    }
    if (kind == SK_RELABEL) {
        for (const auto &rs : relabel(c, g, h->local.n)) {
            if (!owns(c, rs.first)) continue;
            if (c->dryrun()) { c->dry.push_back({0, rs.first, 0, 0, 0, {scale_gate(h->local, rs.second)}}); continue; }
            GatePlan p;
            sv_status s = plan_gate(h->local, scale_gate(h->local, rs.second), false, &p, err);
            if (s == SV_OK) s = launch_on(h, p, slice_of(c, rs.first));
            if (s != SV_OK) return s;
        }
        return SV_OK;
    }
    // local view of the gate (sharded controls become the rank predicate)
    GateSpec gl = g;
    gl.ctrl.clear();
    for (const auto &cs : g.ctrl)
        if (cs.q < h->local.n) gl.ctrl.push_back(cs);
    std::vector<int> done(c->P, 0);
    if (c->transport == kIpc) {           // every rank takes part in the fences, firing or not
        sv_status s = ipc_fence(h);
        if (s != SV_OK) return s;
    }
    for (int r : ranks_of(c)) {
        if (done[r]) continue;
        ShardAction a;   // planned on logical slice indices; partner mapped back to a rank
        sv_status s = shard_plan(h->reg, c->P, c->lrank[r], g.target, g.ctrl, &a, err);
        if (s != SV_OK) return s;
        if (a.action == 1) continue;
        if (a.action == 0) {
            if (c->dryrun()) { c->dry.push_back({0, r, 0, 0, 0, {gl}}); continue; }
            GatePlan p;
            s = plan_gate(h->local, gl, false, &p, err);
            if (s != SV_OK) return s;
            s = launch_on(h, p, slice_of(c, r));
            if (s != SV_OK) return s;
            continue;
        }
        const int lpartner = a.partner;
        a.partner = c->prank[lpartner];
        const uint64_t L = h->local.D;
        if (c->dryrun()) {
            c->dry.push_back({2, a.partner, a.beta, 0, 0, {g}});
            ++h->exchanges;
            continue;
        }
        if (c->loopback()) {
            double2 *mine = c->slices[r], *theirs = c->slices[a.partner];
            s = exchange_fused(h, g, a.beta ? theirs : mine, a.beta ? mine : theirs, 0, L);
            done[a.partner] = 1;
        } else if (c->transport == kIpc) {
            double2 *mine = c->peer[r], *theirs = c->peer[a.partner];
            const uint64_t h0 = L / 2;        // lo rank: local indices [0, L/2), hi rank: the rest
            s = exchange_fused(h, g, a.beta ? theirs : mine, a.beta ? mine : theirs, a.beta ? h0 : 0,
                               a.beta ? L - h0 : h0);
        } else {
            s = exchange_nccl(h, g, a);
        }
        if (s != SV_OK) return s;
    }
    if (c->transport == kIpc) return ipc_fence(h);
    return SV_OK;
}

}  // namespace

sv_status shard_apply(sv_handle h, const GateSpec &g_logical, bool check_unitary) {
    ShardCtx *c = h->shard;
    if (check_unitary) {
        const double ue = unitarity_error(g_logical.U.data(), g_logical.d);
        if (!(ue <= 1e-12)) return fail_msg(SV_ERR_NOT_UNITARY, "U is not unitary");
    }
    GateSpec g = to_phys(c, g_logical);
    if (classify(h->local, g) == SK_EXCHANGE) {                     // rule vi
        bool swapped;
        sv_status s = try_swap(h, g.target - h->local.n, nullptr, 0, &swapped);
        if (s != SV_OK) return s;
        if (swapped) g = to_phys(c, g_logical);
    }
    return apply_phys(h, g);
}

namespace {

// Run a local gate list on one half of a slice: the local register without its top digit (whose
// value is fixed over the half), at buf.  The host plan cache is bypassed (keyed by gates, not
// registers); profiling records half-slice state bytes.
sv_status run_on_half(sv_handle h, const Register &sub, std::vector<GateSpec> gates, uint32_t flags, double2 *buf) {
    const Register keep = h->local;
    const bool cache = h->plan_cache;
    h->local = sub;
    h->plan_cache = false;
    sv_status s = run_local_circuit(h, gates, flags, buf);
    h->local = keep;
    h->plan_cache = cache;
    return s;
}

}  // namespace

// Rule vi with overlap (SV_OPT_SHARD_OVERLAP): the remap of sharded position j with the TOP local
// position k moves the half of each slice whose digit k is 1 - beta (a contiguous half: k is the
// top digit) and keeps the other.  When the pending local run R neither targets nor controls k and
// no gate of it depends on digit j (a sharded control on j, a local phase from a gate on j),
// R commutes with the remap, so: the half that moves is swapped on the comm stream by
// k_pair_swap on `lend` SMs while R runs on the staying half on the remaining SMs; after the
// swap, R runs on the half that arrived (the partner's, which its owner did not update — by the
// same rule).  Every amplitude gets R once; the swap kernel and the passes touch disjoint halves.
sv_status overlapped_remap(sv_handle h, int k, int j, std::vector<std::vector<GateSpec>> &runs,
                           const std::vector<int> &ranks, uint32_t flags) {
    ShardCtx *c = h->shard;
    const uint64_t L = h->local.D, half = L / 2;
    Register sub;
    std::string *err = err_slot();
    sv_status s = make_register(h->local.dims, h->local.n - 1, &sub, err);
    if (s != SV_OK) return s;
    const int lend = h->cfg.shard_overlap;
    const uint32_t lf = flags & (SV_FUSE | SV_BLOCK);
    s = ipc_fence(h);                               // both halves final everywhere before the swap
    if (s != SV_OK) return s;
    cudaError_t e = cudaEventRecord(c->ev_join, h->stream);   // loopback: the swap after earlier work
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->comm_stream, c->ev_join, 0);
    if (e != cudaSuccess) return cuda_fail_h(h, e, "overlapped swap setup");
    // (1) the moving halves, on the comm stream, on `lend` SMs
    auto beta_of = [&](int r) { return (c->lrank[r] >> j) & 1; };
    if (c->transport == kIpc) {
        const int r = c->rank, beta = beta_of(r), p = c->prank[c->lrank[r] ^ (1 << j)];
        const uint64_t q0 = half / 2, n = beta ? half - q0 : q0;
        void *tok;
        prof_begin(h, &tok, c->comm_stream);
        e = launch_pair_swap(at(c->peer[r], (uint64_t)(1 - beta) * half, h->elem), at(c->peer[p], (uint64_t)beta * half, h->elem),
                             half, beta ? q0 : 0, n, c->comm_stream, lend, &h->launches, h->c64);
        prof_end(h, tok, (double)h->elem * (double)L, 2.0 * (double)h->elem * (double)n, 0.0, c->comm_stream);
        ++h->exchanges;
    } else {                                        // loopback: one kernel per slice pair
        for (int r : ranks) {
            const int p = c->prank[c->lrank[r] ^ (1 << j)];
            if (p < r || e != cudaSuccess) continue;
            const int beta = beta_of(r);
            void *tok;
            prof_begin(h, &tok, c->comm_stream);
            e = launch_pair_swap(at(c->slices[r], (uint64_t)(1 - beta) * half, h->elem),
                                 at(c->slices[p], (uint64_t)beta * half, h->elem), half, 0, half, c->comm_stream, lend,
                                 &h->launches, h->c64);
            prof_end(h, tok, 2.0 * (double)h->elem * (double)L, 0.0, 0.0, c->comm_stream);
            ++h->exchanges;
        }
    }
    if (e != cudaSuccess) return cuda_fail_h(h, e, "overlapped qubit swap");
    // (2) the staying halves, on the main stream, on the other SMs
    const int sms = h->cfg.num_sms;
    h->cfg.num_sms = sms - lend;
    for (size_t i = 0; i < ranks.size() && s == SV_OK; ++i)
        if (!runs[i].empty())
            s = run_on_half(h, sub, runs[i], lf, at(slice_of(c, ranks[i]), (uint64_t)beta_of(ranks[i]) * half, h->elem));
    h->cfg.num_sms = sms;
    if (s != SV_OK) return s;
    // join: the swap done on this device; IPC: on every device (the partner writes our half)
    e = cudaEventRecord(c->ev_join, c->comm_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->stream, c->ev_join, 0);
    if (e != cudaSuccess) return cuda_fail_h(h, e, "overlapped swap join");
    s = ipc_fence(h);
    if (s != SV_OK) return s;
    // (3) the arrived halves (digit k = 1 - beta before the relabel of positions)
    for (size_t i = 0; i < ranks.size() && s == SV_OK; ++i)
        if (!runs[i].empty())
            s = run_on_half(h, sub, runs[i], lf, at(slice_of(c, ranks[i]), (uint64_t)(1 - beta_of(ranks[i])) * half, h->elem));
    if (s != SV_OK) return s;
    for (auto &r : runs) r.clear();
    const int q = h->local.n + j;                  // the remap itself (as swap_qubits)
    std::swap(c->log_at[k], c->log_at[q]);
    c->pos_of[c->log_at[k]] = k;
    c->pos_of[c->log_at[q]] = q;
    ++c->overlapped;
    return SV_OK;
}

sv_status shard_apply_circuit(sv_handle h, std::vector<GateSpec> &specs, uint32_t flags) {
    // Runs of gates with a local target go through the local circuit driver on every slice
    // this handle owns (fusion / multi-gate passes included).  Controls on sharded digits are
    // a rank predicate (rule ii): per slice, the gate is dropped when its rank fails them and
    // kept without them otherwise, so they do not break the run.  With SV_BLOCK, gates are first
    // merged across commuting neighbours (merge_commuting, also merging gates on sharded qubits:
    // fewer exchanges), and a local gate moves ahead of pending exchange gates it commutes with,
    // so local runs stay long and exchanges cluster.
    const std::vector<int> ranks = ranks_of(h->shard);
    const int first_sh = h->local.n;
    if ((flags & SV_BLOCK) && h->cfg.pass_merge) specs = merge_commuting(specs, 64);
    std::vector<std::vector<GateSpec>> runs(ranks.size());
    std::vector<GateSpec> pending;                 // exchange gates not applied yet, in order
    bool any = false;
    uint32_t run_dep = 0;                          // sharded positions the pending runs depend on
    auto flush = [&]() -> sv_status {
        if (any) {
            const uint32_t local_flags = flags & (SV_FUSE | SV_BLOCK);
            for (size_t i = 0; i < ranks.size(); ++i) {
                if (runs[i].empty()) continue;
                if (h->shard->dryrun()) {
                    h->shard->dry.push_back({0, ranks[i], 0, 0, 0, runs[i]});
                    runs[i].clear();
                    continue;
                }
                sv_status s = run_local_circuit(h, runs[i], local_flags, slice_of(h->shard, ranks[i]));
                if (s != SV_OK) return s;
                runs[i].clear();
            }
            any = false;
            run_dep = 0;
        }
        for (const GateSpec &g : pending) {
            sv_status s = apply_phys(h, g);
            if (s != SV_OK) return s;
        }
        pending.clear();
        return SV_OK;
    };
    const bool reorder = (flags & SV_BLOCK) != 0;
    ShardCtx *c = h->shard;
    for (size_t gi = 0; gi < specs.size(); ++gi) {
        const GateSpec &gl0 = specs[gi];
        GateSpec g = to_phys(c, gl0);
        ShardKind kind = classify(h->local, g);
        if (kind == SK_EXCHANGE && h->cfg.shard_swap && pick_local(h, g.target - first_sh, &specs, gi) >= 0) {
            const int j = g.target - first_sh, k = pick_local(h, j, &specs, gi);
            const int top = h->local.n - 1;
            bool ov = any && pending.empty() && k == top && h->cfg.shard_overlap > 0 && h->local.n >= 2 &&
                      h->cfg.shard_overlap < h->cfg.num_sms && !((run_dep >> j) & 1u) &&
                      (c->transport == kIpc || c->transport == kLoopback);
            for (size_t i = 0; ov && i < runs.size(); ++i)
                for (const GateSpec &q : runs[i]) {
                    if (q.target + q.span > top) ov = false;          // touches digit k
                    for (const auto &cs : q.ctrl) if (cs.q == top) ov = false;
                }
            sv_status s = SV_OK;
            if (ov) {                               // rule vi overlapped with the pending run
                s = overlapped_remap(h, k, j, runs, ranks, flags);
                any = false;
                run_dep = 0;
            } else {
                s = flush();                        // rule vi: remap, then the gate is local
                bool swapped = false;
                if (s == SV_OK) s = try_swap(h, j, &specs, gi, &swapped);
            }
            if (s != SV_OK) return s;
            g = to_phys(c, gl0);
            kind = classify(h->local, g);
        }
        if (kind == SK_RELABEL) {                   // pending exchanges are planned on the old map
            sv_status s = flush();
            if (s != SV_OK) return s;
            for (const auto &rs : relabel(c, g, first_sh))
                for (size_t i = 0; i < ranks.size(); ++i)
                    if (ranks[i] == rs.first) {
                        runs[i].push_back(scale_gate(h->local, rs.second));
                        any = true;
                        run_dep = ~0u;              // slice-specific scaling: no overlapped remap
                    }
            continue;
        }
        if (kind == SK_EXCHANGE) {
            pending.push_back(g);
            if (!reorder) {
                sv_status s = flush();
                if (s != SV_OK) return s;
            }
            continue;
        }
        bool ahead = true;                          // may this local gate pass the pending ones?
        for (const GateSpec &q : pending) ahead = ahead && commute(q, g);
        if (!ahead) {
            sv_status s = flush();
            if (s != SV_OK) return s;
        }
        for (size_t i = 0; i < ranks.size(); ++i) {
            const int l = c->lrank[ranks[i]];          // bit j of l = digit of q_{n-s+j}
            for (const auto &cs : g.ctrl)
                if (cs.q >= first_sh) run_dep |= 1u << (cs.q - first_sh);   // rank predicate on that digit
            if (!fires_on(g.ctrl, first_sh, l)) continue;
            if (kind == SK_PHASE) {
                run_dep |= 1u << (g.target - first_sh);                    // phase of that digit's value
                GateSpec pl;
                if (phase_local(h->local, g, l, &pl)) {
                    runs[i].push_back(std::move(pl));
                    any = true;
                }
                continue;
            }
            GateSpec lg = g;
            lg.ctrl.clear();
            for (const auto &cs : g.ctrl)
                if (cs.q < first_sh) lg.ctrl.push_back(cs);
            {
                runs[i].push_back(std::move(lg));
                any = true;
            }
        }
    }
    return flush();
}

sv_status shard_reset(sv_handle h, uint64_t idx) {
    ShardCtx *c = h->shard;
    c->identity_map(h->reg.n);
    const uint64_t L = h->local.D;
    const int owner = (int)(idx / L);
    for (int r : ranks_of(c)) {
        cudaError_t e;
        if (r == owner)
            e = launch_set_basis(slice_of(c, r), L, idx - (uint64_t)owner * L, h->stream, &h->launches, h->c64);
        else
            e = cudaMemsetAsync(slice_of(c, r), 0, L * h->elem, h->stream);
        if (e != cudaSuccess) return cuda_fail_h(h, e, "sharded reset");
    }
    return SV_OK;
}

sv_status shard_set_amplitudes(sv_handle h, uint64_t first, uint64_t count, const double *in) {
    ShardCtx *c = h->shard;
    sv_status rs = restore_layout(h);
    if (rs != SV_OK) return rs;
    const uint64_t L = h->local.D;
    for (int r : ranks_of(c)) {
        const uint64_t lo = (uint64_t)c->lrank[r] * L, hi = lo + L;
        const uint64_t a = first > lo ? first : lo, b = (first + count) < hi ? first + count : hi;
        if (a >= b) continue;
        if (h->c64) {                        // complex64: round the ABI's doubles on the host
            const uint64_t chunk = 1ull << 22;
            std::vector<float2> tmp((size_t)((b - a) < chunk ? (b - a) : chunk));
            for (uint64_t o = a; o < b; o += chunk) {
                const uint64_t n = (b - o) < chunk ? b - o : chunk;
                for (uint64_t i = 0; i < n; ++i)
                    tmp[i] = make_float2((float)in[2 * (o - first + i)], (float)in[2 * (o - first + i) + 1]);
                cudaError_t e = cudaMemcpyAsync(at(slice_of(c, r), o - lo, h->elem), tmp.data(), n * h->elem,
                                                cudaMemcpyHostToDevice, h->stream);
                if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
                if (e != cudaSuccess) return cuda_fail_h(h, e, "sharded upload");
            }
            continue;
        }
        cudaError_t e = cudaMemcpyAsync(slice_of(c, r) + (a - lo), in + 2 * (a - first),
                                        (b - a) * sizeof(double2), cudaMemcpyHostToDevice, h->stream);
        if (e != cudaSuccess) return cuda_fail_h(h, e, "sharded upload");
    }
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail_h(h, e, "sharded upload");
    return SV_OK;
}

sv_status shard_amplitudes(sv_handle h, uint64_t first, uint64_t count, double *out) {
    ShardCtx *c = h->shard;
    sv_status rs = restore_layout(h);
    if (rs != SV_OK) return rs;
    rs = ipc_fence(h);                       // IPC: every rank's slice final before anyone reads
    if (rs != SV_OK) return rs;
    const uint64_t L = h->local.D;
    for (int r = 0; r < c->P; ++r) {
        const uint64_t lo = (uint64_t)c->lrank[r] * L, hi = lo + L;
        const uint64_t a = first > lo ? first : lo, b = (first + count) < hi ? first + count : hi;
        if (a >= b) continue;
        // loopback: the slice is in this handle; IPC: read the owner's slice through its mapping
        double2 *src = c->loopback() ? c->slices[r] : (c->transport == kIpc ? c->peer[r] : nullptr);
        if (src && !h->c64) {
            cudaError_t e = cudaMemcpyAsync(out + 2 * (a - first), src + (a - lo),
                                            (b - a) * sizeof(double2), cudaMemcpyDeviceToHost, h->stream);
            if (e != cudaSuccess) return cuda_fail_h(h, e, "sharded readback");
            continue;
        }
        if (src) {                           // complex64: widen to the ABI's doubles on the host
            const uint64_t chunk = 1ull << 22;
            std::vector<float2> tmp((size_t)((b - a) < chunk ? (b - a) : chunk));
            for (uint64_t o = a; o < b; o += chunk) {
                const uint64_t n = (b - o) < chunk ? b - o : chunk;
                cudaError_t e = cudaMemcpyAsync(tmp.data(), at(src, o - lo, h->elem), n * h->elem,
                                                cudaMemcpyDeviceToHost, h->stream);
                if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
                if (e != cudaSuccess) return cuda_fail_h(h, e, "sharded readback");
                for (uint64_t i = 0; i < n; ++i) {
                    out[2 * (o - first + i)] = tmp[i].x;
                    out[2 * (o - first + i) + 1] = tmp[i].y;
                }
            }
            continue;
        }
        for (uint64_t p = a; p < b; p += c->chunk) {     // owner broadcasts, chunk by chunk
            const uint64_t len = (b - p < c->chunk) ? b - p : c->chunk;
            const void *src = (r == c->rank) ? (const void *)at(c->slices[0], p - lo, h->elem) : nullptr;
            ncclResult_t rr = nccl().Broadcast(src ? src : c->stage[0], c->stage[0], 2 * len,
                                               h->c64 ? ncclFloat32 : ncclFloat64, r, c->comm, h->stream);
            if (rr != ncclSuccess) return nccl_fail(h, rr, "ncclBroadcast");
            if (h->c64) {
                std::vector<float2> tmp((size_t)len);
                cudaError_t e = cudaMemcpyAsync(tmp.data(), c->stage[0], len * h->elem, cudaMemcpyDeviceToHost,
                                                h->stream);
                if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
                if (e != cudaSuccess) return cuda_fail_h(h, e, "sharded readback");
                for (uint64_t i = 0; i < len; ++i) {
                    out[2 * (p - first + i)] = tmp[i].x;
                    out[2 * (p - first + i) + 1] = tmp[i].y;
                }
                continue;
            }
            cudaError_t e = cudaMemcpyAsync(out + 2 * (p - first), c->stage[0], len * sizeof(double2),
                                            cudaMemcpyDeviceToHost, h->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
            if (e != cudaSuccess) return cuda_fail_h(h, e, "sharded readback");
        }
    }
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail_h(h, e, "sharded readback");
    return ipc_fence(h);                     // IPC: nobody writes a slice another rank still reads
}

sv_status shard_allreduce_sum(sv_handle h, double *v) {
    ShardCtx *c = h->shard;
    if (c->transport == kIpc) {   // partials through shared memory, summed in rank order
        const int par = c->red_parity;
        c->red_parity ^= 1;
        c->shm->red[par][c->rank] = *v;
        sv_status s = ipc_barrier_raw(c);
        if (s != SV_OK) { h->broken = true; return s; }
        double t = 0.0;
        for (int r = 0; r < c->P; ++r) t += c->shm->red[par][r];
        *v = t;
        return SV_OK;
    }
    if (c->loopback()) {   // local_norm2 covered slice 0; add the others
        double2 *keep = h->psi;
        for (int r = 1; r < c->P; ++r) {
            double s2 = 0.0;
            h->psi = c->slices[r];
            sv_status s = local_norm2(h, &s2);
            h->psi = keep;
            if (s != SV_OK) return s;
            *v += s2;
        }
        return SV_OK;
    }
    cudaError_t e = cudaMemcpyAsync(c->d_scalar, v, sizeof(double), cudaMemcpyHostToDevice, h->stream);
    if (e != cudaSuccess) return cuda_fail_h(h, e, "allreduce");
    ncclResult_t r = nccl().AllReduce(c->d_scalar, c->d_scalar, 1, ncclFloat64, ncclSum, c->comm, h->stream);
    if (r != ncclSuccess) return nccl_fail(h, r, "ncclAllReduce");
    e = cudaMemcpyAsync(v, c->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail_h(h, e, "allreduce");
    return SV_OK;
}

// Wait for the handle's stream while watching the transport: NCCL asynchronous errors abort the
// communicator; an IPC peer that gave up stops this rank too; nothing completes within
// SV_COMM_TIMEOUT_S -> abort.  The handle is unusable after a failure (sticky, like CUDA faults).
sv_status shard_sync(sv_handle h) {
    ShardCtx *c = h->shard;
    const auto t0 = std::chrono::steady_clock::now();
    const double limit = comm_timeout_s();
    for (uint64_t it = 0;; ++it) {
        cudaError_t e = cudaStreamQuery(h->stream);
        if (e == cudaSuccess) break;
        if (e != cudaErrorNotReady) return cuda_fail_h(h, e, "sharded sync");
        if (c->transport == kNccl && c->comm && nccl().CommGetAsyncError) {
            ncclResult_t ae = ncclSuccess;
            if (nccl().CommGetAsyncError(c->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress) {
                if (nccl().CommAbort) nccl().CommAbort(c->comm);
                c->comm = nullptr;
                return nccl_fail(h, ae, "NCCL asynchronous error (communicator aborted)");
            }
        }
        if (c->transport == kIpc && c->shm->failed.load(std::memory_order_relaxed)) {
            h->broken = true;
            return fail_msg(SV_ERR_NCCL, "IPC transport: another rank failed");
        }
        if (it < 256) { sched_yield(); continue; }
        struct timespec ts = {0, 50000};
        nanosleep(&ts, nullptr);
        if ((it & 255) == 0 &&
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
            if (c->transport == kNccl && c->comm && nccl().CommAbort) { nccl().CommAbort(c->comm); c->comm = nullptr; }
            if (c->transport == kIpc) c->shm->failed.store(1, std::memory_order_relaxed);
            h->broken = true;
            return fail_msg(SV_ERR_NCCL, "sharded sync: timeout (SV_COMM_TIMEOUT_S)");
        }
    }
    return SV_OK;
}

}  // namespace svi

using namespace svi;

extern "C" {

sv_status sv_nccl_unique_id(void *out128) {
    if (!out128) return fail_msg(SV_ERR_INVALID_ARG, "null out");
    if (!nccl().ok) return fail_msg(SV_ERR_NCCL, nccl().why);
    ncclUniqueId id;
    ncclResult_t r = nccl().GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(nullptr, r, "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
    return SV_OK;
}

static sv_status create_sharded(const int32_t *dims, int32_t n, sv_dtype dt, int32_t rank, int32_t nranks,
                                int transport, const void *id128, int device, void *cuda_stream, sv_handle *out) {
    if (!out) return fail_msg(SV_ERR_INVALID_ARG, "null out");
    *out = nullptr;
    if (nranks == 1 && rank <= 0)
        return sv_create_ex(dims, n, dt, device, cuda_stream, nullptr, 0, out);
    if (dt != SV_C128 && dt != SV_C64) return fail_msg(SV_ERR_INVALID_ARG, "unknown dtype");
    if (nranks < 1 || (nranks & (nranks - 1))) return fail_msg(SV_ERR_INVALID_ARG, "nranks must be a power of two");
    if (rank < -1 || rank >= nranks) return fail_msg(SV_ERR_INVALID_ARG, "rank out of range");
    if (transport == kIpc && (rank < 0 || nranks > kMaxIpcRanks))
        return fail_msg(SV_ERR_INVALID_ARG, "IPC transport: rank 0..nranks-1, nranks <= 64");
    if (transport != kLoopback && !id128) return fail_msg(SV_ERR_INVALID_ARG, "null unique id");
    sv_handle h = new (std::nothrow) sv_state_s();
    if (!h) return fail_msg(SV_ERR_NOMEM, "host allocation");
    std::string *err = err_slot();
    sv_status s = make_register(dims, n, &h->reg, err);
    if (s != SV_OK) { delete h; return s; }
    int sh = 0;
    while ((1 << sh) < nranks) ++sh;
    if (sh >= n) { delete h; return fail_msg(SV_ERR_UNSUPPORTED, "need at least one local qudit"); }
    for (int k = n - sh; k < n; ++k)
        if (dims[k] != 2) { delete h; return fail_msg(SV_ERR_UNSUPPORTED, "sharded digits must be qubits"); }
    s = make_register(dims, n - sh, &h->local, err);
    if (s != SV_OK) { delete h; return s; }
    h->c64 = dt == SV_C64;
    h->elem = h->c64 ? sizeof(float2) : sizeof(double2);
    ShardCtx *c = new ShardCtx();
    c->P = nranks;
    c->s = sh;
    c->rank = rank;
    c->transport = transport;
    c->identity_map(n);
    h->shard = c;
    if (transport == kIpc) {             // attach the control block before any device work
        char name[129];
        std::memcpy(name, id128, 128);
        name[128] = 0;
        if (name[0] != '/') { state_free(h); return fail_msg(SV_ERR_INVALID_ARG, "bad IPC id"); }
        const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
        if (fd < 0) { state_free(h); return fail_msg(SV_ERR_NCCL, std::string("shm_open ") + name + " failed"); }
        if (ftruncate(fd, sizeof(IpcShm)) != 0) {
            close(fd);
            state_free(h);
            return fail_msg(SV_ERR_NCCL, "ftruncate of the IPC control block failed");
        }
        void *m = mmap(nullptr, sizeof(IpcShm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (m == MAP_FAILED) { state_free(h); return fail_msg(SV_ERR_NCCL, "mmap of the IPC control block failed"); }
        c->shm = reinterpret_cast<IpcShm *>(m);
        std::memcpy(c->shm_name, name, sizeof(name));
    }
    s = state_init_device(h, device, cuda_stream, nullptr, 0);
    if (s != SV_OK) {
        if (c->shm) c->shm->failed.store(1);
        state_free(h);
        return s;
    }
    c->slices.push_back(h->psi);
    const uint64_t L = h->local.D;
    cudaError_t e = cudaSuccess;
    if (transport == kLoopback) {
        for (int r = 1; r < nranks && e == cudaSuccess; ++r) {
            double2 *p = nullptr;
            e = cudaMalloc(&p, L * h->elem);
            if (e == cudaSuccess) c->slices.push_back(p);
        }
        if (e != cudaSuccess) { cudaGetLastError(); state_free(h); return fail_msg(SV_ERR_NOMEM, "slice allocation"); }
    } else if (transport == kIpc) {
        // publish this rank's slice, then map every other rank's (CUDA IPC; across GPUs the
        // mapping enables peer access over NVLink)
        IpcShm *m = c->shm;
        e = cudaIpcGetMemHandle(&m->mem[rank], h->psi);
        m->device[rank] = device;
        if (e != cudaSuccess) { m->failed.store(1); state_free(h); return cuda_fail_h(nullptr, e, "cudaIpcGetMemHandle"); }
        s = ipc_barrier_raw(c);
        if (s != SV_OK) { state_free(h); return s; }
        c->peer.assign(nranks, nullptr);
        c->peer[rank] = h->psi;
        for (int r = 0; r < nranks && e == cudaSuccess; ++r) {
            if (r == rank) continue;
            void *p = nullptr;
            e = cudaIpcOpenMemHandle(&p, m->mem[r], cudaIpcMemLazyEnablePeerAccess);
            if (e == cudaSuccess) c->peer[r] = reinterpret_cast<double2 *>(p);
        }
        if (e != cudaSuccess) { m->failed.store(1); state_free(h); return cuda_fail_h(nullptr, e, "cudaIpcOpenMemHandle"); }
        s = ipc_barrier_raw(c);                   // every rank attached: the name can go
        if (s != SV_OK) { state_free(h); return s; }
        shm_unlink(c->shm_name);                  // every rank; all but the first are no-ops
        c->shm_name[0] = 0;
    } else {
        if (!nccl().ok) { state_free(h); return fail_msg(SV_ERR_NCCL, nccl().why); }
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, id, rank);
        if (r != ncclSuccess) { s = nccl_fail(nullptr, r, "ncclCommInitRank"); c->comm = nullptr; state_free(h); return s; }
    }
    const char *ch = getenv("SV_EXCHANGE_CHUNK");
    c->chunk = ch ? strtoull(ch, nullptr, 10) : (16ull << 20);     // 16 Mi amplitudes = 256 MiB
    if (c->chunk == 0) c->chunk = 16ull << 20;
    if (c->chunk > L) c->chunk = L;
    if (transport == kIpc || transport == kLoopback) {   // the stream an overlapped remap swaps on
        e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
        if (e != cudaSuccess) { cudaGetLastError(); state_free(h); return fail_msg(SV_ERR_NOMEM, "comm stream"); }
    }
    if (transport == kNccl) {                 // staging and the comm stream: the NCCL path only
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaMalloc(&c->stage[i], c->chunk * h->elem);
        if (e == cudaSuccess) e = cudaMalloc(&c->d_scalar, sizeof(double));
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking);
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
            e = cudaEventCreateWithFlags(&c->ev_recv[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming);
        }
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming);
        if (e != cudaSuccess) { cudaGetLastError(); state_free(h); return fail_msg(SV_ERR_NOMEM, "exchange buffers"); }
    }
    s = shard_reset(h, 0);
    if (s != SV_OK) { state_free(h); return s; }
    *out = h;
    return SV_OK;
}

sv_status sv_create_sharded(const int32_t *dims, int32_t n, sv_dtype dt, int32_t rank, int32_t nranks,
                            const void *nccl_unique_id, int device, void *cuda_stream, sv_handle *out) {
    return create_sharded(dims, n, dt, rank, nranks, rank < 0 ? kLoopback : kNccl, nccl_unique_id, device,
                          cuda_stream, out);
}

sv_status sv_ipc_unique_id(void *out128) {
    if (!out128) return fail_msg(SV_ERR_INVALID_ARG, "null out");
    std::random_device rd;
    const uint64_t a = ((uint64_t)rd() << 32) ^ rd(), b = ((uint64_t)rd() << 32) ^ rd();
    char name[128];
    std::memset(name, 0, sizeof(name));
    snprintf(name, sizeof(name), "/sv_ipc_%d_%016llx%016llx", (int)getpid(), (unsigned long long)a,
             (unsigned long long)b);
    std::memcpy(out128, name, sizeof(name));
    return SV_OK;
}

sv_status sv_create_sharded_ipc(const int32_t *dims, int32_t n, sv_dtype dt, int32_t rank, int32_t nranks,
                                const void *ipc_id, int device, void *cuda_stream, sv_handle *out) {
    return create_sharded(dims, n, dt, rank, nranks, kIpc, ipc_id, device, cuda_stream, out);
}

// Host only: the sharded schedule of one rank (sv_shard_schedule in sv.h).
sv_status sv_shard_schedule(const int32_t *dims, int32_t n, int32_t nranks, int32_t rank, const sv_gate *gates,
                            int64_t ngates, uint32_t flags, int32_t shard_swap, double *out, int64_t cap,
                            int64_t *out_len, int32_t *out_lrank) {
    if (!out_len || !out_lrank || (cap > 0 && !out)) return fail_msg(SV_ERR_INVALID_ARG, "null output");
    if (nranks < 2 || (nranks & (nranks - 1)) || rank < 0 || rank >= nranks)
        return fail_msg(SV_ERR_INVALID_ARG, "nranks = 2^s >= 2, 0 <= rank < nranks");
    if (ngates < 0 || (ngates > 0 && !gates)) return fail_msg(SV_ERR_INVALID_ARG, "bad gate list");
    sv_state_s hs;
    sv_handle h = &hs;
    std::string *err = err_slot();
    sv_status s = make_register(dims, n, &h->reg, err);
    if (s != SV_OK) return s;
    int sh = 0;
    while ((1 << sh) < nranks) ++sh;
    if (sh >= n) return fail_msg(SV_ERR_UNSUPPORTED, "need at least one local qudit");
    for (int k = n - sh; k < n; ++k)
        if (dims[k] != 2) return fail_msg(SV_ERR_UNSUPPORTED, "sharded digits must be qubits");
    s = make_register(dims, n - sh, &h->local, err);
    if (s != SV_OK) return s;
    std::vector<GateSpec> specs;
    for (int64_t i = 0; i < ngates; ++i) {
        const sv_gate &g = gates[i];
        s = validate_gate(h->reg, g.target, g.ctrl, g.ctrl_vals, g.nctrl, g.U, err);
        if (s != SV_OK) return s;
        GateSpec q;
        q.target = g.target;
        q.d = h->reg.dims[g.target];
        for (int k = 0; k < g.nctrl; ++k) q.ctrl.push_back({g.ctrl[k], g.ctrl_vals[k]});
        q.U.resize((size_t)q.d * q.d);
        for (int k = 0; k < q.d * q.d; ++k) q.U[k] = make_double2(g.U[2 * k], g.U[2 * k + 1]);
        specs.push_back(std::move(q));
    }
    ShardCtx c;
    c.P = nranks;
    c.s = sh;
    c.rank = rank;
    c.transport = kDryRun;
    c.identity_map(n);
    h->shard = &c;
    h->cfg.shard_swap = shard_swap ? 1 : 0;
    h->cfg.pass_merge = 1;
    h->elem = sizeof(double2);
    s = shard_apply_circuit(h, specs, flags);
    if (s == SV_OK) s = restore_layout(h);          // what a readback does first
    h->shard = nullptr;                              // hs is a stack object: nothing to free
    if (s != SV_OK) return s;
    // serialise: per op [kind, partner, beta, k, j, ngates] then per gate
    // [target, nctrl, ctrl..., vals..., d, re/im of U row-major]
    std::vector<double> buf;
    for (const DryOp &o : c.dry) {
        buf.insert(buf.end(), {(double)o.kind, (double)o.partner, (double)o.beta, (double)o.k, (double)o.j,
                               (double)o.gates.size()});
        for (const GateSpec &g : o.gates) {
            buf.push_back(g.target);
            buf.push_back((double)g.ctrl.size());
            for (const auto &cc : g.ctrl) buf.push_back(cc.q);
            for (const auto &cc : g.ctrl) buf.push_back(cc.v);
            buf.push_back(g.d);
            for (const double2 &u : g.U) { buf.push_back(u.x); buf.push_back(u.y); }
        }
    }
    *out_len = (int64_t)buf.size();
    for (int r = 0; r < nranks; ++r) out_lrank[r] = c.lrank[r];
    if ((int64_t)buf.size() > cap) return fail_msg(SV_ERR_INVALID_ARG, "output buffer too small (see *out_len)");
    std::memcpy(out, buf.data(), buf.size() * sizeof(double));
    return SV_OK;
}

}  // extern "C"
