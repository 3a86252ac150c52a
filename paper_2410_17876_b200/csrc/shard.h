// shard.h — sharded mode: the state is split on its s most-significant
// qubit digits over P = 2^s ranks; rank r owns global indices [r D/P, (r+1) D/P).
#pragma once

#include <vector>

#include "plan.h"

struct sv_state_s;
typedef struct sv_state_s *sv_handle;

namespace svi {

struct ShardCtx;

// implemented in sv_api.cpp
sv_status state_init_device(sv_handle h, int device, void *cuda_stream, void *ext, size_t ext_bytes);
void state_free(sv_handle h);
sv_status local_norm2(sv_handle h, double *out);
sv_status local_apply(sv_handle h, const GatePlan &p);
sv_status launch_on(sv_handle h, const GatePlan &p, double2 *buf);
sv_status run_local_circuit(sv_handle h, std::vector<GateSpec> &specs, uint32_t flags, double2 *buf);
void prof_begin(sv_handle h, void **tok, cudaStream_t st = nullptr);
void prof_end(sv_handle h, void *tok, double hbm_bytes, double nvlink_bytes, double touched,
              cudaStream_t st = nullptr);

// implemented in shard.cpp
void shard_destroy(ShardCtx *c);
int shard_rank(const ShardCtx *c);
int shard_nranks(const ShardCtx *c);
uint64_t shard_overlapped(const ShardCtx *c);
sv_status shard_reset(sv_handle h, uint64_t idx);
sv_status shard_apply(sv_handle h, const GateSpec &g, bool check_unitary);
sv_status shard_apply_circuit(sv_handle h, std::vector<GateSpec> &specs, uint32_t flags);
sv_status shard_amplitudes(sv_handle h, uint64_t first, uint64_t count, double *out);
sv_status shard_set_amplitudes(sv_handle h, uint64_t first, uint64_t count, const double *in);
sv_status shard_allreduce_sum(sv_handle h, double *v);

// device side of the exchange (kernels.cu): psi_loc <- a psi_loc + b psi_partner on the
// local indices [base, base+n) whose local control digits match.
struct CombineCtrl {
    int32_t nctrl;
    uint64_t b[kMaxRem];
    uint64_t mb[kMaxRem];     // magic for division by b
    uint64_t d[kMaxRem];
    uint64_t md[kMaxRem];     // magic for division by d
    uint64_t v[kMaxRem];
};
cudaError_t launch_combine(double2 *loc, const double2 *partner, uint64_t n, uint64_t base,
                           double2 a, double2 b, const CombineCtrl &cc, cudaStream_t st,
                           uint64_t *launches, bool c64 = false);

// peer.cu: fused gate + exchange and in-place qubit swap over peer memory.
// (lo_i, hi_i) <- (u[0] lo_i + u[1] hi_i, u[2] lo_i + u[3] hi_i) for i in [first, first+n) whose
// local control digits match.
cudaError_t launch_pair_update(double2 *lo, double2 *hi, uint64_t first, uint64_t n, const double2 u[4],
                               const CombineCtrl &cc, cudaStream_t st, int num_sms, uint64_t *launches,
                               bool c64 = false);
// a[2 b m + o] <-> c[2 b m + o] for the swap-space elements e in [first, first+n), m = e / b, o = e mod b.
cudaError_t launch_pair_swap(double2 *a, double2 *c, uint64_t b, uint64_t first, uint64_t n, cudaStream_t st,
                             int num_sms, uint64_t *launches, bool c64 = false);

// sv_sync / readback of a sharded handle: wait for its stream while watching the transport
// (NCCL asynchronous errors, the IPC peers); aborts on a fault or after SV_COMM_TIMEOUT_S.
sv_status shard_sync(sv_handle h);

}  // namespace svi
