// plan.h — host-side register model, gate validation/classification and launch planning.
#pragma once

#include <string>
#include <vector>

#include "sv_internal.h"
#include "../../include/sv.h"

namespace svi {

// Register model: dims q_0 first, b_k = prod_{t<k} d_t, D.
struct Register {
    int n = 0;
    int dims[64];
    uint64_t b[64];
    uint64_t D = 0;
};

sv_status make_register(const int32_t *dims, int32_t n, Register *reg, std::string *err);

struct CtrlSpec {
    int q;
    int v;
};

// A gate whose target occupies `span` consecutive qudits starting at `target` (span 2 =
// fused adjacent pair, dimension d_k*d_{k+1}, combined digit j_k + d_k*j_{k+1}).
struct GateSpec {
    int target = 0;
    int span = 1;
    int d = 0;
    std::vector<CtrlSpec> ctrl;
    std::vector<double2> U;   // d*d row-major
};

// Structural validation (ranges, overlap, duplicates, control values).
sv_status validate_gate(const Register &reg, int target, const int32_t *ctrl,
                        const int32_t *vals, int nctrl, const double *U, std::string *err);

// max |U^dag U - I| (NaN/Inf -> +inf)
double unitarity_error(const double2 *U, int d);

// Build the launch plan (classification per PAPER.md §2.1-2.3, fibre decomposer §8 a3).
sv_status plan_gate(const Register &reg, const GateSpec &g, bool check_unitary, GatePlan *out,
                    std::string *err);

// Greedy fusion of consecutive same-qudit / adjacent-qudit gates with identical controls
// into one gate of dimension <= 16.
std::vector<GateSpec> fuse_gates(const Register &reg, const std::vector<GateSpec> &in);

// Sufficient commutation test of two (controlled) single-qudit gates (reading R19).
bool commute(const GateSpec &a, const GateSpec &b);
// Identical control sets (qudits and values, any order).
bool same_controls(const GateSpec &a, const GateSpec &b);

// Consecutive gates on the same target with identical controls -> one matrix product.
std::vector<GateSpec> merge_same_qudit(const std::vector<GateSpec> &in);

// Commutation-aware merging of same-target, same-control gates across gates that commute with
// the later one (a superset of merge_same_qudit); used before multi-gate pass planning.
std::vector<GateSpec> merge_commuting(const std::vector<GateSpec> &in, int window);

// Multi-gate cache-blocked passes.  A pass applies several gates to every
// tile of the state while the tile sits in shared memory: the tile holds all digit values of
// a set Q of "in-tile" qudits (the low prefix q_0..q_{m0-1} whose stride is < 32 is always
// included, so every copied piece is >= 32 amplitudes) and one value of every other digit.
// Gates whose target is in Q can be applied in the pass; their controls may be anywhere.
// Gates are pulled forward past skipped gates only when they commute with them
// (different targets, neither target controls the other).
struct PassPlan {
    std::vector<int> gates;      // indices into the (merged) gate list, in application order
    std::vector<int> H;          // in-tile qudits above the low prefix (ascending)
    int m0 = 0;                  // low prefix q_0..q_{m0-1}
    uint64_t tile = 0;           // amplitudes per tile = b_{m0} * prod_{h in H} d_h
};
// search: choose each pass's in-tile set by scoring every subset of the window's targets
// that fits (else first come, first admitted).
// low_stride: the forced low prefix is every qudit whose stride is below it (in amplitudes; the
// bulk copies of a tile are runs of at least b_{m0} amplitudes)
std::vector<PassPlan> plan_passes(const Register &reg, const std::vector<GateSpec> &g, uint64_t tile_cap,
                                  int max_gates, int window, bool search = true, uint64_t low_stride = 32);

// Work of one multi-gate pass as executed (after merging and pairing), for the roofline:
//   touched      sum of T over the pass's gates (SURVEY.md §8(d) amplitude updates);
//   item_touched amplitudes each executed item (a gate, or a pair gate applied as one 4-member
//                class) reads and writes in shared memory: one round trip per item;
//   flops        FP64 flops of the general items, 8 d flop per touched amplitude (d x d
//                complex matvec per class).
struct PassWork {
    double touched = 0.0;
    double item_touched = 0.0;
    double flops = 0.0;
};

// Launch one multi-gate pass (mgpass.cu).  *handled = false if the pass does not fit the
// kernel (the caller then applies its gates one by one).
cudaError_t run_pass(const Register &reg, const std::vector<GateSpec> &gates, const PassPlan &pp, double2 *psi,
                     cudaStream_t st, const LaunchCfg &cfg, bool *handled, PassWork *work);

// Shard planning.  s = log2(nranks) top digits are sharded qubits.
struct ShardAction {
    int action;    // 0 local, 1 skip, 2 exchange
    int partner;
    int beta;
};
sv_status shard_plan(const Register &reg, int nranks, int rank, int target,
                     const std::vector<CtrlSpec> &ctrl, ShardAction *out, std::string *err);

}  // namespace svi
