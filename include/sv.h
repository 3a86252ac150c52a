/*
 * sv.h — C ABI of the B200 mixed-radix statevector engine (arXiv 2410.17876 hot path).
 *
 * The library applies single-qudit gates, optionally (multi-)controlled, to a dense
 * complex128 statevector resident in HBM by the paper's block method: for a gate on
 * qudit q_k it visits every equivalence class (the d_k amplitudes that differ only in
 * q_k, Table tab:eq_classes), replaces the class vector x by U x
 * (PAPER.md:222), and stores it back in place.  Controlled gates touch only classes whose
 * control digits match.  No tensor product and no D×D operator is
 * ever formed.
 *
 * Conventions (binding for every entry point):
 *   - dims[] lists the qudits q_0 FIRST; q_0 is the least-significant digit.
 *     Basis index i = sum_k q_k * b_k with block size b_k = prod_{t<k} d_t.
 *   - 2 <= d_k <= 16; 1 <= n <= 64; D = prod d_k must fit in uint64.
 *   - Amplitudes are interleaved (re, im) doubles; index arguments are uint64.
 *   - U is d×d complex, ROW-major, interleaved (re, im): y_r = sum_c U[r][c] x_c, so column
 *     c of U is the image of |c>.
 *   - A control (c, v) fires when floor(i / b_c) mod d_c == v; all controls
 *     of a gate are ANDed.  A control may not equal the target or repeat.
 *
 * Ownership: every host input (dims, ctrl, ctrl_vals, U, gates, amplitude buffers) is read
 * or copied before the call returns; the caller keeps ownership.  The library owns the
 * device statevector unless it was adopted with sv_create_ex(ext_device_buf), in which
 * case the caller's buffer must outlive the handle.
 *
 * Errors: every call returns sv_status.  Arguments are validated before any device work,
 * so on a validation error the state is unchanged.  Asynchronous CUDA faults are sticky:
 * the next call on the handle reports SV_ERR_CUDA and the handle is unusable afterwards.
 * sv_last_error() returns a thread-local message for the last failing call.
 *
 * Concurrency: one call at a time per handle.  Gate kernels run asynchronously on the
 * handle's stream; sv_norm, sv_amplitudes, sv_set_amplitudes and sv_sync synchronise it.
 * Sharded handles are SPMD: every rank makes the same calls with identical arguments.
 */
#ifndef SV_H_
#define SV_H_

#include <stddef.h>
#include <stdint.h>

#if defined(SV_BUILD_LIB) && defined(__GNUC__)
#define SV_API __attribute__((visibility("default")))
#else
#define SV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sv_state_s *sv_handle;

/* Element type of the state.  SV_C128: complex128 (the BASELINE configs).  SV_C64: complex64
 * (8 B per amplitude, arithmetic in fp32, also sharded: exchanges move fp32 pairs; SV_BLOCK
 * passes run when the tile's bulk copies are 16-byte aligned, i.e. b_{m0} is even, else the
 * gates fall back to single-gate passes).  The ABI's amplitude buffers and matrices are always
 * doubles; SV_C64 rounds them on the way in and widens them on the way out. */
typedef enum { SV_C128 = 0, SV_C64 = 1 } sv_dtype;

typedef enum {
    SV_OK = 0,
    SV_ERR_INVALID_ARG = 1,   /* null pointer, bad count, bad handle                     */
    SV_ERR_DIM = 2,           /* n < 1, n > 64, or some d < 2 or d > 16                  */
    SV_ERR_OVERFLOW = 3,      /* D = prod d_k overflows uint64                           */
    SV_ERR_QUDIT_RANGE = 4,   /* target or control index outside [0, n)                  */
    SV_ERR_CTRL_OVERLAP = 5,  /* a control equals the target                             */
    SV_ERR_CTRL_DUP = 6,      /* a control qudit repeats                                 */
    SV_ERR_CTRL_VALUE = 7,    /* control value outside [0, d_c)                          */
    SV_ERR_NOT_UNITARY = 8,   /* max |U^dag U - I| > 1e-12, or a non-finite entry        */
    SV_ERR_INDEX_RANGE = 9,   /* basis index / amplitude range outside [0, D)            */
    SV_ERR_NOMEM = 10,        /* device allocation failed                                */
    SV_ERR_CUDA = 11,         /* CUDA error (sticky)                                     */
    SV_ERR_NCCL = 12,         /* communication error in sharded mode: NCCL, or the IPC
                                 transport (a peer failed or timed out); sticky            */
    SV_ERR_UNSUPPORTED = 13   /* valid request outside what this build implements       */
} sv_status;

/* One gate of a circuit (sv_apply_circuit).  Pointers are read during the call only. */
typedef struct {
    int32_t target;
    int32_t nctrl;
    const int32_t *ctrl;
    const int32_t *ctrl_vals;
    const double *U;          /* d_target × d_target complex, row-major, interleaved */
} sv_gate;

/* sv_apply_circuit flags */
#define SV_FUSE      1u   /* merge same-qudit runs and adjacent-qudit pairs (d_k*d_{k+1} <= 16)
                             into one gate each before launching          */
#define SV_NO_CHECK  2u   /* skip the unitarity check (structure checks still run)            */
#define SV_GRAPH     4u   /* capture the launches in a CUDA graph and replay it               */
#define SV_BLOCK     8u   /* multi-gate cache-blocked passes: gates are grouped
                             (commuting gates may be pulled forward) so that one HBM pass applies
                             every gate whose target lies in a shared-memory tile; takes
                             precedence over SV_FUSE's pair fusion                               */

/* ---- lifecycle ------------------------------------------------------------------------ */

/* Create a single-GPU state on the current device with its own stream; state = e_0
 * (PAPER.md:247).  dims: n entries, q_0 first.  *out receives the handle. */
SV_API sv_status sv_create(const int32_t *dims, int32_t n, sv_dtype dt, sv_handle *out);

/* As sv_create, on `device`, launching on `cuda_stream` (a cudaStream_t, or NULL for a new
 * stream owned by the handle).  If ext_device_buf is non-NULL it is adopted as the state
 * (must hold >= 16*D bytes, 16-byte aligned, on `device`; the caller keeps ownership, e.g.
 * a torch tensor).  The state is set to e_0. */
SV_API sv_status sv_create_ex(const int32_t *dims, int32_t n, sv_dtype dt, int device,
                       void *cuda_stream, void *ext_device_buf, size_t ext_bytes,
                       sv_handle *out);

/* Sharded state over nranks = 2^s GPUs (one process per GPU).  The s most-significant
 * digits must be qubits; rank r initially owns global indices [r*D/P, (r+1)*D/P) (SURVEY.md
 * §8(e)).  Gates on a sharded qubit that need no partner data move none: a diagonal gate is a
 * per-slice local phase, and an anti-diagonal gate with no local controls relabels the slices
 * (afterwards rank r may own a different logical slice); any other gate on a sharded qubit
 * swaps that qubit with a local qubit (SV_OPT_SHARD_SWAP) or exchanges slices.  sv_amplitudes
 * / sv_set_amplitudes address global indices either way (they first swap remapped qubits
 * back), and sv_reset restores the initial layout.
 * nccl_unique_id: the 128-byte ncclUniqueId produced by sv_nccl_unique_id on rank 0 and
 * broadcast by the caller (e.g. through torch.distributed).  cuda_stream as in sv_create_ex.
 * rank = -1 creates a LOOPBACK handle: all nranks slices live in this one handle on one
 * device and the pairwise exchange runs through device copies instead of NCCL (same shard
 * planner, rank predicates, chunking and combine kernel; a single-GPU testing aid).
 * nranks = 1 is an ordinary single-GPU state.  Errors: SV_ERR_UNSUPPORTED if the s top
 * digits are not qubits; SV_ERR_NCCL if NCCL cannot be loaded or initialised. */
SV_API sv_status sv_create_sharded(const int32_t *dims, int32_t n, sv_dtype dt, int32_t rank,
                            int32_t nranks, const void *nccl_unique_id, int device,
                            void *cuda_stream, sv_handle *out);
SV_API sv_status sv_nccl_unique_id(void *out128);

/* Sharded state over the fused peer-memory transport (same layout, rules and
 * SPMD contract as sv_create_sharded).  The nranks processes run on ONE node (one GPU each,
 * or several on one GPU): each rank maps every other rank's slice through CUDA IPC, and a gate
 * on a sharded qubit runs as ONE kernel per rank that reads and writes the partner's slice in
 * place over NVLink — rank lo of the pair updates the classes of local indices [0, L/2), rank hi
 * the rest, (lo_i, hi_i) <- U (lo_i, hi_i) — and a qubit remapping swaps the two
 * half-slices element by element; no staging buffer, no combine pass.  Ranks order these
 * accesses with host barriers in POSIX shared memory (the kernels never wait on each other);
 * norms reduce through it in rank order (deterministic).  ipc_id: the 128-byte id produced by
 * sv_ipc_unique_id on one rank and broadcast by the caller (a shared-memory name).  Every
 * rank must create, use and destroy the state together; a rank that stops (timeout
 * SV_COMM_TIMEOUT_S, default 600 s) makes the others fail with SV_ERR_NCCL instead of hanging.
 * Errors: as sv_create_sharded; SV_ERR_NCCL if the control block cannot be created;
 * SV_ERR_CUDA if CUDA IPC fails (e.g. no peer access between the GPUs). */
SV_API sv_status sv_create_sharded_ipc(const int32_t *dims, int32_t n, sv_dtype dt, int32_t rank,
                                       int32_t nranks, const void *ipc_id, int device,
                                       void *cuda_stream, sv_handle *out);
SV_API sv_status sv_ipc_unique_id(void *out128);

SV_API sv_status sv_destroy(sv_handle h);

/* State = basis vector e_{basis_index} (the paper's initial state is e_0 = |0...0>,
 * PAPER.md:247).  SV_ERR_INDEX_RANGE if basis_index >= D. */
SV_API sv_status sv_reset(sv_handle h, uint64_t basis_index);

/* ---- the hot path --------------------------------------------------------------------- */

/* Apply U on qudit `target`, controlled on ctrl[0..nctrl) having values ctrl_vals[...]
 * (ctrl/ctrl_vals may be NULL when nctrl == 0).  Asynchronous on the handle's stream. */
SV_API sv_status sv_apply_gate(sv_handle h, int32_t target, const int32_t *ctrl,
                        const int32_t *ctrl_vals, int32_t nctrl, const double *U);

/* Validate all gates first (state untouched on any error), then apply them in order
 * (gate after gate; SV_BLOCK may reorder commuting gates, which leaves the result
 * unchanged up to rounding).  flags: SV_FUSE | SV_NO_CHECK | SV_GRAPH | SV_BLOCK. */
SV_API sv_status sv_apply_circuit(sv_handle h, const sv_gate *gates, int64_t ngates, uint32_t flags);

/* ---- readback ------------------------------------------------------------------------- */

/* Copy amplitudes [first, first+count) to out (2*count doubles).  Synchronises.
 * Sharded handles: global indices; collective (the owning ranks broadcast). */
SV_API sv_status sv_amplitudes(sv_handle h, uint64_t first, uint64_t count, double *out);

/* Overwrite amplitudes [first, first+count) from in (2*count doubles).  Synchronises.
 * Sharded: global indices; each rank writes the part it owns (collective call). */
SV_API sv_status sv_set_amplitudes(sv_handle h, uint64_t first, uint64_t count, const double *in);

/* *out = sqrt(sum_i |psi_i|^2), fp64, deterministic two-level tree.  Synchronises.
 * Sharded: collective (all-reduce of the squared partial norms). */
SV_API sv_status sv_norm(sv_handle h, double *out);

/* Wait until every kernel queued on the handle's stream has finished (readback and setup
 * calls synchronise on their own; this makes a timed region end on the device
 * semantics of a completed evolution).  SV_ERR_CUDA reports an asynchronous fault (sticky). */
SV_API sv_status sv_sync(sv_handle h);

/* Thread-local message for the last failing call on this thread (empty if none); valid until
 * the next failing call on the same thread.  Mirrors SPEC.md:45, 261, 346's error names. */
SV_API const char *sv_last_error(void);

/* ---- introspection (tests, bench) -------------------------------------------------------- */

typedef struct {
    uint64_t D;              /* global register size                                    */
    uint64_t local_D;        /* amplitudes held by this handle (D / nranks)             */
    int32_t n;
    int32_t rank, nranks;
    void *device_ptr;        /* the device statevector (local slice)                    */
    void *cuda_stream;
    uint64_t kernel_launches;/* number of this library's kernels launched so far        */
    uint64_t exchanges;      /* sharded: cross-rank steps performed (exchanges and qubit remaps;
                                loopback counts slice pairs)                                */
    uint64_t overlapped;     /* sharded: qubit remaps overlapped with a local run (SV_OPT_SHARD_OVERLAP) */
} sv_info;

SV_API sv_status sv_get_info(sv_handle h, sv_info *out);

/* Engine options (tests/bench): SV_OPT_KERNEL selects the gate kernel family. */
#define SV_OPT_KERNEL       1   /* 0 = auto, 1 = direct (per-fibre), 2 = tiled (TMA bulk)      */
#define SV_OPT_TILE_ELEMS   2   /* amplitudes per smem tile (tiled kernel)                       */
#define SV_OPT_TILE_STAGES  3   /* smem pipeline stages (tiled kernel)                           */
#define SV_OPT_CTAS_PER_SM  4   /* resident CTAs per SM (tiled kernel)                           */
#define SV_OPT_PROFILE      5   /* 1 = bracket every gate kernel with CUDA events on the handle's
                                   stream (read back with sv_profile_read)                        */
#define SV_OPT_PASS_TILE    6   /* SV_BLOCK: the planner's cap on a pass tile, in amplitudes (<= 8192;
                                   default 3200)                                                   */
#define SV_OPT_PASS_STAGES  7   /* SV_BLOCK: ring capacity = this many tiles of SV_OPT_PASS_TILE (2..12,
                                   default 4); each pass re-cuts it into as many stages of its own
                                   tile size as fit (at most 8), so smaller tiles get a deeper ring */
#define SV_OPT_PASS_THREADS 8   /* compute threads per CTA of the pass kernel (256, 384, 512 or 576) */
#define SV_OPT_PASS_GATES   9   /* max gates applied per pass (1..32)                              */
#define SV_OPT_PASS_GROUPS 10   /* consumer warp groups of the pass kernel, each on its own tile
                                   (1, 2, 4 or 8 with 512 threads; at most the number of stages)    */
#define SV_OPT_PASS_WINDOW 11   /* gates the pass planner scans ahead (1..4096)                    */
#define SV_OPT_PASS_MERGE  12   /* 1 (default): merge commuting same-target gates before SV_BLOCK passes;
                                   0: keep every gate (per-gate microbenchmarks)                   */
#define SV_OPT_SHARD_SWAP  13   /* sharded handles: 1 (default) = a gate on a sharded qubit that needs
                                   the partner's amplitudes first swaps that qubit with the top local
                                   qubit (half-slice transfer, then a local gate); 0 = pairwise
                                   exchange + combine.  Ignored when no local qubit has long digit runs */
#define SV_OPT_PASS_SEARCH 14   /* 1 (default): each SV_BLOCK pass's in-tile qudit set is the one that
                                   admits the most window gates (subset search); 0: first come, first
                                   admitted */
#define SV_OPT_SHARD_OVERLAP 17 /* sharded handles (IPC, loopback): when a qubit remap (rule vi) swaps the
                                   top local qubit and the pending local gates neither touch it nor
                                   depend on the remapped sharded digit, the half-slice swap runs on a
                                   comm stream on this many SMs while the pending gates run on the
                                   staying half on the others; the moved half gets them afterwards.
                                   0 = off; default 16                                                */
#define SV_OPT_PASS_LOW    18   /* SV_BLOCK: the low prefix every pass tile holds whole = the qudits whose
                                   stride is below this many amplitudes (default 32: tile runs, i.e.
                                   bulk copies, of >= 512 B for complex128)                          */
#define SV_OPT_PASS_ABSORB 19   /* SV_BLOCK (per-gate pass kernel): 1 (default) = a pure permutation gate
                                   (unit coefficients) whose target is a member digit
                                   of the pass tile and whose controls are member digits or constant
                                   over the tile is not a compute item: moved to the front of the pass
                                   (past the earlier gates it commutes with) it relabels which global
                                   member each tile slot is loaded from, else moved to the back it
                                   relabels where each slot is stored; 0 = every gate is an item     */
#define SV_OPT_PASS_KERNEL 16   /* SV_BLOCK pass kernel: 0 (default) = per-gate (k_gate_pass: every gate
                                   sweeps the shared-memory tile, one group barrier per gate); 1 =
                                   register-blocked stages (k_gate_stage: consecutive gates on a pair of
                                   in-tile digits applied to register blocks, one shared-memory round
                                   trip per stage) when the pass fits them (targets d <= 5)            */
#define SV_OPT_PLAN_CACHE  15   /* 1 (default): the SV_BLOCK host plan (merged gates + passes) is
                                   memoised per handle and reused while the same gates and options
                                   come again; 0: plan every call (cold-submission timing)          */
SV_API sv_status sv_set_option(sv_handle h, int32_t option, int64_t value);

/* Per-launch timing of the gate kernels recorded while SV_OPT_PROFILE is on: the summed
 * device time between the events bracketing each gate launch, the number of launches, and
 * the algorithmic bytes those launches move (one read and one write per touched amplitude:
 * 32 B for complex128, 16 B for complex64).  Synchronises; reset != 0 clears
 * the record. */
typedef struct {
    uint64_t launches;
    double kernel_ms;
    double algorithmic_bytes;  /* 2 x element bytes x sum of T over the gates the launches applied */
    double touched;            /* amplitude updates (sum of T over the launched gates)          */
    double state_bytes;        /* bytes the launches must move at least: a single-gate launch
                                  2 x elem x T; a multi-gate pass (SV_BLOCK) 2 x elem x the state */
    /* the multi-gate pass launches (k_gate_pass) among them, as executed (merged, paired): */
    uint64_t pass_launches;
    double pass_ms;
    double pass_touched;       /* sum of T over the gates the passes applied                   */
    double pass_item_touched;  /* amplitudes read + written in shared memory, one round trip per
                                  executed item (a gate, a qubit pair applied as one class, or a
                                  factored pair of general gates with d_a d_b <= 8)               */
    double pass_flops;         /* FP64 flops of the general items: 8 d per touched amplitude
                                  (8 (d_a + d_b) for a factored pair)                            */
    double pass_state_bytes;   /* 2 x elem x the local state per pass                           */
    double plan_ms;            /* host planning time (SV_BLOCK merge + pass planning) since the
                                  last reset                                                    */
    /* sharded handles: the cross-rank kernels (fused exchanges, qubit swaps): */
    uint64_t comm_launches;
    double comm_ms;
    double comm_hbm_bytes;     /* bytes they move through this rank's HBM                       */
    double comm_nvlink_bytes;  /* bytes per direction over this rank's NVLink ports (IPC
                                  transport; 0 for loopback slices on one device)               */
} sv_profile;
SV_API sv_status sv_profile_read(sv_handle h, int32_t reset, sv_profile *out);

/* Host-only gate analysis (no device work; usable without a GPU).  Fills `out` with the
 * classification and launch plan the library would use for this gate on this register. */
typedef struct {
    int32_t kind;            /* 0 = general, 1 = monomial (phase/permutation, §2.1-2.2) */
    int32_t d;               /* target dimension                                           */
    uint64_t b;              /* target block size b_k                                      */
    uint64_t fibres;         /* number of control-satisfying classes F = D/(d*prod d_c)      */
    uint64_t touched;        /* amplitudes that can change (T)               */
    uint32_t active_mask;    /* monomial: members that move or scale                        */
    int32_t sigma[16];       /* monomial: member j goes to sigma[j]                         */
    double unitarity_err;    /* max |U^dag U - I|                                          */
} sv_gate_plan;

SV_API sv_status sv_plan_gate(const int32_t *dims, int32_t n, int32_t target, const int32_t *ctrl,
                       const int32_t *ctrl_vals, int32_t nctrl, const double *U,
                       sv_gate_plan *out);

/* Host-only: the first `count` class representatives (member j = 0 of each
 * control-satisfying class) in the enumeration order the kernels use, starting at class
 * id `first` — the mixed-radix digit-insertion decomposer of SURVEY.md §8 a3. */
SV_API sv_status sv_enumerate_fibres(const int32_t *dims, int32_t n, int32_t target,
                              const int32_t *ctrl, const int32_t *ctrl_vals, int32_t nctrl,
                              uint64_t first, uint64_t count, uint64_t *out);

/* Host-only: run the fusion planner (SV_FUSE) on a gate list and return the fused list.
 * out_gates / out_ctrl / out_vals / out_U are caller arrays with room for ngates gates,
 * sum(nctrl) controls and ngates*256 complex entries; *out_n receives the fused count.
 * out_gates[i].target is the LOWER qudit of a fused adjacent pair; out_dims[i] holds the
 * fused dimension (d_k or d_k*d_{k+1}), out_span[i] = 1 or 2 qudits. */
SV_API sv_status sv_fuse_plan(const int32_t *dims, int32_t n, const sv_gate *gates, int64_t ngates,
                       int32_t *out_target, int32_t *out_span, int32_t *out_dim,
                       int32_t *out_nctrl, int32_t *out_ctrl, int32_t *out_vals,
                       double *out_U, int64_t *out_n);

/* Host-only: the SV_BLOCK pre-pass that merges gates (PAPER.md:256 applies gates one at a time;
 * merging is this build's addition): each gate joins the latest earlier gate with the same
 * target and the same controls when every gate in between commutes with it (different digits
 * and neither target a control of the other unless that target gate is diagonal, or both on one
 * digit and both diagonal), looking back at most `window` gates; merged matrices are products
 * (later gate on the left).  Output layout as sv_fuse_plan (out_span[i] = 1).  Errors as
 * sv_fuse_plan, plus SV_ERR_INVALID_ARG for window < 1. */
SV_API sv_status sv_merge_plan(const int32_t *dims, int32_t n, const sv_gate *gates, int64_t ngates,
                               int32_t window, int32_t *out_target, int32_t *out_span, int32_t *out_dim,
                               int32_t *out_nctrl, int32_t *out_ctrl, int32_t *out_vals,
                               double *out_U, int64_t *out_n);

/* Host-only: run the SV_BLOCK pass planner (without same-qudit merging) on a gate list.
 * out_order[i] = index of the i-th gate in application order; out_pass[i] = its pass id;
 * out_tile[p] = amplitudes per shared-memory tile of pass p (room for ngates entries);
 * *out_npasses = number of passes.  Gates are only reordered across gates they commute with. */
SV_API sv_status sv_block_plan(const int32_t *dims, int32_t n, const sv_gate *gates, int64_t ngates,
                               int64_t tile_cap, int64_t *out_order, int64_t *out_pass,
                               int64_t *out_tile, int64_t *out_npasses);
/* As sv_block_plan with the planner's knobs: at most max_gates (1..32) gates per pass, `window`
 * gates scanned ahead, search != 0 = the in-tile set search (the SV_BLOCK defaults are 32, 256, 1;
 * sv_block_plan uses 24, 64, 1). */
SV_API sv_status sv_block_plan_ex(const int32_t *dims, int32_t n, const sv_gate *gates, int64_t ngates,
                                  int64_t tile_cap, int32_t max_gates, int32_t window, int32_t search,
                                  int64_t *out_order, int64_t *out_pass, int64_t *out_tile,
                                  int64_t *out_npasses);

/* Host-only (sharded planning): what rank `rank` of `nranks` does for a
 * gate.  *action: 0 = local apply, 1 = skip (a sharded control is unmet on this rank),
 * 2 = pairwise exchange with *partner on sharded target qubit.  *beta = this rank's digit
 * of the sharded target (action 2). */
SV_API sv_status sv_shard_plan(const int32_t *dims, int32_t n, int32_t nranks, int32_t rank,
                        int32_t target, const int32_t *ctrl, const int32_t *ctrl_vals,
                        int32_t nctrl, int32_t *action, int32_t *partner, int32_t *beta);

/* Host-only (no GPU): the sharded schedule rank `rank` of `nranks` runs for a circuit — the same
 * planner as sv_apply_circuit on a sharded handle (rules ii-vi of SURVEY.md §8(e) / DESIGN.md §9:
 * sharded-control predicates, local phases, rank relabelling, qubit remapping when shard_swap != 0,
 * pairwise exchanges), followed by the layout restore a readback performs.  For CPU tests that
 * replay it on per-rank slices over gloo.  out (cap doubles) receives, per step,
 * [kind (0 local gates on this rank's slice, 1 qubit swap, 2 exchange), partner, beta, k, j, ngates]
 * and per gate [target, nctrl, ctrl..., vals..., d, U as re/im pairs, row-major]; *out_len = the
 * doubles written (or needed: SV_ERR_INVALID_ARG if cap is too small); out_lrank[nranks] = the
 * final logical slice of every physical rank.  Gate targets/controls are local digit positions
 * (the sharded controls of local gates already resolved).  flags as sv_apply_circuit. */
SV_API sv_status sv_shard_schedule(const int32_t *dims, int32_t n, int32_t nranks, int32_t rank,
                                   const sv_gate *gates, int64_t ngates, uint32_t flags, int32_t shard_swap,
                                   double *out, int64_t cap, int64_t *out_len, int32_t *out_lrank);

SV_API const char *sv_version(void);

/* ---- sparse states (the paper's "Our Method (Sparse)") --
 * The state is the list of basis indices holding a non-zero amplitude (complex128, sorted by
 * index, on the device).  A gate transforms only the classes that hold a stored index: column v
 * of U times the amplitude of each stored member with target digit v, summed per index
 * (PAPER.md:222); entries whose controls do not hold are unchanged; amplitudes
 * with |a| < eps are dropped afterwards.  D must be <= 2^63 (the paper's 64-bit index limit,
 * PAPER.md:489), so GHZ reaches 62 qubits, 39 qutrits, 31 ququads, 27 ququints. */
typedef struct sv_sparse_s *sv_sparse_handle;

/* State = e_0.  eps <= 0 selects 1e-12.  SV_ERR_OVERFLOW if D > 2^63. */
SV_API sv_status sv_sparse_create(const int32_t *dims, int32_t n, double eps, sv_sparse_handle *out);
SV_API sv_status sv_sparse_destroy(sv_sparse_handle h);
SV_API sv_status sv_sparse_reset(sv_sparse_handle h, uint64_t basis_index);
/* Same argument conventions and validation as sv_apply_gate / sv_apply_circuit (flags:
 * SV_NO_CHECK only).  Each gate synchronises (the new entry count sizes the next gate). */
SV_API sv_status sv_sparse_apply_gate(sv_sparse_handle h, int32_t target, const int32_t *ctrl,
                                      const int32_t *ctrl_vals, int32_t nctrl, const double *U);
SV_API sv_status sv_sparse_apply_circuit(sv_sparse_handle h, const sv_gate *gates, int64_t ngates,
                                         uint32_t flags);
SV_API sv_status sv_sparse_nnz(sv_sparse_handle h, uint64_t *out);
/* Copy min(cap, nnz) entries (ascending index) into idx[] and amp[] (2 doubles each);
 * *n receives nnz. */
SV_API sv_status sv_sparse_entries(sv_sparse_handle h, uint64_t cap, uint64_t *idx, double *amp,
                                   uint64_t *n);
SV_API sv_status sv_sparse_launches(sv_sparse_handle h, uint64_t *out);

#ifdef __cplusplus
}
#endif
#endif /* SV_H_ */
