"""bench.py — throughput of the block-simulation hot path on B200.

One step = sv_reset(e_0) + the whole seeded circuit of the workload applied through the
C ABI (every gate kernel of the path).  metric: amplitude-updates/s (sum over gates of the
amplitudes each gate can change, T_g); achieved HBM GB/s = 32 B x that.

  python bench.py [--gpus N --steps K --warmup W] [--config 4] [--impl ours|reference]

N = 1: config 4 (10 qubits + 6 qutrits + 4 ququarts + 2 ququints, D = 4.78e9, 76 GB) on one
GPU — the largest single-GPU config, the one north_star's >= 70 % HBM target is stated on.
N > 1 (torchrun, one process per GPU, NCCL): the same register sharded over N GPUs on its
most-significant qubits (strong scaling), pairwise NVLink exchanges for sharded targets.
--impl reference: the CPU oracle (oracle/blocksim.c, O-2) timed on the host cores on a
bounded sample of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "amplitude-updates/s and achieved HBM GB/s (vs B200 peak) per gate, 1/2/4/8 GPU"
UNIT = "amplitude-updates/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def circuit_work(dims, gates):
    """Per circuit, from the library's host planner: sum_g T_g (touched amplitudes) and the
    FP64 flops of the general gates (8 d flop per touched amplitude: a d x d complex matvec per
    class); monomial gates (phase / permutation, §2.1-2.2) do at most 6 flop per
    moved amplitude and are counted as data movement only."""
    import paper_2410_17876_b200 as P
    T = 0
    flops = 0
    for g in gates:
        pl = P.plan_gate(dims, g.target, g.U, g.ctrl, g.vals)
        T += int(pl.touched)
        if int(pl.kind) == 0:
            flops += 8 * int(pl.d) * int(pl.touched)
    return T, flops


# FP64 peak measured on this pool's B200 (tools/probes/fp64_probe.cu, profiles/r01/fp64_probe.jsonl:
# DFMA 35.7 TFLOP/s, DMMA 37.1); shared memory: 128 B/clk/SM x 148 SMs at the SM clock
FP64_TFLOPS = 35.7
SMEM_B_PER_CLK_SM = 128


def host_info():
    """The host the oracle runs on: logical CPUs, sockets, cores, NUMA nodes, RAM."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k in ("Socket(s)", "Core(s) per socket", "Thread(s) per core", "NUMA node(s)", "Model name"):
                info[k] = v
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal:"):
                    info["ram_gb"] = round(int(line.split()[1]) / 1e6, 1)
    except Exception:
        pass
    return info


def workload_config(cfg: int, dtype: str = "c128", nqubits=None):
    """The workload both arms are quoted on (identical dicts; implementation options go under
    the line's "mode").  nqubits: a reduced register (functional runs), named as such."""
    from sv_inputs import config_circuit, CONFIG_NAMES
    dims = config_circuit(cfg, ngates=0, nqubits=nqubits)[0]
    D = int(np.prod(dims, dtype=object))
    ngates = len(config_circuit(cfg)[1])
    elem = 16 if dtype == "c128" else 8
    return {"workload": CONFIG_NAMES[cfg] + ("" if nqubits is None else f"_reduced_{nqubits}qubits"),
            "dims_q0_first": dims,
            "state_dtype": "complex128" if dtype == "c128" else "complex64", "D": D, "gates": ngates,
            "initial_state": "e_0", "l2": "state (%.1f GB) >> L2 (126 MB): no flush needed" % (elem * D / 1e9)}


def _oracle_sample(cfg: int, budget_s: float, threads: int | None = None):
    """O-2 on a bounded sample of the workload: the same recipe on a register with fewer qubits,
    gates applied in order until ~budget_s of host time.  Work counted by oracle/work.py (the
    metric's definition); the product library is not loaded."""
    from oracle import blocksim as O2
    from oracle import work as W
    from sv_inputs import config_circuit
    nq = {3: 12, 4: 5, 5: 4}.get(cfg, None)        # ~10-20 s of O-2 work on 16 cores
    dims, gates = config_circuit(cfg, nqubits=nq)
    D = int(np.prod(dims))
    psi = np.zeros(D, dtype=np.complex128)
    psi[0] = 1.0
    nt0 = O2.num_threads()
    if threads:
        O2.set_threads(threads)
    try:
        cores = O2.num_threads()
        t0 = time.perf_counter()
        upd, ng = 0, 0
        for g in gates:
            O2.apply(psi, dims, g)
            ng += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
    finally:
        O2.set_threads(nt0)
    upd = W.circuit_touched(dims, gates[:ng])
    return upd / dt, cores, (f"config {cfg} recipe with {nq} qubits (D={D}), first {ng} of {len(gates)} "
                             f"gates, {dt:.1f} s on the host")


def cpu_baseline(cfg: int, budget_s: float = 20.0):
    """O-2 on a bounded sample (all host threads), plus the same sample on one thread."""
    v, cores, sample = _oracle_sample(cfg, budget_s)
    v1, _, sample1 = _oracle_sample(cfg, budget_s / 4, threads=1)
    return {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
            "one_thread": {"value": v1, "sample": sample1}, "host": host_info()}


def run_reference(args, rank, world):
    """The tier's reference arm: the CPU oracle O-2 as it stands, on the host cores.  One step =
    the next few gates of the same recipe on a bounded register (5 qubits instead of 10 for c4)
    so that W + K steps finish in about a minute; only the K steps are timed.  Loads only
    oracle/ and sv_inputs/ (work counted by oracle/work.py)."""
    if rank != 0:
        return
    from oracle import blocksim as O2
    from oracle import work as W
    from sv_inputs import config_circuit
    nq = {3: 7, 4: 5, 5: 4}.get(args.config, None)
    dims, gates = config_circuit(args.config, nqubits=nq)
    D = int(np.prod(dims))
    psi = np.zeros(D, dtype=np.complex128)
    psi[0] = 1.0
    per_step = max(1, min(len(gates) // max(1, args.steps + args.warmup), 6 if args.config >= 3 else 200))
    gi, upd, t = 0, 0, 0.0
    for step in range(args.warmup + args.steps):
        chunk = [gates[(gi + k) % len(gates)] for k in range(per_step)]
        gi += per_step
        t0 = time.perf_counter()
        for g in chunk:
            O2.apply(psi, dims, g)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            t += dt
            upd += W.circuit_touched(dims, chunk)
    value = upd / t
    b = {"value": value, "unit": UNIT, "cores": O2.num_threads(), "kind": "oracle",
         "sample": f"config {args.config} recipe with {nq} qubits (D={D}), {per_step} gates per step, "
                   f"{args.steps} timed steps after {args.warmup} warm-up steps",
         "host": host_info()}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / max(1, args.steps), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(args.config),
            "cpu_baseline": b,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def pairwise_peak(P, ipc_id, rank, world, dev, dtype, allreduce_max, lgl=27, reps=5):
    """In-run NVLink reference for the multi-GPU roofline: the fused exchange kernel alone (H on
    the top sharded qubit with qubit remapping off) on a probe state of 2^lgl amplitudes per
    rank; GB/s per direction per rank = bytes that cross this rank's NVLink ports each way / the
    kernel's event-timed duration, best of `reps`, the slowest rank.  On one GPU (ranks sharing
    cuda:0) this measures HBM, not NVLink, and is labelled so."""
    s = max(1, (world - 1).bit_length())
    dims = [2] * (lgl + s)
    st = P.State.sharded_ipc(dims, rank, world, ipc_id, device=dev, dtype=dtype)
    try:
        st.set_option(P.sv.SV_OPT_SHARD_SWAP, 0)
        from sv_inputs import Gate, hadamard
        gate = [Gate(len(dims) - 1, (), (), hadamard())]
        st.apply_circuit(gate)
        st.sync()
        best = 0.0
        for _ in range(reps):
            st.set_option(P.sv.SV_OPT_PROFILE, 1)
            st.profile_read(reset=True)
            st.apply_circuit(gate)
            pr = st.profile_read(reset=True)
            st.set_option(P.sv.SV_OPT_PROFILE, 0)
            if pr.comm_launches and pr.comm_ms > 0:
                best = max(best, pr.comm_nvlink_bytes / (pr.comm_ms / 1e3) / 1e9)
    finally:
        st.close()
    worst = -allreduce_max(-best)
    return {"gbs_per_direction": worst, "kernel": "k_pair_update (fused exchange)",
            "probe_amplitudes_per_rank": 2 ** lgl}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=None,
                    help="BASELINE config (default: 4 for N <= 4 GPUs; 5, the 391 GB 8-GPU config, for N = 8)")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="N > 1: fused peer-memory kernels over CUDA IPC (default) or NCCL send/recv + combine")
    ap.add_argument("--nqubits", type=int, default=None, help="shrink the register (functional checks only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 direct, 2 tiled")
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--block", action="store_true", help="force multi-gate cache-blocked passes (SV_BLOCK)")
    ap.add_argument("--no-block", action="store_true", help="disable SV_BLOCK on c1-c3")
    ap.add_argument("--graph", action="store_true", help="force a cached CUDA graph (SV_GRAPH)")
    ap.add_argument("--no-graph", action="store_true", help="disable SV_GRAPH on c1/c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ngates", type=int, default=None)
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"],
                    help="state element type (BASELINE configs: c128; c64 = SV_C64, fp32 arithmetic)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config is None:
        args.config = 5 if world >= 8 else 4
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2410_17876_b200 as P
    from sv_inputs import config_circuit

    # one process per GPU; with fewer GPUs than ranks (a functional run of the multi-process
    # path on one GPU: the IPC transport's kernels never wait on another rank) all ranks share
    # cuda:0 and the bootstrap group runs over gloo
    ngpu = torch.cuda.device_count()
    dev = local_rank if ngpu >= world else 0
    torch.cuda.set_device(dev)
    backend = "nccl" if ngpu >= world else "gloo"
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")

    def allreduce_max(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allreduce_sum(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    dims, gates = config_circuit(args.config, ngates=args.ngates, nqubits=args.nqubits)
    # circuit-driver mode per workload (measured, profiles/r01/passbench_*): multi-gate passes
    # (SV_BLOCK) on c1-c5, plus a cached CUDA graph for the launch-bound c1/c2; sharded runs
    # run the same passes on each slice between the cross-rank steps of gates on sharded qubits.
    fuse = not args.no_fuse
    block = args.block or (args.config in (1, 2, 3, 4, 5) and not args.no_block)
    graph = args.graph or (args.config in (1, 2) and not args.no_graph and world == 1)
    T_step, F_step = circuit_work(dims, gates)               # global amplitude updates, flops / step
    D_total = int(np.prod(dims, dtype=object))
    nread = min(4096, D_total)

    nvl_peak = None
    if world > 1:
        if args.transport == "ipc":
            obj = [P.sv.ipc_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, 0)
            nvl_peak = pairwise_peak(P, obj[0], rank, world, dev, args.dtype, allreduce_max)
            obj = [P.sv.ipc_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, 0)
            st = P.State.sharded_ipc(dims, rank, world, obj[0], device=dev, dtype=args.dtype)
        else:
            obj = [P.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, 0)
            st = P.State.sharded(dims, rank, world, obj[0], device=dev, dtype=args.dtype)
    else:
        st = P.State(dims, device=dev, dtype=args.dtype)
    st.set_option(P.sv.SV_OPT_KERNEL, args.kernel)
    ga = P.sv._GateArray(gates)
    info = st.info()
    ext = torch.cuda.ExternalStream(info.cuda_stream)

    def step():
        st.reset(0)
        st.apply_circuit(ga, fuse=fuse, check=False, block=block, graph=graph)

    # ---- cold first submission: a fresh handle's first circuit, host planning included
    st.sync()
    t0 = time.perf_counter()
    step()
    st.sync()
    cold_first_s = time.perf_counter() - t0
    for _ in range(max(0, args.warmup - 1)):
        step()
    st.sync()
    # ---- timed region: K steps, barrier + sync on both sides, CUDA events on the library stream
    st.set_option(P.sv.SV_OPT_PROFILE, 1)
    st.profile_read(reset=True)
    launches0 = st.info().kernel_launches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk:
        e0.record(ext)
        for _ in range(args.steps):
            step()
        e1.record(ext)
        st.sync()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    prof = st.profile_read(reset=True)
    st.set_option(P.sv.SV_OPT_PROFILE, 0)
    launches = st.info().kernel_launches - launches0
    ms_rank = ms
    ms = allreduce_max(ms)
    value = T_step * args.steps / (ms / 1e3)

    # ---- e2e: the public API end to end with host buffers (gate matrices in, norm + the
    # first 4096 amplitudes out), timed on the host around the whole call sequence.  Warm: the
    # handle's memoised host plan is reused (the same circuit every step); cold: the plan cache
    # is off, so every step plans (merge + pass planning) from scratch.
    out = np.empty(nread, dtype=np.complex128)
    h2d = sum(16 * g.U.size + 8 * len(g.ctrl) + 8 for g in gates)

    def e2e_run(cache: bool):
        st.set_option(P.sv.SV_OPT_PLAN_CACHE, 1 if cache else 0)
        st.profile_read(reset=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            st.reset(0)
            st.apply_circuit(gates, fuse=fuse, check=True, block=block, graph=graph)   # host gates each step
            nrm = st.norm()
            st.amplitudes(0, nread, out)
        dt = time.perf_counter() - t0
        plan_ms = st.profile_read(reset=True).plan_ms / args.steps
        st.set_option(P.sv.SV_OPT_PLAN_CACHE, 1)
        dt = allreduce_max(dt)
        return T_step * args.steps / dt, nrm, plan_ms

    v_warm, nrm, plan_warm = e2e_run(True)
    v_cold, _, plan_cold = e2e_run(False)
    e2e = {"value": v_warm, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(8 + 16 * nread), "norm": nrm,
           "host_plan_ms_per_step": plan_warm,
           "cold": {"value": v_cold, "host_plan_ms_per_step": plan_cold,
                    "note": "plan cache off: merge + pass planning on every submission"},
           "first_submission_s": cold_first_s}

    hbm, hbm_src = peaks()
    bpu = 32.0 if args.dtype == "c128" else 16.0      # bytes per amplitude update (read + write)
    traffic_ratio, traffic_note = None, None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            tr = json.load(open(tr_path))["block" if block else "single"]
            traffic_ratio, traffic_note = tr["ratio_dram_to_state_bytes"], tr["source"]
        except Exception:
            pass
    sm_mhz = clk.summary().get("sm_mhz") or 1965.0
    if block and prof.pass_launches:
        # the dominant kernel: k_gate_pass.  Its algorithmic HBM bytes per launch are the state
        # once in and once out (2 x elem x D_local); achieved = that / the mean event-timed launch.
        n_l = prof.pass_launches
        ms_l = prof.pass_ms / n_l
        state_b = prof.pass_state_bytes / n_l
        achieved = state_b / (ms_l / 1e3) / 1e9
        # executed work per launch (merged and paired gates, one smem round trip per item)
        floors = {"hbm": state_b / (hbm * 1e9),
                  "smem": bpu * prof.pass_item_touched / n_l / (SMEM_B_PER_CLK_SM * 148 * sm_mhz * 1e6),
                  "fp64": prof.pass_flops / n_l / (FP64_TFLOPS * 1e12)} if args.dtype == "c128" else None
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "traffic": traffic_ratio * state_b if traffic_ratio else None,
                    "kernel": "k_gate_pass", "algorithmic": "2 x elem bytes x local state per pass (one HBM "
                    "round trip of the state; SURVEY.md 8(d) per-unit 32 B x D amplitudes)",
                    "bytes_per_launch": state_b, "ms_per_launch": ms_l, "launches_timed": int(n_l),
                    "share_of_step": prof.pass_ms / ms if ms else None,
                    "peak_source": hbm_src, "traffic_source": traffic_note}
        pass_roofline = None
        if floors:
            b = max(floors, key=floors.get)
            pass_roofline = {"bound": b, "frac": 1e3 * floors[b] / ms_l, "ms_per_launch": ms_l,
                             "lower_bound_ms_per_launch": {k: 1e3 * v for k, v in floors.items()},
                             "executed_per_launch": {"touched": prof.pass_touched / n_l,
                                                     "smem_round_trip_amplitudes": prof.pass_item_touched / n_l,
                                                     "fp64_flops": prof.pass_flops / n_l},
                             "peaks": {"hbm_gbs": hbm, "fp64_tflops": FP64_TFLOPS,
                                       "smem_bytes_per_clk_per_sm": SMEM_B_PER_CLK_SM, "sm_mhz": sm_mhz},
                             "note": "floors from the executed (merged, paired) gates of each pass"}
    else:
        n_l = max(1, prof.launches)
        ms_l = prof.kernel_ms / n_l
        b_l = prof.algorithmic_bytes / n_l
        achieved = b_l / (ms_l / 1e3) / 1e9 if prof.launches else None
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm if achieved else None,
                    "traffic": traffic_ratio * b_l if traffic_ratio else None,
                    "kernel": "single-gate kernels (k_gate_tiled / k_gate_direct)",
                    "algorithmic": "32 B x touched amplitudes per gate launch (SURVEY.md 8(d))",
                    "bytes_per_launch": b_l, "ms_per_launch": ms_l, "launches_timed": int(prof.launches),
                    "share_of_step": prof.kernel_ms / ms if ms else None,
                    "peak_source": hbm_src, "traffic_source": traffic_note}
        pass_roofline = None
    multi = None
    if world > 1:
        # SURVEY.md 8(d) multi-GPU roofline: per rank, the HBM time of its passes and single-gate
        # launches plus, for the cross-rank kernels, the slower of their HBM and NVLink times;
        # the slowest rank's floor over the slowest rank's measured time
        bw_nvl = (nvl_peak or {}).get("gbs_per_direction") or 770.0
        gate_bytes = max(0.0, prof.algorithmic_bytes - bpu * prof.pass_touched - prof.comm_hbm_bytes)
        floor_s = ((prof.pass_state_bytes + gate_bytes) / (hbm * 1e9) +
                   max(prof.comm_hbm_bytes / (hbm * 1e9), prof.comm_nvlink_bytes / (bw_nvl * 1e9)))
        floor_max = allreduce_max(floor_s)
        nvl_step = prof.comm_nvlink_bytes / args.steps
        multi = {"transport": args.transport if world > 1 else None,
                 "nvlink_bytes_per_step_per_rank": nvl_step,
                 "nvlink_bytes_per_step_max_rank": allreduce_max(nvl_step),
                 "cross_rank_kernels_per_step": prof.comm_launches / args.steps,
                 "cross_rank_ms_per_step": prof.comm_ms / args.steps,
                 "cross_rank_nvlink_gbs": (prof.comm_nvlink_bytes / (prof.comm_ms / 1e3) / 1e9) if prof.comm_ms else None,
                 "pairwise_peak": nvl_peak,
                 "bw_nvlink_gbs_used": bw_nvl,
                 "bw_nvlink_source": "in-run pairwise probe" if nvl_peak else "B200_PROFILING.md peer copy 770 GB/s",
                 "ranks_share_one_gpu": ngpu < world,
                 "roofline_floor_ms_per_step": 1e3 * floor_max / args.steps,
                 "roofline_frac": floor_max / (ms / 1e3)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64" if args.dtype == "c128" else "f32",
            "data": "synthetic",
            "config": workload_config(args.config, args.dtype, args.nqubits),
            "mode": {"fuse": fuse, "block_passes": block, "cuda_graph": graph, "kernel": args.kernel,
                     "sharded_ranks": world, "gates_timed": len(gates)},
            "hbm_gbs": bpu * value / 1e9,
            "effective_hbm_frac": bpu * value / 1e9 / hbm if world == 1 else None,
            "effective_note": "32 B x sum of T over the user's gates / step time, over the measured HBM peak: "
                              "above 1 when a pass applies several gates per HBM round trip",
            "roofline": roofline,
            "pass_roofline": pass_roofline,
            "multi_gpu": multi,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.config)
        print(json.dumps(line), flush=True)
    st.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
