"""Per-gate cost of the multi-gate pass kernel by gate type: circuits of one gate type only
(targets cycling over a set of in-tile qudits so no two neighbours merge), run as SV_BLOCK
passes on a c4-shaped register.  Prints ms per gate application and the FP64 / shared-memory
floors of that gate (8 d flop and 32 B of shared-memory traffic per touched amplitude)."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

FP64 = 37.0e12        # measured DFMA / DMMA peak (tools/probes/fp64_probe.cu)
SMEM = 128 * 148 * 1.965e9   # 128 B/clk/SM


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nqubits", type=int, default=3)
    ap.add_argument("--ngates", type=int, default=240)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--only", default=None, help="comma-separated mix names")
    args = ap.parse_args()
    import torch
    import paper_2410_17876_b200 as P
    from sv_inputs import Gate, config_dims, haar_unitary, shift_x, clock_z
    dims = config_dims(4, nqubits=args.nqubits)
    n = len(dims)
    D = int(np.prod(dims, dtype=object))
    rng = np.random.default_rng(5)
    qutrits = [q for q in range(n) if dims[q] == 3]
    qubits = [q for q in range(n) if dims[q] == 2]

    def cyc(targets, make):
        return [make(targets[i % len(targets)], i) for i in range(args.ngates)]

    mixes = {
        "general_low_q0q1q2": cyc([0, 1, 2], lambda t, i: Gate(t, (), (), haar_unitary(dims[t], rng))),
        "general_qutrits_H": cyc(qutrits[:3], lambda t, i: Gate(t, (), (), haar_unitary(3, rng))),
        "general_qubits_H": cyc(qubits[:3], lambda t, i: Gate(t, (), (), haar_unitary(2, rng))),
        "general_d4_H": cyc([3, 4], lambda t, i: Gate(t, (), (), haar_unitary(4, rng))),
        "perm_qutrits_H": cyc(qutrits[:3], lambda t, i: Gate(t, (), (), shift_x(3, 1))),
        "cinc_qutrits_ctrl_out": cyc(qutrits[:3], lambda t, i: Gate(t, (n - 1,), (1,), shift_x(3, 1))),
        "cinc_qutrits_ctrl_H": cyc(qutrits[:3], lambda t, i: Gate(t, (qutrits[(qutrits.index(t) + 1) % 3],), (2,), shift_x(3, 1))),
        "cinc_qutrits_ctrl_low": cyc(qutrits[:3], lambda t, i: Gate(t, (0,), (4,), shift_x(3, 1))),
        "phase_qutrits_H": cyc(qutrits[:3], lambda t, i: Gate(t, (), (), clock_z(3))),
    }
    st = P.State(dims)
    st.set_option(P.sv.SV_OPT_PASS_MERGE, 0)       # one application per listed gate
    ext = torch.cuda.ExternalStream(st.info().cuda_stream)
    for name, gates in mixes.items():
        if args.only and name not in args.only.split(","):
            continue
        ga = P.sv._GateArray(gates)
        T = sum(int(P.plan_gate(dims, g.target, g.U, g.ctrl, g.vals).touched) for g in gates)
        flop = 0
        for g in gates:
            p = P.plan_gate(dims, g.target, g.U, g.ctrl, g.vals)
            if int(p.kind) == 0:
                flop += 8 * int(p.d) * int(p.touched)
        st.reset(0)
        st.apply_circuit(ga, check=False, block=True)
        st.sync()
        n0 = st.info().kernel_launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        for _ in range(args.reps):
            st.apply_circuit(ga, check=False, block=True)
        e1.record(ext)
        st.sync()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        launches = (st.info().kernel_launches - n0) // args.reps
        per_gate = ms / len(gates)
        print(json.dumps({"mix": name, "D": D, "gates": len(gates), "launches": launches, "ms": ms,
                          "us_per_gate": 1e3 * per_gate,
                          "fp64_floor_us": 1e6 * flop / len(gates) / FP64,
                          "smem_floor_us": 1e6 * 32.0 * T / len(gates) / SMEM,
                          "hbm_state_us_per_gate": 1e6 * 32.0 * D * launches / len(gates) / 6.55e12}), flush=True)
    st.close()


if __name__ == "__main__":
    main()
