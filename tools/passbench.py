"""Sweep the multi-gate pass kernel's configuration on a config circuit: one JSON line per
(tile, stages, threads, max gates) with ms per circuit and the number of launches."""
from __future__ import annotations

import argparse
import itertools
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--nqubits", type=int, default=None)
    ap.add_argument("--ngates", type=int, default=None)
    ap.add_argument("--tiles", default="4096,2048")
    ap.add_argument("--stages", default="3,2")
    ap.add_argument("--threads", default="512,256")
    ap.add_argument("--gates", default="24,8,4,2")
    ap.add_argument("--groups", default="1")
    ap.add_argument("--windows", default="64")
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"])
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--search", type=int, default=1, help="SV_OPT_PASS_SEARCH (in-tile set search)")
    ap.add_argument("--skip-noblock", action="store_true", help="do not time the single-gate mode")
    ap.add_argument("--low", type=int, default=32, help="SV_OPT_PASS_LOW (low-prefix stride threshold)")
    ap.add_argument("--absorb", type=int, default=1, help="SV_OPT_PASS_ABSORB (permutations as load / store relabelling)")
    ap.add_argument("--pass-kernel", type=int, default=0, help="SV_OPT_PASS_KERNEL: 0 per-gate, 1 register-blocked stages")
    args = ap.parse_args()
    import torch
    import paper_2410_17876_b200 as P
    from sv_inputs import config_circuit
    dims, gates = config_circuit(args.config, ngates=args.ngates, nqubits=args.nqubits)
    T = sum(int(P.plan_gate(dims, g.target, g.U, g.ctrl, g.vals).touched) for g in gates)
    D = int(np.prod(dims, dtype=object))
    st = P.State(dims, dtype=args.dtype)
    ext = torch.cuda.ExternalStream(st.info().cuda_stream)
    ga = P.sv._GateArray(gates)
    cases = [] if args.skip_noblock else [("noblock", 0, 0, 0, 0)]
    for te, s, nt, ng, gr, wi in itertools.product(*[[int(x) for x in a.split(",")] for a in
                                                     (args.tiles, args.stages, args.threads, args.gates, args.groups,
                                                      args.windows)]):
        if te * (16 if args.dtype == 'c128' else 8) * s > 210 * 1024 or (gr == 3 and nt % 96):
            continue
        cases.append(("block", te, s, nt, ng, gr, wi))
    for kind, te, s, nt, ng, *rest in cases:
        block = kind == "block"
        if block:
            st.set_option(P.sv.SV_OPT_PASS_TILE, te)
            st.set_option(P.sv.SV_OPT_PASS_STAGES, s)
            st.set_option(P.sv.SV_OPT_PASS_THREADS, nt)
            st.set_option(P.sv.SV_OPT_PASS_GATES, ng)
            st.set_option(P.sv.SV_OPT_PASS_GROUPS, rest[0])
            st.set_option(P.sv.SV_OPT_PASS_WINDOW, rest[1])
            st.set_option(P.sv.SV_OPT_PASS_SEARCH, args.search)
            st.set_option(P.sv.SV_OPT_PASS_KERNEL, args.pass_kernel)
            st.set_option(P.sv.SV_OPT_PASS_LOW, args.low)
            if args.absorb >= 0:
                st.set_option(P.sv.SV_OPT_PASS_ABSORB, args.absorb)
        st.reset(0)
        st.apply_circuit(ga, fuse=True, check=False, block=block)
        st.sync()
        n0 = st.info().kernel_launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        for _ in range(args.reps):
            st.apply_circuit(ga, fuse=True, check=False, block=block)
        e1.record(ext)
        st.sync()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        launches = (st.info().kernel_launches - n0) // args.reps
        print(json.dumps({"config": args.config, "D": D, "gates": len(gates), "mode": kind, "tile": te,
                          "stages": s, "threads": nt, "groups": rest[0] if rest else 0, "window": rest[1] if rest else 0, "max_gates": ng, "pass_kernel": args.pass_kernel, "absorb": args.absorb, "ms": ms, "launches": launches,
                          "updates_per_s": T / (ms / 1e3), "equiv_GBps": 32.0 * T / (ms / 1e3) / 1e9,
                          "pass_GBps": 32.0 * D * launches / (ms / 1e3) / 1e9}), flush=True)
    st.close()


if __name__ == "__main__":
    main()
