"""Per-gate microbenchmark: every target qudit of a config register x {general (Haar),
controlled increment, phase} x kernel family, timed with CUDA events on the library stream.
Prints one JSON line per case: algorithmic GB/s = 32 B x touched / time."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--nqubits", type=int, default=None)
    ap.add_argument("--kernels", default="1,2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--kinds", default="haar,cinc,phase")
    ap.add_argument("--targets", default=None)
    ap.add_argument("--te", type=int, default=None)
    ap.add_argument("--stages", type=int, default=None)
    ap.add_argument("--cps", type=int, default=None)
    args = ap.parse_args()
    import torch
    import paper_2410_17876_b200 as P
    from sv_inputs import config_circuit, haar_unitary, shift_x, phase_gate
    dims = config_circuit(args.config, ngates=0, nqubits=args.nqubits)[0]
    n = len(dims)
    rng = np.random.default_rng(0)
    st = P.State(dims)
    ext = torch.cuda.ExternalStream(st.info().cuda_stream)
    targets = range(n) if args.targets is None else [int(x) for x in args.targets.split(",")]
    if args.te:
        st.set_option(P.sv.SV_OPT_TILE_ELEMS, args.te)
    if args.stages:
        st.set_option(P.sv.SV_OPT_TILE_STAGES, args.stages)
    if args.cps:
        st.set_option(P.sv.SV_OPT_CTAS_PER_SM, args.cps)
    for kernel in [int(k) for k in args.kernels.split(",")]:
        st.set_option(P.sv.SV_OPT_KERNEL, kernel)
        for t in targets:
            d = dims[t]
            for kind in args.kinds.split(","):
                ctrl, vals = (), ()
                if kind == "pair":           # two gates on (t, t+1) fused into one d_t*d_{t+1} launch
                    if t + 1 >= n or dims[t] * dims[t + 1] > 16:
                        continue
                    from sv_inputs import Gate
                    pair = [Gate(t, (), (), haar_unitary(d, rng)), Gate(t + 1, (), (), haar_unitary(dims[t + 1], rng))]
                    ga = P.sv._GateArray(pair)
                    st.apply_circuit(ga, fuse=True)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    st.sync()
                    e0.record(ext)
                    for _ in range(args.reps):
                        st.apply_circuit(ga, fuse=True, check=False)
                    e1.record(ext)
                    st.sync()
                    ms = e0.elapsed_time(e1) / args.reps
                    T = int(np.prod(dims, dtype=object))
                    print(json.dumps({"config": args.config, "kernel": kernel, "te": args.te, "stages": args.stages,
                                      "cps": args.cps, "target": t, "d": d * dims[t + 1],
                                      "b": int(np.prod(dims[:t], dtype=object)), "kind": "pair", "ctrl": [],
                                      "touched": T, "ms": ms, "GBps": 32.0 * T / (ms / 1e3) / 1e9}), flush=True)
                    continue
                if kind == "haar":
                    U = haar_unitary(d, rng)
                elif kind == "phase":
                    U = phase_gate(rng.uniform(0, 6, size=d))
                else:
                    c = (t + 1) % n if t != n - 1 else 0
                    U, ctrl, vals = shift_x(d, 1), (c,), (dims[c] - 1,)
                T = P.plan_gate(dims, t, U, ctrl, vals).touched
                st.apply_gate(t, U, ctrl, vals)          # warm
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                st.sync()
                e0.record(ext)
                for _ in range(args.reps):
                    st.apply_gate(t, U, ctrl, vals)
                e1.record(ext)
                st.sync()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / args.reps
                print(json.dumps({"config": args.config, "kernel": kernel, "te": args.te, "stages": args.stages, "cps": args.cps, "target": t, "d": d,
                                  "b": int(np.prod(dims[:t], dtype=object)), "kind": kind,
                                  "ctrl": list(ctrl), "touched": int(T), "ms": ms,
                                  "GBps": 32.0 * T / (ms / 1e3) / 1e9}), flush=True)
    st.close()


if __name__ == "__main__":
    main()
