"""Sharded mode on one GPU through the loopback transport (all P slices on this device, device
copies instead of NCCL): ms per circuit for P = 1 (plain state) and P = 2/4/8, the same circuit
and driver flags as bench.py.  A proxy for the per-GPU work of an N-GPU run: each slice runs the
local passes its rank would, exchanges become device copies."""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--nqubits", type=int, default=None)
    ap.add_argument("--block", type=int, default=1)
    ap.add_argument("--swap", type=int, default=1, help="SV_OPT_SHARD_SWAP: qubit remapping (1) or exchange (0)")
    ap.add_argument("--overlap", type=int, default=16, help="SV_OPT_SHARD_OVERLAP: SMs lent to overlapped remaps (0 off)")
    args = ap.parse_args()
    import torch
    import paper_2410_17876_b200 as P
    from sv_inputs import config_circuit
    dims, gates = config_circuit(args.config, nqubits=args.nqubits)
    ga = P.sv._GateArray(gates)
    for nr in [int(x) for x in args.ranks.split(",")]:
        st = P.State(dims) if nr == 1 else P.State.loopback(dims, nr)
        if nr > 1:
            st.set_option(P.sv.SV_OPT_SHARD_SWAP, args.swap)
            st.set_option(P.sv.SV_OPT_SHARD_OVERLAP, args.overlap)
        ext = torch.cuda.ExternalStream(st.info().cuda_stream)
        st.reset(0)
        st.apply_circuit(ga, fuse=True, check=False, block=bool(args.block))
        st.sync()
        x0, o0 = st.info().exchanges, st.info().overlapped
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        for _ in range(args.reps):
            st.reset(0)
            st.apply_circuit(ga, fuse=True, check=False, block=bool(args.block))
        e1.record(ext)
        st.sync()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        print(json.dumps({"config": args.config, "ranks": nr, "swap": args.swap, "overlap": args.overlap,
                          "overlapped_per_circuit": (st.info().overlapped - o0) / args.reps, "ms_per_circuit": ms,
                          "ms_per_rank_slice": ms / nr,
                          "exchanges_per_circuit": (st.info().exchanges - x0) / args.reps}), flush=True)
        st.close()


if __name__ == "__main__":
    main()
