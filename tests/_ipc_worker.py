"""One rank of a multi-process sharded run over the IPC transport (sv_create_sharded_ipc),
driven by tests/test_gpu_ipc.py: every rank is its own process (one CUDA context each; on the
one-GPU test box all ranks share cuda:0).  Not a test module (no test_ prefix).

argv[1] = a pickle with the job: dims, gates, psi0 (or None for e_0), nranks, ipc_id, mode,
swap, dtype, extra (a second gate list applied after the first readback), and out (where rank
0 stores its results).  argv[2] = this rank.
"""
import os
import pickle
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    job = pickle.load(open(sys.argv[1], "rb"))
    rank = int(sys.argv[2])
    import paper_2410_17876_b200 as P
    dims, gates = job["dims"], job["gates"]
    res = {}
    dev = rank if job.get("device_per_rank") else 0
    st = P.State.sharded_ipc(dims, rank, job["nranks"], job["ipc_id"], device=dev, dtype=job.get("dtype", "c128"))
    try:
        st.set_option(P.sv.SV_OPT_SHARD_SWAP, job.get("swap", 1))
        st.set_option(P.sv.SV_OPT_SHARD_OVERLAP, job.get("overlap", 16))
        if job.get("psi0") is not None:
            st.set_amplitudes(0, job["psi0"])      # each rank writes the part it owns
        mode = job.get("mode", "block")
        if mode == "gate":
            for g in gates:
                st.apply_gate(g.target, g.U, g.ctrl, g.vals)
        else:
            st.apply_circuit(gates, fuse=mode == "fuse", block=mode == "block")
        res["norm"] = st.norm()                    # collective: partials in rank order
        if job.get("adjoint"):                     # full-size: circuit + adjoint back to e_0
            st.apply_circuit(job["adjoint"], fuse=mode == "fuse", block=mode == "block")
            D = st.info().D
            res["norm2"] = st.norm()
            res["head"] = st.amplitudes(0, 4096)
            res["tail"] = st.amplitudes(D - 4096, 4096)
        else:
            res["psi"] = st.amplitudes()           # collective: reads every slice
        res["exchanges"] = int(st.info().exchanges)
        res["overlapped"] = int(st.info().overlapped)
        if job.get("extra"):
            st.apply_circuit(job["extra"], block=True)
            res["psi_extra"] = st.amplitudes()
        st.sync()
    finally:
        st.close()                                 # collective: fences before freeing the slice
    if rank == 0:
        pickle.dump(res, open(job["out"], "wb"))
    print(f"rank {rank} ok", flush=True)


if __name__ == "__main__":
    main()
