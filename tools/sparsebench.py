"""Sparse GHZ benchmark at the paper's maxima (62 qubits ~0.15 ms, 39 qutrits
0.188 ms, 31 ququads 0.2 ms, 27 ququints ~0.21 ms on an i5-1135G7): wall time per GHZ circuit
through the C ABI (sv_sparse_reset + sv_sparse_apply_circuit + sv_sparse_nnz), median of reps,
plus the oracle O-3 (Python dict) on the same circuit."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2410_17876_b200 as P
    from oracle import sparse as O3
    from sv_inputs import ghz_circuit
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    paper = {(2, 62): 0.15, (3, 39): 0.188, (4, 31): 0.2, (5, 27): 0.21}
    for (d, n), pms in paper.items():
        dims, gates = ghz_circuit(d, n)
        ga = P.sv._GateArray(gates)
        with P.sv.SparseState(dims) as st:
            for _ in range(5):
                st.reset(0)
                st.apply_circuit(ga, check=False)
                st.nnz()
            ts = []
            l0 = st.launches()
            for _ in range(reps):
                t0 = time.perf_counter()
                st.reset(0)
                st.apply_circuit(ga, check=False)
                nnz = st.nnz()
                ts.append(time.perf_counter() - t0)
            launches = (st.launches() - l0) / reps
            idx, amp = st.entries()
        t0 = time.perf_counter()
        ref = O3.run(dims, gates)
        t_or = time.perf_counter() - t0
        ok = sorted(ref) == [int(i) for i in idx] and all(abs(ref[int(i)] - a) < 1e-15 for i, a in zip(idx, amp))
        print(json.dumps({"d": d, "n": n, "gates": len(gates), "nnz": nnz, "median_ms": 1e3 * float(np.median(ts)),
                          "p10_ms": 1e3 * float(np.percentile(ts, 10)), "launches_per_circuit": launches,
                          "paper_ms_i5_1135G7": pms, "oracle_py_ms": 1e3 * t_or, "matches_oracle": ok}), flush=True)


if __name__ == "__main__":
    main()
