"""Small invocations of every synchronising kernel of the path, for compute-sanitizer
(racecheck / synccheck / memcheck, one tool per run):

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py

  * k_gate_pass (per-gate multi-gate passes: mbarrier ring, consumer groups, named barriers)
    for consumer groups 1 / 2 / 4 and ring stages 2..4, full and ragged tiles, in-tile and
    run-digit controls;
  * k_gate_stage (register-blocked stages) with 1 and 2 groups;
  * k_gate_tiled (single-gate TMA tiles, modes N and W) and k_gate_direct;
  * the loopback peer kernels (fused exchange k_pair_update, qubit swap k_pair_swap);
  * the sparse small-state kernel.
Registers are tiny (sanitizers slow kernels down by 100-1000x).  Every case is also checked
against the oracle so a run that completes is a parity run too.  Exits non-zero on a mismatch.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2410_17876_b200 as P
    from oracle import blocksim as O2
    from oracle import sparse as O3
    from sv_inputs import random_circuit, random_state, ghz_circuit, Gate, hadamard, haar_unitary

    S = P.sv
    fails = 0

    def check(name, got, ref, tol=1e-11):
        nonlocal fails
        err = float(np.max(np.abs(got - ref)))
        ok = err <= tol
        fails += 0 if ok else 1
        print(f"{name}: max|d| = {err:.2e} {'ok' if ok else 'FAIL'}", flush=True)

    dims = [3, 2, 4, 2, 3, 2, 2]                      # D = 1152: several tiles of 256 amplitudes
    D = int(np.prod(dims))
    _, gates = random_circuit(4242, dims, 40, max_ctrl=2)
    psi0 = random_state(D, 1)
    ref = O2.run(dims, gates, psi0)
    # per-gate pass kernel: (threads, groups, stages)
    for nt, g, s in ((256, 1, 2), (512, 2, 3), (512, 4, 4), (384, 2, 2)):
        with P.State(dims) as st:
            st.set_option(S.SV_OPT_PASS_KERNEL, 0)
            st.set_option(S.SV_OPT_PASS_TILE, 256)
            st.set_option(S.SV_OPT_PASS_THREADS, nt)
            st.set_option(S.SV_OPT_PASS_GROUPS, g)
            st.set_option(S.SV_OPT_PASS_STAGES, s)
            st.set_amplitudes(0, psi0)
            st.apply_circuit(gates, block=True)
            check(f"k_gate_pass nt={nt} groups={g} stages={s}", st.amplitudes(), ref)
    for nt, g in ((256, 1), (384, 2)):
        with P.State(dims) as st:
            st.set_option(S.SV_OPT_PASS_KERNEL, 1)
            st.set_option(S.SV_OPT_PASS_TILE, 256)
            st.set_option(S.SV_OPT_PASS_THREADS, nt)
            st.set_option(S.SV_OPT_PASS_GROUPS, g)
            st.set_amplitudes(0, psi0)
            st.apply_circuit(gates, block=True)
            check(f"k_gate_stage nt={nt} groups={g}", st.amplitudes(), ref)
    for kern in (1, 2):                               # direct, tiled (single-gate kernels)
        with P.State(dims) as st:
            st.set_option(S.SV_OPT_KERNEL, kern)
            st.set_option(S.SV_OPT_TILE_ELEMS, 256)
            st.set_amplitudes(0, psi0)
            st.apply_circuit(gates)
            check(f"single-gate kernel {kern}", st.amplitudes(), ref)
    # loopback peer kernels: exchanges (remapping off) and qubit swaps (on)
    sdims = [3, 2, 2, 2, 2, 2]
    rng = np.random.default_rng(3)
    sg = [Gate(5, (), (), hadamard()), Gate(4, (0,), (1,), haar_unitary(2, rng)), Gate(1, (5,), (1,), hadamard()),
          Gate(5, (1,), (0,), haar_unitary(2, rng))]
    sp0 = random_state(int(np.prod(sdims)), 2)
    sref = O2.run(sdims, sg, sp0)
    for swap in (0, 1):
        with P.State.loopback(sdims, 4) as st:
            st.set_option(S.SV_OPT_SHARD_SWAP, swap)
            st.set_amplitudes(0, sp0)
            st.apply_circuit(sg, block=True)
            check(f"loopback peer kernels swap={swap}", st.amplitudes(), sref)
    # sparse small-state kernel: GHZ_3 on 6 qutrits
    gd, gg = ghz_circuit(3, 6)
    with P.sv.SparseState(gd) as sst:
        sst.apply_circuit(gg)
        idx, amp = sst.entries()
    ref3 = O3.run(gd, gg)
    got = dict(zip([int(i) for i in idx], amp))
    err = max(abs(got.get(i, 0) - a) for i, a in ref3.items())
    fails += 0 if err <= 1e-12 else 1
    print(f"sparse GHZ_3: max|d| = {err:.2e} {'ok' if err <= 1e-12 else 'FAIL'}", flush=True)
    print("sanitize cases:", "FAIL" if fails else "all ok", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
