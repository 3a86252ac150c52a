"""Host-side tests of the C-ABI library (no GPU needed): the library loads and exports every
symbol include/sv.h declares; validation, classification, the fibre decomposer, the fusion
planner and the shard planner are checked against independent definitions / the oracle."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2410_17876_b200 as P
from paper_2410_17876_b200 import sv as S
from oracle import blocksim as O2
from sv_inputs import (Gate, shift_x, clock_z, fourier, hadamard, t_gate, haar_unitary,
                       permutation_matrix, phase_gate, random_circuit, random_state, config_circuit)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "sv.h")).read()
    declared = set(re.findall(r"^SV_API\s+[^(]*?\b(sv_\w+)\s*\(", hdr, flags=re.M))
    assert len(declared) >= 20
    out = subprocess.check_output(["nm", "-D", "--defined-only", S.LIB_PATH]).decode()
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert declared <= exported, declared - exported
    assert set(S.EXPORTS) == declared
    assert "sm_100a" in P.sv.version()


def test_library_is_sm100a_only():
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", S.LIB_PATH]).decode()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def _err(fn, *a, **k):
    with pytest.raises(P.SVError) as e:
        fn(*a, **k)
    return e.value.name


def test_register_validation_before_device_work():
    assert _err(P.State, [2, 1]) == "SV_ERR_DIM"
    assert _err(P.State, [2, 17]) == "SV_ERR_DIM"
    assert _err(P.State, []) == "SV_ERR_DIM"
    assert _err(P.State, [2] * 65) == "SV_ERR_DIM"
    assert _err(P.plan_gate, [16] * 16 + [2], 0, np.eye(16)) == "SV_ERR_OVERFLOW"


def test_gate_validation_codes():
    dims = [2, 3, 4]
    H = hadamard()
    assert _err(P.plan_gate, dims, 3, H) == "SV_ERR_QUDIT_RANGE"
    assert _err(P.plan_gate, dims, 0, H, ctrl=[0], vals=[1]) == "SV_ERR_CTRL_OVERLAP"
    assert _err(P.plan_gate, dims, 0, H, ctrl=[1, 1], vals=[0, 0]) == "SV_ERR_CTRL_DUP"
    assert _err(P.plan_gate, dims, 0, H, ctrl=[1], vals=[3]) == "SV_ERR_CTRL_VALUE"
    assert _err(P.plan_gate, dims, 0, H, ctrl=[5], vals=[0]) == "SV_ERR_QUDIT_RANGE"
    p = P.plan_gate(dims, 0, np.array([[1, 0], [0, 2]], complex))
    assert abs(p.unitarity_err - 3.0) < 1e-15          # |4 - 1|


def test_classification_and_touched_counts():
    dims = [2, 3, 4, 5]
    D = 120
    # permutation X_{+1} on q2 (d=4): monomial, sigma = j+1, every member moves
    p = P.plan_gate(dims, 2, shift_x(4, 1))
    assert p.kind == 1 and list(p.sigma[:4]) == [1, 2, 3, 0] and p.active_mask == 0b1111
    assert p.fibres == D // 4 and p.touched == D and p.b == 6
    # clock Z_3 on q1: diagonal; member 0 has phase exactly 1 -> untouched (T = D (d-1)/d)
    p = P.plan_gate(dims, 1, clock_z(3, 1))
    assert p.kind == 1 and p.active_mask == 0b110 and p.touched == D * 2 // 3
    # T gate on a qubit: only the |1> block
    p = P.plan_gate(dims, 0, t_gate())
    assert p.kind == 1 and p.active_mask == 0b10 and p.touched == D // 2
    # general gates
    assert P.plan_gate(dims, 3, fourier(5)).kind == 0
    assert P.plan_gate(dims, 3, haar_unitary(5, np.random.default_rng(0))).kind == 0
    # CINC qubit->ququint: fibres D/(5*2), touched D/2
    p = P.plan_gate(dims, 3, shift_x(5, 1), ctrl=[0], vals=[1])
    assert p.fibres == D // 10 and p.touched == D // 2
    # identity: nothing to do
    assert P.plan_gate(dims, 1, np.eye(3)).fibres == 0
    # monomial with phases (Y-like) is still monomial: y_{sigma(j)} = c_j x_j
    Y = np.array([[0, -1j], [1j, 0]])
    assert P.plan_gate(dims, 0, Y).kind == 1


def _brute_bases(dims, target, ctrl, vals):
    D = int(np.prod(dims))
    i = np.arange(D)
    digits, rest = [], i.copy()
    for d in dims:
        digits.append(rest % d)
        rest //= d
    ok = digits[target] == 0
    for c, v in zip(ctrl, vals):
        ok &= digits[c] == v
    return i[ok]


def test_fibre_decomposer_matches_brute_force():
    """digit insertion yields exactly the satisfying class representatives,
    in ascending order, for random registers and up to 3 controls (incl. adjacent runs)."""
    rng = np.random.default_rng(123)
    for trial in range(300):
        n = int(rng.integers(1, 7))
        dims = [int(x) for x in rng.integers(2, 7, size=n)]
        while np.prod(dims) > 20000:
            dims = dims[:-1]
        n = len(dims)
        t = int(rng.integers(n))
        others = [q for q in range(n) if q != t]
        nc = int(rng.integers(0, min(3, len(others)) + 1))
        ctrl = [int(c) for c in rng.choice(others, size=nc, replace=False)] if nc else []
        vals = [int(rng.integers(dims[c])) for c in ctrl]
        got = P.enumerate_fibres(dims, t, ctrl, vals)
        exp = _brute_bases(dims, t, ctrl, vals)
        assert np.array_equal(got.astype(np.int64), exp), (dims, t, ctrl, vals)


def test_fibre_decomposer_64bit_offsets():
    """Class ids beyond 2^32 on the c4 register (D = 4.78e9): spot-check against the digits."""
    dims = config_circuit(4, ngates=0)[0]
    b = np.cumprod([1] + dims[:-1]).astype(object)
    for t, ctrl, vals in ((0, [], []), (21, [3], [2]), (7, [0, 21], [4, 1]), (12, [13, 14], [1, 0])):
        F = int(np.prod(dims, dtype=object)) // (dims[t] * int(np.prod([dims[c] for c in ctrl], dtype=object)))
        for first in (0, F // 3, F - 5):
            got = P.enumerate_fibres(dims, t, ctrl, vals, first=first, count=5)
            for x in got:
                x = int(x)
                dg = [(x // int(b[k])) % dims[k] for k in range(len(dims))]
                assert dg[t] == 0 and all(dg[c] == v for c, v in zip(ctrl, vals))
            if first == F - 5 and t != 21:
                assert int(got[-1]) > 2 ** 32            # representatives need 64-bit math


def _merged_apply(psi, dims, fused):
    """Apply one fused gate with the oracle: a span-2 gate on (k, k+1) is a single-qudit gate
    on the register whose qudits k and k+1 are merged into one digit of dim d_k d_{k+1}
    (same memory layout: stride b_k, digit j_k + d_k j_{k+1})."""
    t, span, k, ctrl, vals, U = fused
    if span == 1:
        O2.apply(psi, dims, Gate(t, ctrl, vals, U))
        return
    md = dims[:t] + [dims[t] * dims[t + 1]] + dims[t + 2:]
    mc = tuple(c if c < t else c - 1 for c in ctrl)
    O2.apply(psi, md, Gate(t, mc, vals, U))


def test_fusion_planner_preserves_the_circuit():
    rng = np.random.default_rng(31)
    for s in range(25):
        dims = [int(x) for x in rng.integers(2, 5, size=5)]
        _, gates = random_circuit(500 + s, dims, 40, max_ctrl=1)
        # add same-qudit and adjacent runs so fusion actually fires
        extra = []
        for g in gates:
            extra.append(g)
            if rng.random() < 0.5 and g.target + 1 < len(dims) and (g.target + 1) not in g.ctrl:
                extra.append(Gate(g.target + 1, g.ctrl, g.vals, haar_unitary(dims[g.target + 1], rng)))
        gates = extra
        fused = P.fuse_plan(dims, gates)
        assert len(fused) < len(gates)
        assert all(f[2] <= 16 for f in fused)
        psi0 = random_state(int(np.prod(dims)), 900 + s)
        ref = O2.run(dims, gates, psi0)
        got = psi0.copy()
        for f in fused:
            _merged_apply(got, dims, f)
        assert np.max(np.abs(got - ref)) < 1e-13


def test_shard_plan_rules():
    """sharded controls -> rank predicate; sharded target -> partner r^2^j."""
    dims = [3, 3, 2, 2, 2, 2]          # P = 4 shards on q_4, q_5
    P_ = 4
    for r in range(P_):
        assert P.shard_plan(dims, P_, r, 0) == (0, r, 0)
        a, p, b = P.shard_plan(dims, P_, r, 4)
        assert a == 2 and p == r ^ 1 and b == (r & 1)
        a, p, b = P.shard_plan(dims, P_, r, 5)
        assert a == 2 and p == r ^ 2 and b == (r >> 1) & 1
        a, _, _ = P.shard_plan(dims, P_, r, 1, ctrl=[5], vals=[1])
        assert a == (0 if (r >> 1) & 1 == 1 else 1)
        a, p, _ = P.shard_plan(dims, P_, r, 4, ctrl=[5, 0], vals=[0, 2])
        assert a == (2 if (r >> 1) & 1 == 0 else 1)
    assert _err(P.shard_plan, [3, 3, 3], 2, 0, 0) == "SV_ERR_UNSUPPORTED"   # top digit not a qubit
    assert _err(P.shard_plan, dims, 3, 0, 0) == "SV_ERR_INVALID_ARG"


def test_block_planner_reorders_only_commuting_gates():
    """SV_BLOCK's pass planner: applying the gates in its order (O-2) reproduces the original
    circuit; every pass's tile fits the cap; the planner actually groups gates."""
    rng = np.random.default_rng(77)
    for cfg, nq in ((4, 2), (3, 5), (2, None), (1, None)):
        dims, gates = config_circuit(cfg, nqubits=nq) if cfg in (3, 4) else config_circuit(cfg)
        gates = gates[:120]
        for cap in (4096, 2048):
            order, pid, tiles = P.block_plan(dims, gates, cap)
            assert sorted(order.tolist()) == list(range(len(gates)))
            assert all(t <= cap for t in tiles) or len(tiles) == len(gates)
            assert len(tiles) < len(gates)          # grouping happened
            assert np.all(np.diff(pid) >= 0)
            D = int(np.prod(dims))
            if D > 2_000_000:
                continue
            psi0 = random_state(D, 5)
            ref = O2.run(dims, gates, psi0)
            got = O2.run(dims, [gates[i] for i in order], psi0)
            assert np.max(np.abs(got - ref)) < 1e-12
    # random circuits with controls everywhere
    for s in range(30):
        dims = [int(x) for x in rng.integers(2, 6, size=6)]
        _, gates = random_circuit(800 + s, dims, 60, max_ctrl=2)
        order, pid, tiles = P.block_plan(dims, gates, 256)
        psi0 = random_state(int(np.prod(dims)), s)
        ref = O2.run(dims, gates, psi0)
        got = O2.run(dims, [gates[i] for i in order], psi0)
        assert np.max(np.abs(got - ref)) < 1e-12


def test_block_planner_subset_search_pass_count():
    """The in-tile set search (plan.cpp best_in_tile_set): on the full c4 circuit after merging,
    the pass count stays at or below the searched plan's 23 (first-come admission: 30 at this
    window), and every tile fits."""
    from sv_inputs import Gate
    dims, gates = config_circuit(4)
    merged = [Gate(t, c, v, U) for (t, sp, k, c, v, U) in P.merge_plan(dims, gates, 64)]
    order, pid, tiles = P.block_plan(dims, merged, 4096)
    assert sorted(order.tolist()) == list(range(len(merged)))
    assert len(tiles) <= 23
    assert all(t <= 4096 for t in tiles)


def test_merge_planner_preserves_the_circuit():
    """The SV_BLOCK pre-pass (sv_merge_plan): gates move back across gates they commute with and
    merge with an earlier same-target, same-control gate.  The merged list must give the same
    state as the original (O-2), and must merge where the commutation rules allow it."""
    from sv_inputs import t_gate, hadamard
    rng = np.random.default_rng(41)
    for s in range(30):
        dims = [int(x) for x in rng.integers(2, 5, size=5)]
        _, gates = random_circuit(700 + s, dims, 50, max_ctrl=2)
        # diagonal gates and repeats so the diagonal rules and merges fire
        extra = []
        for g in gates:
            extra.append(g)
            r = rng.random()
            if r < 0.25:
                extra.append(Gate(g.target, (), (), np.diag(np.exp(1j * rng.random(dims[g.target])))))
            elif r < 0.5:
                extra.append(Gate(g.target, g.ctrl, g.vals, haar_unitary(dims[g.target], rng)))
        gates = extra
        merged = P.merge_plan(dims, gates, 64)
        assert len(merged) < len(gates)
        assert all(m[1] == 1 for m in merged)
        psi0 = random_state(int(np.prod(dims)), 300 + s)
        ref = O2.run(dims, gates, psi0)
        got = psi0.copy()
        for m in merged:
            _merged_apply(got, dims, m)
        assert np.max(np.abs(got - ref)) < 1e-13


def test_merge_planner_commutation_rules():
    """Closed cases: H on q0, CNOT(q1 -> q2), H on q0 merges (disjoint); T on q1 passes a gate
    controlled on q1 (diagonal); a non-diagonal gate on q1 does not; same-digit diagonals commute."""
    from sv_inputs import t_gate, hadamard, shift_x
    dims = [2, 2, 2]
    H, T, X = hadamard(), t_gate(), shift_x(2, 1)
    cnot = Gate(2, (1,), (1,), X)
    m = P.merge_plan(dims, [Gate(0, (), (), H), cnot, Gate(0, (), (), H)])
    assert len(m) == 2 and np.allclose(m[0][5], np.eye(2))          # H H = I merged past the CNOT
    m = P.merge_plan(dims, [Gate(1, (), (), T), cnot, Gate(1, (), (), T)])
    assert len(m) == 2 and np.allclose(m[0][5], T @ T)              # T commutes with a control on q1
    m = P.merge_plan(dims, [Gate(1, (), (), H), cnot, Gate(1, (), (), H)])
    assert len(m) == 3                                              # H does not
    Z = np.diag([1.0, -1.0]).astype(np.complex128)
    m = P.merge_plan(dims, [Gate(1, (), (), T), Gate(1, (0,), (1,), Z), Gate(1, (), (), T)])
    assert len(m) == 2                                              # diagonals on one digit commute
    m = P.merge_plan(dims, [Gate(0, (), (), H), cnot, Gate(0, (), (), H)], window=1)
    assert len(m) == 3                                              # the window bounds the scan


def test_bench_reference_arm_line():
    """bench.py --impl reference (the oracle timed on the host, the tier's reference arm) prints
    one JSON line with the contract's keys; the config names the full c4 workload."""
    import json
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                         cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1
    assert d["config"]["dims_q0_first"] == [5, 5, 4, 4, 4, 4] + [3] * 6 + [2] * 10
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["host"]["nproc"] >= 1


def test_bench_reference_arm_does_not_load_the_product():
    """The oracle arms count work with oracle/work.py: the reference-arm process maps the
    oracle's library and never the product's libsv.so."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','1'];"
            "runpy.run_path('bench.py', run_name='__main__');"
            "maps=open('/proc/self/maps').read(); print('LIBSV' if 'libsv.so' in maps else 'NOLIBSV');"
            "print('PKG' if 'paper_2410_17876_b200' in sys.modules else 'NOPKG')")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "NOLIBSV" in out.stdout and "NOPKG" in out.stdout, out.stdout[-500:]


def test_block_planner_order_is_equivalent():
    """sv_block_plan (the SV_BLOCK pass planner): gates are pulled into a pass only past gates
    they commute with, so applying them in the planner's order gives the same state (O-2) —
    with diagonal gates, whose commutation with gates controlled on their digit the planner
    uses (R19).  Every gate appears exactly once and pass ids are non-decreasing."""
    rng = np.random.default_rng(77)
    for s in range(20):
        dims = [int(x) for x in rng.integers(2, 5, size=6)]
        _, gates = random_circuit(900 + s, dims, 60, max_ctrl=2)
        extra = []
        for g in gates:
            extra.append(g)
            if rng.random() < 0.3:
                t = int(rng.integers(len(dims)))
                extra.append(Gate(t, (), (), np.diag(np.exp(1j * rng.random(dims[t])))))
        gates = extra
        order, pid, tiles = P.block_plan(dims, gates, 256)
        assert sorted(order.tolist()) == list(range(len(gates)))
        assert all(np.diff(pid) >= 0)
        psi0 = random_state(int(np.prod(dims)), 1000 + s)
        ref = O2.run(dims, gates, psi0)
        got = O2.run(dims, [gates[i] for i in order], psi0)
        assert np.max(np.abs(got - ref)) < 1e-13


def test_bench_reference_arm_under_torchrun():
    """The driver launches N > 1 through torch.distributed.run; for the reference arm rank 0
    alone runs and prints one JSON line, the other ranks exit 0 without work."""
    import json
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_oracle_work_count_matches_planner_and_closed_forms():
    """The metric's work count T has two independent implementations: the
    product planner (sv_plan_gate, used by bench.py's GPU arm) and oracle/work.py (used by the
    oracle arms, which must not load the product).  Pinned by closed forms, then equal on every
    gate of every config circuit."""
    from oracle import work as W
    dims = [5, 4, 3, 2, 2]
    D = int(np.prod(dims))
    assert W.touched(dims, Gate(2, (), (), haar_unitary(3, np.random.default_rng(1)))) == D
    assert W.touched(dims, Gate(1, (), (), shift_x(4, 1))) == D                   # X_d: every member
    assert W.touched(dims, Gate(0, (), (), clock_z(5))) == D * 4 // 5             # Z_d: j = 0 fixed
    assert W.touched(dims, Gate(4, (), (), t_gate())) == D // 2                    # T: |0> fixed
    assert W.touched(dims, Gate(2, (3,), (1,), shift_x(3, 1))) == D // 2           # CINC: D / d_c
    assert W.touched(dims, Gate(0, (1, 3), (3, 0), haar_unitary(5, np.random.default_rng(2)))) == D // 8
    assert W.touched(dims, Gate(3, (), (), np.eye(2))) == 0
    for cfg in (1, 2, 3, 4, 5):
        cd, gates = config_circuit(cfg, ngates=None if cfg != 2 else 600)
        for g in gates:
            assert W.touched(cd, g) == int(P.plan_gate(cd, g.target, g.U, g.ctrl, g.vals).touched), (cfg, g)
