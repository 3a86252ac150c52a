"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Tolerances (north_star): max |dpsi| <= 1e-10 and | ||psi|| - 1 | <= 1e-10 on normalised
states; bit-exact (==) for index mappings (permutation-only circuits on an index-labelled
state).  Every case runs for each gate-kernel family (1 = direct per-class, 2 = TMA-tiled)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import blocksim as O2  # noqa: E402
from oracle import kron as O1  # noqa: E402
from _circuits import overlap_circuit as _overlap_circuit  # noqa: E402
from sv_inputs import (Gate, shift_x, clock_z, fourier, hadamard, t_gate, haar_unitary,  # noqa: E402
                       permutation_matrix, phase_gate, ghz_circuit, worked_example,
                       random_circuit, adjoint_circuit, labelled_state, random_state,
                       config_circuit)

KERNELS = [1, 2]


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2410_17876_b200 as P
    return P


def run_gpu(P, dims, gates, psi0=None, kernel=0, fuse=False, graph=False, per_gate=False, block=False,
            pass_tile=None, pass_cfg=None, pass_kernel=0):
    with P.State(dims) as st:
        st.set_option(P.sv.SV_OPT_KERNEL, kernel)
        st.set_option(P.sv.SV_OPT_PASS_KERNEL, pass_kernel)
        if pass_tile:
            st.set_option(P.sv.SV_OPT_PASS_TILE, pass_tile)
        if pass_cfg:
            threads, groups, stages = pass_cfg
            st.set_option(P.sv.SV_OPT_PASS_THREADS, threads)
            st.set_option(P.sv.SV_OPT_PASS_GROUPS, groups)
            st.set_option(P.sv.SV_OPT_PASS_STAGES, stages)
        if psi0 is not None:
            st.set_amplitudes(0, psi0)
        n0 = st.info().kernel_launches
        if per_gate:
            for g in gates:
                st.apply_gate(g.target, g.U, g.ctrl, g.vals)
        else:
            st.apply_circuit(gates, fuse=fuse, graph=graph, block=block)
        out = st.amplitudes()
        nrm = st.norm()
        launched = st.info().kernel_launches - n0
    return out, nrm, launched


@pytest.mark.parametrize("kernel", KERNELS)
def test_worked_example(P, kernel):
    dims, gates = worked_example()
    got, nrm, _ = run_gpu(P, dims, gates, kernel=kernel)
    s = 1.0 / np.sqrt(3.0)
    exp = np.zeros(6, complex)
    exp[[0, 2, 5]] = s
    assert np.max(np.abs(got - exp)) < 1e-15
    assert np.flatnonzero(got).tolist() == [0, 2, 5]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("d,n", [(2, 20), (3, 12), (4, 10), (5, 8), (7, 6), (16, 4)])
def test_ghz_exact(P, kernel, d, n):
    dims, gates = ghz_circuit(d, n)
    got, nrm, _ = run_gpu(P, dims, gates, kernel=kernel)
    rep = sum(d ** k for k in range(n))
    idx = [v * rep for v in range(d)]
    s = 1.0 / np.sqrt(d)
    assert np.flatnonzero(got).tolist() == idx
    assert all(got[i].real == s and got[i].imag == 0.0 for i in idx)
    assert abs(nrm - 1.0) <= 1e-10


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("mode", ["plain", "fuse", "graph", "per_gate", "block", "block_graph"])
def test_c1_against_kronecker(P, kernel, mode):
    dims, gates = config_circuit(1)
    ref = O1.run(dims, gates)
    got, nrm, launched = run_gpu(P, dims, gates, kernel=kernel, fuse=mode in ("fuse", "graph"),
                                 graph=mode in ("graph", "block_graph"), per_gate=mode == "per_gate",
                                 block=mode.startswith("block"))
    assert np.max(np.abs(got - ref)) <= 1e-10
    assert abs(nrm - 1.0) <= 1e-10
    assert launched > 0


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("fuse", [False, True, "block"])
def test_c2_against_blocksim(P, kernel, fuse):
    dims, gates = config_circuit(2)
    ref = O2.run(dims, gates)
    got, nrm, _ = run_gpu(P, dims, gates, kernel=kernel, fuse=fuse is True, graph=bool(fuse),
                          block=fuse == "block")
    assert np.max(np.abs(got - ref)) <= 1e-10
    assert abs(nrm - 1.0) <= 1e-10


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("block", [False, True])
def test_c3_reduced_register(P, kernel, block):
    dims, gates = config_circuit(3, nqubits=6)
    ref = O2.run(dims, gates)
    got, nrm, _ = run_gpu(P, dims, gates, kernel=kernel, fuse=True, block=block)
    assert np.max(np.abs(got - ref)) <= 1e-10
    assert abs(nrm - 1.0) <= 1e-10


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("block", [False, True])
def test_c4_reduced_register(P, kernel, block):
    dims, gates = config_circuit(4, nqubits=1)        # D = 9.3e6, every dimension class
    ref = O2.run(dims, gates)
    got, nrm, _ = run_gpu(P, dims, gates, kernel=kernel, block=block)
    assert np.max(np.abs(got - ref)) <= 1e-10
    assert abs(nrm - 1.0) <= 1e-10


# ------------------------------------------------ (dimension x stride x kind x controls)
REGISTERS = {
    # name: (dims, target) -> target stride b_k
    "b1": lambda d: ([d, 3, 4, 2, 5], 0),                 # b = 1
    "b5": lambda d: ([5, d, 3, 2, 4], 1),                 # b = 5 (odd, narrow)
    "b30": lambda d: ([5, 6, d, 3, 2], 2),                # b = 30 (narrow, < 32)
    "b64": lambda d: ([4, 16, d, 3, 5], 2),               # b = 64
    "b2304": lambda d: ([16, 16, 9, d, 3], 3),            # b = 2304 (wide, > tile)
    "top": lambda d: ([3, 16, 5, 7, d], 4),               # most significant, r = 1
}


def _gate_for(kind, d, rng):
    if kind == "haar":
        return haar_unitary(d, rng)
    if kind == "fourier":
        return fourier(d)
    if kind == "phase":
        return phase_gate(rng.uniform(0, 2 * np.pi, size=d))
    if kind == "perm":
        return permutation_matrix(rng.permutation(d))
    if kind == "clock":
        return clock_z(d, 1)
    raise ValueError(kind)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("reg", sorted(REGISTERS))
@pytest.mark.parametrize("d", [2, 3, 4, 5, 7, 16])
def test_kernel_matrix(P, kernel, reg, d):
    rng = np.random.default_rng(1000 + d)
    dims, t = REGISTERS[reg](d)
    n = len(dims)
    D = int(np.prod(dims))
    psi0 = random_state(D, 77 + d)
    others = [q for q in range(n) if q != t]
    below = [q for q in others if q < t]
    above = [q for q in others if q > t]
    ctrl_sets = [[]]
    if below:
        ctrl_sets.append([below[0]])
        ctrl_sets.append([below[-1]])                     # adjacent below
    if above:
        ctrl_sets.append([above[0]])                      # adjacent above
        ctrl_sets.append([above[-1]])
    if below and above:
        ctrl_sets.append([below[0], above[-1]])
    if len(others) >= 3:
        ctrl_sets.append(others[:3])
    with P.State(dims) as st:
        st.set_option(P.sv.SV_OPT_KERNEL, kernel)
        for kind in ("haar", "fourier", "phase", "perm", "clock"):
            for ctrl in ctrl_sets:
                vals = [int(rng.integers(dims[c])) for c in ctrl]
                U = _gate_for(kind, d, rng)
                st.set_amplitudes(0, psi0)
                st.apply_gate(t, U, ctrl, vals)
                got = st.amplitudes()
                ref = psi0.copy()
                O2.apply(ref, dims, Gate(t, tuple(ctrl), tuple(vals), U))
                err = np.max(np.abs(got - ref))
                assert err <= 1e-12, (kind, ctrl, vals, err)
                if kind in ("perm", "clock") or not ctrl:
                    pass
                # untouched classes are bit-exact
                if ctrl:
                    digits = [(np.arange(D) // int(np.prod(dims[:q]))) % dims[q] for q in ctrl]
                    off = np.ones(D, bool)
                    for dg, v in zip(digits, vals):
                        off &= dg == v
                    assert np.array_equal(got[~off], psi0[~off])


@pytest.mark.parametrize("kernel", KERNELS)
def test_fused_dimensions(P, kernel):
    """Adjacent-pair fusion produces every combined dimension 4..16 (2x2 ... 4x4, 3x5)."""
    rng = np.random.default_rng(5)
    for dims in ([2, 2, 3, 5, 4, 4, 3], [3, 3, 2, 4, 5, 2, 2], [4, 4, 2, 3, 3, 5]):
        D = int(np.prod(dims))
        gates = []
        for k in range(len(dims) - 1):
            gates.append(Gate(k, (), (), haar_unitary(dims[k], rng)))
            gates.append(Gate(k + 1, (), (), haar_unitary(dims[k + 1], rng)))
            c = (k + 3) % len(dims)
            if c not in (k, k + 1):
                gates.append(Gate(k, (c,), (1,), haar_unitary(dims[k], rng)))
                gates.append(Gate(k + 1, (c,), (1,), haar_unitary(dims[k + 1], rng)))
        psi0 = random_state(D, 3)
        ref = O2.run(dims, gates, psi0)
        fused = P.fuse_plan(dims, gates)
        assert len(fused) < len(gates)
        for graph in (False, True):
            got, _, _ = run_gpu(P, dims, gates, psi0, kernel=kernel, fuse=True, graph=graph)
            assert np.max(np.abs(got - ref)) <= 1e-12


@pytest.mark.parametrize("kernel", KERNELS)
def test_labelled_permutation_circuits_bit_exact(P, kernel):
    """Index mappings are bit-exact: X_d, CINC, CNOT, multi-controlled X on the labelled state,
    compared with == to O-2 and to the closed-form map i -> i + (sigma(v) - v) b_k."""
    rng = np.random.default_rng(17)
    for cfg in (1, 3, 4):
        dims = config_circuit(cfg, ngates=0, nqubits=3 if cfg in (3, 4) else None)[0]
        n, D = len(dims), int(np.prod(dims))
        gates = []
        for _ in range(60):
            t = int(rng.integers(n))
            others = [q for q in range(n) if q != t]
            nc = int(rng.integers(0, 4))
            ctrl = tuple(int(c) for c in rng.choice(others, size=nc, replace=False))
            vals = tuple(int(rng.integers(dims[c])) for c in ctrl)
            U = shift_x(dims[t], int(rng.integers(1, dims[t]))) if rng.random() < 0.6 else \
                permutation_matrix(rng.permutation(dims[t]))
            gates.append(Gate(t, ctrl, vals, U))
        psi0 = labelled_state(0, D)
        ref = O2.run(dims, gates, psi0)
        got, _, _ = run_gpu(P, dims, gates, psi0, kernel=kernel)
        assert np.array_equal(got, ref)
        # closed form for a single gate
        g = gates[0]
        one, _, _ = run_gpu(P, dims, [g], psi0, kernel=kernel)
        b = int(np.prod(dims[:g.target]))
        i = np.arange(D)
        dg = lambda q: (i // int(np.prod(dims[:q]))) % dims[q]
        ok = np.ones(D, bool)
        for c, v in zip(g.ctrl, g.vals):
            ok &= dg(c) == v
        sig = np.argmax(np.abs(g.U), axis=0)
        v = dg(g.target)
        dest = np.where(ok, i + (sig[v] - v) * b, i)
        exp = np.empty_like(psi0)
        exp[dest] = psi0
        assert np.array_equal(one, exp)


@pytest.mark.parametrize("kernel", KERNELS)
def test_random_sweep_against_kronecker(P, kernel):
    """SPEC.md:587-style sweep: seeded random circuits, n <= 4, dims 2..5, <= 2 controls."""
    rng = np.random.default_rng(2024)
    for s in range(60):
        n = int(rng.integers(1, 5))
        dims = [int(x) for x in rng.integers(2, 6, size=n)]
        _, gates = random_circuit(30_000 + s, dims, int(rng.integers(1, 21)), max_ctrl=2)
        ref = O1.run(dims, gates)
        got, nrm, _ = run_gpu(P, dims, gates, kernel=kernel)
        assert np.max(np.abs(got - ref)) <= 1e-10
        assert abs(nrm - 1.0) <= 1e-10


def test_adjoint_returns_to_basis_state(P):
    dims, gates = config_circuit(3, nqubits=8)
    with P.State(dims) as st:
        st.apply_circuit(gates + adjoint_circuit(gates), fuse=True)
        a = st.amplitudes()
    assert abs(a[0] - 1.0) <= 1e-10 and np.max(np.abs(a[1:])) <= 1e-10


def test_validation_leaves_state_untouched(P):
    dims = [2, 3, 4]
    with P.State(dims) as st:
        st.apply_gate(1, fourier(3))
        before = st.amplitudes()
        bad = [
            lambda: st.apply_gate(3, hadamard()),
            lambda: st.apply_gate(0, hadamard(), [0], [1]),
            lambda: st.apply_gate(0, hadamard(), [1, 1], [0, 0]),
            lambda: st.apply_gate(0, hadamard(), [1], [3]),
            lambda: st.apply_gate(0, np.array([[1, 0], [0, 2]], complex)),
            lambda: st.apply_circuit([Gate(0, (), (), hadamard()), Gate(1, (), (), np.eye(3) * 2)]),
            lambda: st.amplitudes(20, 10),
            lambda: st.reset(24),
        ]
        names = []
        for f in bad:
            with pytest.raises(P.SVError) as e:
                f()
            names.append(e.value.name)
        assert names == ["SV_ERR_QUDIT_RANGE", "SV_ERR_CTRL_OVERLAP", "SV_ERR_CTRL_DUP",
                         "SV_ERR_CTRL_VALUE", "SV_ERR_NOT_UNITARY", "SV_ERR_NOT_UNITARY",
                         "SV_ERR_INDEX_RANGE", "SV_ERR_INDEX_RANGE"]
        assert np.array_equal(st.amplitudes(), before)
        st.reset(23)
        a = st.amplitudes()
        assert a[23] == 1.0 and np.count_nonzero(a) == 1


def test_external_torch_buffer_and_stream(P):
    import torch
    dims, gates = config_circuit(1)
    buf = torch.empty(2 * 144, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with P.State(dims, ext_buffer=buf.data_ptr(), ext_bytes=buf.numel() * 8,
                 stream=s.cuda_stream) as st:
        st.apply_circuit(gates)
        st.sync()
        got = torch.view_as_complex(buf.view(-1, 2)).cpu().numpy()
    ref = O1.run(dims, gates)
    assert np.max(np.abs(got - ref)) <= 1e-10


def _sharded_free_circuit(dims, nranks, seed):
    """Gates whose sharded-target members move no data (rules iv, v of shard.cpp): diagonal
    gates (with and without local controls) and X-like gates with only sharded controls,
    interleaved with local gates controlled on sharded qubits."""
    rng = np.random.default_rng(seed)
    n = len(dims)
    s = nranks.bit_length() - 1
    sh = list(range(n - s, n))
    loc = list(range(n - s))
    y = np.array([[0, -1j], [1j, 0]])
    mono = np.array([[0, np.exp(0.3j)], [np.exp(-1.1j), 0]])
    gates = []
    for i in range(60):
        k = i % 6
        t = int(rng.choice(sh))
        others = [q for q in sh if q != t]
        if k == 0:
            gates.append(Gate(t, (), (), shift_x(2, 1)))
        elif k == 1:
            c = tuple(int(x) for x in others[:1])
            gates.append(Gate(t, c, tuple(int(rng.integers(2)) for _ in c), y if i % 12 else mono))
        elif k == 2:
            gates.append(Gate(t, (), (), t_gate() if i % 12 else np.diag([1, -1]).astype(complex)))
        elif k == 3:
            c = int(rng.choice(loc))
            gates.append(Gate(t, (c,), (int(rng.integers(dims[c])),), np.diag(np.exp(1j * rng.random(2)))))
        elif k == 4:
            q = int(rng.choice(loc))
            gates.append(Gate(q, (t,), (int(rng.integers(2)),), haar_unitary(dims[q], rng)))
        else:
            q = int(rng.choice(loc))
            gates.append(Gate(q, (), (), haar_unitary(dims[q], rng)))
    return gates


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_loopback_relabel_and_phase_move_no_data(P, nranks):
    """Rank relabelling and local phases for gates on sharded qubits: the
    result matches the oracle in every driver mode and through apply_gate, no exchange runs,
    and readback, partial uploads and reset see the relabelled slices."""
    dims = [3, 2, 4, 2, 2, 2, 2, 2]
    D = int(np.prod(dims))
    gates = _sharded_free_circuit(dims, nranks, 7 + nranks)
    psi0 = random_state(D, 11)
    ref = O2.run(dims, gates, psi0)
    for mode in ("gate", False, True, "block"):
        with P.State.loopback(dims, nranks) as st:
            st.set_amplitudes(0, psi0)
            if mode == "gate":
                for g in gates:
                    st.apply_gate(g.target, g.U, g.ctrl, g.vals)
            else:
                st.apply_circuit(gates, fuse=mode is True, block=mode == "block")
            got = st.amplitudes()
            assert st.info().exchanges == 0, mode
            # partial reads and a partial upload across relabelled slice boundaries
            L = D // nranks
            lo, cnt = L // 2, L + 3
            assert np.array_equal(st.amplitudes(lo, cnt), got[lo:lo + cnt])
            patch = random_state(cnt, 3)
            st.set_amplitudes(lo, patch)
            full = got.copy()
            full[lo:lo + cnt] = patch
            assert np.array_equal(st.amplitudes(), full)
            # a following exchange gate pairs the right slices
            hx = [Gate(len(dims) - 1, (), (), hadamard())]
            st.apply_circuit(hx)
            assert st.info().exchanges == nranks // 2       # loopback counts slice pairs
            assert np.max(np.abs(st.amplitudes() - O2.run(dims, hx, full))) <= 1e-12
            st.reset(D - 5)
            a = st.amplitudes()
            assert a[D - 5] == 1.0 and np.count_nonzero(a) == 1
        assert np.max(np.abs(got - ref)) <= 1e-12, mode
    # bit-exact labelled permutations mixing relabels, exchanges and sharded predicates
    perm = [g for g in gates if np.count_nonzero(g.U) == g.U.shape[0]
            and np.all(np.abs(g.U[np.nonzero(g.U)] - 1) == 0)]
    perm += [Gate(0, (len(dims) - 1,), (1,), shift_x(3, 2)), Gate(len(dims) - 1, (1,), (1,), shift_x(2, 1))]
    lab = labelled_state(0, D)
    with P.State.loopback(dims, nranks) as st:
        st.set_amplitudes(0, lab)
        st.apply_circuit(perm, block=True)
        assert np.array_equal(st.amplitudes(), O2.run(dims, perm, lab))


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_loopback_sharded_matches_single_state(P, nranks):
    """Sharded mode with the loopback transport: sharded targets exchange,
    sharded controls predicate, local gates run per slice; small chunks force pipelining."""
    import os
    os.environ["SV_EXCHANGE_CHUNK"] = "1000"
    try:
        rng = np.random.default_rng(nranks)
        dims = [3, 3, 4, 2, 2, 2, 2, 2]
        n, D = len(dims), int(np.prod(dims))
        _, gates = random_circuit(99 + nranks, dims, 120, max_ctrl=2)
        gates += [Gate(7, (), (), hadamard()), Gate(6, (0,), (2,), haar_unitary(2, rng)),
                  Gate(5, (7,), (1,), shift_x(2, 1)), Gate(1, (6, 7), (1, 0), fourier(3))]
        psi0 = random_state(D, 5)
        ref = O2.run(dims, gates, psi0)
        for swap in (1, 0):            # qubit remapping (default) / pairwise exchange + combine
            for fuse in ("gate", False, True, "block"):
                with P.State.loopback(dims, nranks) as st:
                    st.set_option(P.sv.SV_OPT_SHARD_SWAP, swap)
                    st.set_amplitudes(0, psi0)
                    if fuse == "gate":
                        for g in gates:
                            st.apply_gate(g.target, g.U, g.ctrl, g.vals)
                    else:
                        st.apply_circuit(gates, fuse=fuse is True, block=fuse == "block")
                    nrm = st.norm()             # before readback: on the remapped layout
                    got = st.amplitudes()
                    assert st.info().exchanges > 0
                    # readback restored the layout: more gates continue correctly from there
                    st.apply_circuit(gates[:40], block=True)
                    again = st.amplitudes()
                assert np.max(np.abs(got - ref)) <= 1e-12, (swap, fuse)
                assert abs(nrm - 1.0) <= 1e-10
                assert np.max(np.abs(again - O2.run(dims, gates[:40], ref))) <= 1e-12, (swap, fuse)
            # bit-exact labelled permutations across shards
            perm = [Gate(7, (), (), shift_x(2, 1)), Gate(6, (2,), (3,), shift_x(2, 1)),
                    Gate(2, (7,), (1,), shift_x(4, 3)), Gate(5, (6, 0), (0, 1), shift_x(2, 1)),
                    Gate(7, (2,), (1,), shift_x(2, 1)), Gate(6, (0,), (2,), shift_x(2, 1)),
                    Gate(2, (6,), (1,), shift_x(4, 1)), Gate(5, (7,), (0,), shift_x(2, 1))]
            lab = labelled_state(0, D)
            with P.State.loopback(dims, nranks) as st:
                st.set_option(P.sv.SV_OPT_SHARD_SWAP, swap)
                st.set_amplitudes(0, lab)
                for g in perm:
                    st.apply_gate(g.target, g.U, g.ctrl, g.vals)
                got = st.amplitudes()
            assert np.array_equal(got, O2.run(dims, perm, lab))
    finally:
        del os.environ["SV_EXCHANGE_CHUNK"]


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_loopback_c5_recipe_reduced_register(P, nranks):
    """BASELINE config 5's recipe on a register reduced to 13 qubits, sharded P ways on one device
    (loopback: the fused exchange / swap kernels over slice pairs), both remap settings, vs O-2."""
    dims, gates = config_circuit(5, nqubits=13)
    ref = O2.run(dims, gates)
    for swap in (1, 0):
        with P.State.loopback(dims, nranks) as st:
            st.set_option(P.sv.SV_OPT_SHARD_SWAP, swap)
            st.apply_circuit(gates, fuse=True, block=True)
            got = st.amplitudes()
            nrm = st.norm()
            assert st.info().exchanges > 0
        assert np.max(np.abs(got - ref)) <= 1e-10, swap
        assert abs(nrm - 1.0) <= 1e-10


@pytest.mark.parametrize("nranks", [2, 4])
def test_loopback_overlapped_remap(P, nranks):
    """Remaps overlapped with the pending local run (the half that moves swapped on a comm stream
    while the run updates the staying half, then the arrived half): same state as O-2 and as the
    non-overlapped schedule; the overlap path actually runs."""
    dims = [3, 3, 4, 2, 2, 2, 2, 2, 2]
    gates = _overlap_circuit(dims, 31 + nranks, nranks)
    psi0 = random_state(int(np.prod(dims)), 9)
    ref = O2.run(dims, gates, psi0)
    for ov, block in ((16, True), (0, True), (16, False)):
        with P.State.loopback(dims, nranks) as st:
            st.set_option(P.sv.SV_OPT_SHARD_OVERLAP, ov)
            st.set_amplitudes(0, psi0)
            st.apply_circuit(gates, block=block)
            got = st.amplitudes()
            over = st.info().overlapped
        assert np.max(np.abs(got - ref)) <= 1e-12, (ov, block)
        assert (over > 0) == (ov > 0), (ov, block, over)


# (compute threads, consumer groups, stages) of the pass kernel
PASS_CFGS = [(256, 1, 2), (384, 1, 2), (512, 1, 2), (384, 2, 2), (256, 2, 3), (384, 2, 3), (512, 2, 3), (512, 4, 4),
             (512, 4, 5), (512, 8, 9), (576, 3, 4), (576, 2, 3)]


@pytest.mark.parametrize("pass_cfg", PASS_CFGS)
@pytest.mark.parametrize("pass_tile", [6144, 4096, 1024, 256])
def test_block_passes_random_sweep(P, pass_tile, pass_cfg):
    """SV_BLOCK multi-gate passes on random registers and circuits with controls inside the
    tile (in-tile high digits, low digits) and outside it (per-tile predicate), ragged tiles,
    tiny registers; against O-2."""
    rng = np.random.default_rng(pass_tile)
    for s in range(25):
        n = int(rng.integers(2, 9))
        dims = [int(x) for x in rng.integers(2, 6, size=n)]
        while np.prod(dims) > 3_000_000:
            dims = dims[:-1]
        _, gates = random_circuit(70_000 + s, dims, 80, max_ctrl=3)
        psi0 = random_state(int(np.prod(dims)), s)
        ref = O2.run(dims, gates, psi0)
        if pass_tile * 16 * pass_cfg[2] > 200 * 1024:
            pytest.skip("tile ring does not fit shared memory")
        got, nrm, _ = run_gpu(P, dims, gates, psi0, block=True, pass_tile=pass_tile, pass_cfg=pass_cfg)
        assert np.max(np.abs(got - ref)) <= 1e-12, (dims, s)


@pytest.mark.parametrize("pass_cfg", [(512, 4, 4), (512, 2, 3), (256, 1, 2)])
@pytest.mark.parametrize("dims", [[2, 3, 2, 4, 3, 2, 2, 3], [4, 2, 2, 3, 2, 4, 2], [3, 2, 3, 2, 2, 2, 3, 2, 2]])
def test_block_passes_factored_pairs(P, dims, pass_cfg):
    """Factored pair items (two general gates on different in-tile digits with the same controls,
    d_a d_b <= 8: U_a then U_b on the class held in registers): layers of uncontrolled and
    identically controlled Haar gates on qubit / qutrit / ququart targets, interleaved with
    permutations that do or do not commute with them; ragged tiles (small tile caps); against
    O-2, and the pass work shows fewer shared-memory round trips than gates."""
    rng = np.random.default_rng(sum(dims) * 7 + pass_cfg[1])
    n, D = len(dims), int(np.prod(dims))
    gates = []
    for layer in range(12):
        ctrl = () if layer % 3 else (int(rng.integers(n)),)
        vals = tuple(int(rng.integers(dims[c])) for c in ctrl)
        for t in rng.permutation([q for q in range(n) if q not in ctrl]):
            gates.append(Gate(int(t), ctrl, vals, haar_unitary(dims[int(t)], rng)))
        t = int(rng.integers(n))
        c = (t + 1) % n
        gates.append(Gate(t, (c,), (dims[c] - 1,), shift_x(dims[t], 1)))
    psi0 = random_state(D, 11)
    ref = O2.run(dims, gates, psi0)
    for tile in (512, 1280, 3200):
        with P.State(dims) as st:
            threads, groups, stages = pass_cfg
            st.set_option(P.sv.SV_OPT_PASS_TILE, tile)
            st.set_option(P.sv.SV_OPT_PASS_THREADS, threads)
            st.set_option(P.sv.SV_OPT_PASS_GROUPS, groups)
            st.set_option(P.sv.SV_OPT_PASS_STAGES, stages)
            st.set_option(P.sv.SV_OPT_PASS_MERGE, 0)          # keep every gate (pairs, not products)
            st.set_option(P.sv.SV_OPT_PROFILE, 1)
            st.set_amplitudes(0, psi0)
            st.apply_circuit(gates, block=True)
            got = st.amplitudes()
            prof = st.profile_read()
        assert np.max(np.abs(got - ref)) <= 1e-12, tile
        assert prof.pass_launches > 0
        assert prof.pass_item_touched < 0.9 * prof.pass_touched, (prof.pass_item_touched, prof.pass_touched)


@pytest.mark.parametrize("pass_cfg", PASS_CFGS)
def test_block_passes_labelled_bit_exact(P, pass_cfg):
    """Permutation-only circuits through multi-gate passes: bit-exact against O-2."""
    rng = np.random.default_rng(3)
    dims = config_circuit(4, ngates=0, nqubits=4)[0]
    n, D = len(dims), int(np.prod(dims))
    gates = []
    for _ in range(150):
        t = int(rng.integers(n))
        others = [q for q in range(n) if q != t]
        nc = int(rng.integers(0, 3))
        ctrl = tuple(int(c) for c in rng.choice(others, size=nc, replace=False))
        vals = tuple(int(rng.integers(dims[c])) for c in ctrl)
        gates.append(Gate(t, ctrl, vals, permutation_matrix(rng.permutation(dims[t]))))
    psi0 = labelled_state(0, D)
    ref = O2.run(dims, gates, psi0)
    tile = {2: 6144, 3: 4096, 4: 3072, 5: 2560}.get(pass_cfg[2], 1280)   # the ring fits shared memory
    got, _, launched = run_gpu(P, dims, gates, psi0, block=True, pass_tile=tile, pass_cfg=pass_cfg)
    assert launched < len(gates)
    assert np.array_equal(got, ref)


def _absorb_circuit(rng, dims, ngates, general_frac=0.4):
    """Haar gates mixed with permutations (random sigma or X_{+1}) carrying 0-2 controls of any
    value: permutations whose target and controls are member digits or out-of-tile digits get
    absorbed at the load (front) or store (back) of their pass; the rest stay items."""
    n = len(dims)
    gates = []
    for _ in range(ngates):
        t = int(rng.integers(n))
        if rng.random() < general_frac:
            gates.append(Gate(t, (), (), haar_unitary(dims[t], rng)))
            continue
        others = [q for q in range(n) if q != t]
        nc = int(rng.integers(0, 3))
        ctrl = tuple(int(c) for c in rng.choice(others, size=nc, replace=False))
        vals = tuple(int(rng.integers(dims[c])) for c in ctrl)
        U = shift_x(dims[t], 1) if rng.random() < 0.5 else permutation_matrix(rng.permutation(dims[t]))
        gates.append(Gate(t, ctrl, vals, U))
    return gates


def _run_absorb(P, dims, gates, psi0, absorb, tile, pass_cfg=(512, 4, 4), dtype="c128"):
    with P.State(dims, dtype=dtype) as st:
        threads, groups, stages = pass_cfg
        st.set_option(P.sv.SV_OPT_PASS_TILE, tile)
        st.set_option(P.sv.SV_OPT_PASS_THREADS, threads)
        st.set_option(P.sv.SV_OPT_PASS_GROUPS, groups)
        st.set_option(P.sv.SV_OPT_PASS_STAGES, stages)
        st.set_option(P.sv.SV_OPT_PASS_ABSORB, absorb)
        st.set_option(P.sv.SV_OPT_PROFILE, 1)
        st.set_amplitudes(0, psi0)
        st.apply_circuit(gates, block=True)
        got = st.amplitudes()
        prof = st.profile_read()
    return got, prof


@pytest.mark.parametrize("pass_cfg", [(512, 4, 4), (512, 2, 3), (256, 1, 2)])
@pytest.mark.parametrize("tile", [3200, 1280, 512])
def test_block_passes_absorbed_permutations(P, tile, pass_cfg):
    """Permutations absorbed into the pass tile's load / store member addressing
    (SV_OPT_PASS_ABSORB): random registers (c4-like low prefixes and qubit-only ones), Haar gates
    mixed with controlled permutations; against O-2 with absorption on and off, the same applied
    work either way, and fewer shared-memory round trips with it on (absorbed gates are no
    compute items)."""
    rng = np.random.default_rng(tile + pass_cfg[1])
    regs = [[5, 5, 4, 4, 3, 3, 2, 2, 2, 2], [2] * 16, [3, 2, 4, 2, 2, 3, 2, 2, 3], [4, 3, 2, 2, 2, 2, 5, 2]]
    work = np.zeros(2)
    for r, dims in enumerate(regs):
        D = int(np.prod(dims))
        gates = _absorb_circuit(rng, dims, 120)
        psi0 = random_state(D, r)
        ref = O2.run(dims, gates, psi0)
        on, pon = _run_absorb(P, dims, gates, psi0, 1, tile, pass_cfg)
        off, poff = _run_absorb(P, dims, gates, psi0, 0, tile, pass_cfg)
        assert np.max(np.abs(on - ref)) <= 1e-12, (dims, tile)
        assert np.max(np.abs(off - ref)) <= 1e-12, (dims, tile)
        assert pon.pass_launches > 0
        assert pon.pass_touched == poff.pass_touched          # absorbed gates still count as applied
        assert pon.pass_item_touched <= poff.pass_item_touched
        work += [pon.pass_item_touched, poff.pass_item_touched]
    # a small register's tile may be all run and low prefix, with no member digit to absorb on
    assert work[0] < work[1], work


def test_block_passes_absorbed_permutations_bit_exact(P):
    """Permutation-only circuits on an index-labelled state with absorption: bit-exact against
    O-2, including passes whose every gate is absorbed (no compute item at all)."""
    rng = np.random.default_rng(17)
    for dims in ([5, 5, 4, 2, 2, 3, 2, 2], [2] * 14):
        D = int(np.prod(dims))
        gates = _absorb_circuit(rng, dims, 100, general_frac=0.0)
        lab = labelled_state(0, D)
        ref = O2.run(dims, gates, lab)
        work = np.zeros(2)
        for tile in (3200, 640):
            got, pon = _run_absorb(P, dims, gates, lab, 1, tile)
            assert np.array_equal(got, ref), (dims, tile)
            _, poff = _run_absorb(P, dims, gates, lab, 0, tile)
            assert pon.pass_touched == poff.pass_touched
            work += [pon.pass_item_touched, poff.pass_item_touched]
        assert work[0] < work[1], (dims, work)


@pytest.mark.parametrize("pass_cfg", [(256, 1, 3), (384, 2, 3), (512, 2, 3)])
@pytest.mark.parametrize("pass_tile", [4096, 1024, 256])
def test_stage_kernel_random_sweep(P, pass_tile, pass_cfg):
    """The register-blocked stage kernel (SV_OPT_PASS_KERNEL = 1): stages of gates on digit pairs,
    passive partners, controls on the partner digit / in-tile digits / run digits / outside the
    tile, diagonal, cyclic-shift and general gates, ragged tiles; against O-2."""
    rng = np.random.default_rng(pass_tile + 7)
    for s in range(20):
        n = int(rng.integers(2, 9))
        dims = [int(x) for x in rng.integers(2, 6, size=n)]
        while np.prod(dims) > 3_000_000:
            dims = dims[:-1]
        _, gates = random_circuit(80_000 + s, dims, 80, max_ctrl=3)
        psi0 = random_state(int(np.prod(dims)), s)
        ref = O2.run(dims, gates, psi0)
        got, _, _ = run_gpu(P, dims, gates, psi0, block=True, pass_tile=pass_tile, pass_cfg=pass_cfg, pass_kernel=1)
        assert np.max(np.abs(got - ref)) <= 1e-12, (dims, s)


def test_stage_kernel_labelled_bit_exact(P):
    """Permutations through the stage kernel (cyclic shifts as register moves, other
    permutations through the general rule with exact 0/1 entries): bit-exact against O-2."""
    rng = np.random.default_rng(5)
    dims = config_circuit(4, ngates=0, nqubits=4)[0]
    n, D = len(dims), int(np.prod(dims))
    gates = []
    for _ in range(150):
        t = int(rng.integers(n))
        others = [q for q in range(n) if q != t]
        nc = int(rng.integers(0, 3))
        ctrl = tuple(int(c) for c in rng.choice(others, size=nc, replace=False))
        vals = tuple(int(rng.integers(dims[c])) for c in ctrl)
        U = shift_x(dims[t], int(rng.integers(1, dims[t]))) if rng.random() < 0.5 else \
            permutation_matrix(rng.permutation(dims[t]))
        gates.append(Gate(t, ctrl, vals, U))
    psi0 = labelled_state(0, D)
    ref = O2.run(dims, gates, psi0)
    got, _, launched = run_gpu(P, dims, gates, psi0, block=True, pass_tile=4096, pass_cfg=(384, 2, 3),
                               pass_kernel=1)
    assert launched < len(gates)
    assert np.array_equal(got, ref)


def test_graph_cache_replays_same_circuit_and_recaptures_changes(P):
    """SV_GRAPH keeps the instantiated graph of the last circuit and replays it when the
    same circuit (same matrices, controls, flags) is submitted again; any change recaptures."""
    dims, gates = config_circuit(2, ngates=300)
    ref = O2.run(dims, gates)
    ref2 = O2.run(dims, gates + gates)
    with P.State(dims) as st:
        for block in (False, True):
            st.reset(0)
            st.apply_circuit(gates, graph=True, block=block)
            assert np.max(np.abs(st.amplitudes() - ref)) <= 1e-10
            st.apply_circuit(gates, graph=True, block=block)       # replay on the evolved state
            assert np.max(np.abs(st.amplitudes() - ref2)) <= 1e-10
        changed = list(gates)
        changed[7] = Gate(changed[7].target, changed[7].ctrl, changed[7].vals, changed[7].U.conj().T)
        st.reset(0)
        st.apply_circuit(changed, graph=True)
        assert np.max(np.abs(st.amplitudes() - O2.run(dims, changed))) <= 1e-10


def test_pass_groups_stage_reuse_regression(P):
    """Two consumer groups share the pass kernel's stage ring; a group that finishes a cheap tile
    must not start on a stage whose previous tile (the other group's) has not been loaded yet.
    Found as a hang (or silently wrong tiles) on a c4-shaped register with a pass whose tiles are
    cheap: gates with an in-tile low control and with an out-of-tile control on the same qutrit.
    Every consumer-group setting is compared with O-2 on the whole register (a
    self-comparison is no race check), and the settings with one another bit for bit (the
    per-class arithmetic is the same)."""
    from sv_inputs import config_dims
    dims = config_dims(4, nqubits=6)
    _, gates7 = config_circuit(4, nqubits=7)
    gates = [gates7[179], gates7[181], gates7[179], gates7[181]]
    assert all(g.target < len(dims) and all(c < len(dims) for c in g.ctrl) for g in gates)
    D = int(np.prod(dims, dtype=object))
    states = []
    try:
        for groups, stages in ((1, 3), (2, 3), (4, 4)):
            st = P.State(dims)
            states.append(st)
            st.set_option(P.sv.SV_OPT_PASS_GROUPS, groups)
            st.set_option(P.sv.SV_OPT_PASS_STAGES, stages)
            st.set_amplitudes(0, labelled_state(0, 1 << 20))       # non-zero, exact values
            st.apply_circuit(gates, check=False, block=True)
            st.sync()
        ref = np.zeros(D, dtype=np.complex128)
        ref[:1 << 20] = labelled_state(0, 1 << 20)
        O2.run_inplace(ref, dims, gates)
        scale = float(np.max(np.abs(ref)))
        chunk = 1 << 24
        for first in range(0, D, chunk):
            n = min(chunk, D - first)
            a0 = states[0].amplitudes(first, n)
            assert np.max(np.abs(a0 - ref[first:first + n])) <= 1e-12 * scale, first
            for other in states[1:]:
                assert np.array_equal(a0, other.amplitudes(first, n)), first
    finally:
        for st in states:
            st.close()


MODES = [dict(), dict(fuse=True), dict(block=True), dict(block=True, graph=True), dict(fuse=True, graph=True)]


@pytest.mark.parametrize("mode", range(len(MODES)))
def test_edge_cases_every_driver_mode(P, mode):
    """Degenerate inputs through every circuit-driver mode against the oracle: the empty
    circuit, one-qudit registers (d = 2 and 16), identity gates (no class to visit), a d = 16
    qudit among small ones (the generic path inside passes), gates with 4 controls (the pass
    kernel's maximum) and 5 controls (a single-gate fallback)."""
    kw = MODES[mode]
    rng = np.random.default_rng(mode)
    # empty circuit: e_0 stays e_0
    dims = [3, 2, 4]
    got, nrm, _ = run_gpu(P, dims, [], **kw)
    assert got[0] == 1.0 and np.count_nonzero(got) == 1 and nrm == 1.0
    # one-qudit registers
    for d in (2, 16):
        gates = [Gate(0, (), (), haar_unitary(d, rng)) for _ in range(5)]
        got, nrm, _ = run_gpu(P, [d], gates, **kw)
        assert np.max(np.abs(got - O1.run([d], gates))) <= 1e-12
    # identity gates, a 16-dimensional qudit, many controls
    dims = [2, 3, 16, 2, 2, 3, 2, 2]
    gates = [Gate(1, (), (), np.eye(3, dtype=np.complex128)),
             Gate(2, (), (), haar_unitary(16, rng)),
             Gate(0, (2,), (7,), haar_unitary(2, rng)),
             Gate(2, (0, 1), (1, 2), haar_unitary(16, rng)),
             Gate(4, (0, 1, 3, 5), (1, 0, 1, 2), haar_unitary(2, rng)),
             Gate(6, (0, 1, 3, 4, 7), (1, 2, 0, 1, 1), haar_unitary(2, rng)),
             Gate(5, (6, 7, 0, 2), (1, 1, 1, 15), shift_x(3, 1)),
             Gate(3, (), (), np.eye(2, dtype=np.complex128))]
    gates += [Gate(int(t), (), (), haar_unitary(dims[int(t)], rng)) for t in rng.integers(0, len(dims), 12)]
    psi0 = random_state(int(np.prod(dims)), 17 + mode)
    ref = O2.run(dims, gates, psi0)
    got, nrm, _ = run_gpu(P, dims, gates, psi0, **kw)
    assert np.max(np.abs(got - ref)) <= 1e-12
    assert abs(nrm - 1.0) <= 1e-10


def test_block_plan_cache_follows_the_gates(P):
    """The SV_BLOCK host plan is memoised per handle: resubmitting a circuit reuses it, while a
    changed matrix, gate order or option plans afresh (results against the oracle each time)."""
    rng = np.random.default_rng(5)
    dims = [3, 2, 4, 2, 3, 2, 2, 5, 2]
    D = int(np.prod(dims))
    _, gates = random_circuit(55, dims, 150, max_ctrl=2)
    other = list(gates)
    other[10] = Gate(other[10].target, other[10].ctrl, other[10].vals, haar_unitary(dims[other[10].target], rng))
    psi = random_state(D, 2)
    with P.State(dims) as st:
        st.set_amplitudes(0, psi)
        for circ in (gates, gates, other, gates[::-1], gates, "opt", gates):
            if circ == "opt":
                st.set_option(P.sv.SV_OPT_PASS_SEARCH, 0)
                continue
            st.apply_circuit(circ, block=True)
            psi = O2.run(dims, circ, psi)
            assert np.max(np.abs(st.amplitudes() - psi)) <= 1e-11
