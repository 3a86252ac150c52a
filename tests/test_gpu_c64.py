"""complex64 states (SV_C64) against the fp64 oracle.

Tolerance (R17): one gate rounds every class output y = U x in fp32 with at most
2d FMAs per component plus the fp32 rounding of U, so ||dy||_2 <= (2d + 1) sqrt(d) u ||x||_2
with u = 2^-24; unitary gates carry earlier errors unchanged, so after G gates
||psi_c64 - psi_exact||_2 <= G (2 d_max + 1) sqrt(d_max) 2^-24 (plus the fp32 rounding of the
input state when one is uploaded).  Permutations move values without arithmetic: bit-exact
on labelled states whose labels are exact in fp32 (D < 2^24)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import blocksim as O2  # noqa: E402
from sv_inputs import (Gate, config_circuit, random_circuit, random_state, labelled_state,  # noqa: E402
                       permutation_matrix, shift_x, haar_unitary, ghz_circuit)

U32 = 2.0 ** -24


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2410_17876_b200 as P
    return P


def bound(gates, dims, extra=0.0):
    dmax = max(dims[g.target] for g in gates) if gates else 2
    return len(gates) * (2 * dmax + 1) * np.sqrt(dmax) * U32 + extra


def run_c64(P, dims, gates, psi0=None, kernel=0, fuse=False, block=False):
    with P.State(dims, dtype="c64") as st:
        st.set_option(P.sv.SV_OPT_KERNEL, kernel)
        if psi0 is not None:
            st.set_amplitudes(0, psi0)
        st.apply_circuit(gates, fuse=fuse, block=block)
        return st.amplitudes(), st.norm()


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_configs_c64_against_fp64_oracle(P, kernel, cfg):
    nq = {3: 6, 4: 1}.get(cfg)
    dims, gates = config_circuit(cfg, nqubits=nq) if nq else config_circuit(cfg)
    if cfg == 2:
        gates = gates[:1200]
    ref = O2.run(dims, gates)
    got, nrm = run_c64(P, dims, gates, kernel=kernel, fuse=True, block=True)
    err = float(np.linalg.norm(got - ref))
    tol = bound(gates, dims)
    assert err <= tol, (err, tol)
    assert abs(nrm - 1.0) <= tol


def test_random_sweep_c64(P):
    rng = np.random.default_rng(64)
    for s in range(30):
        n = int(rng.integers(2, 7))
        dims = [int(x) for x in rng.integers(2, 6, size=n)]
        _, gates = random_circuit(64_000 + s, dims, 40, max_ctrl=2)
        psi0 = random_state(int(np.prod(dims)), s)
        ref = O2.run(dims, gates, psi0)
        for kernel, block in ((1, False), (2, False), (0, True)):
            got, _ = run_c64(P, dims, gates, psi0, kernel=kernel, block=block)
            # input rounding to fp32 adds at most sqrt(2) u per amplitude (||.||_2 <= sqrt(2) u)
            assert np.linalg.norm(got - ref) <= bound(gates, dims, np.sqrt(2) * U32), (kernel, block)


def test_labelled_permutations_bit_exact_c64(P):
    rng = np.random.default_rng(7)
    dims = [5, 3, 4, 2, 3, 2, 2, 3]
    n, D = len(dims), int(np.prod(dims))
    assert D < 2 ** 24
    gates = []
    for _ in range(80):
        t = int(rng.integers(n))
        others = [q for q in range(n) if q != t]
        nc = int(rng.integers(0, 3))
        ctrl = tuple(int(c) for c in rng.choice(others, size=nc, replace=False))
        vals = tuple(int(rng.integers(dims[c])) for c in ctrl)
        gates.append(Gate(t, ctrl, vals, permutation_matrix(rng.permutation(dims[t]))))
    lab = labelled_state(0, D)
    ref = O2.run(dims, gates, lab)
    for kernel, block in ((1, False), (2, False), (0, True)):      # block: the c64 pass kernel (L = 60)
        got, _ = run_c64(P, dims, gates, lab, kernel=kernel, block=block)
        assert np.array_equal(got, ref), (kernel, block)


def test_ghz_c64_exact_to_fp32(P):
    for d, n in ((2, 20), (3, 12), (5, 8)):
        dims, gates = ghz_circuit(d, n)
        got, _ = run_c64(P, dims, gates)
        rep = sum(d ** k for k in range(n))
        idx = [v * rep for v in range(d)]
        s = np.float32(1.0 / np.sqrt(d))
        assert np.flatnonzero(got).tolist() == idx
        assert all(got[i].real == float(s) and got[i].imag == 0.0 for i in idx)


def test_c64_state_is_half_the_bytes(P):
    import torch
    dims = [3] * 12
    before = torch.cuda.mem_get_info()[0]
    st = P.State(dims, dtype="c64")
    used = before - torch.cuda.mem_get_info()[0]
    st.close()
    D = 3 ** 12
    assert used < 16 * D          # 8 B per amplitude (+ small scratch), not 16


def test_c64_pass_kernel_used_and_matches(P):
    """The complex64 pass kernel runs when the tile is 16-byte aligned (even L = b_{m0}): a
    c4-shaped register (L = 100) in block mode launches fewer kernels than gates and matches the
    fp64 oracle within the fp32 bound; an odd-L register (c3 shape, L = 81) falls back to the
    single-gate kernels with the same result quality."""
    for cfg, nq in ((4, 1), (3, 4)):
        dims, gates = config_circuit(cfg, nqubits=nq)
        gates = gates[:200]
        ref = O2.run(dims, gates)
        with P.State(dims, dtype="c64") as st:
            n0 = st.info().kernel_launches
            st.apply_circuit(gates, block=True)
            got = st.amplitudes()
            launched = st.info().kernel_launches - n0
        assert np.linalg.norm(got - ref) <= bound(gates, dims)
        if cfg == 4:
            assert launched < len(gates) // 4, launched


@pytest.mark.parametrize("nranks", [2, 4])
def test_loopback_sharded_c64(P, nranks):
    """Sharded complex64 (loopback transport on one GPU): sharded targets exchange fp32 slices,
    sharded controls predicate, local runs use the complex64 pass kernel; against the fp64
    oracle within the fp32 bound, and labelled permutations bit-exact across shards."""
    import os
    os.environ["SV_EXCHANGE_CHUNK"] = "1000"
    try:
        from sv_inputs import hadamard, fourier
        dims = [4, 5, 2, 2, 2, 2, 2, 2]
        n, D = len(dims), int(np.prod(dims))
        rng = np.random.default_rng(40 + nranks)
        _, gates = random_circuit(640 + nranks, dims, 100, max_ctrl=2)
        gates += [Gate(7, (), (), hadamard()), Gate(6, (0,), (2,), haar_unitary(2, rng)),
                  Gate(5, (7,), (1,), shift_x(2, 1)), Gate(1, (6, 7), (1, 0), fourier(5))]
        psi0 = random_state(D, 9)
        ref = O2.run(dims, gates, psi0)
        for block in (False, True):
            with P.State.loopback(dims, nranks, dtype="c64") as st:
                st.set_amplitudes(0, psi0)
                st.apply_circuit(gates, block=block)
                got = st.amplitudes()
                assert st.info().exchanges > 0
            assert np.linalg.norm(got - ref) <= bound(gates, dims, np.sqrt(2) * U32), block
        perm = [Gate(7, (), (), shift_x(2, 1)), Gate(6, (2,), (1,), shift_x(2, 1)),
                Gate(1, (7,), (1,), shift_x(5, 3)), Gate(5, (6, 0), (0, 1), shift_x(2, 1))]
        lab = labelled_state(0, D)
        with P.State.loopback(dims, nranks, dtype="c64") as st:
            st.set_amplitudes(0, lab)
            st.apply_circuit(perm, block=True)
            got = st.amplitudes()
        assert np.array_equal(got, O2.run(dims, perm, lab))
    finally:
        del os.environ["SV_EXCHANGE_CHUNK"]


@pytest.mark.parametrize("nranks", [2, 8])
def test_loopback_relabel_and_phase_c64(P, nranks):
    """complex64 sharded state: gates on sharded qubits that move no data (relabelled slices,
    local phases) against the fp64 oracle within the fp32 bound, with no exchange."""
    from test_gpu_parity import _sharded_free_circuit
    dims = [3, 2, 4, 2, 2, 2, 2, 2]
    D = int(np.prod(dims))
    gates = _sharded_free_circuit(dims, nranks, 70 + nranks)
    psi0 = random_state(D, 12)
    ref = O2.run(dims, gates, psi0)
    for block in (False, True):
        with P.State.loopback(dims, nranks, dtype="c64") as st:
            st.set_amplitudes(0, psi0)
            st.apply_circuit(gates, block=block)
            got = st.amplitudes()
            assert st.info().exchanges == 0
        assert np.linalg.norm(got - ref) <= bound(gates, dims, np.sqrt(2) * U32), block


def test_c64_absorbed_permutations(P):
    """Permutations absorbed into the complex64 pass kernel's load / store addressing
    (SV_OPT_PASS_ABSORB): a labelled permutation circuit bit-exact, and Haar gates mixed with
    controlled permutations within the fp32 bound, with fewer shared-memory round trips."""
    dims = [4, 2, 2, 3, 2, 4, 2, 2, 2]          # L = 48: 16-byte aligned complex64 tiles
    rng = np.random.default_rng(33)
    n, D = len(dims), int(np.prod(dims))

    def circuit(general_frac, ngates):
        gates = []
        for _ in range(ngates):
            t = int(rng.integers(n))
            if rng.random() < general_frac:
                gates.append(Gate(t, (), (), haar_unitary(dims[t], rng)))
                continue
            others = [q for q in range(n) if q != t]
            ctrl = tuple(int(c) for c in rng.choice(others, size=int(rng.integers(0, 3)), replace=False))
            vals = tuple(int(rng.integers(dims[c])) for c in ctrl)
            gates.append(Gate(t, ctrl, vals, permutation_matrix(rng.permutation(dims[t]))))
        return gates

    for general_frac in (0.0, 0.4):
        gates = circuit(general_frac, 90)
        psi0 = labelled_state(0, D) if general_frac == 0.0 else random_state(D, 9)
        ref = O2.run(dims, gates, psi0)
        with P.State(dims, dtype="c64") as st:
            st.set_option(P.sv.SV_OPT_PASS_ABSORB, 1)
            st.set_option(P.sv.SV_OPT_PROFILE, 1)
            st.set_amplitudes(0, psi0)
            st.apply_circuit(gates, block=True)
            got = st.amplitudes()
            prof = st.profile_read()
        if general_frac == 0.0:
            assert np.array_equal(got, ref)
        else:
            assert np.linalg.norm(got - ref) <= bound(gates, dims)
        assert prof.pass_launches > 0
        assert prof.pass_item_touched < prof.pass_touched


def test_c64_factored_pairs(P):
    """Factored pair items in the complex64 pass kernel (two general gates on different in-tile
    digits with the same controls, U_a then U_b on the class in registers): against the fp64
    oracle within the fp32 bound (each factor rounds like a separate gate), with fewer
    shared-memory round trips than gates in the pass work."""
    dims = [4, 2, 2, 3, 2, 4, 2, 2]            # L = b_4 = 48: 16-byte aligned complex64 tiles
    rng = np.random.default_rng(21)
    n, D = len(dims), int(np.prod(dims))
    gates = []
    for layer in range(10):
        ctrl = () if layer % 3 else (int(rng.integers(n)),)
        vals = tuple(int(rng.integers(dims[c])) for c in ctrl)
        for t in rng.permutation([q for q in range(n) if q not in ctrl]):
            gates.append(Gate(int(t), ctrl, vals, haar_unitary(dims[int(t)], rng)))
    psi0 = random_state(D, 5)
    ref = O2.run(dims, gates, psi0)
    with P.State(dims, dtype="c64") as st:
        st.set_option(P.sv.SV_OPT_PASS_MERGE, 0)
        st.set_option(P.sv.SV_OPT_PROFILE, 1)
        st.set_amplitudes(0, psi0)
        st.apply_circuit(gates, block=True)
        got = st.amplitudes()
        prof = st.profile_read()
    assert np.linalg.norm(got - ref) <= bound(gates, dims, np.sqrt(2) * U32)
    assert prof.pass_launches > 0
    assert prof.pass_item_touched < 0.9 * prof.pass_touched
