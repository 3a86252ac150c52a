"""Pins for the oracle (CPU only).  Each test fixes the oracle to something other than
itself: a value the paper prints or narrates, a closed form, an invariant, a special case
that reduces to a textbook operation, or the independent Kronecker definition (O-1)."""
import os

import numpy as np
import pytest

from oracle import blocksim as O2
from oracle import kron as O1
from sv_inputs import (Gate, shift_x, clock_z, fourier, hadamard, haar_unitary,
                       permutation_matrix, phase_gate, ghz_circuit, worked_example,
                       random_circuit, labelled_state, random_state)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_example.txt")


def _digits(i, dims):
    """Mixed-radix digits of index array i (q_0 least significant), written out directly."""
    out = []
    rest = np.asarray(i, dtype=np.int64).copy()
    for d in dims:
        out.append(rest % d)
        rest //= d
    return out


def _golden():
    rows = {}
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        st, i, re, im = line.split()
        rows.setdefault(st, {})[int(i)] = complex(float(re), float(im))
    return rows


# ---------------------------------------------------------------- index model
def test_strides_examples():
    assert O2.strides([2, 3]) == ([1, 2], 6)          # SPEC.md:47 (PAPER §2.5 register)
    assert O2.strides([2, 3, 2]) == ([1, 2, 6], 12)
    assert O2.strides([5, 5, 5])[0][2] == 25
    assert O2.strides([2] * 63)[1] == 2 ** 63
    with pytest.raises(OverflowError):
        O2.strides([2] * 64)


# ----------------------------------------------------------- §2.5 worked example (golden)
@pytest.mark.parametrize("impl", ["O1", "O2"])
def test_worked_example_golden(impl):
    dims, gates = worked_example()
    gold = _golden()
    run = O1.run if impl == "O1" else O2.run
    for stage, gs in (("after_h", gates[:1]), ("final", gates)):
        psi = run(dims, gs)
        exp = np.zeros(6, dtype=np.complex128)
        for i, a in gold[stage].items():
            exp[i] = a
        assert np.flatnonzero(np.abs(psi) > 1e-14).tolist() == sorted(gold[stage])
        assert np.max(np.abs(psi - exp)) < 1e-15


# ------------------------------------------------------------- O-1 vs O-2
def test_o1_vs_o2_random_sweep():
    rng = np.random.default_rng(7)
    worst = 0.0
    for s in range(150):
        n = int(rng.integers(1, 5))
        dims = [int(x) for x in rng.integers(2, 6, size=n)]
        while np.prod(dims) > 625:
            dims = dims[:-1]
        _, gates = random_circuit(10_000 + s, dims, int(rng.integers(1, 21)), max_ctrl=2)
        psi0 = random_state(int(np.prod(dims)), 20_000 + s)
        a = O1.run(dims, gates, psi0)
        b = O2.run(dims, gates, psi0)
        worst = max(worst, float(np.max(np.abs(a - b))))
    assert worst < 1e-13, worst


def test_o2_single_gates_match_full_operator_every_position():
    """Every (dims, target, control placement) on a 3-qudit register, against O-1."""
    rng = np.random.default_rng(3)
    for dims in ([2, 3, 4], [5, 2, 3], [3, 3, 3], [4, 5, 2]):
        D = int(np.prod(dims))
        for t in range(3):
            U = haar_unitary(dims[t], rng)
            others = [q for q in range(3) if q != t]
            for ctrl in ([], [others[0]], [others[1]], others):
                vals = [int(rng.integers(dims[c])) for c in ctrl]
                g = Gate(t, tuple(ctrl), tuple(vals), U)
                psi = random_state(D, 5)
                ref = O1.full_operator(dims, t, ctrl, vals, U) @ psi
                O2.apply(psi, dims, g)
                assert np.max(np.abs(psi - ref)) < 1e-14


# --------------------------------------------------------------------- closed forms
@pytest.mark.parametrize("d", [2, 3, 4, 5, 7, 16])
def test_shift_power_d_is_identity_bit_exact(d):
    dims = [3, d, 2]
    psi0 = random_state(int(np.prod(dims)), d)
    psi = psi0.copy()
    for _ in range(d):
        O2.apply(psi, dims, Gate(1, (), (), shift_x(d, 1)))
    assert np.array_equal(psi, psi0)


@pytest.mark.parametrize("d", [2, 3, 4, 5, 16])
def test_clock_and_fourier_powers(d):
    dims = [2, d]
    psi0 = random_state(2 * d, 11 + d)
    psi = psi0.copy()
    for _ in range(d):
        O2.apply(psi, dims, Gate(1, (), (), clock_z(d, 1)))
    assert np.max(np.abs(psi - psi0)) < 2e-14                    # Z_d^d = I
    psi = psi0.copy()
    for _ in range(2):
        O2.apply(psi, dims, Gate(1, (), (), fourier(d)))
    # F_d^2 = parity: |j> -> |-j mod d>, i.e. the q_1 digit is negated (closed form)
    q0, q1 = _digits(np.arange(2 * d), dims)
    exp = np.empty_like(psi0)
    exp[q0 + 2 * ((-q1) % d)] = psi0
    assert np.max(np.abs(psi - exp)) < 2e-14
    for _ in range(2):
        O2.apply(psi, dims, Gate(1, (), (), fourier(d)))
    assert np.max(np.abs(psi - psi0)) < 2e-14                    # F_d^4 = I


def test_hadamard_on_one():
    psi = np.array([0, 1], dtype=np.complex128)
    O2.apply(psi, [2], Gate(0, (), (), hadamard()))
    assert np.allclose(psi, [1 / np.sqrt(2), -1 / np.sqrt(2)], atol=1e-16, rtol=0)


def test_fourier_on_every_qutrit_is_uniform():
    """F_3 on all 12 qutrits of e_0: every amplitude is (1/sqrt 3)^12 = 1/729 (closed form)."""
    dims = [3] * 12
    psi = O2.run(dims, [Gate(q, (), (), fourier(3)) for q in range(12)])
    assert np.max(np.abs(psi - 1.0 / 729.0)) < 2.4e-18


@pytest.mark.parametrize("d,n", [(2, 14), (3, 9), (4, 7), (5, 6), (7, 5)])
def test_ghz_amplitudes_exact(d, n):
    """GHZ_d: exactly d nonzeros at |v v .. v>, each bit-equal to fl(1/sqrt d) (north_star)."""
    dims, gates = ghz_circuit(d, n)
    psi = O2.run(dims, gates)
    rep = sum(d ** k for k in range(n))              # index of |1 1 .. 1>
    idx = [v * rep for v in range(d)]
    assert np.flatnonzero(psi != 0).tolist() == idx
    s = 1.0 / np.sqrt(d)
    assert all(psi[i].real == s and psi[i].imag == 0.0 for i in idx)


def test_toffoli_truth_table():
    dims = [2, 2, 2]
    g = Gate(0, (2, 1), (1, 1), shift_x(2, 1))
    for i in range(8):
        psi = np.zeros(8, dtype=np.complex128)
        psi[i] = 1.0
        O2.apply(psi, dims, g)
        exp = i ^ 1 if i in (6, 7) else i
        assert psi[exp] == 1.0 and np.count_nonzero(psi) == 1


def _kron_vecs(vecs_q0_first):
    out = np.ones(1, dtype=np.complex128)
    for v in reversed(vecs_q0_first):       # q_{n-1} is the left factor
        out = np.kron(out, v)
    return out


def test_product_state_factorisation():
    """U on q_k of a product state replaces factor k by U phi_k (tensor identity); with a
    control in basis state v the gate fires iff v equals the control value."""
    rng = np.random.default_rng(9)
    for dims in ([2, 3, 5], [4, 2, 3, 2], [3, 5]):
        n = len(dims)
        for t in range(n):
            phis = [random_state(d, 100 + 7 * k + t) for k, d in enumerate(dims)]
            U = haar_unitary(dims[t], rng)
            psi = _kron_vecs(phis)
            O2.apply(psi, dims, Gate(t, (), (), U))
            exp = _kron_vecs([U @ p if k == t else p for k, p in enumerate(phis)])
            assert np.max(np.abs(psi - exp)) < 1e-14
            # controlled on a basis-state qudit
            c = (t + 1) % n
            for v_state in range(dims[c]):
                phis_c = list(phis)
                phis_c[c] = np.eye(dims[c], dtype=np.complex128)[v_state]
                psi = _kron_vecs(phis_c)
                psi_in = psi.copy()
                O2.apply(psi, dims, Gate(t, (c,), (1 % dims[c],), U))
                if v_state == 1 % dims[c]:
                    exp = _kron_vecs([U @ p if k == t else p for k, p in enumerate(phis_c)])
                    assert np.max(np.abs(psi - exp)) < 1e-14
                else:
                    assert np.array_equal(psi, psi_in)


def test_labelled_permutation_index_map_bit_exact():
    """Permutation gates move amplitude i to i + (sigma(v) - v) b_k."""
    rng = np.random.default_rng(21)
    dims = [3, 2, 5, 4]
    D = int(np.prod(dims))
    b = [1, 3, 6, 30]
    for _ in range(40):
        t = int(rng.integers(4))
        d = dims[t]
        sigma = rng.permutation(d)
        others = [q for q in range(4) if q != t]
        nc = int(rng.integers(0, 3))
        ctrl = [int(c) for c in rng.choice(others, size=nc, replace=False)]
        vals = [int(rng.integers(dims[c])) for c in ctrl]
        psi = labelled_state(0, D)
        inp = psi.copy()
        O2.apply(psi, dims, Gate(t, tuple(ctrl), tuple(vals), permutation_matrix(sigma)))
        i = np.arange(D)
        dg = _digits(i, dims)
        ok = np.ones(D, dtype=bool)
        for c, v in zip(ctrl, vals):
            ok &= dg[c] == v
        dest = np.where(ok, i + (sigma[dg[t]] - dg[t]) * b[t], i)
        exp = np.empty_like(inp)
        exp[dest] = inp
        assert np.array_equal(psi, exp)


def test_phase_closed_form_and_block_rules():
    """General rule on a diagonal U == psi_i * diag[digit(i,k)] == the §2.1 block rule; the
    §2.2 block rotation == the general rule on X_{+a} (bit-exact)."""
    rng = np.random.default_rng(5)
    dims = [2, 5, 3, 4]
    D = int(np.prod(dims))
    for t in range(4):
        d = dims[t]
        diag = np.exp(1j * rng.uniform(0, 2 * np.pi, size=d))
        psi0 = random_state(D, 40 + t)
        dg = _digits(np.arange(D), dims)
        exp = psi0 * diag[dg[t]]
        a = psi0.copy()
        O2.apply(a, dims, Gate(t, (), (), np.diag(diag)))
        b_ = psi0.copy()
        O2.apply_phase(b_, dims, t, diag)
        assert np.max(np.abs(a - exp)) < 1e-15 and np.max(np.abs(b_ - exp)) < 1e-15
        for sh in range(1, d):
            c = (t + 1) % 4
            x = psi0.copy()
            O2.apply(x, dims, Gate(t, (c,), (1,), shift_x(d, sh)))
            y = psi0.copy()
            O2.apply_shift(y, dims, t, sh, (c,), (1,))
            assert np.array_equal(x, y)


def test_norm_preserved_and_norm_function():
    dims = [3, 4, 2, 5]
    _, gates = random_circuit(77, dims, 60, max_ctrl=2)
    psi = O2.run(dims, gates)
    assert abs(O2.norm(psi) - 1.0) < 1e-13
    assert abs(O2.norm(np.array([0.6, 0.8j])) - 1.0) < 1e-16     # 3-4-5
    assert O2.norm(np.zeros(4, dtype=np.complex128)) == 0.0


def test_sampled_gate_output_matches_full_apply():
    """The one-index evaluator used for full-size sampled checks == the full class sweep."""
    rng = np.random.default_rng(8)
    dims = [5, 4, 3, 2, 3]
    D = int(np.prod(dims))
    for t in range(5):
        U = haar_unitary(dims[t], rng)
        for ctrl, vals in (((), ()), (((t + 2) % 5,), (1,))):
            g = Gate(t, ctrl, vals, U)
            psi = labelled_state(0, D)
            O2.apply(psi, dims, g)
            idx = rng.choice(D, size=200, replace=False)
            got = O2.gate_output_labelled(dims, g, idx)
            assert np.max(np.abs(got - psi[idx]) / np.abs(psi[idx])) < 1e-15


def test_sampled_circuit_output_matches_kronecker():
    """The short-circuit evaluator used for sampled full-size checks of multi-gate passes ==
    O-1 (the Kronecker operators, independent of O-2) on the labelled state, every index."""
    from oracle import kron as O1
    rng = np.random.default_rng(9)
    for s in range(40):
        n = int(rng.integers(2, 5))
        dims = [int(x) for x in rng.integers(2, 6, size=n)]
        D = int(np.prod(dims))
        _, gates = random_circuit(9_000 + s, dims, int(rng.integers(1, 4)), max_ctrl=2)
        ref = O1.run(dims, gates, psi0=labelled_state(0, D))
        got = O2.circuit_output_labelled(dims, gates, np.arange(D))
        assert np.max(np.abs(got - ref) / np.abs(ref).max()) < 1e-14, (dims, s)
    assert O2.circuit_output_labelled([2, 3], [], [4])[0] == labelled_state(4, 1)[0]


# ------------------------------------------------------------------ O-3 (sparse, §2.3)
def test_sparse_oracle_matches_dense_oracle():
    from oracle import sparse as O3
    rng = np.random.default_rng(33)
    for s in range(60):
        n = int(rng.integers(1, 6))
        dims = [int(x) for x in rng.integers(2, 6, size=n)]
        _, gates = random_circuit(40_000 + s, dims, int(rng.integers(1, 25)), max_ctrl=2)
        dense = O2.run(dims, gates)
        sp = O3.run(dims, gates)
        rebuilt = np.zeros_like(dense)
        for i, a in sp.items():
            rebuilt[i] = a
        assert np.max(np.abs(rebuilt - dense)) < 1e-12           # pruned entries are < 1e-12
        assert all(abs(a) >= O3.EPS for a in sp.values())


@pytest.mark.parametrize("d,n", [(2, 62), (3, 39), (4, 31), (5, 27)])
def test_sparse_oracle_ghz_at_the_papers_maxima(d, n):
    """GHZ reaches 62 qubits, 39 qutrits, 31 ququads, 27 ququints (the 64-bit
    index limit); the state has exactly d entries at v*(1+d+...+d^{n-1}), each fl(1/sqrt d)."""
    from oracle import sparse as O3
    dims, gates = ghz_circuit(d, n)
    st = O3.run(dims, gates)
    rep = sum(d ** k for k in range(n))
    assert sorted(st) == [v * rep for v in range(d)]
    assert max(st) < 2 ** 63
    assert all(a == 1.0 / np.sqrt(d) for a in st.values())
