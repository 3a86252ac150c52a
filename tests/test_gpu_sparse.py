"""GPU sparse states against the sparse oracle O-3 and closed forms.

Tolerance: |a_gpu - a_oracle| <= 1e-12 per index (entries missing on one side count as 0;
both sides drop |a| < 1e-12, so a pruning-boundary disagreement is itself below 1e-12).
Permutation circuits are bit-exact (values only move)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import sparse as O3  # noqa: E402
from oracle import blocksim as O2  # noqa: E402
from sv_inputs import (Gate, ghz_circuit, random_circuit, worked_example, shift_x,  # noqa: E402
                       permutation_matrix, hadamard, fourier, haar_unitary)


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2410_17876_b200 as P
    return P


def run_sparse(P, dims, gates, per_gate=False):
    with P.sv.SparseState(dims) as st:
        if per_gate:
            for g in gates:
                st.apply_gate(g.target, g.U, g.ctrl, g.vals)
        else:
            st.apply_circuit(gates)
        idx, amp = st.entries()
    return {int(i): complex(a) for i, a in zip(idx, amp)}, idx


def diff(a: dict, b: dict) -> float:
    keys = set(a) | set(b)
    return max((abs(a.get(k, 0) - b.get(k, 0)) for k in keys), default=0.0)


def test_worked_example_sparse(P):
    dims, gates = worked_example()
    got, idx = run_sparse(P, dims, gates)
    assert sorted(got) == [0, 2, 5]
    assert all(abs(a - 1 / np.sqrt(3)) < 1e-15 for a in got.values())
    assert np.all(np.diff(idx.astype(np.int64)) > 0)          # sorted, unique


@pytest.mark.parametrize("d,n", [(2, 62), (3, 39), (4, 31), (5, 27), (2, 20), (7, 10)])
def test_ghz_sparse_at_the_papers_maxima(P, d, n):
    dims, gates = ghz_circuit(d, n)
    got, _ = run_sparse(P, dims, gates)
    rep = sum(d ** k for k in range(n))
    assert sorted(got) == [v * rep for v in range(d)]
    assert all(a == 1.0 / np.sqrt(d) for a in got.values())     # bit-equal to fl(1/sqrt d)


def test_sparse_overflow_rule(P):
    with pytest.raises(P.SVError) as e:
        P.sv.SparseState([2] * 64)
    assert e.value.name == "SV_ERR_OVERFLOW"
    P.sv.SparseState([2] * 63).close()


def test_sparse_random_circuits_against_oracles(P):
    rng = np.random.default_rng(11)
    for s in range(40):
        n = int(rng.integers(2, 9))
        dims = [int(x) for x in rng.integers(2, 6, size=n)]
        _, gates = random_circuit(90_000 + s, dims, int(rng.integers(5, 40)), max_ctrl=2)
        ref = O3.run(dims, gates)
        got, _ = run_sparse(P, dims, gates, per_gate=bool(s % 2))
        assert diff(got, ref) <= 1e-12, s
        if int(np.prod(dims)) <= 200_000:                        # and the dense oracle
            dense = O2.run(dims, gates)
            rebuilt = np.zeros_like(dense)
            for i, a in got.items():
                rebuilt[i] = a
            assert np.max(np.abs(rebuilt - dense)) <= 1e-12


def test_sparse_wide_register_permutations_bit_exact(P):
    """40 qudits (D ~ 1e19 would overflow; here 2^20 * 3^12 * 5^3 ~ 7e13): controlled shifts and
    permutations from a few seeds of F on low qubits; bit-exact against O-3."""
    rng = np.random.default_rng(5)
    dims = [2] * 20 + [3] * 12 + [5] * 3
    n = len(dims)
    gates = [Gate(q, (), (), hadamard()) for q in range(8)]            # 256 entries
    for _ in range(200):
        t = int(rng.integers(n))
        others = [q for q in range(n) if q != t]
        nc = int(rng.integers(0, 3))
        ctrl = tuple(int(c) for c in rng.choice(others, size=nc, replace=False))
        vals = tuple(int(rng.integers(dims[c])) for c in ctrl)
        U = shift_x(dims[t], int(rng.integers(1, dims[t]))) if rng.random() < 0.5 else \
            permutation_matrix(rng.permutation(dims[t]))
        gates.append(Gate(t, ctrl, vals, U))
    ref = O3.run(dims, gates)
    got, _ = run_sparse(P, dims, gates)
    assert len(got) == 256
    assert got == ref


def test_sparse_growth_and_interference(P):
    """F on 14 qutrits (4.8e6 entries), then the inverse: back to e_0 (interference cancels,
    pruning removes the ~1e-16 residues)."""
    dims = [3] * 14
    fwd = [Gate(q, (), (), fourier(3)) for q in range(14)]
    inv = [Gate(q, (), (), fourier(3).conj().T) for q in range(14)]
    with P.sv.SparseState(dims) as st:
        st.apply_circuit(fwd)
        assert st.nnz() == 3 ** 14
        st.apply_circuit(inv)
        idx, amp = st.entries()
    assert idx.tolist() == [0] and abs(amp[0] - 1.0) < 1e-12
