"""Full-size parity at BASELINE.json's configs c3 (6.9 GB) and c4 (76.4 GB) against the oracle,
in two circuit-driver modes: single-gate kernels (auto kernel policy, SV_FUSE) and the mode
bench.py times on c1-c4 (SV_BLOCK multi-gate passes with the default pass configuration):

  * the state after a prefix of the seeded circuit, compared element by element with O-2
    run on the host (streamed back in 2 GB chunks); with SV_BLOCK a 48-gate prefix forms
    merged gates, pair gates and multi-gate passes;
  * multi-gate passes whose in-tile set has no high digit (a run spans the whole register,
    D > 2^32), with run-digit controls on the top qubits, on the labelled state against the
    oracle's short-circuit evaluator;
  * every target qudit x {Haar U(d), controlled increment with a high / low-stride control,
    phase} applied to the index-labelled state, checked at sampled windows against the
    oracle's one-index evaluator (O-2, PAPER.md:222 row v of U times the class vector), then
    undone with the adjoint (back to the labels);
  * the whole circuit followed by its adjoint returns to e_0 (closed form), norm preserved.
Tolerances: normalised states 1e-10 (north_star); the labelled state (values up to 4.8e9)
relative 1e-13 (R15), permutations bit-exact."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

from oracle import blocksim as O2  # noqa: E402
from sv_inputs import (Gate, config_circuit, adjoint_circuit, haar_unitary, shift_x,  # noqa: E402
                       phase_gate, labelled_state)

CHUNK = 1 << 27          # 2 GB of complex128


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2410_17876_b200 as P
    return P


def _upload_labelled(st, D):
    for first in range(0, D, CHUNK):
        st.set_amplitudes(first, labelled_state(first, min(CHUNK, D - first)))


def _compare_full(st, ref):
    D = ref.size
    worst = 0.0
    buf = np.empty(CHUNK, dtype=np.complex128)
    for first in range(0, D, CHUNK):
        n = min(CHUNK, D - first)
        got = st.amplitudes(first, n, buf[:n])
        worst = max(worst, float(np.max(np.abs(got - ref[first:first + n]))))
    return worst


def _windows(D, rng, nwin=48, width=1024):
    starts = np.sort(rng.integers(0, D - width, size=nwin))
    starts[0], starts[-1] = 0, D - width          # include both ends of the register
    return starts, width


def _sample(st, starts, width):
    return np.concatenate([st.amplitudes(int(s), width) for s in starts])


def _idx(starts, width):
    return (starts[:, None] + np.arange(width)[None, :]).ravel().astype(np.uint64)


def _prefix_parity(P, cfg, ngates, block=False):
    dims, gates = config_circuit(cfg, ngates=ngates)
    ref = O2.run(dims, gates)                       # host O-2 on the full register
    with P.State(dims) as st:
        st.apply_circuit(gates, fuse=True, block=block)
        err = _compare_full(st, ref)
        nrm = st.norm()
    del ref
    assert err <= 1e-10, err
    assert abs(nrm - 1.0) <= 1e-10


def _labelled_gates(P, cfg):
    dims = config_circuit(cfg, ngates=0)[0]
    n, D = len(dims), int(np.prod(dims))
    rng = np.random.default_rng(100 + cfg)
    starts, width = _windows(D, rng)
    idx = _idx(starts, width)
    exp_lab = np.empty(idx.size, dtype=np.complex128)
    exp_lab.real = idx.astype(np.float64) + 1.0
    exp_lab.imag = -(idx.astype(np.float64) + 1.0) / 2.0
    b = np.cumprod([1] + dims[:-1]).astype(np.float64)
    with P.State(dims) as st:
        _upload_labelled(st, D)
        assert np.array_equal(_sample(st, starts, width), exp_lab)
        # pass 1: permutations (state stays exactly labelled); pass 2: general and phase gates
        for t in [t for t in range(n)] + [t + n for t in range(n)]:
            general = t >= n
            t = t % n
            d = dims[t]
            # rounding scale of a class: its largest label (members differ by multiples of b_t)
            scale = idx.astype(np.float64) + d * b[t] + 1.0
            hi = (t + 1) % n if (t + 1) % n != t else 0
            if general:
                cases = [Gate(t, (), (), haar_unitary(d, rng), "haar"),
                         Gate(t, (), (), phase_gate(rng.uniform(0, 6.28, size=d)), "phase")]
            else:
                cases = [Gate(t, (hi,), (dims[hi] - 1,), shift_x(d, 1), "cinc_hi"),
                         Gate(t, (0 if t != 0 else 1,), (1,), shift_x(d, 1), "cinc_lo")]
            for g in cases:
                st.apply_gate(g.target, g.U, g.ctrl, g.vals)
                got = _sample(st, starts, width)
                exp = O2.gate_output_labelled(dims, g, idx)
                if g.name.startswith("cinc"):
                    assert np.array_equal(got, exp), (t, g.name)
                else:
                    rel = np.max(np.abs(got - exp) / scale)
                    assert rel <= 1e-13, (t, g.name, rel)
                # undo with the adjoint: back to the labels
                st.apply_gate(g.target, g.U.conj().T, g.ctrl, g.vals)
                back = _sample(st, starts, width)
                if g.name.startswith("cinc"):
                    assert np.array_equal(back, exp_lab), (t, g.name)
                else:
                    assert np.max(np.abs(back - exp_lab) / scale) <= 1e-13, (t, g.name)
            if general and t % 8 == 7:
                _upload_labelled(st, D)      # reset the accumulated rounding of the round trips


def _adjoint_return(P, cfg, block=False):
    dims, gates = config_circuit(cfg)
    with P.State(dims) as st:
        st.apply_circuit(gates, fuse=True, block=block)
        nrm = st.norm()
        st.apply_circuit(adjoint_circuit(gates), fuse=True, block=block)
        a0 = st.amplitudes(0, 4096)
        D = int(np.prod(dims))
        tail = st.amplitudes(D - 4096, 4096)
        nrm2 = st.norm()
    assert abs(nrm - 1.0) <= 1e-10 and abs(nrm2 - 1.0) <= 1e-10
    assert abs(a0[0] - 1.0) <= 1e-10
    assert np.max(np.abs(a0[1:])) <= 1e-10 and np.max(np.abs(tail)) <= 1e-10


def test_c3_prefix_parity_full_register(P):
    _prefix_parity(P, 3, 60)


def test_c3_labelled_every_target(P):
    _labelled_gates(P, 3)


def test_c3_circuit_then_adjoint(P):
    _adjoint_return(P, 3)


def test_c4_prefix_parity_full_register(P):
    _prefix_parity(P, 4, 4)


def test_c4_labelled_every_target(P):
    _labelled_gates(P, 4)


def test_c4_circuit_then_adjoint(P):
    _adjoint_return(P, 4)


def test_c4_block_prefix_parity_full_register(P):
    """The bench's circuit-driver mode (SV_BLOCK, default pass configuration) on the first 48
    gates of c4 (merges, pair gates, multi-gate passes) vs O-2 on the whole register."""
    _prefix_parity(P, 4, 48, block=True)


def test_c4_block_circuit_then_adjoint(P):
    """The bench's whole timed circuit (SV_BLOCK) and its adjoint return to e_0."""
    _adjoint_return(P, 4, block=True)


def test_c3_block_circuit_then_adjoint(P):
    _adjoint_return(P, 3, block=True)


def test_c4_block_run_digit_controls_labelled(P):
    """Two-gate SV_BLOCK passes whose targets all lie in the low prefix (q_0..q_2), so the
    in-tile set has no high digit and a tile run spans the register (D = 4.78e9 > 2^32):
    controls on q_20 / q_21 have b_c d_c >= 2^31 (per-tile threshold), on q_6 / q_13 below it.
    Windows straddle the digit changes of q_20 and q_21 (D/4, D/2, 3D/4), where a tile holds
    both control values.  Checked on the labelled state against the oracle's short-circuit
    evaluator; regression for the 32-bit control modulus."""
    dims = config_circuit(4, ngates=0)[0]
    D = int(np.prod(dims))
    rng = np.random.default_rng(404)
    starts, width = _windows(D, rng, nwin=24)
    extra = np.array([D // 4 - width // 2, D // 2 - width // 2, 3 * D // 4 - width // 2,
                      D // 2 - 4000, D // 2 + 3000], dtype=np.int64)
    starts = np.sort(np.concatenate([starts, extra]))
    idx = _idx(starts, width)
    b = np.cumprod([1] + dims[:-1]).astype(np.float64)
    scale = idx.astype(np.float64) + float(np.sum(np.array(dims) * b)) + 1.0
    H = lambda d: haar_unitary(d, rng)                  # noqa: E731
    cases = [
        ("cinc_q21", [Gate(0, (), (), H(5)), Gate(1, (21,), (1,), shift_x(5, 1))]),
        ("haar_q20_v0", [Gate(1, (), (), H(5)), Gate(2, (20,), (0,), H(4))]),
        ("haar_q13_q21", [Gate(2, (), (), shift_x(4, 1)), Gate(0, (13, 21), (1, 0), H(5))]),
        ("haar_q6_q20", [Gate(0, (), (), H(5)), Gate(1, (6, 20), (2, 1), H(5))]),
    ]
    exp_lab = np.concatenate([labelled_state(int(s0), width) for s0 in starts])
    with P.State(dims) as st:
        _upload_labelled(st, D)                     # once: each case is undone by its adjoint
        for name, gates in cases:
            l0 = st.info().kernel_launches
            st.apply_circuit(gates, fuse=True, block=True)
            assert st.info().kernel_launches - l0 == 1, name       # one multi-gate pass
            got = _sample(st, starts, width)
            exp = O2.circuit_output_labelled(dims, gates, idx)
            rel = float(np.max(np.abs(got - exp) / scale))
            assert rel <= 1e-13, (name, rel)
            st.apply_circuit(adjoint_circuit(gates), fuse=True, block=True)
            back = _sample(st, starts, width)
            assert float(np.max(np.abs(back - exp_lab) / scale)) <= 1e-13, name


def test_c3_many_controls_labelled(P):
    """multi-controlled gates (3 and 4 controls, on low-stride and high-stride
    digits, with values other than the top one) at full c3 size, through the single-gate kernels
    and through SV_BLOCK passes, on the index-labelled state against the oracle's one-index
    evaluator (only control-satisfying classes change)."""
    dims = config_circuit(3, ngates=0)[0]                # [3]*8 + [2]*16
    n, D = len(dims), int(np.prod(dims))
    rng = np.random.default_rng(303)
    starts, width = _windows(D, rng)
    idx = _idx(starts, width)
    exp_lab = np.empty(idx.size, dtype=np.complex128)
    exp_lab.real = idx.astype(np.float64) + 1.0
    exp_lab.imag = -(idx.astype(np.float64) + 1.0) / 2.0
    b = np.cumprod([1] + dims[:-1]).astype(np.float64)
    # permutations first: they keep the state exactly labelled (the general gates' round
    # trips leave rounding behind)
    cases = [
        Gate(5, (1, 4, 17), (0, 2, 1), shift_x(3, 2), "perm_3ctrl"),
        Gate(22, (0, 1, 2, 15), (2, 2, 0, 1), shift_x(2, 1), "perm_4ctrl"),
        Gate(9, (0, 3, 20), (2, 1, 1), haar_unitary(2, rng), "haar_3ctrl"),
        Gate(2, (0, 8, 12, 23), (1, 1, 0, 1), haar_unitary(3, rng), "haar_4ctrl"),
    ]
    with P.State(dims) as st:
        for block in (False, True):
            _upload_labelled(st, D)
            for g in cases:
                if block:
                    st.apply_circuit([g], block=True)
                else:
                    st.apply_gate(g.target, g.U, g.ctrl, g.vals)
                got = _sample(st, starts, width)
                exp = O2.gate_output_labelled(dims, g, idx)
                if g.name.startswith("perm"):
                    assert np.array_equal(got, exp), (block, g.name)
                else:
                    scale = idx.astype(np.float64) + dims[g.target] * b[g.target] + 1.0
                    assert np.max(np.abs(got - exp) / scale) <= 1e-13, (block, g.name)
                st.apply_gate(g.target, g.U.conj().T, g.ctrl, g.vals)       # undo
                back = _sample(st, starts, width)
                if g.name.startswith("perm"):
                    assert np.array_equal(back, exp_lab), (block, g.name)
