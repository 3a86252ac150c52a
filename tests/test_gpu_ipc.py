"""Sharded mode in real processes: P = 2 / 4 ranks, each its own process and CUDA context, over
the fused peer-memory transport (sv_create_sharded_ipc).  On the one-GPU
box every rank's slice lives on cuda:0 and the ranks reach each other's slices through CUDA IPC
mappings, exactly as on an 8-GPU node where the mappings go over NVLink.  The kernels never
wait on one another (host barriers order them), so ranks sharing one GPU are safe.

Covered: exchanges (rule iii, fused gate + exchange), rank relabelling (v), local phases (iv),
qubit remapping (vi, SV_OPT_SHARD_SWAP on / off), sharded-control predicates (ii), the
collective readback and norm, a second circuit after a readback (layout restored), complex64;
against O-2 on the whole register (1e-12; permutations on the labelled state bit-exact)."""
import os
import pickle
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import blocksim as O2  # noqa: E402
from sv_inputs import (Gate, hadamard, haar_unitary, shift_x, fourier, t_gate, random_circuit,  # noqa: E402
                       random_state, labelled_state, config_circuit, adjoint_circuit)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "_ipc_worker.py")


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2410_17876_b200 as P
    return P


def _run(P, job, nranks, timeout=300):
    job = dict(job)
    job["nranks"] = nranks
    job["ipc_id"] = P.sv.ipc_unique_id()
    with tempfile.TemporaryDirectory() as td:
        job["out"] = os.path.join(td, "out.pkl")
        jp = os.path.join(td, "job.pkl")
        pickle.dump(job, open(jp, "wb"))
        env = dict(os.environ, SV_COMM_TIMEOUT_S="120")
        procs = [subprocess.Popen([sys.executable, WORKER, jp, str(r)], stdout=subprocess.PIPE,
                                  stderr=subprocess.PIPE, text=True, env=env) for r in range(nranks)]
        outs = []
        for p in procs:
            try:
                o, e = p.communicate(timeout=timeout)
            except subprocess.TimeoutExpired:
                for q in procs:
                    q.kill()
                raise
            outs.append((p.returncode, o, e))
        for r, (rc, o, e) in enumerate(outs):
            assert rc == 0, f"rank {r} failed:\n{e[-3000:]}"
        return pickle.load(open(job["out"], "rb"))


def _mixed_circuit(dims, nranks, seed):
    """Random gates over every qudit (sharded targets and controls included) plus the explicit
    sharded cases: Haar / H on sharded qubits (exchange or remap), X on a sharded qubit (relabel),
    T / Z on sharded qubits (local phase), local gates controlled on sharded qubits."""
    rng = np.random.default_rng(seed)
    n = len(dims)
    _, gates = random_circuit(seed, dims, 90, max_ctrl=2)
    top = n - 1
    gates += [Gate(top, (), (), hadamard()), Gate(top - 1, (0,), (2,), haar_unitary(2, rng)),
              Gate(top, (), (), shift_x(2, 1)), Gate(top - 1, (), (), t_gate()),
              Gate(1, (top, top - 1), (1, 0), fourier(dims[1])), Gate(top, (top - 1,), (1,), shift_x(2, 1)),
              Gate(top - 1, (2,), (1,), haar_unitary(2, rng))]
    return gates


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("swap", [1, 0])
def test_ipc_sharded_matches_oracle(P, nranks, swap):
    dims = [3, 3, 4, 2, 2, 2, 2, 2, 2]
    D = int(np.prod(dims))
    gates = _mixed_circuit(dims, nranks, 500 + nranks)
    psi0 = random_state(D, 21)
    ref = O2.run(dims, gates, psi0)
    extra = gates[:30]
    for mode in ("block", "gate"):
        res = _run(P, {"dims": dims, "gates": gates, "psi0": psi0, "swap": swap, "mode": mode,
                       "extra": extra}, nranks)
        assert np.max(np.abs(res["psi"] - ref)) <= 1e-12, (mode, swap)
        assert abs(res["norm"] - 1.0) <= 1e-10
        assert res["exchanges"] > 0
        assert np.max(np.abs(res["psi_extra"] - O2.run(dims, extra, ref))) <= 1e-12, (mode, swap)


@pytest.mark.parametrize("nranks", [2, 4])
def test_ipc_labelled_permutations_bit_exact(P, nranks):
    """Permutations across shards (exchanges, relabels, remaps, sharded predicates) on the
    index-labelled state: bit-exact against O-2."""
    dims = [3, 3, 4, 2, 2, 2, 2, 2]
    D = int(np.prod(dims))
    n = len(dims)
    perm = [Gate(n - 1, (), (), shift_x(2, 1)), Gate(n - 2, (2,), (3,), shift_x(2, 1)),
            Gate(2, (n - 1,), (1,), shift_x(4, 3)), Gate(5, (n - 2, 0), (0, 1), shift_x(2, 1)),
            Gate(n - 1, (2,), (1,), shift_x(2, 1)), Gate(n - 2, (0,), (2,), shift_x(2, 1)),
            Gate(2, (n - 2,), (1,), shift_x(4, 1)), Gate(5, (n - 1,), (0,), shift_x(2, 1))]
    lab = labelled_state(0, D)
    for swap in (1, 0):
        res = _run(P, {"dims": dims, "gates": perm, "psi0": lab, "swap": swap, "mode": "gate"}, nranks)
        assert np.array_equal(res["psi"], O2.run(dims, perm, lab)), swap


def test_ipc_sharded_complex64(P):
    """complex64 slices over the fused transport, within the derived fp32 bound (DESIGN R17)."""
    dims = [3, 4, 2, 2, 2, 2, 2, 2]
    D = int(np.prod(dims))
    gates = _mixed_circuit(dims, 4, 77)
    psi0 = random_state(D, 8)
    ref = O2.run(dims, gates, psi0)
    res = _run(P, {"dims": dims, "gates": gates, "psi0": psi0, "swap": 1, "mode": "block", "dtype": "c64"}, 4)
    bound = len(gates) * (2 * 4 + 1) * 2.0 * 2.0 ** -24 + 2 ** 0.5 * 2.0 ** -24
    assert np.linalg.norm(res["psi"] - ref) <= bound


def test_ipc_rank_failure_is_reported_not_hung(P):
    """A rank that never shows up: the others fail with SV_ERR_NCCL after SV_COMM_TIMEOUT_S
    instead of hanging (transport fault handling)."""
    code = ("import sys; sys.path.insert(0, %r); import paper_2410_17876_b200 as P\n"
            "try:\n    P.State.sharded_ipc([2, 2, 2], 0, 2, P.sv.ipc_unique_id())\n"
            "except P.SVError as e:\n    print('ERR', e.name)\n" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120,
                         env=dict(os.environ, SV_COMM_TIMEOUT_S="3"))
    assert "ERR SV_ERR_NCCL" in out.stdout, (out.stdout, out.stderr[-2000:])


@pytest.mark.parametrize("nranks", [2, 4])
def test_ipc_c5_recipe_reduced_register(P, nranks):
    """BASELINE config 5's recipe (6 qutrits + qubits, 200 gates, 20 % on the 3 top qubits,
    CNOTs controlled on sharded qubits) on a register reduced to 14 qubits (D = 1.2e7), sharded
    over P processes: vs O-2 on the whole register (SURVEY.md §8(c) fallback for c5)."""
    dims, gates = config_circuit(5, nqubits=14)
    ref = O2.run(dims, gates)
    for swap in (1, 0):
        res = _run(P, {"dims": dims, "gates": gates, "psi0": None, "swap": swap, "mode": "block"}, nranks,
                   timeout=600)
        assert np.max(np.abs(res["psi"] - ref)) <= 1e-10, swap
        assert abs(res["norm"] - 1.0) <= 1e-10


def test_ipc_c5_full_size_adjoint_return(P):
    """The full 391 GB config 5 on 8 GPUs (48.9 GB per rank; 4 GPUs: 97.8 GB): the circuit and its
    adjoint return to e_0 within 1e-10 (SURVEY.md §8(c) fallback when the host cannot hold O-2's
    copy).  Needs >= 4 GPUs (skipped on the one-GPU box)."""
    import torch
    ng = torch.cuda.device_count()
    if ng < 4:
        pytest.skip("needs 4 or 8 GPUs")
    nranks = 8 if ng >= 8 else 4
    dims, gates = config_circuit(5)
    res = _run(P, {"dims": dims, "gates": gates, "psi0": None, "swap": 1, "mode": "block",
                   "adjoint": adjoint_circuit(gates), "device_per_rank": True}, nranks, timeout=3000)
    assert abs(res["norm"] - 1.0) <= 1e-10 and abs(res["norm2"] - 1.0) <= 1e-10
    assert abs(res["head"][0] - 1.0) <= 1e-10
    assert np.max(np.abs(res["head"][1:])) <= 1e-10 and np.max(np.abs(res["tail"])) <= 1e-10


@pytest.mark.parametrize("nranks", [2, 4])
def test_ipc_overlapped_remap(P, nranks):
    """The overlapped remap across processes: the swap kernel on the comm stream reads and writes
    the partner's moving half while each rank's passes update its staying half; vs O-2."""
    from _circuits import overlap_circuit as _overlap_circuit
    dims = [3, 3, 4, 2, 2, 2, 2, 2, 2]
    gates = _overlap_circuit(dims, 41 + nranks, nranks)
    psi0 = random_state(int(np.prod(dims)), 10)
    ref = O2.run(dims, gates, psi0)
    res = _run(P, {"dims": dims, "gates": gates, "psi0": psi0, "swap": 1, "mode": "block", "overlap": 16}, nranks)
    assert np.max(np.abs(res["psi"] - ref)) <= 1e-12
    assert res["overlapped"] > 0
