"""Seeded synthetic registers, circuits and states (BASELINE.json configs).

The paper measures on named algorithm circuits that are not available
here and whose gate lists the paper does not give; these seeded synthetic circuits stand
in for them.  Generator: numpy Generator(PCG64(seed)),
seed = 1000 + config number.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from .gates import (Gate, shift_x, clock_z, fourier, hadamard, t_gate, haar_unitary,
                    special_unitary, adjoint_gate, permutation_matrix, phase_gate)

CONFIG_NAMES = {
    1: "c1_hybrid_2x4_3x2_200g",
    2: "c2_12qutrits_depth500",
    3: "c3_16qubits_8qutrits_1000g",
    4: "c4_mixed_22qudits_300g",
    5: "c5_25qubits_6qutrits_200g_sharded",
}


def config_dims(cfg: int, nqubits: int | None = None) -> List[int]:
    """q_0-first dims; qubits are the most-significant digits."""
    if cfg == 1:
        return [2, 2, 2, 2, 3, 3]
    if cfg == 2:
        return [3] * 12
    if cfg == 3:
        return [3] * 8 + [2] * (16 if nqubits is None else nqubits)
    if cfg == 4:
        return [5, 5, 4, 4, 4, 4, 3, 3, 3, 3, 3, 3] + [2] * (10 if nqubits is None else nqubits)
    if cfg == 5:
        return [3] * 6 + [2] * (25 if nqubits is None else nqubits)
    raise ValueError(cfg)


def register_size(dims: Sequence[int]) -> int:
    D = 1
    for d in dims:
        D *= int(d)
    return D


def _cinc(c: int, t: int, dims) -> Gate:
    """Controlled increment: X_{+1} on t when q_c = d_c - 1 (reading R3)."""
    return Gate(t, (c,), (dims[c] - 1,), shift_x(dims[t], 1), "cinc")


def _c1(rng):
    dims = config_dims(1)
    n = len(dims)
    gates = []
    for _ in range(200):
        kind = int(rng.integers(5))
        t = int(rng.integers(n))
        d = dims[t]
        if kind == 0:
            gates.append(Gate(t, (), (), haar_unitary(d, rng), "haar"))
        elif kind == 1:
            gates.append(Gate(t, (), (), shift_x(d, int(rng.integers(1, d))), "x"))
        elif kind == 2:
            gates.append(Gate(t, (), (), clock_z(d, int(rng.integers(1, d))), "z"))
        elif kind == 3:
            gates.append(Gate(t, (), (), fourier(d), "f"))
        else:
            c, t = (int(x) for x in rng.choice(n, size=2, replace=False))
            gates.append(_cinc(c, t, dims))
    return dims, gates


def _c2(rng, layers=500):
    dims = config_dims(2)
    n = len(dims)
    gates = []
    for layer in range(layers):
        if layer % 2 == 0:
            for q in range(n):
                if rng.random() < 0.5:
                    gates.append(Gate(q, (), (), fourier(3), "f"))
                else:
                    gates.append(Gate(q, (), (), special_unitary(3, rng), "su3"))
        else:
            for _ in range(n):
                c, t = (int(x) for x in rng.choice(n, size=2, replace=False))
                gates.append(_cinc(c, t, dims))
    return dims, gates


def _c3(rng, ngates=1000, nqubits=None):
    dims = config_dims(3, nqubits)
    qutrits = list(range(8))
    qubits = list(range(8, len(dims)))
    gates = []
    for _ in range(ngates):
        kind = int(rng.integers(8))
        if kind == 0:
            gates.append(Gate(int(rng.choice(qubits)), (), (), hadamard(), "h"))
        elif kind == 1:
            gates.append(Gate(int(rng.choice(qubits)), (), (), t_gate(), "t"))
        elif kind == 2:
            c, t = (int(x) for x in rng.choice(qubits, size=2, replace=False))
            gates.append(_cinc(c, t, dims))
        elif kind == 3:
            gates.append(Gate(int(rng.choice(qutrits)), (), (), fourier(3), "f"))
        elif kind == 4:
            gates.append(Gate(int(rng.choice(qutrits)), (), (), shift_x(3, int(rng.integers(1, 3))), "x"))
        elif kind == 5:
            gates.append(Gate(int(rng.choice(qutrits)), (), (), special_unitary(3, rng), "su3"))
        elif kind == 6:
            gates.append(_cinc(int(rng.choice(qubits)), int(rng.choice(qutrits)), dims))
        else:
            c, t = (int(x) for x in rng.choice(qutrits, size=2, replace=False))
            gates.append(_cinc(c, t, dims))
    return dims, gates


def _c4(rng, ngates=300, nqubits=None):
    dims = config_dims(4, nqubits)
    n = len(dims)
    gates = []
    for _ in range(ngates):
        if rng.random() < 0.5:
            t = int(rng.integers(n))
            gates.append(Gate(t, (), (), haar_unitary(dims[t], rng), "haar"))
        else:
            t = int(rng.integers(n))
            others = [q for q in range(n) if q != t]
            c = int(rng.choice(others))
            gates.append(_cinc(c, t, dims))
    return dims, gates


def _c5(rng, ngates=200, nqubits=None, nsharded=3):
    dims = config_dims(5, nqubits)
    n = len(dims)
    qutrits = list(range(6))
    qubits = list(range(6, n))
    sharded = qubits[-nsharded:]
    local_q = qubits[:-nsharded]
    n_sh = ngates // 5
    is_sh = np.zeros(ngates, dtype=bool)
    is_sh[rng.choice(ngates, size=n_sh, replace=False)] = True
    gates = []
    for i in range(ngates):
        if is_sh[i]:
            t = int(rng.choice(sharded))
            kind = int(rng.integers(3))
            if kind == 0:
                gates.append(Gate(t, (), (), hadamard(), "h"))
            elif kind == 1:
                gates.append(Gate(t, (), (), haar_unitary(2, rng), "haar"))
            else:
                gates.append(_cinc(int(rng.choice(local_q)), t, dims))
        else:
            kind = int(rng.integers(5))
            if kind == 0:
                gates.append(Gate(int(rng.choice(qutrits)), (), (), fourier(3), "f"))
            elif kind == 1:
                gates.append(Gate(int(rng.choice(qutrits)), (), (), special_unitary(3, rng), "su3"))
            elif kind == 2:
                t = int(rng.choice(local_q))
                c = int(rng.choice([q for q in qubits if q != t]))
                gates.append(_cinc(c, t, dims))
            elif kind == 3:
                gates.append(_cinc(int(rng.choice(qubits)), int(rng.choice(qutrits)), dims))
            else:
                c, t = (int(x) for x in rng.choice(qutrits, size=2, replace=False))
                gates.append(_cinc(c, t, dims))
    return dims, gates


def config_circuit(cfg: int, ngates: int | None = None, nqubits: int | None = None):
    """(dims, gates) for BASELINE.json config cfg (1-based), seed 1000+cfg.

    ngates / nqubits shrink the circuit / register (same recipe) for bounded samples.
    """
    rng = np.random.Generator(np.random.PCG64(1000 + cfg))
    if cfg == 1:
        dims, g = _c1(rng)
    elif cfg == 2:
        dims, g = _c2(rng)
    elif cfg == 3:
        dims, g = _c3(rng, nqubits=nqubits)
    elif cfg == 4:
        dims, g = _c4(rng, nqubits=nqubits)
    elif cfg == 5:
        dims, g = _c5(rng, nqubits=nqubits)
    else:
        raise ValueError(cfg)
    if ngates is not None:
        g = g[:ngates]
    return dims, g


def ghz_circuit(d: int, n: int):
    """Generalised GHZ fan (reading R5): F_d on q_0, then for k=1..n-1, v=1..d-1:
    X_{+v} on q_k controlled by q_{k-1} = v.  Final state sum_v |v..v>/sqrt(d)."""
    dims = [d] * n
    gates = [Gate(0, (), (), fourier(d), "f")]
    for k in range(1, n):
        for v in range(1, d):
            gates.append(Gate(k, (k - 1,), (v,), shift_x(d, v), "cx"))
    return dims, gates


def worked_example():
    """PAPER.md:246-296 (§2.5): dims [2,3]; generalised Hadamard on q_1 (depth 0), then CX
    with control q_1 at its highest state 2 and target q_0 incremented by +1 (depth 1)."""
    dims = [2, 3]
    gates = [Gate(1, (), (), fourier(3), "f"),
             Gate(0, (1,), (2,), shift_x(2, 1), "cx")]
    return dims, gates


def random_circuit(seed: int, dims: Sequence[int], depth: int, max_ctrl: int = 2):
    """Seeded random circuit over all gate kinds (phase / permutation / general), each with
    0..max_ctrl value controls (SPEC.md:587 acceptance-sweep recipe)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = len(dims)
    gates = []
    for _ in range(depth):
        t = int(rng.integers(n))
        d = dims[t]
        kind = int(rng.integers(6))
        if kind == 0:
            U, nm = haar_unitary(d, rng), "haar"
        elif kind == 1:
            U, nm = permutation_matrix(rng.permutation(d)), "perm"
        elif kind == 2:
            U, nm = phase_gate(rng.uniform(0, 2 * np.pi, size=d)), "phase"
        elif kind == 3:
            U, nm = fourier(d), "f"
        elif kind == 4:
            U, nm = shift_x(d, int(rng.integers(1, d))), "x"
        else:
            U, nm = clock_z(d, int(rng.integers(1, d))), "z"
        nc = int(rng.integers(0, min(max_ctrl, n - 1) + 1))
        others = [q for q in range(n) if q != t]
        ctrl = tuple(int(c) for c in rng.choice(others, size=nc, replace=False)) if nc else ()
        vals = tuple(int(rng.integers(dims[c])) for c in ctrl)
        gates.append(Gate(t, ctrl, vals, U, nm))
    return list(dims), gates


def adjoint_circuit(gates):
    return [adjoint_gate(g) for g in reversed(gates)]


def labelled_state(first: int, count: int) -> np.ndarray:
    """Index-labelled state: Re psi_i = i+1, Im psi_i = -(i+1)/2 (exact in fp64 for i < 2^52,
    no zero component).  Not normalised; used for bit-exact index-mapping tests."""
    i = np.arange(first, first + count, dtype=np.float64)
    out = np.empty(count, dtype=np.complex128)
    out.real = i + 1.0
    out.imag = -(i + 1.0) / 2.0
    return out


def random_state(D: int, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    v = rng.standard_normal(D) + 1j * rng.standard_normal(D)
    return (v / np.linalg.norm(v)).astype(np.complex128)
