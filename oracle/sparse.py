"""O-3: the paper's sparse block method as a plain Python dict simulator.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Follows PAPER.md:222 (§2.3) step by step:
"we first identify all basis states with non-zero amplitudes in a given class.  Each of these
basis states will correspond to a particular column of the unitary U ... select columns
corresponding to non-zero basis states in a given class, perform the scalar product of the
columns with the corresponding state amplitudes, and find the sum of these column vectors."
Classes are keyed by their member with target digit 0 (i - v b_k, v = floor(i/b_k) mod d_k,
PAPER.md:235), controls are checked per stored key (only states satisfying the
control conditions are transformed), and amplitudes with |a| < eps are dropped afterwards
(reading R18: the paper gives no threshold; eps = 1e-12 as in SPEC.md:128).

Pinned by tests/test_oracle_pins.py against O-2 (dense) on small registers and against the
GHZ closed form at the paper's maxima (62 qubits, 39 qutrits, 31 ququads, 27 ququints).
"""
from __future__ import annotations

EPS = 1e-12


def strides(dims):
    b, p = [], 1
    for d in dims:
        b.append(p)
        p *= int(d)
    return b, p


def apply(state: dict, dims, gate, eps: float = EPS) -> dict:
    b, _ = strides(dims)
    t = gate.target
    d, bt = int(dims[t]), b[t]
    U = gate.U
    out: dict = {}
    classes: dict = {}
    for i, a in state.items():
        ok = all((i // b[c]) % dims[c] == v for c, v in zip(gate.ctrl, gate.vals))
        if not ok:                                   # unmet controls: untouched
            out[i] = out.get(i, 0) + a
            continue
        v = (i // bt) % d
        classes.setdefault(i - v * bt, {})[v] = a
    for base, members in classes.items():
        for k in range(d):                           # sum over the non-zero members' columns
            y = 0j
            for j, xj in members.items():
                y += complex(U[k, j]) * xj
            if y != 0:
                out[base + k * bt] = out.get(base + k * bt, 0) + y
    return {i: a for i, a in out.items() if abs(a) >= eps}


def run(dims, gates, init: int = 0, eps: float = EPS) -> dict:
    state = {int(init): 1.0 + 0j}
    for g in gates:
        state = apply(state, dims, g, eps)
    return state
