"""Work count of the benchmark metric, written from its definition.  TEST INFRASTRUCTURE ONLY
(see oracle/__init__.py): bench.py's cpu_baseline leg and `--impl reference` count the
amplitude updates of the oracle's runs with it, so neither loads the product library.

SURVEY.md §8 (notation): a gate on q_t with controls C visits F = D / (d_t * prod_{c in C} d_c)
control-satisfying classes; the amplitudes it can change are
T = F * (number of class members that move or scale).  For a general gate every member does
(T = F d_t); a gate whose every column of U has exactly one non-zero entry (the §2.1 phase and
§2.2 permutation gates) leaves member j unchanged when U maps |j> to itself
with coefficient exactly 1.  The metric is amplitude-updates/s = sum_g T_g / time
(BASELINE.json metric); algorithmic HBM bytes are 32 B x T for complex128.
"""
from __future__ import annotations

import numpy as np


def touched(dims, gate) -> int:
    """T of one gate on the register `dims` (q_0 first)."""
    d = int(dims[gate.target])
    D = 1
    for x in dims:
        D *= int(x)
    cprod = 1
    for c in gate.ctrl:
        cprod *= int(dims[c])
    F = D // (d * cprod)
    U = np.asarray(gate.U, dtype=np.complex128).reshape(d, d)
    nz = U != 0
    monomial = bool(np.all(nz.sum(axis=0) == 1) and np.all(nz.sum(axis=1) == 1))
    if not monomial:
        return F * d
    moving = 0
    for j in range(d):
        i = int(np.flatnonzero(nz[:, j])[0])       # U|j> = U[i, j] |i>
        if i != j or U[i, j] != 1.0:
            moving += 1
    return F * moving


def circuit_touched(dims, gates) -> int:
    return sum(touched(dims, g) for g in gates)
