"""O-1: Kronecker brute force — the plain definition psi_out = M_G ... M_1 psi_0.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The block method "completely eliminated tensor products and matrix multiplications"
 but must reach exactly the state the full D×D operators give.  This file
builds those operators on purpose, for D <= 4096:

  uncontrolled gate on q_k:  M = I_{r_k} ⊗ U ⊗ I_{b_k}
  controlled gate:           M = I_D + ⊗_{t=n-1..0} B_t,  B_t = |v_t><v_t| on a control,
                             (U - I) on the target, I elsewhere

The Kronecker order runs from q_{n-1} (left factor) down to q_0 (right factor), which is
what "q_0 is the least significant qudit" means for the index i = sum q_k b_k.
"""
from __future__ import annotations

import numpy as np

CAP = 4096


def _kron_all(factors):
    M = np.ones((1, 1), dtype=np.complex128)
    for F in factors:
        M = np.kron(M, F)
    return M


def full_operator(dims, target, ctrl, vals, U):
    dims = [int(d) for d in dims]
    n = len(dims)
    D = int(np.prod(dims))
    if D > CAP:
        raise ValueError("Kronecker oracle capped at D <= %d" % CAP)
    U = np.asarray(U, dtype=np.complex128)
    if len(ctrl) == 0:
        factors = [U if t == target else np.eye(dims[t], dtype=np.complex128)
                   for t in range(n - 1, -1, -1)]
        return _kron_all(factors)
    cmap = dict(zip(ctrl, vals))
    factors = []
    for t in range(n - 1, -1, -1):
        if t == target:
            factors.append(U - np.eye(dims[t], dtype=np.complex128))
        elif t in cmap:
            P = np.zeros((dims[t], dims[t]), dtype=np.complex128)
            P[cmap[t], cmap[t]] = 1.0
            factors.append(P)
        else:
            factors.append(np.eye(dims[t], dtype=np.complex128))
    return np.eye(D, dtype=np.complex128) + _kron_all(factors)


def run(dims, gates, psi0=None):
    """Apply the gates one after another as full matrix-vector products."""
    D = int(np.prod(dims))
    if psi0 is None:
        psi = np.zeros(D, dtype=np.complex128)
        psi[0] = 1.0
    else:
        psi = np.array(psi0, dtype=np.complex128, copy=True)
    for g in gates:
        psi = full_operator(dims, g.target, g.ctrl, g.vals, g.U) @ psi
    return psi
