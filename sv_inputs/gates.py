"""Gate-matrix constructors (inputs only).

Matrices are d×d complex128, row-major, acting as y = U x on a fibre x whose j-th
entry is the amplitude with the target digit equal to j.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Tuple

import numpy as np


@dataclass(frozen=True)
class Gate:
    """A (multi-)controlled single-qudit gate: two control lists as in PAPER.md:230."""
    target: int
    ctrl: Tuple[int, ...]
    vals: Tuple[int, ...]
    U: np.ndarray = field(compare=False)
    name: str = "u"

    @property
    def d(self) -> int:
        return int(self.U.shape[0])


def shift_x(d: int, a: int = 1) -> np.ndarray:
    """Generalised NOT X_{+a}: |j> -> |(j+a) mod d> (§2.2)."""
    U = np.zeros((d, d), dtype=np.complex128)
    for j in range(d):
        U[(j + a) % d, j] = 1.0
    return U


def clock_z(d: int, power: int = 1) -> np.ndarray:
    """Generalised Z (clock) = diag(w^{j*power}), w = exp(2*pi*i/d) (PAPER.md:188 names it;
    matrix per DESIGN.md reading R2)."""
    j = np.arange(d)
    return np.diag(np.exp(2j * np.pi * j * power / d)).astype(np.complex128)


def fourier(d: int) -> np.ndarray:
    """Generalised Hadamard F_d[k][j] = w^{jk}/sqrt(d) (PAPER.md:198 names it; reading R2).
    Entries of column 0 are exactly 1/sqrt(d) (built as 1.0/np.sqrt(d))."""
    k = np.arange(d).reshape(-1, 1)
    j = np.arange(d).reshape(1, -1)
    U = np.exp(2j * np.pi * ((j * k) % d) / d) / np.sqrt(d)
    U[:, 0] = 1.0 / np.sqrt(d)
    U[0, :] = 1.0 / np.sqrt(d)
    return U.astype(np.complex128)


def hadamard() -> np.ndarray:
    s = 1.0 / np.sqrt(2.0)
    return np.array([[s, s], [s, -s]], dtype=np.complex128)


def t_gate() -> np.ndarray:
    return np.diag([1.0, np.exp(1j * np.pi / 4)]).astype(np.complex128)


def phase_gate(angles) -> np.ndarray:
    return np.diag(np.exp(1j * np.asarray(angles, dtype=np.float64))).astype(np.complex128)


def permutation_matrix(sigma) -> np.ndarray:
    """Column j has its single 1 in row sigma[j]: |j> -> |sigma(j)>."""
    d = len(sigma)
    U = np.zeros((d, d), dtype=np.complex128)
    for j, s in enumerate(sigma):
        U[s, j] = 1.0
    return U


def haar_unitary(d: int, rng: np.random.Generator) -> np.ndarray:
    """Haar-random U(d): QR of a complex Ginibre matrix with the R-diagonal phase fix
    (reading R12)."""
    z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / np.sqrt(2.0)
    q, r = np.linalg.qr(z)
    ph = np.diagonal(r) / np.abs(np.diagonal(r))
    return (q * ph[np.newaxis, :]).astype(np.complex128)


def special_unitary(d: int, rng: np.random.Generator) -> np.ndarray:
    """Haar U(d) rescaled to det 1 (principal branch of det^{-1/d})."""
    U = haar_unitary(d, rng)
    det = np.linalg.det(U)
    return (U * np.exp(-1j * np.angle(det) / d)).astype(np.complex128)


def adjoint_gate(g: Gate) -> Gate:
    return Gate(g.target, g.ctrl, g.vals, np.ascontiguousarray(g.U.conj().T), g.name + "^dag")
