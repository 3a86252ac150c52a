"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the block-simulation method (§2): it only
builds the *inputs* the method consumes — registers (dims lists), gate matrices and
circuits (ordered gate lists), and initial states.  Both sides (oracle/ and the CUDA
path in paper_2410_17876_b200/) receive exactly the same objects from here; neither
side imports the other.

Conventions (SURVEY.md §0, C1–C6):
  * dims are listed q_0 first; q_0 is the least-significant digit.
  * a gate is (target, ctrl, vals, U) with U a d×d complex128 matrix, y = U x
    (column j of U is the image of |j>).
  * a control (c, v) fires when digit c of the basis index equals v.
"""
from .gates import (Gate, shift_x, clock_z, fourier, hadamard, t_gate, phase_gate,
                    haar_unitary, special_unitary, permutation_matrix, adjoint_gate)
from .circuits import (config_dims, config_circuit, CONFIG_NAMES, ghz_circuit,
                       worked_example, random_circuit, adjoint_circuit, labelled_state,
                       random_state, register_size)

__all__ = [
    "Gate", "shift_x", "clock_z", "fourier", "hadamard", "t_gate", "phase_gate",
    "haar_unitary", "special_unitary", "permutation_matrix", "adjoint_gate",
    "config_dims", "config_circuit", "CONFIG_NAMES", "ghz_circuit", "worked_example",
    "random_circuit", "adjoint_circuit", "labelled_state", "random_state", "register_size",
]
