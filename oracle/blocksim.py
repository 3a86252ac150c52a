"""ctypes binding of O-2 (oracle/blocksim.c).  TEST INFRASTRUCTURE ONLY (see __init__.py)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "blocksim.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_up = C.POINTER(C.c_uint64)


def build(force: bool = False) -> str:
    """Compile the oracle with the host compiler (plain -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-Wall", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        L.orc_apply.argtypes = [_dp, C.c_int, _ip, C.c_int, C.c_int, _ip, _ip, _dp]
        L.orc_apply_phase.argtypes = [_dp, C.c_int, _ip, C.c_int, C.c_int, _ip, _ip, _dp]
        L.orc_apply_shift.argtypes = [_dp, C.c_int, _ip, C.c_int, C.c_int, _ip, _ip, C.c_int]
        L.orc_run.argtypes = [_dp, C.c_int, _ip, C.c_int64, _ip, _ip, _ip, _ip, _dp]
        L.orc_norm.argtypes = [_dp, C.c_uint64]
        L.orc_norm.restype = C.c_double
        L.orc_strides.argtypes = [C.c_int, _ip, _up, _up]
        L.orc_gate_output_labelled.argtypes = [C.c_int, _ip, C.c_int, C.c_int, _ip, _ip, _dp,
                                               _up, C.c_int64, _dp]
        L.orc_circuit_output_labelled.argtypes = [C.c_int, _ip, C.c_int64, _ip, _ip, _ip, _ip, _dp,
                                                  _up, C.c_int64, _dp]
        L.orc_num_threads.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _c128(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    return a


def strides(dims):
    dims = _i32(dims)
    b = np.zeros(len(dims), dtype=np.uint64)
    D = np.zeros(1, dtype=np.uint64)
    if lib().orc_strides(len(dims), _ptr(dims, _ip), _ptr(b, _up), _ptr(D, _up)):
        raise OverflowError("register size overflows uint64")
    return [int(x) for x in b], int(D[0])


def apply(psi: np.ndarray, dims, gate) -> None:
    """In place: one (controlled) gate by the general §2.3 class rule."""
    assert psi.dtype == np.complex128 and psi.flags.c_contiguous
    dims_a = _i32(dims)
    ctrl = _i32(gate.ctrl if len(gate.ctrl) else [0])
    vals = _i32(gate.vals if len(gate.vals) else [0])
    U = _c128(gate.U)
    rc = lib().orc_apply(_ptr(psi.view(np.float64), _dp), len(dims_a), _ptr(dims_a, _ip),
                         int(gate.target), len(gate.ctrl), _ptr(ctrl, _ip), _ptr(vals, _ip),
                         _ptr(U.view(np.float64), _dp))
    if rc:
        raise ValueError("oracle rejected gate")


def apply_phase(psi, dims, target, diag, ctrl=(), vals=()):
    dims_a = _i32(dims)
    c = _i32(ctrl if len(ctrl) else [0])
    v = _i32(vals if len(vals) else [0])
    dg = _c128(diag)
    lib().orc_apply_phase(_ptr(psi.view(np.float64), _dp), len(dims_a), _ptr(dims_a, _ip),
                          int(target), len(ctrl), _ptr(c, _ip), _ptr(v, _ip),
                          _ptr(dg.view(np.float64), _dp))


def apply_shift(psi, dims, target, a, ctrl=(), vals=()):
    dims_a = _i32(dims)
    c = _i32(ctrl if len(ctrl) else [0])
    v = _i32(vals if len(vals) else [0])
    lib().orc_apply_shift(_ptr(psi.view(np.float64), _dp), len(dims_a), _ptr(dims_a, _ip),
                          int(target), len(ctrl), _ptr(c, _ip), _ptr(v, _ip), int(a))


def run(dims, gates, psi0=None) -> np.ndarray:
    """Apply a circuit from e_0 (or psi0) and return the final state."""
    _, D = strides(dims)
    if psi0 is None:
        psi = np.zeros(D, dtype=np.complex128)
        psi[0] = 1.0
    else:
        psi = np.array(psi0, dtype=np.complex128, copy=True)
    run_inplace(psi, dims, gates)
    return psi


def run_inplace(psi, dims, gates) -> None:
    if not gates:
        return
    dims_a = _i32(dims)
    targets = _i32([g.target for g in gates])
    nctrls = _i32([len(g.ctrl) for g in gates])
    cf = _i32([c for g in gates for c in g.ctrl] or [0])
    vf = _i32([v for g in gates for v in g.vals] or [0])
    Uf = np.ascontiguousarray(np.concatenate([np.asarray(g.U, np.complex128).ravel() for g in gates]))
    rc = lib().orc_run(_ptr(psi.view(np.float64), _dp), len(dims_a), _ptr(dims_a, _ip),
                       len(gates), _ptr(targets, _ip), _ptr(nctrls, _ip), _ptr(cf, _ip),
                       _ptr(vf, _ip), _ptr(Uf.view(np.float64), _dp))
    if rc:
        raise ValueError("oracle rejected circuit")


def norm(psi) -> float:
    return float(lib().orc_norm(_ptr(psi.view(np.float64), _dp), psi.size))


def gate_output_labelled(dims, gate, idx) -> np.ndarray:
    """Sampled outputs of one gate applied to the labelled state (sv_inputs.labelled_state)."""
    dims_a = _i32(dims)
    ctrl = _i32(gate.ctrl if len(gate.ctrl) else [0])
    vals = _i32(gate.vals if len(gate.vals) else [0])
    U = _c128(gate.U)
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.uint64))
    out = np.zeros(idx.size, dtype=np.complex128)
    lib().orc_gate_output_labelled(len(dims_a), _ptr(dims_a, _ip), int(gate.target),
                                   len(gate.ctrl), _ptr(ctrl, _ip), _ptr(vals, _ip),
                                   _ptr(U.view(np.float64), _dp), _ptr(idx, _up), idx.size,
                                   _ptr(out.view(np.float64), _dp))
    return out


def circuit_output_labelled(dims, gates, idx) -> np.ndarray:
    """Sampled outputs of a short circuit (<= 8 gates) applied to the labelled state."""
    dims_a = _i32(dims)
    targets = _i32([g.target for g in gates] or [0])
    nctrls = _i32([len(g.ctrl) for g in gates] or [0])
    cf = _i32([c for g in gates for c in g.ctrl] or [0])
    vf = _i32([v for g in gates for v in g.vals] or [0])
    Uf = np.ascontiguousarray(np.concatenate([np.asarray(g.U, np.complex128).ravel() for g in gates]
                                             or [np.zeros(1, np.complex128)]))
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.uint64))
    out = np.zeros(idx.size, dtype=np.complex128)
    rc = lib().orc_circuit_output_labelled(len(dims_a), _ptr(dims_a, _ip), len(gates), _ptr(targets, _ip),
                                           _ptr(nctrls, _ip), _ptr(cf, _ip), _ptr(vf, _ip),
                                           _ptr(Uf.view(np.float64), _dp), _ptr(idx, _up), idx.size,
                                           _ptr(out.view(np.float64), _dp))
    if rc:
        raise ValueError("oracle rejected circuit")
    return out


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))
