"""Thin ctypes binding of the C ABI (include/sv.h) — argument marshalling only.

Every step of the hot path runs in libsv.so's CUDA kernels.  There is no CPU fallback:
if libsv.so is missing or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Iterable, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SV_LIB_PATH: an alternative in-tree build (A/B kernel experiments, tools/build_variant.py)
LIB_PATH = os.environ.get("SV_LIB_PATH") or os.path.join(_HERE, "libsv.so")

SV_C128, SV_C64 = 0, 1
SV_FUSE, SV_NO_CHECK, SV_GRAPH, SV_BLOCK = 1, 2, 4, 8
SV_OPT_KERNEL, SV_OPT_TILE_ELEMS, SV_OPT_TILE_STAGES, SV_OPT_CTAS_PER_SM, SV_OPT_PROFILE, SV_OPT_PASS_TILE = 1, 2, 3, 4, 5, 6
SV_OPT_PASS_STAGES, SV_OPT_PASS_THREADS, SV_OPT_PASS_GATES, SV_OPT_PASS_GROUPS = 7, 8, 9, 10
SV_OPT_PASS_WINDOW, SV_OPT_PASS_MERGE, SV_OPT_SHARD_SWAP, SV_OPT_PASS_SEARCH = 11, 12, 13, 14
SV_OPT_PLAN_CACHE, SV_OPT_PASS_KERNEL, SV_OPT_SHARD_OVERLAP, SV_OPT_PASS_LOW = 15, 16, 17, 18
SV_OPT_PASS_ABSORB = 19

STATUS = {0: "SV_OK", 1: "SV_ERR_INVALID_ARG", 2: "SV_ERR_DIM", 3: "SV_ERR_OVERFLOW",
          4: "SV_ERR_QUDIT_RANGE", 5: "SV_ERR_CTRL_OVERLAP", 6: "SV_ERR_CTRL_DUP",
          7: "SV_ERR_CTRL_VALUE", 8: "SV_ERR_NOT_UNITARY", 9: "SV_ERR_INDEX_RANGE",
          10: "SV_ERR_NOMEM", 11: "SV_ERR_CUDA", 12: "SV_ERR_NCCL", 13: "SV_ERR_UNSUPPORTED"}


class SVError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class sv_gate(C.Structure):
    _fields_ = [("target", C.c_int32), ("nctrl", C.c_int32),
                ("ctrl", C.POINTER(C.c_int32)), ("ctrl_vals", C.POINTER(C.c_int32)),
                ("U", C.POINTER(C.c_double))]


class sv_info(C.Structure):
    _fields_ = [("D", C.c_uint64), ("local_D", C.c_uint64), ("n", C.c_int32),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("device_ptr", C.c_void_p),
                ("cuda_stream", C.c_void_p), ("kernel_launches", C.c_uint64),
                ("exchanges", C.c_uint64), ("overlapped", C.c_uint64)]


class sv_profile(C.Structure):
    _fields_ = [("launches", C.c_uint64), ("kernel_ms", C.c_double),
                ("algorithmic_bytes", C.c_double), ("touched", C.c_double), ("state_bytes", C.c_double),
                ("pass_launches", C.c_uint64), ("pass_ms", C.c_double), ("pass_touched", C.c_double),
                ("pass_item_touched", C.c_double), ("pass_flops", C.c_double),
                ("pass_state_bytes", C.c_double), ("plan_ms", C.c_double),
                ("comm_launches", C.c_uint64), ("comm_ms", C.c_double), ("comm_hbm_bytes", C.c_double),
                ("comm_nvlink_bytes", C.c_double)]


class sv_gate_plan(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d", C.c_int32), ("b", C.c_uint64), ("fibres", C.c_uint64),
                ("touched", C.c_uint64), ("active_mask", C.c_uint32), ("sigma", C.c_int32 * 16),
                ("unitarity_err", C.c_double)]


_i32p = C.POINTER(C.c_int32)
_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_h = C.c_void_p

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)


def _sig(name, args, res=C.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_sig("sv_create", [_i32p, C.c_int32, C.c_int, C.POINTER(_h)])
_sig("sv_create_ex", [_i32p, C.c_int32, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(_h)])
_sig("sv_create_sharded", [_i32p, C.c_int32, C.c_int, C.c_int32, C.c_int32, C.c_void_p, C.c_int,
                           C.c_void_p, C.POINTER(_h)])
_sig("sv_nccl_unique_id", [C.c_void_p])
_sig("sv_create_sharded_ipc", [_i32p, C.c_int32, C.c_int, C.c_int32, C.c_int32, C.c_void_p, C.c_int,
                               C.c_void_p, C.POINTER(_h)])
_sig("sv_ipc_unique_id", [C.c_void_p])
_sig("sv_destroy", [_h])
_sig("sv_reset", [_h, C.c_uint64])
_sig("sv_apply_gate", [_h, C.c_int32, _i32p, _i32p, C.c_int32, _dp])
_sig("sv_apply_circuit", [_h, C.POINTER(sv_gate), C.c_int64, C.c_uint32])
_sig("sv_amplitudes", [_h, C.c_uint64, C.c_uint64, _dp])
_sig("sv_set_amplitudes", [_h, C.c_uint64, C.c_uint64, _dp])
_sig("sv_norm", [_h, _dp])
_sig("sv_sync", [_h])
_sig("sv_last_error", [], C.c_char_p)
_sig("sv_get_info", [_h, C.POINTER(sv_info)])
_sig("sv_set_option", [_h, C.c_int32, C.c_int64])
_sig("sv_plan_gate", [_i32p, C.c_int32, C.c_int32, _i32p, _i32p, C.c_int32, _dp, C.POINTER(sv_gate_plan)])
_sig("sv_enumerate_fibres", [_i32p, C.c_int32, C.c_int32, _i32p, _i32p, C.c_int32, C.c_uint64,
                             C.c_uint64, _u64p])
_sig("sv_fuse_plan", [_i32p, C.c_int32, C.POINTER(sv_gate), C.c_int64, _i32p, _i32p, _i32p, _i32p,
                      _i32p, _i32p, _dp, C.POINTER(C.c_int64)])
_sig("sv_merge_plan", [_i32p, C.c_int32, C.POINTER(sv_gate), C.c_int64, C.c_int32, _i32p, _i32p, _i32p, _i32p,
                       _i32p, _i32p, _dp, C.POINTER(C.c_int64)])
_sig("sv_shard_plan", [_i32p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _i32p, _i32p, C.c_int32,
                       _i32p, _i32p, _i32p])
_sig("sv_version", [], C.c_char_p)
_sig("sv_profile_read", [_h, C.c_int32, C.POINTER(sv_profile)])
_sig("sv_sparse_create", [_i32p, C.c_int32, C.c_double, C.POINTER(_h)])
_sig("sv_sparse_destroy", [_h])
_sig("sv_sparse_reset", [_h, C.c_uint64])
_sig("sv_sparse_apply_gate", [_h, C.c_int32, _i32p, _i32p, C.c_int32, _dp])
_sig("sv_sparse_apply_circuit", [_h, C.POINTER(sv_gate), C.c_int64, C.c_uint32])
_sig("sv_sparse_nnz", [_h, C.POINTER(C.c_uint64)])
_sig("sv_sparse_entries", [_h, C.c_uint64, _u64p, _dp, C.POINTER(C.c_uint64)])
_sig("sv_sparse_launches", [_h, C.POINTER(C.c_uint64)])
_sig("sv_block_plan", [_i32p, C.c_int32, C.POINTER(sv_gate), C.c_int64, C.c_int64, C.POINTER(C.c_int64),
                       C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)])
_sig("sv_shard_schedule", [_i32p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(sv_gate), C.c_int64, C.c_uint32,
                           C.c_int32, _dp, C.c_int64, C.POINTER(C.c_int64), _i32p])
_sig("sv_block_plan_ex", [_i32p, C.c_int32, C.POINTER(sv_gate), C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                          C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                          C.POINTER(C.c_int64)])

EXPORTS = ["sv_create", "sv_create_ex", "sv_create_sharded", "sv_nccl_unique_id", "sv_destroy",
           "sv_create_sharded_ipc", "sv_ipc_unique_id",
           "sv_reset", "sv_apply_gate", "sv_apply_circuit", "sv_amplitudes", "sv_set_amplitudes",
           "sv_norm", "sv_sync", "sv_last_error", "sv_get_info", "sv_set_option", "sv_plan_gate",
           "sv_enumerate_fibres", "sv_fuse_plan", "sv_merge_plan", "sv_shard_plan", "sv_version", "sv_profile_read", "sv_block_plan",
           "sv_sparse_create", "sv_sparse_destroy", "sv_sparse_reset", "sv_sparse_apply_gate",
           "sv_sparse_apply_circuit", "sv_sparse_nnz", "sv_sparse_entries", "sv_sparse_launches",
           "sv_block_plan_ex", "sv_shard_schedule"]


def _check(rc: int):
    if rc != 0:
        raise SVError(rc, (_lib.sv_last_error() or b"").decode())


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(list(a) if not isinstance(a, np.ndarray) else a,
                                           dtype=np.int32).reshape(-1))


def _cplx(U) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(U, dtype=np.complex128))


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None and a.size else None


def version() -> str:
    return _lib.sv_version().decode()


class _GateArray:
    """Marshals gate objects (target, ctrl, vals, U attributes) into an sv_gate array."""

    def __init__(self, gates: Iterable):
        gates = list(gates)
        self.keep = []
        self.arr = (sv_gate * max(1, len(gates)))()
        for i, g in enumerate(gates):
            c, v, U = _i32(g.ctrl), _i32(g.vals), _cplx(g.U)
            self.keep += [c, v, U]
            self.arr[i].target = int(g.target)
            self.arr[i].nctrl = int(c.size)
            self.arr[i].ctrl = _p(c, _i32p)
            self.arr[i].ctrl_vals = _p(v, _i32p)
            self.arr[i].U = U.view(np.float64).ctypes.data_as(_dp)
        self.n = len(gates)


class State:
    """A dense complex128 statevector on one B200 (or one shard of a sharded state)."""

    def __init__(self, dims: Sequence[int], device: int = 0, stream=None, ext_buffer=None,
                 ext_bytes: int = 0, _handle=None, dtype: str = "c128"):
        self.dims = [int(d) for d in dims]
        if _handle is not None:
            self._h = _handle
            return
        if dtype not in ("c128", "c64"):
            raise ValueError("dtype must be 'c128' or 'c64'")
        d = _i32(self.dims)
        h = _h()
        _check(_lib.sv_create_ex(d.ctypes.data_as(_i32p), d.size, SV_C128 if dtype == "c128" else SV_C64, int(device),
                                 C.c_void_p(stream) if stream else None,
                                 C.c_void_p(ext_buffer) if ext_buffer else None,
                                 int(ext_bytes), C.byref(h)))
        self._h = h

    @classmethod
    def sharded(cls, dims, rank: int, nranks: int, nccl_id: bytes | None, device: int = 0,
                stream=None, dtype: str = "c128") -> "State":
        d = _i32(dims)
        h = _h()
        idbuf = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id else None
        dt = {"c128": SV_C128, "c64": SV_C64}[dtype]
        _check(_lib.sv_create_sharded(d.ctypes.data_as(_i32p), d.size, dt, int(rank), int(nranks),
                                      idbuf, int(device), C.c_void_p(stream) if stream else None,
                                      C.byref(h)))
        return cls(dims, _handle=h)

    @classmethod
    def sharded_ipc(cls, dims, rank: int, nranks: int, ipc_id: bytes, device: int = 0,
                    stream=None, dtype: str = "c128") -> "State":
        """One rank of a sharded state over the fused peer-memory transport (sv_create_sharded_ipc)."""
        d = _i32(dims)
        h = _h()
        idbuf = C.create_string_buffer(bytes(ipc_id), 128)
        dt = {"c128": SV_C128, "c64": SV_C64}[dtype]
        _check(_lib.sv_create_sharded_ipc(d.ctypes.data_as(_i32p), d.size, dt, int(rank), int(nranks),
                                          idbuf, int(device), C.c_void_p(stream) if stream else None,
                                          C.byref(h)))
        return cls(dims, _handle=h)

    @classmethod
    def loopback(cls, dims, nranks: int, device: int = 0, dtype: str = "c128") -> "State":
        return cls.sharded(dims, -1, nranks, None, device, dtype=dtype)

    def close(self):
        if getattr(self, "_h", None):
            _check(_lib.sv_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def reset(self, index: int = 0):
        _check(_lib.sv_reset(self._h, int(index)))

    def apply_gate(self, target: int, U, ctrl=(), vals=()):
        c, v, Uc = _i32(ctrl), _i32(vals), _cplx(U)
        _check(_lib.sv_apply_gate(self._h, int(target), _p(c, _i32p), _p(v, _i32p), int(c.size),
                                  Uc.view(np.float64).ctypes.data_as(_dp)))

    def apply_circuit(self, gates, fuse: bool = False, check: bool = True, graph: bool = False,
                      block: bool = False):
        ga = gates if isinstance(gates, _GateArray) else _GateArray(gates)
        flags = (SV_FUSE if fuse else 0) | (0 if check else SV_NO_CHECK) | (SV_GRAPH if graph else 0) | \
            (SV_BLOCK if block else 0)
        _check(_lib.sv_apply_circuit(self._h, ga.arr, ga.n, flags))

    def amplitudes(self, first: int = 0, count: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
        if count is None:
            count = self.info().D - first
        if out is None:
            out = np.empty(int(count), dtype=np.complex128)
        _check(_lib.sv_amplitudes(self._h, int(first), int(count), out.view(np.float64).ctypes.data_as(_dp)))
        return out

    def set_amplitudes(self, first: int, values) -> None:
        v = _cplx(values).reshape(-1)
        _check(_lib.sv_set_amplitudes(self._h, int(first), v.size, v.view(np.float64).ctypes.data_as(_dp)))

    def norm(self) -> float:
        out = C.c_double()
        _check(_lib.sv_norm(self._h, C.byref(out)))
        return out.value

    def sync(self):
        _check(_lib.sv_sync(self._h))

    def info(self) -> sv_info:
        i = sv_info()
        _check(_lib.sv_get_info(self._h, C.byref(i)))
        return i

    def set_option(self, option: int, value: int):
        _check(_lib.sv_set_option(self._h, int(option), int(value)))

    def profile_read(self, reset: bool = True) -> sv_profile:
        p = sv_profile()
        _check(_lib.sv_profile_read(self._h, 1 if reset else 0, C.byref(p)))
        return p


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.sv_nccl_unique_id(buf))
    return buf.raw


def ipc_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.sv_ipc_unique_id(buf))
    return buf.raw


def plan_gate(dims, target, U, ctrl=(), vals=()) -> sv_gate_plan:
    d, c, v, Uc = _i32(dims), _i32(ctrl), _i32(vals), _cplx(U)
    out = sv_gate_plan()
    _check(_lib.sv_plan_gate(d.ctypes.data_as(_i32p), d.size, int(target), _p(c, _i32p), _p(v, _i32p),
                             int(c.size), Uc.view(np.float64).ctypes.data_as(_dp), C.byref(out)))
    return out


def enumerate_fibres(dims, target, ctrl=(), vals=(), first: int = 0, count: int | None = None) -> np.ndarray:
    d, c, v = _i32(dims), _i32(ctrl), _i32(vals)
    if count is None:
        D = int(np.prod([int(x) for x in dims], dtype=object))
        cp = 1
        for q in c:
            cp *= int(dims[int(q)])
        count = D // (int(dims[int(target)]) * cp) - first
    out = np.zeros(max(1, int(count)), dtype=np.uint64)
    _check(_lib.sv_enumerate_fibres(d.ctypes.data_as(_i32p), d.size, int(target), _p(c, _i32p),
                                    _p(v, _i32p), int(c.size), int(first), int(count),
                                    out.ctypes.data_as(_u64p)))
    return out[:int(count)]


def _host_plan(fn, dims, gates, *extra):
    gates = list(gates)
    ga = _GateArray(gates)
    n = max(1, len(gates))
    tot_c = max(1, sum(len(g.ctrl) for g in gates))
    t, sp, dm, nc = (np.zeros(n, np.int32) for _ in range(4))
    oc, ov = np.zeros(tot_c, np.int32), np.zeros(tot_c, np.int32)
    U = np.zeros(n * 512, np.float64)
    nout = C.c_int64()
    d = _i32(dims)
    _check(fn(d.ctypes.data_as(_i32p), d.size, ga.arr, ga.n, *extra, _p(t, _i32p), _p(sp, _i32p),
              _p(dm, _i32p), _p(nc, _i32p), _p(oc, _i32p), _p(ov, _i32p), U.ctypes.data_as(_dp), C.byref(nout)))
    res, co = [], 0
    for i in range(nout.value):
        k = int(dm[i])
        u = U[i * 512: i * 512 + 2 * k * k].view(np.complex128).reshape(k, k).copy()
        res.append((int(t[i]), int(sp[i]), k, tuple(int(x) for x in oc[co:co + nc[i]]),
                    tuple(int(x) for x in ov[co:co + nc[i]]), u))
        co += int(nc[i])
    return res


def fuse_plan(dims, gates):
    """Host fusion planner: list of (target, span, dim, ctrl tuple, vals tuple, U ndarray)."""
    return _host_plan(_lib.sv_fuse_plan, dims, gates)


def merge_plan(dims, gates, window: int = 64):
    """Host commutation-aware merge (the SV_BLOCK pre-pass): same output layout as fuse_plan."""
    return _host_plan(_lib.sv_merge_plan, dims, gates, C.c_int32(int(window)))


def block_plan(dims, gates, tile_cap: int = 4096, max_gates: int | None = None, window: int = 64,
               search: bool = False):
    """Host pass planner: (order, pass_id, tiles) — gate indices in application order.
    max_gates=None: sv_block_plan (24 gates, window 64, search); else sv_block_plan_ex."""
    gates = list(gates)
    ga = _GateArray(gates)
    n = max(1, len(gates))
    order, pid, tiles = (np.zeros(n, np.int64) for _ in range(3))
    npass = C.c_int64()
    d = _i32(dims)
    p64 = C.POINTER(C.c_int64)
    if max_gates is None:
        _check(_lib.sv_block_plan(d.ctypes.data_as(_i32p), d.size, ga.arr, ga.n, int(tile_cap),
                                  order.ctypes.data_as(p64), pid.ctypes.data_as(p64), tiles.ctypes.data_as(p64),
                                  C.byref(npass)))
    else:
        _check(_lib.sv_block_plan_ex(d.ctypes.data_as(_i32p), d.size, ga.arr, ga.n, int(tile_cap), int(max_gates),
                                     int(window), 1 if search else 0, order.ctypes.data_as(p64),
                                     pid.ctypes.data_as(p64), tiles.ctypes.data_as(p64), C.byref(npass)))
    return order[:len(gates)], pid[:len(gates)], tiles[:npass.value]


class SparseState:
    """A sparse complex128 state on the GPU (the paper's sparse variant): sorted (index, amplitude)
    entries; gates touch only the classes holding a stored index."""

    def __init__(self, dims: Sequence[int], eps: float = 1e-12):
        self.dims = [int(d) for d in dims]
        d = _i32(self.dims)
        h = _h()
        _check(_lib.sv_sparse_create(d.ctypes.data_as(_i32p), d.size, float(eps), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _check(_lib.sv_sparse_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def reset(self, index: int = 0):
        _check(_lib.sv_sparse_reset(self._h, int(index)))

    def apply_gate(self, target: int, U, ctrl=(), vals=()):
        c, v, Uc = _i32(ctrl), _i32(vals), _cplx(U)
        _check(_lib.sv_sparse_apply_gate(self._h, int(target), _p(c, _i32p), _p(v, _i32p), int(c.size),
                                         Uc.view(np.float64).ctypes.data_as(_dp)))

    def apply_circuit(self, gates, check: bool = True):
        ga = gates if isinstance(gates, _GateArray) else _GateArray(gates)
        _check(_lib.sv_sparse_apply_circuit(self._h, ga.arr, ga.n, 0 if check else SV_NO_CHECK))

    def nnz(self) -> int:
        out = C.c_uint64()
        _check(_lib.sv_sparse_nnz(self._h, C.byref(out)))
        return out.value

    def entries(self):
        n = self.nnz()
        idx = np.zeros(max(1, n), dtype=np.uint64)
        amp = np.zeros(max(1, n), dtype=np.complex128)
        got = C.c_uint64()
        _check(_lib.sv_sparse_entries(self._h, n, idx.ctypes.data_as(_u64p), amp.view(np.float64).ctypes.data_as(_dp),
                                      C.byref(got)))
        return idx[:n], amp[:n]

    def launches(self) -> int:
        out = C.c_uint64()
        _check(_lib.sv_sparse_launches(self._h, C.byref(out)))
        return out.value


def shard_plan(dims, nranks, rank, target, ctrl=(), vals=()):
    d, c, v = _i32(dims), _i32(ctrl), _i32(vals)
    a, p, b = C.c_int32(), C.c_int32(), C.c_int32()
    _check(_lib.sv_shard_plan(d.ctypes.data_as(_i32p), d.size, int(nranks), int(rank), int(target),
                              _p(c, _i32p), _p(v, _i32p), int(c.size), C.byref(a), C.byref(p), C.byref(b)))
    return a.value, p.value, b.value


def shard_schedule(dims, nranks: int, rank: int, gates, block: bool = True, fuse: bool = False, swap: bool = True):
    """Host-only sharded schedule of one rank (sv_shard_schedule): (ops, final lrank).  ops are
    dicts {kind: 'local'|'swap'|'exchange', partner, beta, k, j, gates: [(target, ctrl, vals, U)]}."""
    gates = list(gates)
    ga = _GateArray(gates)
    d = _i32(dims)
    flags = (SV_BLOCK if block else 0) | (SV_FUSE if fuse else 0) | SV_NO_CHECK
    n_out = C.c_int64()
    lrank = np.zeros(nranks, np.int32)
    cap = 1 << 16
    while True:
        buf = np.zeros(cap, np.float64)
        rc = _lib.sv_shard_schedule(d.ctypes.data_as(_i32p), d.size, int(nranks), int(rank), ga.arr, ga.n, flags,
                                    1 if swap else 0, buf.ctypes.data_as(_dp), cap, C.byref(n_out),
                                    lrank.ctypes.data_as(_i32p))
        if rc != 0 and n_out.value > cap:
            cap = int(n_out.value)
            continue
        _check(rc)
        break
    ops, i = [], 0
    kinds = {0: "local", 1: "swap", 2: "exchange"}
    while i < n_out.value:
        kind, partner, beta, k, j, ng = (int(x) for x in buf[i:i + 6])
        i += 6
        gl = []
        for _ in range(ng):
            t, nc = int(buf[i]), int(buf[i + 1])
            i += 2
            ctrl = tuple(int(x) for x in buf[i:i + nc]); i += nc
            vals = tuple(int(x) for x in buf[i:i + nc]); i += nc
            dd = int(buf[i]); i += 1
            U = buf[i:i + 2 * dd * dd].view(np.complex128).reshape(dd, dd).copy(); i += 2 * dd * dd
            gl.append((t, ctrl, vals, U))
        ops.append({"kind": kinds[kind], "partner": partner, "beta": beta, "k": k, "j": j, "gates": gl})
    return ops, [int(x) for x in lrank]
