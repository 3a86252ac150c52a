"""B200-native mixed-radix statevector engine: the hot path of arXiv 2410.17876's block
simulation (direct-evolution gate application on a dense complex128 statevector).

The product is libsv.so (C ABI, include/sv.h) with hand-written sm_100a kernels;
`paper_2410_17876_b200.sv` is a thin ctypes binding with the same entry points.
"""
from . import sv  # noqa: F401  (raises ImportError if libsv.so is missing: no CPU fallback)
from .sv import State, SVError, plan_gate, enumerate_fibres, fuse_plan, merge_plan, shard_plan, block_plan, nccl_unique_id, ipc_unique_id  # noqa: F401

__all__ = ["sv", "State", "SVError", "plan_gate", "enumerate_fibres", "fuse_plan", "merge_plan", "shard_plan",
           "nccl_unique_id", "ipc_unique_id"]
