"""Build libsv.so in-tree: all CUDA/C++ sources of the C ABI, compiled for sm_100a only."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.environ.get("SV_BUILD_CSRC") or os.path.join(HERE, "csrc")    # override: variant builds
LIB = os.environ.get("SV_BUILD_OUT") or os.path.join(HERE, "libsv.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_paths():
    try:
        import nvidia.nccl  # the wheel torch itself uses (NCCL 2.28)
        base = list(nvidia.nccl.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib", "libnccl.so.2")
    except Exception:
        return "/usr/include", "libnccl.so.2"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "sv.h"),
                                                              os.path.abspath(__file__)]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    inc, nccl_lib = _nccl_paths()
    objdir = os.path.join(os.path.dirname(LIB), "build") if os.environ.get("SV_BUILD_OUT") else os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include"), "-I", inc,
              f'-DSV_NCCL_WHEEL_LIB="{nccl_lib}"', "-DSV_BUILD_LIB"]
    if verbose:
        common += ["-Xptxas", "-v"]
    common += os.environ.get("SV_BUILD_FLAGS", "").split()      # e.g. -DSV_DEBUG_CHECKS (debug variant)
    objs, procs = [], []
    for src in sources():                       # one nvcc per translation unit, in parallel
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = common + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd)))
    failed = [s for s, p in procs if p.wait() != 0]
    if failed:
        raise RuntimeError("nvcc failed for " + ", ".join(failed))
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-ldl"])
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
