"""Build an alternative libsv.so from a modified copy of csrc/ for A/B kernel measurements:

  python tools/build_variant.py NAME FILE=PATH [FILE=PATH ...]

copies paper_2410_17876_b200/csrc to variants/NAME/pkg/csrc, replaces the named source files and
builds variants/NAME/libsv.so (git-ignored build output).  Select it at run time with
SV_LIB_PATH=variants/NAME/libsv.so."""
import importlib.util
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    name, repl = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "variants", name)
    csrc = os.path.join(out, "pkg", "csrc")          # csrc includes ../../include/sv.h
    shutil.rmtree(out, ignore_errors=True)
    shutil.copytree(os.path.join(ROOT, "paper_2410_17876_b200", "csrc"), csrc)
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(out, "include"))
    for r in repl:
        f, path = r.split("=", 1)
        shutil.copy(path, os.path.join(csrc, f))
    os.environ["SV_BUILD_CSRC"] = csrc
    os.environ["SV_BUILD_OUT"] = os.path.join(out, "libsv.so")
    spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_2410_17876_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    print(b.build(force=True))
    shutil.rmtree(os.path.join(out, "build"), ignore_errors=True)     # objects: keep the gpurun snapshot small


if __name__ == "__main__":
    main()
