"""Build the test-only checkers (see oracle/oracle.c header).

* ``oracle/liboracle.so``   — the C restatement (oracle.c), gcc -fopenmp.
* ``oracle/_ref/libmerit_ref.so`` — the UNMODIFIED reference compiled from
  its own headers where they lie (/root/reference/proj/include) through the
  extern "C" shim ref_shim.cpp.  Only when /root/reference exists (this
  container); the GPU box uses the prebuilt file that travels with gpurun.
  The reference's own CMake build is not used (it needs doctest / CLI11,
  which are absent); the engine path is header-only and needs neither.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
REF_INCLUDE = Path(os.environ.get("MERIT_REF_INCLUDE", "/root/reference/proj/include"))
LIB = HERE / "liboracle.so"
REF_DIR = HERE / "_ref"
REF_LIB = REF_DIR / "libmerit_ref.so"


def _stale(target: Path, deps) -> bool:
    return not target.exists() or any(d.stat().st_mtime > target.stat().st_mtime for d in deps)


def build_oracle(verbose: bool = False) -> Path:
    src = HERE / "oracle.c"
    hdr = ROOT / "include" / "merit_dev.h"
    if _stale(LIB, [src, hdr]):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
               "-fno-fast-math", f"-I{ROOT / 'include'}", str(src), "-o", str(LIB), "-lm"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


def build_ref(verbose: bool = False) -> Path | None:
    if not (REF_INCLUDE / "merit" / "engine.hpp").exists():
        return REF_LIB if REF_LIB.exists() else None
    REF_DIR.mkdir(exist_ok=True)
    src = HERE / "ref_shim.cpp"
    deps = [src, ROOT / "include" / "merit_dev.h", *sorted((REF_INCLUDE / "merit").glob("*.hpp"))]
    if _stale(REF_LIB, deps):
        cmd = ["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-ffp-contract=off",
               f"-I{REF_INCLUDE}", f"-I{ROOT / 'include'}", str(src), "-o", str(REF_LIB)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return REF_LIB


def build_dropin_test(verbose: bool = False) -> Path | None:
    """tests/cpp/test_device_header.cpp: reference engine vs include/merit/device.hpp."""
    if not (REF_INCLUDE / "merit" / "engine.hpp").exists():
        exe = REF_DIR / "test_device_header"
        return exe if exe.exists() else None
    REF_DIR.mkdir(exist_ok=True)
    src = ROOT / "tests" / "cpp" / "test_device_header.cpp"
    exe = REF_DIR / "test_device_header"
    lib = ROOT / "paper_1911_03458_b200" / "libmerit_dev.so"
    deps = [src, ROOT / "include" / "merit_dev.h", ROOT / "include" / "merit" / "device.hpp", lib]
    if _stale(exe, deps):
        cmd = ["g++", "-O2", "-std=c++20", f"-I{REF_INCLUDE}", f"-I{ROOT / 'include'}", str(src), "-o", str(exe),
               f"-L{lib.parent}", "-lmerit_dev", "-Wl,-rpath,$ORIGIN/../../paper_1911_03458_b200"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return exe


def build(verbose: bool = False):
    return build_oracle(verbose), build_ref(verbose), build_dropin_test(verbose)


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
