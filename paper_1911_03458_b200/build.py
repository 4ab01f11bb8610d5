"""Build the in-tree C-ABI library ``libmerit_dev.so`` for sm_100a.

Plain nvcc (no torch extension machinery): every ``csrc/*.cu`` and
``csrc/*.cpp`` is compiled with ``-gencode arch=compute_100a,code=sm_100a``
and linked into one shared library next to this file, with the CUDA runtime
linked statically so the library does not depend on which libcudart the host
process (e.g. torch) loaded.  Cross-compiles without a GPU.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = PKG / "_build"
LIB = PKG / "libmerit_dev.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
              "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the device library cannot be built")


def _sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers():
    return sorted(list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h")))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


# Diagnostic build (-DMERIT_DEV_DEBUG): the MERIT_*_DEBUG / MERIT_SAD_DBG
# timing knobs exist only here.  Load it with MERIT_DEV_LIB=<path>.
DEBUG_BUILD = PKG / "_build_debug"
DEBUG_LIB = PKG / "libmerit_dev_debug.so"


def build(verbose: bool = False, force: bool = False, debug: bool = False) -> Path:
    bdir, lib = (DEBUG_BUILD, DEBUG_LIB) if debug else (BUILD, LIB)
    bdir.mkdir(exist_ok=True)
    cc = nvcc()
    headers = _headers()
    objs, cmds = [], []
    for src in _sources():
        obj = bdir / (src.name + ".o")
        objs.append(obj)
        if force or _stale(obj, [src, *headers, Path(__file__)]):
            cmds.append([cc, *ARCH, *NVCC_FLAGS, *(["-DMERIT_DEV_DEBUG"] if debug else []), f"-I{INCLUDE}",
                         f"-I{CSRC}", "-c", str(src), "-o", str(obj)])

    def compile_one(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)

    # translation units are independent: compile them concurrently
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        list(ex.map(compile_one, cmds))
    if force or _stale(lib, objs):
        cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs), "-lcuda", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if not debug:
        build_cli(verbose, force)
    return lib


CLI_SRC = PKG / "cli" / "merit_dev.cpp"
CLI = PKG / "bin" / "merit-dev"


def build_cli(verbose: bool = False, force: bool = False) -> Path:
    """bin/merit-dev: the reference CLI's `run --manifest` path over the C ABI
    (host C++, linked to libmerit_dev.so through an $ORIGIN rpath)."""
    CLI.parent.mkdir(exist_ok=True)
    if force or _stale(CLI, [CLI_SRC, LIB, INCLUDE / "merit_dev.h"]):
        cxx = shutil.which("g++") or "g++"
        cmd = [cxx, "-O2", "-std=c++17", "-Wall", f"-I{INCLUDE}", str(CLI_SRC), "-o", str(CLI),
               f"-L{PKG}", "-l:libmerit_dev.so", "-Wl,-rpath,$ORIGIN/.."]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return CLI


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv, debug="--debug" in sys.argv))
