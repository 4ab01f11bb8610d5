"""Builds tests/cuda/libpoison.so (the shared-memory poisoning helper of
tests/test_gpu_determinism.py) with nvcc for sm_100a.  Test infrastructure:
nothing in the product imports it."""
import shutil
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "poison.cu"
LIB = HERE / "libpoison.so"


def build(verbose: bool = False) -> Path:
    if LIB.exists() and LIB.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared", "-Xcompiler", "-fPIC",
           "-cudart", "static", str(SRC), "-o", str(LIB)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
