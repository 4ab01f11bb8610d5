"""Build an experiment variant of the device library (A/B timing on the GPU).

  python tools/build_variant.py NAME SOURCE.cu [-DMACRO=1 ...]

Recompiles one translation unit with extra flags and links it with the other
objects of the product build (paper_1911_03458_b200/_build) into
paper_1911_03458_b200/variants/libmerit_dev_NAME.so; select it on the GPU
box with MERIT_DEV_LIB=<path>.  Experiments only: the product library is the
one build.py makes.
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1911_03458_b200 import build as B  # noqa: E402

name, src, *flags = sys.argv[1:]
out_dir = B.PKG / "variants"
out_dir.mkdir(exist_ok=True)
obj = out_dir / f"{name}_{Path(src).name}.o"
cmd = [B.nvcc(), *B.ARCH, *B.NVCC_FLAGS, *flags, f"-I{B.INCLUDE}", f"-I{B.CSRC}", "-c", str(B.CSRC / src), "-o", str(obj)]
subprocess.run(cmd, check=True)
objs = [o for o in sorted(B.BUILD.glob("*.o")) if o.name != Path(src).name + ".o"] + [obj]
lib = out_dir / f"libmerit_dev_{name}.so"
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs), "-lcuda", "-ldl"],
               check=True)
print(lib)
