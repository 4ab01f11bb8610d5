"""Randomised shape sweeps, each in a fresh process (GPU).

tools/conv_sweep.py draws convolution shapes (Cin 3..192, Cout 8..300, odd
sizes, stride 1 / 2, fp32 / bf16, relu) and runs each through six dispatch
variants against the oracle; tools/misc_sweep.py does the same for max-pool
views, SAD maps + argmin (single and batched pairs), the fused 16x16 + 8x8
search and correlation (bit-exact).  Fresh processes matter: the fault these
sweeps found in round 2 (a raw slot handed back to the TMA engine before its
loads had returned) showed on the first launch of a process far
more often than on later ones."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _run(script, *args):
    cmd = [sys.executable, str(ROOT / "tools" / script), *map(str, args)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    if "initialization error" in r.stdout + r.stderr:
        # the CUDA driver occasionally refuses a context to a process started
        # right after another one exited (seen once in ~150 starts): not a
        # result of the kernels under test, so start the process once more
        r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return r.stdout


@pytest.mark.parametrize("seed", [7, 23])
def test_conv_sweep(cuda, seed):
    out = _run("conv_sweep.py", 100, seed)
    assert "ERROR" not in out and out.strip().splitlines()[-1].endswith("bad 0"), out[-2000:]


@pytest.mark.parametrize("seed", [5, 6])
def test_misc_sweep(cuda, seed):
    out = _run("misc_sweep.py", 20, seed)
    assert "ERROR" not in out and "BAD" not in out, out[-2000:]
    assert out.strip().splitlines()[-1].startswith("cases 20 bad {'maxpool': 0, 'sad': 0, 'fused': 0, 'corr': 0}"), out[-500:]


@pytest.mark.parametrize("args", ["3 70 37 28 80 3 1 1 0", "3 128 37 28 64 3 1 1 0", "6 70 37 28 16 3 1 0 0"])
def test_conv_first_launch_of_a_process(cuda, args):
    """The first convolution launch of a fresh process, four times per shape
    (the Cout = 80 shape failed 7 times in 8 before the raw-slot release waited
    for its loads)."""
    for _ in range(4):
        out = _run("conv_case.py", *args.split(), 1)
        assert " bad 0 " in out.strip().splitlines()[-1], out[-500:]
