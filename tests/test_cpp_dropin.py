"""The C++ header swap (include/merit/device.hpp) against the unmodified
reference engine, driven by the reference's own templates and RNG: the
compiled driver oracle/_ref/test_device_header (built from
tests/cpp/test_device_header.cpp where /root/reference exists)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "oracle" / "_ref" / "test_device_header"


@pytest.mark.gpu
def test_cpp_header_swap_matches_reference_engine(cuda):
    if not EXE.exists():
        pytest.skip("drop-in driver not built (needs /root/reference at build time)")
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout
