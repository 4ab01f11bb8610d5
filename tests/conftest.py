import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case at config scale")


@pytest.fixture(scope="session")
def devlib():
    from paper_1911_03458_b200 import _capi
    return _capi.load()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for @pytest.mark.gpu tests (no CPU fallback exists)")
    return torch.device("cuda:0")


_POISON = None
_FLUSH = None


def poison_shared_memory(pattern: int = 0xFFFFFFFF) -> None:
    """Fill every SM's shared memory with `pattern` (tests/cuda/poison.cu), in
    stream order on the default stream: a kernel launched next that reads
    shared memory before its own (asynchronous) writes landed computes with
    NaNs / 255s instead of with bytes an earlier launch happened to leave."""
    global _POISON
    if _POISON is None:
        import ctypes
        sys.path.insert(0, str(ROOT / "tests" / "cuda"))
        import build_helpers
        _POISON = ctypes.CDLL(str(build_helpers.build()))
        _POISON.poison_shared_memory.argtypes = [ctypes.c_uint32, ctypes.c_void_p]
        _POISON.poison_shared_memory.restype = ctypes.c_int
    rc = _POISON.poison_shared_memory(pattern, None)
    assert rc == 0, f"poison kernel launch failed (cudaError {rc})"


@pytest.fixture
def smem_poison():
    """The poisoning call itself, for tests that poison between launches."""
    return poison_shared_memory


@pytest.fixture(autouse=True)
def _poisoned_shared_memory(request):
    """Every GPU test starts with poisoned shared memory on all SMs, so the
    first launch of each shape runs as it would after an unrelated kernel."""
    if request.node.get_closest_marker("gpu") is not None:
        import torch
        if torch.cuda.is_available():
            torch.cuda.init()
            # primary context current on this thread; the write pass over 2 x L2
            # also leaves the test's first staging copies to come from DRAM
            global _FLUSH
            if _FLUSH is None:
                _FLUSH = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
            _FLUSH.add_(1)
            poison_shared_memory()
    yield
