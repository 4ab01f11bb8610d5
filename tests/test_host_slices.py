"""Host-side slicing of pipelined run_host calls (CPU, no device).

merit_dev_plan_slices reports how merit_dev_run_host cuts a plan; the GPU
tests (test_host_pipeline.py) check the sliced results bit for bit.  Here:
the output and argmin ranges tile [0, bytes) in order with no gaps, source
prefixes never shrink and the last one covers everything, no slice is empty,
and plans that cannot slice (the exact interpreter, GEMM views, one image)
run unsliced.
"""
import pytest

from paper_1911_03458_b200 import FLAG_ARGMIN, FLAG_EXACT, FLAG_NO_MAP, Plan
from paper_1911_03458_b200 import workloads as W


def _check(plan, expect_sliced=True):
    sl = plan.host_slices()
    info = plan.info
    if not expect_sliced:
        assert sl == []
        return sl
    assert 2 <= len(sl) <= 16
    out_b, aux_b = int(info.out_bytes), int(info.aux_elems) * 4
    o = x = a = b = 0
    for s in sl:
        assert s["out_lo"] == o and s["aux_lo"] == x
        assert s["out_hi"] >= s["out_lo"] and s["aux_hi"] >= s["aux_lo"]
        assert (s["out_hi"] - s["out_lo"]) + (s["aux_hi"] - s["aux_lo"]) > 0 or out_b + aux_b == 0
        assert s["a_need"] >= a and s["b_need"] >= b
        o, x, a, b = s["out_hi"], s["aux_hi"], s["a_need"], s["b_need"]
    assert (o, x) == (out_b, aux_b)
    assert (a, b) == (int(info.src_a_bytes), int(info.src_b_bytes))
    return sl


@pytest.mark.parametrize("name,flags", [("C1", 0), ("C2", FLAG_ARGMIN), ("C3", 0), ("C4", 0)])
def test_config_plans_slice(name, flags):
    w = W.config_workload(name, with_inputs=False)
    _check(Plan(w, flags))


def test_c5_pair_slices():
    w = W.me_view(2160, 3840, 16, 32, pairs=64)
    sl = _check(Plan(w, FLAG_ARGMIN | FLAG_NO_MAP))
    assert all(s["out_hi"] == 0 for s in sl)   # no map: argmin records only


def test_c2_band_slices_reach_the_window_below():
    # a band of block rows reads its reference window: by_end * 16 + oy + WY + margin rows
    w = W.config_workload("C2", with_inputs=False)
    sl = _check(Plan(w, FLAG_ARGMIN))
    first = sl[0]
    out_row = 120 * 33 * 33 * 4
    rows = first["out_hi"] // out_row        # block rows in the first band
    assert first["b_need"] >= min(1080, rows * 16 - 16 + 33 + 15) * 1920
    assert first["a_need"] >= rows * 16 * 1920


@pytest.mark.parametrize("chunks", [2, 3, 7])
def test_forced_slice_counts(monkeypatch, chunks):
    monkeypatch.setenv("MERIT_HOST_CHUNKS", str(chunks))
    w = W.maxpool_nchw_view(3, 5, 17, 23, 3, 2, 1)   # 15 planes
    sl = _check(Plan(w))
    assert len(sl) == chunks


def test_unsliced_plans(monkeypatch):
    monkeypatch.setenv("MERIT_HOST_CHUNKS", "4")
    w = W.conv_nchw_view(4, 3, 9, 9, 4, 3, 1, 1)
    _check(Plan(w, FLAG_EXACT), expect_sliced=False)            # exact interpreter
    _check(Plan(W.build_template("gemm", {"m": 64, "n": 32, "k": 16})), expect_sliced=False)
    _check(Plan(W.conv_nchw_view(1, 64, 14, 14, 64, 3, 1, 1)), expect_sliced=False)  # one image
    monkeypatch.setenv("MERIT_HOST_CHUNKS", "1")
    _check(Plan(W.config_workload("C1", with_inputs=False)), expect_sliced=False)
