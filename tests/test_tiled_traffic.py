"""Device run_tiled (engine.hpp:289-295): the TrafficReport of a TilingPlan.

The device path computes the reference's report in closed form
(merit_dev_tiled_traffic, csrc/traffic.cpp); these CPU tests pin it to the
reference's own run_tiled (oracle/_ref, compiled from the unmodified headers)
on template and config-shaped workloads, including the reference's KAT
(tests/test_engine.cpp:91-107: a 5x5 conv pass reads 240 words, 3,200
unrolled).  Plan creation needs no GPU.
"""
import numpy as np
import pytest

from oracle import binding as O
from paper_1911_03458_b200 import Error, ErrorCode, Plan
from paper_1911_03458_b200 import workloads as W

FIELDS = ["dram_read_words_a", "dram_read_words_b", "dram_write_words", "scratchpad_peak_words_a",
          "scratchpad_peak_words_b", "passes", "macs"]

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not built")


def _template(name, prm, seed=3):
    w = W.build_template(name, prm)
    W.fill_random(w, seed, seed + 1)
    return w


CASES = [
    # (workload factory, t_p, t_a)
    (lambda: _template("conv2d", {"h": 68, "w": 68, "k": 5, "pad": 0}), [16, 8], [5, 5]),
    (lambda: _template("conv2d", {"h": 20, "w": 17, "k": 3}), [7, 5], [3, 3]),        # partial p tiles
    (lambda: _template("conv2d", {"h": 12, "w": 12, "k": 3}), [12, 12], [2, 3]),      # outer a split
    (lambda: _template("maxpool", {"h": 9, "w": 11, "k": 3}), [2, 2], [3, 3]),
    (lambda: _template("motion_estimation", {"h": 32, "w": 48, "blk": 8, "r": 4}), [1, 4, 2, 3], [8, 8]),
]


def _nchw_conv():
    w = W.conv_nchw_view(2, 8, 10, 9, 4, 3, 2, 1)
    w.src_a = W.gen_uniform([2, 8, 10, 9], 5)
    w.src_b = W.gen_normal([4, 8, 3, 3], 6, 0.2)
    return w


CASES.append((_nchw_conv, [1, 3, 2, 4], [5, 3, 3]))


@needs_ref
@pytest.mark.parametrize("idx", range(len(CASES)))
def test_traffic_matches_reference_run_tiled(idx):
    make, t_p, t_a = CASES[idx]
    w = make()
    got = Plan(w).tiled_traffic(t_p, t_a)
    _, ref = O.ref_run_tiled(w, t_p, t_a)
    assert [got[k] for k in FIELDS] == [int(v) for v in ref]


def test_traffic_known_answer_240_vs_3200():
    # tests/test_engine.cpp:91-107
    w = _template("conv2d", {"h": 68, "w": 68, "k": 5, "pad": 0})
    rep = Plan(w).tiled_traffic([16, 8], [5, 5])
    assert rep["scratchpad_peak_words_a"] == 240
    assert rep["dram_read_words_a"] == 240 * rep["passes"]
    assert 16 * 8 * 25 == 3200
    assert rep["dram_read_words_a"] < 64 * 64 * 25  # traffic_naive_unrolled
    assert rep["macs"] == 64 * 64 * 25 and rep["dram_write_words"] == 64 * 64


def test_traffic_config_scale_closed_form():
    # C4's batched view with the device's tile shape (4 output rows x all
    # columns, all output channels): passes and per-pass Eq. 6 boxes
    w = W.config_workload("C4", with_inputs=False)
    rep = Plan(w).tiled_traffic([1, 256, 4, 28], [128, 3, 3])
    assert rep["passes"] == 256 * 7
    # input box per pass: 1 image x 128 ch x (1 + 3*2 + 2) rows x (1 + 27*2 + 2) cols
    assert rep["scratchpad_peak_words_a"] == 128 * 9 * 57
    assert rep["macs"] == 256 * 256 * 28 * 28 * 128 * 9


@pytest.mark.parametrize("t_p,t_a,why", [
    ([0, 8], [5, 5], "p tile extent out of range"),
    ([16, 65], [5, 5], "p tile extent out of range"),
    ([16, 8], [5, 4], "only the outermost a dimension may be tiled"),
    ([16, 8], [6, 5], "a tile extent out of range"),
])
def test_invalid_plans_raise_bad_params(t_p, t_a, why):
    # TilingPlan::validate (engine.hpp:50-63)
    w = _template("conv2d", {"h": 68, "w": 68, "k": 5, "pad": 0})
    with pytest.raises(Error) as e:
        Plan(w).tiled_traffic(t_p, t_a)
    assert e.value.code == ErrorCode.BadParams and why in str(e.value)


def test_rank_mismatch_raises_bad_params():
    w = _template("conv2d", {"h": 12, "w": 12, "k": 3})
    with pytest.raises(Error) as e:
        Plan(w).tiled_traffic([4], [3, 3])
    assert e.value.code == ErrorCode.BadParams


@needs_ref
@pytest.mark.parametrize("idx", range(len(CASES)))
@pytest.mark.parametrize("caps", [(8192, 4096), (200, 100), (1 << 40, 10)])
def test_scratchpad_overflow_like_reference(idx, caps):
    # EngineConfig capacities (engine.hpp:82-87): the reference throws
    # ScratchpadOverflow from Scratchpad::load (:154-155); device run_tiled
    # raises the same code before touching the device
    from paper_1911_03458_b200 import run_tiled
    make, t_p, t_a = CASES[idx]
    w = make()
    try:
        O.ref_run_tiled(w, t_p, t_a, caps)
        ref_code = None
    except Error as e:
        ref_code = e.code
    rep = Plan(w).tiled_traffic(t_p, t_a)
    dev_over = rep["scratchpad_peak_words_a"] > caps[0] or rep["scratchpad_peak_words_b"] > caps[1]
    assert (ref_code == ErrorCode.ScratchpadOverflow) == dev_over
    if dev_over:
        with pytest.raises(Error) as ei:
            run_tiled(w, t_p, t_a, scratch_words_a=caps[0], scratch_words_b=caps[1])
        assert ei.value.code == ErrorCode.ScratchpadOverflow
