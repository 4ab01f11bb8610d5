"""Measured traffic: run_tiled's TrafficReport is the
reference's word count for a TilingPlan (engine.hpp:233-241, pinned on CPU in
test_tiled_traffic.py); merit_dev_measure_traffic reads what the device run
actually moved from HBM (GPU counters through CUPTI, L2 flushed first).  The
device stages each footprint once per tile and keeps the halo reuse in L2 /
shared memory, so DRAM reads are the compulsory source bytes — below the
reference's tiled count whenever its tiles re-read halos."""
import numpy as np
import pytest

from oracle import binding as O
from paper_1911_03458_b200 import FLAG_ARGMIN, Error, Plan, run_tiled
from paper_1911_03458_b200 import workloads as W

pytestmark = pytest.mark.gpu

UNAVAILABLE = "measure_traffic unavailable on this system"


def _skip_if_profiler_refused(e):
    """Some GPU hosts refuse a CUPTI profiling session (counters held by a
    monitoring agent, profiling restricted): the library reports that with a
    fixed message prefix (merit_dev.h), and there is nothing to measure.  Any
    other failure of the call is a failure of this test."""
    if UNAVAILABLE in str(e):
        pytest.skip(str(e))
    raise e


def _measure(cuda, plan, a, b):
    import torch
    ta = torch.from_numpy(np.ascontiguousarray(a)).to(cuda)
    tb = torch.from_numpy(np.ascontiguousarray(b)).to(cuda)
    out = torch.empty(max(1, int(plan.info.out_bytes)), dtype=torch.uint8, device=cuda)
    aux = torch.empty(max(1, int(plan.info.aux_elems)), dtype=torch.int32, device=cuda)
    try:
        return plan.measure_traffic(ta, tb, out, aux if plan.info.aux_elems else None)
    except Error as e:
        _skip_if_profiler_refused(e)


@pytest.mark.parametrize("config", ["C1", "C2", "C3", "C4"])
def test_measured_reads_are_compulsory_bytes(cuda, config):
    scale = {"C1": 1, "C2": 1, "C3": 1, "C4": 8}[config]
    w = W.config_workload(config, scale=scale) if config != "C2" else W.config_workload("C2")
    flags = FLAG_ARGMIN if config == "C2" else 0
    plan = Plan(w, flags)
    m = _measure(cuda, plan, w.src_a, w.src_b)
    print(config, m)
    src = float(plan.info.src_a_bytes + plan.info.src_b_bytes)
    assert m["ranges"] >= 1 and m["range_time_ns"] > 0
    # every source byte comes from HBM once; small re-reads (tile halos
    # evicted from L2 before their neighbour ran) stay within 15%
    assert 0.85 * src <= m["dram_read_bytes"] <= 1.15 * src + (4 << 20)
    assert m["dram_write_bytes"] <= 1.05 * plan.info.out_bytes + plan.info.aux_elems * 4 + (8 << 20)


def test_run_tiled_report_with_measurement(cuda):
    # a 5x5 conv over a 1-channel 512 x 512 image with 16 x 8 output tiles:
    # the reference's plan reads every tile's (20 x 12) footprint box, the
    # device reads the image once
    w = W.build_template("conv2d", {"h": 516, "w": 516, "k": 5, "pad": 0})
    W.fill_random(w, 3, 4)
    try:
        out, rep = run_tiled(w, [16, 8], [5, 5], measure=True)
    except Error as e:
        _skip_if_profiler_refused(e)
    _, ref_traffic = O.ref_run_tiled(w, [16, 8], [5, 5])
    assert int(ref_traffic[0]) == rep["dram_read_words_a"]   # the reference's own count
    m = rep["measured"]
    words_read_measured = m["dram_read_bytes"] / 4
    print("reference tiled words", rep["dram_read_words_a"] + rep["dram_read_words_b"], "measured words", words_read_measured)
    assert words_read_measured < rep["dram_read_words_a"]
    assert words_read_measured >= 0.85 * (516 * 516 + 25)
