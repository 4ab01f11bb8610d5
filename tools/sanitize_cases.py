"""Every device kernel once, at reduced config shapes, for compute-sanitizer
(memcheck / synccheck / racecheck / initcheck): each config's production
kernel (C1 max-pool, C2 SAD + map + argmin, C3 stride-1 conv, C4 stride-2
conv pairs, C5 fused 8x8 + 16x16 and the two separate SAD kernels), plus the
correlation kernel, the exact interpreter and the narrowed REAL32 SAD path,
each checked against the C oracle.

  compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import binding as O  # noqa: E402
from paper_1911_03458_b200 import (FLAG_ARGMIN, FLAG_NO_MAP, Plan, PlanGroup, run_full,  # noqa: E402
                                   run_full_argmin)
from paper_1911_03458_b200 import _capi  # noqa: E402
from paper_1911_03458_b200 import workloads as W  # noqa: E402


def rel(got, want):
    return float(np.max(np.abs(got.astype(np.float64) - want) / (1 + np.abs(want))))


def main():
    lib = _capi.load()
    done = []

    def note(name):
        done.append(f"{name}: {(lib.merit_dev_last_kernel() or b'').decode()}")

    w = W.config_workload("C1", scale=4)
    assert np.array_equal(run_full(w).view(np.uint32), O.maxpool(w.src_a, 56, 56).view(np.uint32))
    note("C1 (2 images)")
    w = W.config_workload("C2")
    sad, mv = run_full_argmin(w)
    want = O.me_sad(w.src_a, w.src_b, 16, 16)
    assert np.array_equal(sad, want) and np.array_equal(mv, O.me_argmin(want, 16))
    note("C2 (full frame)")
    w = W.config_workload("C3", scale=8)
    assert rel(run_full(w), O.conv2d(w.src_a, w.src_b, 1, 1)) <= 1e-4
    note("C3 (4 images)")
    w = W.config_workload("C4", scale=32)
    assert rel(run_full(w), O.conv2d(*w.fp32_inputs, 2, 1)) <= 1e-2
    note("C4 (8 images)")
    w16 = W.config_workload("C5", pairs=1)
    w8 = W.me_view(2160, 3840, 8, 32, pairs=1)
    w8.src_a, w8.src_b = w16.src_a, w16.src_b
    res = PlanGroup([w16, w8], FLAG_ARGMIN | FLAG_NO_MAP).run_host(w16.src_a, w16.src_b)
    note("C5 fused (1 pair)")
    for (_, got), w in zip(res, (w16, w8)):
        _, sep = Plan(w, FLAG_ARGMIN | FLAG_NO_MAP).run_host(w.src_a, w.src_b)
        assert np.array_equal(got, sep)
        note(f"C5 {w.view_a.a_shape[0]}x{w.view_a.a_shape[1]} (1 pair)")
    w = W.build_template("correlation", {"c": 16, "h": 24, "w": 32, "d": 7})
    W.fill_random(w, 3, 4)
    assert np.array_equal(run_full(w).view(np.uint32), O.run_full(w).view(np.uint32))
    note("correlation")
    w = W.build_template("bilateral", {"h": 12, "w": 10, "k": 3})
    W.fill_random(w, 5, 6)
    w.src_b = w.src_a
    assert np.array_equal(run_full(w).view(np.uint32), O.run_full(w).view(np.uint32))
    note("generic (bilateral)")
    cur, ref = W.gen_me_pair(48, 96, 7)
    w = W.me_view(48, 96, 16, 16)
    w.src_a, w.src_b = cur.astype(np.float32), ref.astype(np.float32)
    w.dtype_a = w.dtype_b = w.dtype_out = W.Dtype.Real32
    assert np.array_equal(run_full(w), O.me_sad(cur, ref, 16, 16).astype(np.float32))
    note("narrowed REAL32 SAD")
    print("sanitize cases ok:", "; ".join(done))


if __name__ == "__main__":
    main()
