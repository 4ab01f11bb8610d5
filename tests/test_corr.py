"""K4 displacement correlation (§8(f) row 4) against the reference engine.

The kernel folds channels in the engine's order with the engine's REAL32 MAC
(fl(r + fl(a * b)), rip.hpp:161-178), so every case is BIT-EXACT with
merit::run_full (oracle/_ref, the compiled reference) or, where the reference
engine would take minutes, with the exact device interpreter (FLAG_EXACT),
itself bit-exact with the engine (test_gpu_parity.py).  Cases follow the
reference's random correlation instances (tests/test_workloads.cpp:169-176),
plus the shapes the template does not produce: centred (negative)
displacement offsets with zero-padded edges, swapped ports, a relu Post_1 and
a FlowNet-sized layer.
"""
import numpy as np
import pytest

from oracle import binding as O
from paper_1911_03458_b200 import FLAG_EXACT, Kernel, Plan, run_full
from paper_1911_03458_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _exact(w):
    if O.ref_available() and np.prod(w.view_a.p_shape) * w.view_a.a_shape[0] < 3e6:
        return O.ref_run_full(w)
    plan = Plan(w, FLAG_EXACT)
    assert plan.kernel == Kernel.GENERIC
    out, _ = plan.run_host(w.src_a, w.src_b)
    return out


def _check(w):
    plan = Plan(w)
    assert plan.kernel == Kernel.CORR, plan.description
    got = run_full(w)
    want = _exact(w)
    assert got.shape == tuple(w.view_a.p_shape)
    assert np.array_equal(got.view(np.uint32), np.asarray(want, np.float32).reshape(got.shape).view(np.uint32))


@pytest.mark.parametrize("t", range(10))
def test_random_instances_like_reference(cuda, t):
    rng = np.random.default_rng(4000 + t)
    prm = {"c": int(rng.integers(1, 7)), "h": int(rng.integers(2, 13)), "w": int(rng.integers(2, 13)),
           "d": int(rng.integers(1, 6))}
    w = W.build_template("correlation", prm)
    W.fill_random(w, 2 * (4000 + t) + 1, 2 * (4000 + t) + 2)
    _check(w)


@pytest.mark.parametrize("c,h,wd,d,off", [
    (32, 20, 27, 9, -4),    # centred 9x9 window: zero padding on every edge
    (7, 5, 33, 11, -5),     # windows wider than the image
    (64, 24, 24, 21, -10),  # FlowNet-like 21x21 (441 displacements)
])
def test_centred_windows(cuda, c, h, wd, d, off):
    w = W.build_template("correlation", {"c": c, "h": h, "w": wd, "d": d})
    for term in w.view_b.terms:
        if term.axis in (1, 2) and term.component in (2, 3):
            term.offset = off
    w.src_a = W.gen_uniform([c, h, wd], 11)
    w.src_b = W.gen_uniform([c, h, wd], 12)
    _check(w)


def test_swapped_ports_and_relu(cuda):
    w = W.build_template("correlation", {"c": 16, "h": 9, "w": 14, "d": 7})
    for term in w.view_b.terms:
        if term.component in (2, 3):
            term.offset = -3
    w.view_a, w.view_b = w.view_b, w.view_a
    w.src_a = W.gen_uniform([16, 9, 14], 21)
    w.src_b = W.gen_uniform([16, 9, 14], 22)
    W.relu_post(w.program)
    plan = Plan(w)
    assert plan.kernel == Kernel.CORR and plan.description.endswith("relu")
    _check(w)


def test_flownet_layer_matches_interpreter(cuda):
    # FlowNetC's correlation: 256 channels, 48x48, +/-10 displacements
    w = W.build_template("correlation", {"c": 256, "h": 48, "w": 48, "d": 21})
    for term in w.view_b.terms:
        if term.component in (2, 3):
            term.offset = -10
    w.src_a = W.gen_uniform([256, 48, 48], 31)
    w.src_b = W.gen_uniform([256, 48, 48], 32)
    _check(w)
