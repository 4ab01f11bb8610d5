"""Pin the C restatement (oracle/oracle.c) to the reference: golden vectors
produced by the reference itself (tests/golden/make_golden.py), the reference
tests' known-answer cases, and — where /root/reference is present — a live
comparison against the compiled reference engine."""
import numpy as np
import pytest

from oracle import binding as O
from paper_1911_03458_b200 import workloads as W
from tests.golden_io import load, load_case

GOLD = load()


def _workload_for(key):
    name, rest = key.split("|", 1)
    prm = {}
    for kv in rest.split("|")[0].split(","):
        k, v = kv.split("=")
        prm[k] = float(v) if "." in v else int(v)
    return name, prm


RANDOM_KEYS = [str(k) for k in GOLD["random_index"]]


@pytest.mark.parametrize("key", RANDOM_KEYS)
def test_engine_restatement_matches_reference_engine(key):
    """reference tests/test_workloads.cpp:123-216 instances (same parameter draws,
    same fill_random seeds); the restated engine must equal merit::run_full
    bit for bit, and stay within the reference's own 1e-5 check of its oracle."""
    name, prm = _workload_for(key.split("random/", 1)[1])
    case = load_case(None, key=key)
    w = W.build_template(name, prm)
    w.src_a = case["src_a"].reshape(w.view_a.source_shape)
    w.src_b = case["src_b"].reshape(w.view_b.source_shape)
    got = O.run_full(w).ravel()
    if case["fix"]:
        assert np.array_equal(got, case["engine"])
    else:
        assert np.array_equal(got.view(np.uint32), case["engine"].view(np.uint32))
        want = case["oracle"].astype(np.float64)
        assert np.all(np.abs(got - want) <= 1e-5 * (1 + np.abs(want)))


def test_known_answers():
    # maxpool 4x4 k2 ramp -> {5,7,13,15}   (tests/test_workloads.cpp:115-121)
    w = W.build_template("maxpool", {"h": 4, "w": 4, "k": 2})
    w.src_a = np.arange(16, dtype=np.float32).reshape(4, 4)
    assert O.run_full(w).ravel().tolist() == [5, 7, 13, 15]
    # 1x1 kernel of value 2 doubles the image  (:60-69)
    w = W.build_template("conv2d", {"h": 6, "w": 5, "k": 1})
    w.src_a = W.gen_uniform([6, 5], 102)
    w.src_b = np.array([[2.0]], np.float32)
    assert np.array_equal(O.run_full(w), 2.0 * w.src_a)
    # identical frames: SAD 0 at zero displacement  (:95-104)
    w = W.build_template("motion_estimation", {"h": 8, "w": 8, "blk": 4, "win": 3})
    w.src_a = W.gen_uniform([8, 8], 103)
    w.src_b = w.src_a.copy()
    out = O.run_full(w)
    assert np.all(out[:, :, 1, 1] == 0)
    # identity gemm returns the input  (:47-57)
    w = W.build_template("gemm", {"m": 4, "n": 4, "k": 4})
    w.src_a = W.gen_uniform([4, 4], 101)
    w.src_b = np.eye(4, dtype=np.float32)
    assert np.array_equal(O.run_full(w), w.src_a)


def test_boundary_modes_view_algebra():
    # tests/test_view.cpp:37-47: ZERO_PAD -> 0, CLAMP -> edge value, REJECT throws
    from paper_1911_03458_b200 import Boundary, Error
    w = W.build_template("maxpool", {"h": 3, "w": 3, "k": 2})
    w.src_a = -(np.arange(9, dtype=np.float32).reshape(3, 3) + 1)
    w.view_a.terms[1].offset = -1           # window rows start at -1
    w.view_a.boundary = Boundary.ZeroPad
    assert O.run_full(w)[0, 0] == 0.0       # max(0, 0, -1, -2)
    w.view_a.boundary = Boundary.Clamp
    assert O.run_full(w)[0, 0] == -1.0      # row -1 clamps to row 0
    w.view_a.boundary = Boundary.Reject
    with pytest.raises(Error):
        O.run_full(w)


def test_config_slices_match_reference_engine():
    g = load("configs.npz")
    # C1: engine semantics == restated max-pool (bit-exact)
    x = g["C1::src_a"]
    assert np.array_equal(O.maxpool(x, 56, 56).view(np.uint32), g["C1::engine"].view(np.uint32))
    # C2: int SAD == REAL32 engine (exact integers)
    sad = O.me_sad(g["C2::src_a"], g["C2::src_b"], 16, 16)
    assert np.array_equal(sad.astype(np.float32), g["C2::engine"])
    # C3 / C4: double-accumulating oracle within 1e-5 of the fp32 engine chain
    for c, s in (("C3", 1), ("C4", 2)):
        got = O.conv2d(g[c + "::src_a"], g[c + "::src_b"], s, 1)
        want = g[c + "::engine"].astype(np.float64)
        assert np.max(np.abs(got - want) / (1 + np.abs(want))) <= 1e-5


def test_argmin_tie_break():
    sad = np.array([[[[5, 3, 3], [3, 9, 3], [7, 7, 3]]]], np.int32)
    mv = O.me_argmin(sad, 1)
    assert mv.tolist() == [[-1, 0, 3]]   # first raster index holding the minimum


@pytest.mark.skipif(not O.ref_available(), reason="reference not present")
def test_restatement_vs_live_reference_on_fresh_cases():
    rng = np.random.default_rng(0)
    for t in range(6):
        n, c, h, wd = 1 + t % 2, 2 + t, 9 + t, 7 + 2 * t
        w = W.maxpool_nchw_view(n, c, h, wd, 3, 2, 1)
        w.src_a = rng.standard_normal((n, c, h, wd)).astype(np.float32)
        assert np.array_equal(O.ref_run_full(w).view(np.uint32),
                              O.maxpool(w.src_a, *w.view_a.p_shape[2:]).view(np.uint32))
        cur, ref = W.gen_me_pair(32, 48, t)
        w = W.me_view(32, 48, 8, 4 + t)
        w.src_a, w.src_b = cur, ref
        assert np.array_equal(O.ref_run_full(w), O.me_sad(cur, ref, 8, 4 + t).astype(np.float32))


def test_oracle_generators_match_device_library_generators():
    # the CPU baseline arms generate their inputs with liboracle (they never
    # load the device library); the bytes must be the GPU arm's bytes
    for h, wd, seed in ((1080, 1920, 2), (37, 61, 9)):
        a = O.gen_me_pair(h, wd, seed)
        b = W.gen_me_pair(h, wd, seed)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(O.gen_normal([64, 64, 3, 3], 1003, (2.0 / 576) ** 0.5),
                          W.gen_normal([64, 64, 3, 3], 1003, (2.0 / 576) ** 0.5))
    assert np.array_equal(O.gen_uniform([3, 5, 7], 4), W.gen_uniform([3, 5, 7], 4))
    x = O.gen_uniform([1000], 5, -3.0, 3.0)
    x[:3] = [np.nan, np.inf, -0.0]
    assert np.array_equal(O.to_bf16_bits(x), W.to_bf16_bits(x))
