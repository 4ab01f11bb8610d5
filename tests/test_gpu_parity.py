"""Device parity: every kernel through the C ABI against the oracle / golden.

Bars: max-pool, SAD and argmin bit-exact; the generic
interpreter bit-exact with the reference engine; convolution within
|got - ref| <= tol * (1 + |ref|) (the reference's own check,
tools/merit.cpp:88-91) with tol = 1e-4 for the fp32 path (3-term bf16
split) and tol = 1e-2 for bf16 data (C4, stated in BASELINE.json).
"""
import numpy as np
import pytest

from oracle import binding as O
from paper_1911_03458_b200 import (FLAG_ARGMIN, FLAG_EXACT, FLAG_FAST_BF16, FLAG_NO_MAP, Boundary,
                                   Error, ErrorCode, Kernel, Plan, run_full, run_full_argmin)
from paper_1911_03458_b200 import _capi
from paper_1911_03458_b200 import workloads as W

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-4
TOL_BF16 = 1e-2


def rel_err(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want) / (1.0 + np.abs(want)))) if want.size else 0.0


# ------------------------------------------------------------- max-pool ---
def test_maxpool_known_answer(cuda):
    # reference tests/test_workloads.cpp:115-121
    w = W.build_template("maxpool", {"h": 4, "w": 4, "k": 2})
    w.src_a = np.arange(16, dtype=np.float32).reshape(4, 4)
    assert Plan(w).kernel == Kernel.MAXPOOL
    assert run_full(w).ravel().tolist() == [5, 7, 13, 15]


def test_maxpool_c1_full_bit_exact(cuda):
    w = W.config_workload("C1")
    plan = Plan(w)
    assert plan.kernel == Kernel.MAXPOOL and "fast3x3s2" in plan.description
    got = run_full(w)
    want = O.maxpool(w.src_a, 56, 56)
    assert got.shape == (8, 64, 56, 56)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("shape,k,s,pad,boundary", [
    ((3, 5, 17, 23), 3, 2, 1, Boundary.Clamp),
    ((2, 3, 16, 16), 3, 2, 1, Boundary.Clamp),   # fast path, odd plane count
    ((1, 2, 9, 300), 3, 2, 1, Boundary.Clamp),   # W > 128: multi-segment fast path
    ((2, 8, 60, 60), 3, 2, 1, Boundary.Clamp),   # 14-row bands, ragged last band, Wo % 4 != 0
    ((1, 4, 112, 64), 3, 2, 1, Boundary.Clamp),  # 14-row bands, 16-byte output stores
    ((2, 2, 11, 13), 2, 1, 0, Boundary.Clamp),
    ((2, 2, 11, 13), 3, 3, 1, Boundary.ZeroPad),
    ((1, 1, 7, 7), 5, 1, 2, Boundary.Clamp),
])
def test_maxpool_views_bit_exact(cuda, shape, k, s, pad, boundary):
    n, c, h, wd = shape
    w = W.maxpool_nchw_view(n, c, h, wd, k, s, pad)
    w.view_a.boundary = boundary
    w.src_a = W.gen_uniform(list(shape), 77)
    ho, wo = w.view_a.p_shape[2:]
    got = run_full(w)
    want = O.maxpool(w.src_a, ho, wo, k, s, pad, clamp=boundary == Boundary.Clamp)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    # and the reference engine itself on the same workload
    if O.ref_available():
        assert np.array_equal(got.view(np.uint32), O.ref_run_full(w).view(np.uint32))


def test_maxpool_signed_zero_and_constant(cuda):
    # Post_1 is ADD r + 0.0f (rip.hpp:167-168): a -0.0 maximum is emitted as +0.0,
    # and a window of values below the MOVC constant returns the constant.
    w = W.maxpool_nchw_view(1, 1, 4, 4, 3, 2, 1)
    x = np.full((1, 1, 4, 4), -0.0, np.float32)
    x[0, 0, 3, 3] = -np.inf
    w.src_a = x
    got = run_full(w)
    assert np.all(got.view(np.uint32) == np.float32(0.0).view(np.uint32))
    w.src_a = np.full((1, 1, 4, 4), -np.inf, np.float32)
    got = run_full(w)
    assert np.all(got == np.float32(-3.0e38))


# -------------------------------------------------------------------- SAD --
def test_sad_c2_full_bit_exact(cuda):
    w = W.config_workload("C2")
    plan = Plan(w, FLAG_ARGMIN)
    assert plan.kernel == Kernel.SAD
    sad, mv = run_full_argmin(w)
    want = O.me_sad(w.src_a, w.src_b, 16, 16)
    assert sad.shape == (67, 120, 33, 33)
    assert np.array_equal(sad, want)
    assert np.array_equal(mv, O.me_argmin(want, 16))
    # no-map mode returns the same argmin
    _, mv2 = run_full_argmin(w, with_map=False)
    assert np.array_equal(mv2, mv)


@pytest.mark.parametrize("h,wd,blk,r,boundary", [
    (48, 64, 16, 16, Boundary.ZeroPad),
    (40, 72, 8, 16, Boundary.ZeroPad),
    (64, 96, 16, 32, Boundary.ZeroPad),
    (72, 80, 8, 32, Boundary.ZeroPad),
    (50, 70, 8, 5, Boundary.ZeroPad),      # frame not a block multiple, odd radius
    (48, 64, 16, 16, Boundary.Clamp),
    (37, 61, 8, 3, Boundary.Clamp),        # unaligned width: byte staging path
])
def test_sad_small_bit_exact(cuda, h, wd, blk, r, boundary):
    cur, ref = W.gen_me_pair(h, wd, 9, blk, min(r, 16), 4)
    w = W.me_view(h, wd, blk, r)
    w.view_b.boundary = boundary
    w.src_a, w.src_b = cur, ref
    sad, mv = run_full_argmin(w)
    want = O.me_sad(cur, ref, blk, r, clamp=boundary == Boundary.Clamp)
    assert np.array_equal(sad, want)
    assert np.array_equal(mv, O.me_argmin(want, r))


# staging: TMA boxes with the barrier-free kernel / TMA boxes with one tile
# barrier per tile / cp.async
@pytest.mark.parametrize("mode", ["1", "1-sync", "0"])
@pytest.mark.parametrize("blk", [8, 16])
def test_sad_staging_modes_unaligned_windows(cuda, monkeypatch, mode, blk):
    # windows that start at every byte offset mod 16 (radius r: x0 = bx*blk - r),
    # the case TMA boxes cannot start at (tools/microbench/tma_u8.cu)
    monkeypatch.setenv("MERIT_SAD_TMA", mode[0])
    monkeypatch.setenv("MERIT_SAD_ASYNC", "0" if mode == "1-sync" else "1")
    for (h, wd, r) in [(64, 96, 2), (48, 128, 5), (80, 160, 7), (72, 112, 12), (88, 80, 23)]:  # BY odd for 8x8 in the last two
        cur, ref = W.gen_me_pair(h, wd, 17, blk, min(r, 16), 4)
        w = W.me_view(h, wd, blk, r)
        w.src_a, w.src_b = cur, ref
        sad, mv = run_full_argmin(w)
        want = O.me_sad(cur, ref, blk, r)
        assert np.array_equal(sad, want), (h, wd, r)
        assert np.array_equal(mv, O.me_argmin(want, r)), (h, wd, r)


# warp-per-block kernels (16x16 +/-16 and +/-32, 8x8 +/-32, >= 8 block columns)
# on every staging path: TMA (ZERO_PAD), cp.async words (CLAMP), bytes
# (unaligned width), with ragged tiles, odd block rows and a pair axis
@pytest.mark.parametrize("h,wd,blk,r,boundary,pairs", [
    (64, 160, 16, 16, Boundary.ZeroPad, 2),   # 10 block columns: a 2-block tail tile
    (48, 128, 16, 16, Boundary.Clamp, 1),     # cp.async word staging
    (40, 131, 16, 16, Boundary.ZeroPad, 1),   # unaligned width: byte staging
    (96, 144, 16, 32, Boundary.ZeroPad, 1),   # two warps per block
    (64, 128, 16, 32, Boundary.Clamp, 1),
    (88, 96, 8, 32, Boundary.ZeroPad, 2),     # 8x8, 11 block rows: odd pair of rows
    (72, 72, 8, 32, Boundary.Clamp, 1),
])
def test_sad_warp_per_block_paths(cuda, h, wd, blk, r, boundary, pairs):
    if pairs > 1:
        cur = np.empty((pairs, h, wd), np.uint8)
        ref = np.empty((pairs, h, wd), np.uint8)
        for i in range(pairs):
            cur[i], ref[i] = W.gen_me_pair(h, wd, 40 + i, blk, min(r, 16), 4)
    else:
        cur, ref = W.gen_me_pair(h, wd, 40, blk, min(r, 16), 4)
    w = W.me_view(h, wd, blk, r, pairs=pairs if pairs > 1 else None)
    w.view_b.boundary = boundary
    w.src_a, w.src_b = cur, ref
    sad, mv = run_full_argmin(w)
    assert "warp per block" in _capi.load().merit_dev_last_kernel().decode()
    want = O.me_sad(cur, ref, blk, r, clamp=boundary == Boundary.Clamp)
    assert np.array_equal(sad, want)
    assert np.array_equal(mv, O.me_argmin(want, r))
    w.dtype_out = W.Dtype.Real32
    assert np.array_equal(run_full(w), want.astype(np.float32))


def test_sad_ties_lowest_raster(cuda):
    # Flat frames: every displacement that stays inside the frame ties at 0;
    # the lowest raster index (dy*WX + dx) must win.
    h, wd = 64, 64
    cur = np.full((h, wd), 7, np.uint8)
    ref = np.full((h, wd), 7, np.uint8)
    w = W.me_view(h, wd, 16, 16)
    w.src_a, w.src_b = cur, ref
    sad, mv = run_full_argmin(w)
    want = O.me_sad(cur, ref, 16, 16)
    assert np.array_equal(sad, want)
    assert np.array_equal(mv, O.me_argmin(want, 16))


def test_sad_identical_frames_zero_at_centre(cuda):
    # reference tests/test_workloads.cpp:95-104, on u8 frames
    cur, _ = W.gen_me_pair(64, 64, 3)
    w = W.me_view(64, 64, 16, 16)
    w.src_a, w.src_b = cur, cur.copy()
    sad, _ = run_full_argmin(w)
    assert np.all(sad[:, :, 16, 16] == 0)


def test_sad_pairs_axis_and_float_output(cuda):
    pairs = 3
    cur = np.empty((pairs, 64, 96), np.uint8)
    ref = np.empty((pairs, 64, 96), np.uint8)
    for i in range(pairs):
        cur[i], ref[i] = W.gen_me_pair(64, 96, 100 + i)
    w = W.me_view(64, 96, 16, 16, pairs=pairs)
    w.src_a, w.src_b = cur, ref
    sad, mv = run_full_argmin(w)
    want = O.me_sad(cur, ref, 16, 16)
    assert np.array_equal(sad, want)
    assert np.array_equal(mv, O.me_argmin(want, 16))
    w.dtype_out = W.Dtype.Real32
    got = run_full(w)
    assert got.dtype == np.float32 and np.array_equal(got, want.astype(np.float32))


@pytest.mark.slow
@pytest.mark.parametrize("blk", [16, 8])
def test_sad_c5_pairs_bit_exact(cuda, blk):
    w = W.config_workload("C5", pairs=2, blk=blk)
    _, mv = run_full_argmin(w, with_map=False)
    want = O.me_sad(w.src_a, w.src_b, blk, 32)
    assert np.array_equal(mv, O.me_argmin(want, 32))
    sad, mv2 = run_full_argmin(w, with_map=True)
    assert np.array_equal(sad, want)
    assert np.array_equal(mv2, mv)


# ------------------------------------------------------------------- conv --
def test_conv_c3_full_fp32_tol(cuda):
    w = W.config_workload("C3")
    plan = Plan(w)
    assert plan.kernel == Kernel.CONV_TC and "split=3" in plan.description
    got = run_full(w)
    want = O.conv2d(w.src_a, w.src_b, 1, 1)
    e = rel_err(got, want)
    print("C3 max |d|/(1+|ref|) =", e)
    assert e <= TOL_F32


def test_conv_c4_bf16_tol(cuda):
    w = W.config_workload("C4", scale=16)  # 16 images: the full-size run is in test_full_sizes
    got = run_full(w)
    x, wt = w.fp32_inputs
    want = O.conv2d(x, wt, 2, 1)
    e = rel_err(got, want)
    print("C4 (16 images) max |d|/(1+|ref|) =", e)
    assert e <= TOL_BF16
    # against the oracle fed the same bf16-rounded inputs the error is accumulation only
    want_b = O.conv2d(W.bf16_bits_to_f32(w.src_a), W.bf16_bits_to_f32(w.src_b), 2, 1)
    assert rel_err(got, want_b) <= 1e-4


@pytest.mark.parametrize("n,cin,h,wd,cout,k,s,pad,dil,relu", [
    (2, 64, 9, 11, 64, 3, 1, 1, 1, False),
    (1, 3, 20, 20, 16, 3, 1, 1, 1, False),        # Cin < 64 (zero-padded k-block)
    (3, 70, 8, 8, 40, 3, 2, 1, 1, True),          # Cin % 64 != 0, Cout % 16 != 0, relu
    (2, 32, 15, 13, 300, 3, 1, 1, 1, False),      # Cout > 256: two N tiles
    (1, 16, 17, 19, 32, 3, 1, 2, 2, False),       # dilation 2
    (5, 8, 7, 6, 8, 1, 1, 0, 1, False),           # 1x1
    (1, 3, 35, 35, 48, 11, 4, 5, 1, False),       # alexnet-like 11x11 s4
])
def test_conv_variants_fp32(cuda, n, cin, h, wd, cout, k, s, pad, dil, relu):
    w = W.conv_nchw_view(n, cin, h, wd, cout, k, s, pad, dil, relu)
    w.src_a = W.gen_uniform([n, cin, h, wd], 11)
    w.src_b = W.gen_normal([cout, cin, k, k], 12, (2.0 / (cin * k * k)) ** 0.5)
    plan = Plan(w)
    assert plan.kernel == Kernel.CONV_TC
    got = run_full(w)
    want = O.conv2d(w.src_a, w.src_b, s, pad, dil, relu)
    assert rel_err(got, want) <= TOL_F32
    if relu:
        assert np.all(got >= 0)


@pytest.mark.parametrize("variant", ["s1", "no_s1"])
@pytest.mark.parametrize("n,cin,h,wd,cout,relu", [
    (2, 64, 56, 56, 64, False),    # C3 geometry, 64 slots / row, 2 rows / tile
    (1, 3, 20, 20, 16, False),     # Cin < 64, N = 48
    (2, 64, 28, 28, 80, True),     # Cout = 80 -> N = 240: A in shared memory, relu
    (3, 70, 37, 28, 80, True),     # the same with two / three channel blocks (conv_sweep seed 7 case 95:
    (3, 192, 37, 28, 80, False),   # a raw slot was handed back before its loads had returned)
    (3, 70, 20, 56, 80, False),
    (1, 128, 13, 12, 48, False),   # two channel blocks, 32 slots (4 rows / tile), Ho % 4 != 0
    (3, 32, 30, 28, 32, False),    # 32 slots
    (1, 16, 9, 124, 16, False),    # 128 slots: segments of 31 > 30 columns -> general kernel
    (1, 16, 9, 120, 16, False),    # 128 slots, 1 row / tile: four segments of 30 columns
    (1, 32, 6, 60, 32, False),     # 64 slots: two segments of 30 columns
])
def test_conv_fp32_stride1_tap_stacked(cuda, monkeypatch, variant, n, cin, h, wd, cout, relu):
    if variant == "no_s1":
        monkeypatch.setenv("MERIT_CONV_S1", "0")
    w = W.conv_nchw_view(n, cin, h, wd, cout, 3, 1, 1, 1, relu)
    w.src_a = W.gen_uniform([n, cin, h, wd], 41)
    w.src_b = W.gen_normal([cout, cin, 3, 3], 42, (2.0 / (cin * 9)) ** 0.5)
    got = run_full(w)
    kern = (_capi.load().merit_dev_last_kernel() or b"").decode()
    if variant == "s1":  # K3d takes every shape whose row segments fit 30 columns
        assert ("conv_s1" in kern) == (wd != 124), kern
    assert rel_err(got, O.conv2d(w.src_a, w.src_b, 1, 1, 1, relu)) <= TOL_F32


CONV_VARIANTS = {
    "default": {},                                  # TMA gather, CTA pairs where eligible
    "single": {"MERIT_CONV_PAIR": "0"},             # TMA gather, one CTA per tile
    "quad": {"MERIT_CONV_QUAD": "1"},               # two CTA pairs per cluster, weight multicast
    "tap3": {"MERIT_CONV_TMA": "0"},                # register gather, tap-shared planes
    "general": {"MERIT_CONV_KERNEL": "general"},    # per-tap gather
}


@pytest.mark.parametrize("variant", sorted(CONV_VARIANTS))
@pytest.mark.parametrize("n,cin,h,cout", [
    (2, 128, 16, 256),    # small image: tap3 path, two channel blocks
    (2, 128, 32, 256),
    (3, 128, 56, 256),    # C4 geometry, 21 M tiles: odd -> ghost tile in pair mode
    (5, 128, 56, 256),    # 35 M tiles: three ghost tiles in quad mode
    (1, 192, 56, 96),     # three channel blocks, BN = 96
    (2, 64, 56, 320),     # two N tiles (BN = 160)
])
def test_conv_bf16_stride2_kernel_variants(cuda, monkeypatch, variant, n, cin, h, cout):
    for k, v in CONV_VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    w = W.conv_nchw_view(n, cin, h, h, cout, 3, 2, 1)
    x = W.gen_uniform([n, cin, h, h], 31)
    wt = W.gen_normal([cout, cin, 3, 3], 32, (2.0 / (9 * cin)) ** 0.5)
    w.src_a, w.src_b = W.to_bf16_bits(x), W.to_bf16_bits(wt)
    w.dtype_a = w.dtype_b = W.Dtype.BF16
    got = run_full(w)
    assert rel_err(got, O.conv2d(x, wt, 2, 1)) <= TOL_BF16
    want_b = O.conv2d(W.bf16_bits_to_f32(w.src_a), W.bf16_bits_to_f32(w.src_b), 2, 1)
    assert rel_err(got, want_b) <= 1e-4


def test_conv_fast_bf16_flag(cuda):
    w = W.conv_nchw_view(2, 64, 12, 12, 64, 3, 1, 1)
    w.src_a = W.gen_uniform([2, 64, 12, 12], 5)
    w.src_b = W.gen_normal([64, 64, 3, 3], 6, (2.0 / 576) ** 0.5)
    plan = Plan(w, FLAG_FAST_BF16)
    assert "split=1" in plan.description
    got, _ = plan.run_host(w.src_a, w.src_b)
    want = O.conv2d(w.src_a, w.src_b, 1, 1)
    assert rel_err(got, want) <= TOL_BF16


def test_conv_exact_flag_matches_reference_engine(cuda):
    # FLAG_EXACT runs the MAC chain in the engine's order with its rounding:
    # bit-exact with merit::run_full.
    w = W.conv_nchw_view(1, 3, 9, 8, 4, 3, 2, 1)
    w.src_a = W.gen_uniform([1, 3, 9, 8], 21)
    w.src_b = W.gen_uniform([4, 3, 3, 3], 22)
    plan = Plan(w, FLAG_EXACT)
    assert plan.kernel == Kernel.GENERIC
    got, _ = plan.run_host(w.src_a, w.src_b)
    want = O.run_full(w)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_conv_device_buffers_and_prepacked_weights(cuda):
    import torch
    w = W.config_workload("C3", scale=8)
    plan = Plan(w)
    x = torch.from_numpy(w.src_a).to(cuda)
    wt = torch.from_numpy(w.src_b).to(cuda)
    out = torch.empty(plan.out_shape, dtype=torch.float32, device=cuda)
    plan.pack_b(wt)
    plan.run(x, None, out)          # weights come from the packed copy
    torch.cuda.synchronize()
    want = O.conv2d(w.src_a, w.src_b, 1, 1)
    assert rel_err(out.cpu().numpy(), want) <= TOL_F32


# ---------------------------------------------------- generic interpreter --
TEMPLATE_CASES = [
    ("gemm", {"m": 5, "n": 7, "k": 9}),
    ("gemm", {"m": 4, "n": 3, "k": 6, "fix": 1, "frac": 6}),
    ("conv2d", {"h": 9, "w": 8, "k": 3, "stride": 2, "cin": 2, "cout": 3}),
    ("conv2d", {"h": 7, "w": 10, "k": 3, "stride": 1, "cin": 1, "cout": 1, "fix": 1, "frac": 5}),
    ("relu_fused_conv", {"h": 8, "w": 8, "k": 3, "cin": 2, "cout": 2}),
    ("dilated", {"h": 10, "w": 9, "k": 3}),
    ("dilated", {"h": 10, "w": 9, "k": 2, "fix": 1, "frac": 8}),
    ("correlation", {"c": 3, "h": 7, "w": 6, "d": 3}),
    ("motion_estimation", {"blk": 4, "h": 12, "w": 8, "win": 5}),
    ("motion_estimation", {"blk": 2, "h": 6, "w": 4, "win": 3, "fix": 1}),
    ("bilateral", {"h": 7, "w": 9, "k": 5, "sigma_r": 0.7, "sigma_s": 1.3}),
    ("maxpool", {"h": 9, "w": 7, "k": 3, "stride": 2}),
    ("maxpool", {"h": 8, "w": 8, "k": 2, "fix": 1}),
]


@pytest.mark.parametrize("name,prm", TEMPLATE_CASES)
def test_templates_match_golden(cuda, name, prm):
    """Reference templates filled like the reference tests (fill_random(2s+1),
    fill_random(2s+2)); the device result must equal the reference ENGINE's
    output (golden, produced by the reference) bit for bit, except for the
    tensor-core conv path, which is held to the tolerance."""
    from tests.golden_io import load_case
    case = load_case(name, prm)
    w = W.build_template(name, prm)
    w.src_a = case["src_a"].reshape(w.view_a.source_shape)
    w.src_b = case["src_b"].reshape(w.view_b.source_shape)
    plan = Plan(w)
    got = run_full(w).ravel()
    if plan.kernel == Kernel.CONV_TC:
        assert rel_err(got, case["engine"]) <= TOL_F32
    elif case["fix"]:
        assert np.array_equal(got, case["engine"])
    else:
        assert np.array_equal(got.view(np.uint32), case["engine"].view(np.uint32)), \
            f"{plan.kernel.name} differs from the reference engine"


def test_generic_errors_raise_like_reference(cuda):
    # REJECT gather outside the source -> OutOfRange (view.hpp:77-78)
    w = W.build_template("maxpool", {"h": 4, "w": 4, "k": 2})
    w.view_a.terms[1].offset = -1   # window now starts at row -1
    w.src_a = np.zeros((4, 4), np.float32)
    with pytest.raises(Error) as ei:
        run_full(w, FLAG_EXACT)
    assert ei.value.code == ErrorCode.OutOfRange
    # DIV by zero (rip.hpp:190-191): bilateral on an all-zero image divides 0/wsum;
    # build a program that divides by a zero register instead.
    w = W.build_template("bilateral", {"h": 4, "w": 4, "k": 3})
    w.program.segments[w.program.post(1)][0].b = W.Operand.r(9)  # r9 is never written
    w.src_a = np.ones((4, 4), np.float32)
    w.src_b = w.src_a
    with pytest.raises(Error) as ei:
        run_full(w)
    assert ei.value.code == ErrorCode.DivByZero


# ------------------------------------------------------------ run_tiled --
def test_run_tiled_output_and_report(cuda):
    # engine.hpp:289-295: the device result equals run_full's, the report is
    # the plan's (pinned on CPU in tests/test_tiled_traffic.py)
    from paper_1911_03458_b200 import run_tiled
    w = W.maxpool_nchw_view(2, 4, 16, 16)
    w.src_a = W.gen_uniform([2, 4, 16, 16], 91)
    out, rep = run_tiled(w, [1, 2, 4, 8], [3, 3])
    assert np.array_equal(out.view(np.uint32), run_full(w).view(np.uint32))
    assert rep["passes"] == 2 * 2 * 2 * 1 and rep["macs"] == 2 * 4 * 8 * 8 * 9


def test_conv_random_shapes_all_dispatch_paths(cuda):
    # a compact run of tools/conv_sweep.py (1,250 case x variant runs clean at
    # seed 11): random shapes / strides / dtypes / Cout through every kernel
    import subprocess, sys
    r = subprocess.run([sys.executable, "tools/conv_sweep.py", "24", "5"], capture_output=True, text=True,
                       cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("bad 0"), r.stdout[-2000:]


@pytest.mark.parametrize("m,n,k", [(9, 7, 11), (300, 70, 129), (128, 300, 64), (1, 1, 1), (517, 256, 200)])
def test_gemm_template_on_tensor_cores(cuda, m, n, k):
    # workloads.hpp:122-136 lowered onto the general tcgen05 kernel through
    # operand strides; fp32 data: 3-term split, tol 1e-4
    w = W.build_template("gemm", {"m": m, "n": n, "k": k})
    W.fill_random(w, 2 * m + 1, 2 * n + 2)
    plan = Plan(w)
    assert plan.kernel == Kernel.CONV_TC and "gemm" in plan.description
    got = run_full(w)
    want = (np.asarray(w.src_a, np.float64) @ np.asarray(w.src_b, np.float64)).astype(np.float32)
    assert got.shape == (m, n)
    assert rel_err(got, want) <= TOL_F32


def test_device_buffer_checks(cuda):
    import torch
    w = W.maxpool_nchw_view(1, 2, 8, 8)
    plan = Plan(w)
    a = torch.zeros(2 * 8 * 8, device="cuda")
    out = torch.zeros(2 * 4 * 4, device="cuda")
    plan.run(a, None, out)
    with pytest.raises(Error):
        plan.run(a[:10], None, out)                      # too small
    with pytest.raises(Error):
        plan.run(a.cpu(), None, out)                     # host tensor


# ------------------------------------------- REAL32 frames on the SAD kernel --
@pytest.mark.parametrize("integer", [True, False])
@pytest.mark.parametrize("blk,r", [(16, 16), (8, 32), (16, 3)])
def test_sad_real32_frames_narrowed_bit_exact(cuda, integer, blk, r):
    # the reference's Tensor is REAL32 / FIX16 only (tensor.hpp:67), so a
    # reference caller's motion-estimation frames arrive as floats: they are
    # narrowed to 8 bits on the device and matched by K2; a frame holding any
    # non-integer (or out-of-range) value re-runs on the exact interpreter.
    # Either way the result is the engine's, bit for bit.
    cur, ref = W.gen_me_pair(48, 96, 51, blk, 8, 4)
    w = W.me_view(48, 96, blk, r)
    w.src_a = cur.astype(np.float32)
    w.src_b = ref.astype(np.float32)
    if not integer:
        w.src_b[5, 7] = 12.5
    w.dtype_a = w.dtype_b = w.dtype_out = W.Dtype.Real32
    plan = Plan(w)
    assert plan.kernel == Kernel.SAD and "narrowed" in plan.description
    got = run_full(w)
    want = O.run_full(w)
    assert got.dtype == np.float32
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    if integer:
        assert np.array_equal(got, O.me_sad(cur, ref, blk, r).astype(np.float32))


@pytest.mark.parametrize("h,wd,blk,r", [(1080, 1920, 16, 16), (72, 80, 8, 32), (64, 96, 16, 32)])
def test_sad_u16_map_bit_exact(cuda, h, wd, blk, r):
    cur, ref = W.gen_me_pair(h, wd, 61, blk, min(r, 16), 4)
    w = W.me_view(h, wd, blk, r)
    w.src_a, w.src_b = cur, ref
    w.dtype_out = W.Dtype.U16
    sad, mv = run_full_argmin(w)
    want = O.me_sad(cur, ref, blk, r)
    assert sad.dtype == np.uint16 and np.array_equal(sad.astype(np.int32), want)
    assert np.array_equal(mv, O.me_argmin(want, r))
