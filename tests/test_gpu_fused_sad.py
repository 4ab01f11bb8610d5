"""The fused 8x8 + 16x16 block search (multi-workload plans, K2 fused mode):
one byte-SIMD pass over the frames yields both workloads' argmin records,
bit-identical to running the two Workloads separately (the reference runs
each with run_full) and to the C oracle (oracle_motion_estimation,
workloads.hpp:548-585, + the caller-side argmin)."""
import numpy as np
import pytest

from oracle import binding as O
from paper_1911_03458_b200 import FLAG_ARGMIN, FLAG_NO_MAP, Kernel, Plan, PlanGroup, run_full_many
from paper_1911_03458_b200 import _capi
from paper_1911_03458_b200 import workloads as W

pytestmark = pytest.mark.gpu
FLAGS = FLAG_ARGMIN | FLAG_NO_MAP


def _frames(h, wd, pairs, seed):
    cur = np.empty((pairs, h, wd), np.uint8)
    ref = np.empty((pairs, h, wd), np.uint8)
    for i in range(pairs):
        cur[i], ref[i] = W.gen_me_pair(h, wd, seed + i, 16, 16, 4)
    return cur, ref


def _group(h, wd, pairs, cur, ref, order=(16, 8)):
    ws = []
    for blk in order:
        w = W.me_view(h, wd, blk, 32, pairs=pairs)
        w.src_a, w.src_b = cur, ref
        ws.append(w)
    return ws


@pytest.mark.parametrize("h,wd,pairs", [
    (80, 128, 1),      # one tile row of 16x16 blocks, full 8-block tiles
    (96, 96, 2),       # partial last tile (12 8x8 columns = 8 + 4)
    (160, 256, 3),     # several tiles / tile rows / pairs
    (2160, 3840, 1),   # C5 geometry
])
@pytest.mark.parametrize("order", [(16, 8), (8, 16)])
def test_fused_equals_oracle_and_separate_runs(cuda, h, wd, pairs, order):
    cur, ref = _frames(h, wd, pairs, 300)
    ws = _group(h, wd, pairs, cur, ref, order)
    g = PlanGroup(ws, FLAGS)
    assert g.kernel == Kernel.SAD and "fused" in g.description
    res = g.run_host(cur, ref)
    assert "fused" in (_capi.load().merit_dev_last_kernel() or b"").decode()
    for (_, mv), blk, w in zip(res, order, ws):
        _, want = Plan(w, FLAGS).run_host(cur, ref)
        assert np.array_equal(mv, want)
        if h * wd <= 160 * 256:
            assert np.array_equal(mv, O.me_argmin(O.me_sad(cur, ref, blk, 32), 32))


def test_fused_device_buffers_many_tiles_per_cta(cuda, monkeypatch):
    import torch
    monkeypatch.setenv("MERIT_GRID_CAP", "3")
    cur, ref = _frames(160, 512, 2, 310)
    g = PlanGroup(_group(160, 512, 2, cur, ref), FLAGS)
    a, b = torch.from_numpy(cur).to(cuda), torch.from_numpy(ref).to(cuda)
    aux = torch.full((int(g.info.aux_elems),), -5, dtype=torch.int32, device=cuda)
    g.run(a, b, None, aux)
    torch.cuda.synchronize()
    got = aux.cpu().numpy()
    off = g.members[1]["aux_offset"]
    assert np.array_equal(got[:off].reshape(-1, 3), O.me_argmin(O.me_sad(cur, ref, 16, 32), 32))
    assert np.array_equal(got[off:].reshape(-1, 3), O.me_argmin(O.me_sad(cur, ref, 8, 32), 32))


def test_fused_ties_on_flat_frames(cuda):
    # every in-frame displacement ties: lowest raster index wins at both levels
    cur = np.full((1, 96, 128), 9, np.uint8)
    ref = np.full((1, 96, 128), 9, np.uint8)
    res = run_full_many(_group(96, 128, 1, cur, ref), FLAGS)
    for (_, mv), blk in zip(res, (16, 8)):
        assert np.array_equal(mv, O.me_argmin(O.me_sad(cur, ref, blk, 32), 32))


def test_unfusable_group_runs_members(cuda):
    cur, ref = _frames(72, 128, 1, 320)       # 9 rows of 8x8 blocks: no 2 x 2 grid
    ws = _group(72, 128, 1, cur, ref)
    g = PlanGroup(ws, FLAGS)
    assert g.kernel == Kernel.MULTI
    for (_, mv), blk in zip(g.run_host(cur, ref), (16, 8)):
        assert np.array_equal(mv, O.me_argmin(O.me_sad(cur, ref, blk, 32), 32))


@pytest.mark.slow
def test_fused_c5_all_64_pairs_as_benched(cuda):
    """bench.py's C5 step: one fused launch over 64 device-resident pairs."""
    import torch
    from tests.test_gpu_config_scale import me_argmin_checker
    w16 = W.config_workload("C5")
    w8 = W.me_view(2160, 3840, 8, 32, pairs=64)
    g = PlanGroup([w16, w8], FLAGS)
    assert g.kernel == Kernel.SAD and g.info.launches_per_run == 1
    cur = torch.from_numpy(w16.src_a).to(cuda)
    ref = torch.from_numpy(w16.src_b).to(cuda)
    aux = torch.full((int(g.info.aux_elems),), -7, dtype=torch.int32, device=cuda)
    g.run(cur, ref, None, aux)
    torch.cuda.synchronize()
    got = aux.cpu().numpy()
    off = g.members[1]["aux_offset"]
    for blk, recs in ((16, got[:off].reshape(-1, 3)), (8, got[off:].reshape(-1, 3))):
        nb = recs.shape[0] // 64
        for p0 in range(0, 64, 8):
            want = me_argmin_checker(cur[p0:p0 + 8], ref[p0:p0 + 8], blk, 32)
            assert np.array_equal(recs[p0 * nb:(p0 + 8) * nb], want), (blk, p0)


def test_multi_plan_of_convolutions_runs_members(cuda):
    # two Workloads over the same input and weights (plain and relu-fused
    # conv): one MULTI plan, outputs back to back, each equal to its own run
    from paper_1911_03458_b200 import run_full
    ws = [W.conv_nchw_view(2, 16, 12, 10, 8, 3, 1, 1, 1, relu) for relu in (False, True)]
    x = W.gen_uniform([2, 16, 12, 10], 500)
    wt = W.gen_normal([8, 16, 3, 3], 501, 0.1)
    for w in ws:
        w.src_a, w.src_b = x, wt
    g = PlanGroup(ws)
    assert g.kernel == Kernel.MULTI and g.info.launches_per_run >= 2
    res = g.run_host(x, wt)
    for (out, aux), w in zip(res, ws):
        assert aux is None
        assert np.array_equal(out.view(np.uint32), run_full(w).view(np.uint32))


def test_multi_plan_error_from_a_member(cuda):
    # a REJECT gather out of range in the second member raises OutOfRange,
    # as the reference's run_full of that Workload would
    from paper_1911_03458_b200 import Error, ErrorCode
    w1 = W.build_template("maxpool", {"h": 9, "w": 9, "k": 3})
    W.fill_random(w1, 1, 2)
    w2 = W.build_template("maxpool", {"h": 9, "w": 9, "k": 3})
    w2.src_a, w2.src_b = w1.src_a, w1.src_b
    w2.view_a.p_shape = [5, 4]
    w2.view_b.p_shape = [5, 4]
    g = PlanGroup([w1, w2])
    with pytest.raises(Error) as ei:
        g.run_host(w1.src_a, w1.src_b)
    assert ei.value.code == ErrorCode.OutOfRange


def test_u16_maps_in_a_multi_plan(cuda):
    cur, ref = _frames(64, 128, 2, 330)
    ws = []
    for blk in (16, 8):
        w = W.me_view(64, 128, blk, 32, pairs=2)
        w.dtype_out = W.Dtype.U16
        ws.append(w)
    g = PlanGroup(ws, FLAG_ARGMIN)          # maps requested: members run one by one
    assert g.kernel == Kernel.MULTI
    for (sad, mv), blk in zip(g.run_host(cur, ref), (16, 8)):
        want = O.me_sad(cur, ref, blk, 32)
        assert sad.dtype == np.uint16 and np.array_equal(sad.astype(np.int32), want)
        assert np.array_equal(mv, O.me_argmin(want, 32))


def test_narrowed_real32_frames_with_pairs_axis_and_clamp(cuda):
    from paper_1911_03458_b200 import run_full
    cur, ref = _frames(48, 64, 3, 340)
    w = W.me_view(48, 64, 16, 8, pairs=3)
    w.view_b.boundary = W.Boundary.Clamp
    w.src_a, w.src_b = cur.astype(np.float32), ref.astype(np.float32)
    w.dtype_a = w.dtype_b = w.dtype_out = W.Dtype.Real32
    assert Plan(w).kernel == Kernel.SAD
    got = run_full(w)
    assert np.array_equal(got, O.me_sad(cur, ref, 16, 8, clamp=True).astype(np.float32))
