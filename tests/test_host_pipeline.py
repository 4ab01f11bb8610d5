"""Pipelined host-buffer runs (csrc/host_pipeline.cpp).

merit_dev_run_host cuts a plan into slices along its outermost independent
axis (max-pool planes, conv images, SAD frame pairs or block-row bands) and
overlaps H2D / kernel / D2H per slice.  Each slice runs the plan's own kernel
on a sub-range, so the result must equal the single-shot run bit for bit,
for any slice count, including ragged slices, and the oracle where the bar
is bit-exact.  MERIT_HOST_CHUNKS is read when a plan first slices.
"""
import numpy as np
import pytest

from oracle import binding as O
from paper_1911_03458_b200 import FLAG_ARGMIN, FLAG_FAST_BF16, FLAG_NO_MAP, Plan
from paper_1911_03458_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _run(w, flags, chunks, monkeypatch):
    monkeypatch.setenv("MERIT_HOST_CHUNKS", str(chunks))
    plan = Plan(w, flags)
    out, aux = plan.run_host(w.src_a, w.src_b)
    return out.copy(), (aux.copy() if aux is not None else None)


def _same(x, y):
    if x is None or y is None:
        return x is None and y is None
    return x.tobytes() == y.tobytes()


@pytest.mark.parametrize("chunks", [2, 3, 7])
def test_maxpool_plane_slices(cuda, monkeypatch, chunks):
    w = W.maxpool_nchw_view(3, 5, 17, 23, 3, 2, 1)          # 15 planes: ragged slices
    w.src_a = W.gen_uniform([3, 5, 17, 23], 5)
    one, _ = _run(w, 0, 1, monkeypatch)
    got, _ = _run(w, 0, chunks, monkeypatch)
    assert _same(got, one)
    assert np.array_equal(got.view(np.uint32), O.maxpool(w.src_a, 9, 12).view(np.uint32))


def test_maxpool_c1_sliced(cuda, monkeypatch):
    w = W.config_workload("C1")
    got, _ = _run(w, 0, 5, monkeypatch)
    assert np.array_equal(got.view(np.uint32), O.maxpool(w.src_a, 56, 56).view(np.uint32))


@pytest.mark.parametrize("n,cin,hw,cout,stride,flags", [
    (5, 64, 14, 64, 1, 0),                 # stride-1 fp32 (tap-stacked kernel)
    (3, 128, 14, 128, 2, FLAG_FAST_BF16),  # stride-2 bf16 TMA kernel
    (4, 3, 11, 8, 1, 0),                   # general kernel
])
@pytest.mark.parametrize("chunks", [2, 3])
def test_conv_image_slices(cuda, monkeypatch, n, cin, hw, cout, stride, flags, chunks):
    w = W.conv_nchw_view(n, cin, hw, hw, cout, 3, stride, 1)
    w.src_a = W.gen_uniform([n, cin, hw, hw], 31)
    w.src_b = W.gen_normal([cout, cin, 3, 3], 32, (2.0 / (9 * cin)) ** 0.5)
    one, _ = _run(w, flags, 1, monkeypatch)
    got, _ = _run(w, flags, chunks, monkeypatch)
    assert _same(got, one)


@pytest.mark.parametrize("blk,h,wd,r,chunks", [
    (16, 160, 192, 16, 3),
    (16, 176, 208, 7, 4),   # 11 block rows -> ragged bands
    (8, 72, 96, 12, 4),     # 8x8 (two block rows per tile) bands with odd starts
    (8, 64, 64, 32, 5),
])
def test_sad_band_slices(cuda, monkeypatch, blk, h, wd, r, chunks):
    cur, ref = W.gen_me_pair(h, wd, 9, blk, min(r, 16), 4)
    w = W.me_view(h, wd, blk, r)
    w.src_a, w.src_b = cur, ref
    one = _run(w, FLAG_ARGMIN, 1, monkeypatch)
    got = _run(w, FLAG_ARGMIN, chunks, monkeypatch)
    assert _same(got[0], one[0]) and _same(got[1], one[1])
    sad = O.me_sad(cur, ref, blk, r)
    assert np.array_equal(got[0].reshape(sad.shape).astype(np.int64), sad.astype(np.int64))


@pytest.mark.parametrize("flags", [FLAG_ARGMIN, FLAG_ARGMIN | FLAG_NO_MAP])
def test_sad_pair_slices(cuda, monkeypatch, flags):
    pairs, h, wd, blk, r = 5, 64, 96, 16, 16
    w = W.me_view(h, wd, blk, r, pairs=pairs)
    a = np.empty((pairs, h, wd), np.uint8)
    b = np.empty((pairs, h, wd), np.uint8)
    for i in range(pairs):
        a[i], b[i] = W.gen_me_pair(h, wd, 40 + i, blk, 16, 4)
    w.src_a, w.src_b = a, b
    one = _run(w, flags, 1, monkeypatch)
    got = _run(w, flags, 3, monkeypatch)
    assert _same(got[0], one[0]) and _same(got[1], one[1])


def test_c2_sliced_matches_golden_argmin(cuda, monkeypatch):
    w = W.config_workload("C2")
    sad, mv = _run(w, FLAG_ARGMIN, 9, monkeypatch)
    one = _run(w, FLAG_ARGMIN, 1, monkeypatch)
    assert _same(sad, one[0]) and _same(mv, one[1])
