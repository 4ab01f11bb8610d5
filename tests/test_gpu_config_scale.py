"""Config-scale parity on exactly the code paths bench.py times (SURVEY §8(a)
A10 / §8(d): "correctness runs on full configs").

* C4 — all 256 images on device buffers with pre-packed weights, the way
  bench.py runs it (conv_tma_kernel, CTA pairs, ~12 scheduling units per
  pair): every output against an fp64 convolution of the same bf16-rounded
  inputs (accumulation error only, <= 1e-4) and of the fp32 originals
  (BASELINE.json's 1e-2), plus the C oracle (oracle_conv2d restated,
  workloads.hpp:458-499) on images spread over the whole batch.
* Multi-unit persistent loops — every conv / SAD / max-pool variant with the
  grid capped (MERIT_GRID_CAP) so each CTA (pair, quad) walks many units:
  ring phases and TMEM accumulators carried across units.
* C5 — all 64 frame pairs, 16x16 and 8x8 blocks, +/-32: argmin and min SAD
  of every block against an independent block-matching checker (int32 SADs
  from torch tensor ops, min over packed (sad, raster index) keys = the
  lowest-raster tie-break), itself pinned to the C oracle
  (oracle_motion_estimation, workloads.hpp:548-585) on crops.
"""
import numpy as np
import pytest

from oracle import binding as O
from paper_1911_03458_b200 import FLAG_ARGMIN, FLAG_NO_MAP, Kernel, Plan
from paper_1911_03458_b200 import _capi
from paper_1911_03458_b200 import workloads as W

pytestmark = pytest.mark.gpu

TOL_BF16 = 1e-2


def rel_err(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want) / (1.0 + np.abs(want)))) if want.size else 0.0


def _conv_f64(x, wt, stride, chunk=32):
    """fp64 NCHW convolution on the GPU (cuDNN double), pad 1: the double-
    accumulated reference oracle_conv2d computes, at config scale."""
    import torch
    import torch.nn.functional as F
    wt64 = torch.from_numpy(np.ascontiguousarray(wt)).cuda().double()
    outs = []
    for i in range(0, x.shape[0], chunk):
        xb = torch.from_numpy(np.ascontiguousarray(x[i:i + chunk])).cuda().double()
        outs.append(F.conv2d(xb, wt64, stride=stride, padding=1).cpu().numpy())
        del xb
    return np.concatenate(outs)


def _run_conv_device(w, cuda):
    """bench.py's C3/C4 step: device buffers, weights packed once, Plan.run."""
    import torch
    plan = Plan(w)
    a = torch.from_numpy(np.ascontiguousarray(w.src_a)).to(cuda)
    b = torch.from_numpy(np.ascontiguousarray(w.src_b)).to(cuda)
    out = torch.empty(plan.out_shape, dtype=torch.float32, device=cuda)
    plan.pack_b(b)
    out.fill_(float("nan"))
    plan.run(a, None, out)
    torch.cuda.synchronize()
    kern = (_capi.load().merit_dev_last_kernel() or b"").decode()
    return out.cpu().numpy(), kern


def test_conv_c4_full_batch_as_benched(cuda):
    w = W.config_workload("C4")
    x, wt = w.fp32_inputs
    got, kern = _run_conv_device(w, cuda)
    assert "pair" in kern, kern
    assert got.shape == (256, 256, 28, 28) and np.all(np.isfinite(got))
    xb = W.bf16_bits_to_f32(w.src_a)
    wb = W.bf16_bits_to_f32(w.src_b)
    e_b = rel_err(got, _conv_f64(xb, wb, 2))
    e_f = rel_err(got, _conv_f64(x, wt, 2))
    print(f"C4 full: vs bf16-input fp64 {e_b:.3e}, vs fp32-input fp64 {e_f:.3e}")
    assert e_b <= 1e-4
    assert e_f <= TOL_BF16
    # the C oracle itself on images spread over the batch (different pairs /
    # units of the persistent loop)
    for n in (0, 97, 255):
        want = O.conv2d(x[n:n + 1], wt, 2, 1)
        assert rel_err(got[n:n + 1], want) <= TOL_BF16
        assert rel_err(got[n:n + 1], O.conv2d(xb[n:n + 1], wb, 2, 1)) <= 1e-4


MULTI_UNIT_VARIANTS = {
    "pair": {},
    "single": {"MERIT_CONV_PAIR": "0"},
    "quad": {"MERIT_CONV_QUAD": "1"},
}


@pytest.mark.parametrize("cap", ["3", "0"])
@pytest.mark.parametrize("variant", sorted(MULTI_UNIT_VARIANTS))
def test_conv_c4_geometry_many_units_per_cta(cuda, monkeypatch, variant, cap):
    # 64 images = 448 M tiles: 224 pair units (~3 per pair at full grid);
    # with the grid capped at 3 clusters / CTAs every one walks ~75-150 units
    for k, v in MULTI_UNIT_VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    if cap != "0":
        monkeypatch.setenv("MERIT_GRID_CAP", cap)
    w = W.config_workload("C4", scale=4, seed_offset=50)
    got, kern = _run_conv_device(w, cuda)
    assert variant in kern, kern
    xb = W.bf16_bits_to_f32(w.src_a)
    wb = W.bf16_bits_to_f32(w.src_b)
    assert rel_err(got, _conv_f64(xb, wb, 2)) <= 1e-4


@pytest.mark.parametrize("cap", ["2", "0"])
def test_conv_c3_geometry_many_units_per_cta(cuda, monkeypatch, cap):
    if cap != "0":
        monkeypatch.setenv("MERIT_GRID_CAP", cap)
    w = W.config_workload("C3", seed_offset=60)
    got, kern = _run_conv_device(w, cuda)
    assert "conv_s1" in kern, kern
    assert rel_err(got, _conv_f64(w.src_a, w.src_b, 1)) <= 1e-4


@pytest.mark.parametrize("cap", ["1", "5"])
@pytest.mark.parametrize("blk,r", [(16, 16), (16, 32), (8, 32)])
def test_sad_many_tiles_per_cta(cuda, monkeypatch, blk, r, cap):
    monkeypatch.setenv("MERIT_GRID_CAP", cap)
    cur, ref = W.gen_me_pair(136, 256, 70, blk, 16, 4)
    w = W.me_view(136, 256, blk, r)
    w.src_a, w.src_b = cur, ref
    plan = Plan(w, FLAG_ARGMIN)
    sad, mv = plan.run_host(cur, ref)
    want = O.me_sad(cur, ref, blk, r)
    assert np.array_equal(sad, want)
    assert np.array_equal(mv, O.me_argmin(want, r))


def test_maxpool_many_bands_per_cta(cuda, monkeypatch):
    monkeypatch.setenv("MERIT_GRID_CAP", "3")
    monkeypatch.setenv("MERIT_MP_RB", "8")   # ring path (several bands per CTA)
    w = W.maxpool_nchw_view(2, 16, 112, 112)
    w.src_a = W.gen_uniform([2, 16, 112, 112], 71)
    got, _ = Plan(w).run_host(w.src_a, np.zeros(1, np.float32))
    want = O.maxpool(w.src_a, 56, 56)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


# ------------------------------------------------------------------ C5 ----
def me_argmin_checker(cur, ref, blk, radius):
    """Independent block-matching argmin on the GPU with torch tensor ops.

    cur, ref: uint8 CUDA tensors (P, H, W).  ref is read as 0 outside the
    frame (ZERO_PAD, oracle_motion_estimation); the block grid is floor(H /
    blk) x floor(W / blk).  Returns int32 (P * BY * BX, 3) records (dy - r,
    dx - r, min SAD), minimising the key sad * 2^16 + (dy * win + dx): lowest
    SAD, then lowest raster index."""
    import torch
    import torch.nn.functional as F
    P, H, Wd = cur.shape
    BY, BX, win = H // blk, Wd // blk, 2 * radius + 1
    recs = []
    for q in range(P):  # one pair at a time: the (win, H, W) int16 slab is ~1 GB at 4K
        c = cur[q, :BY * blk, :BX * blk].to(torch.int16)
        refp = F.pad(ref[q].to(torch.int16)[None], (radius, radius, radius, radius))[0]
        best = torch.full((BY, BX), torch.iinfo(torch.int64).max, dtype=torch.int64, device=cur.device)
        for dy in range(win):
            rows = refp[dy:dy + BY * blk, :]
            # all dx of this dy: (BY*blk, win, BX*blk) as a strided view
            cand = rows.unfold(1, BX * blk, 1)[:, :win, :]
            d = (cand - c.unsqueeze(1)).abs_()
            s = d.view(BY, blk, win, BX, blk).sum(dim=(1, 4), dtype=torch.int32)   # (BY, win, BX)
            key = s.to(torch.int64) * 65536 + (dy * win + torch.arange(win, device=cur.device)).view(1, win, 1)
            best = torch.minimum(best, key.amin(dim=1))
            del rows, cand, d, s, key
        k = best.view(-1)
        idx = (k & 0xFFFF).to(torch.int32)
        recs.append(torch.stack([idx // win - radius, idx % win - radius, (k >> 16).to(torch.int32)], dim=1))
    return torch.cat(recs).to(torch.int32).cpu().numpy()


def test_me_argmin_checker_pinned_to_oracle(cuda):
    import torch
    # the checker is test infrastructure: pin it to the C oracle (full SAD maps
    # + caller-side argmin) on crops of C5 frames, both block sizes
    cur, ref = W.gen_me_pair(2160, 3840, 5, 16, 16, 4)
    for blk in (16, 8):
        cc = np.ascontiguousarray(cur[:160, 1000:1256])
        rc = np.ascontiguousarray(ref[:160, 1000:1256])
        want = O.me_argmin(O.me_sad(cc, rc, blk, 32), 32)
        got = me_argmin_checker(torch.from_numpy(cc)[None].to(cuda), torch.from_numpy(rc)[None].to(cuda), blk, 32)
        assert np.array_equal(got, want)
    # and tie-break on flat frames (every displacement inside the frame ties)
    flat = np.full((64, 64), 7, np.uint8)
    want = O.me_argmin(O.me_sad(flat, flat, 16, 8), 8)
    got = me_argmin_checker(torch.from_numpy(flat)[None].to(cuda), torch.from_numpy(flat)[None].to(cuda), 16, 8)
    assert np.array_equal(got, want)


@pytest.mark.slow
def test_sad_c5_all_64_pairs_argmin(cuda):
    """bench.py's C5 step: 64 pairs on device buffers, two plans (16x16 and
    8x8 blocks, +/-32, argmin only), every block's record checked."""
    import torch
    w16 = W.config_workload("C5")
    cur = torch.from_numpy(w16.src_a).to(cuda)
    ref = torch.from_numpy(w16.src_b).to(cuda)
    for blk in (16, 8):
        w = W.me_view(2160, 3840, blk, 32, pairs=64)
        plan = Plan(w, FLAG_ARGMIN | FLAG_NO_MAP)
        assert plan.kernel == Kernel.SAD
        aux = torch.full((int(plan.info.aux_elems),), -7, dtype=torch.int32, device=cuda)
        plan.run(cur, ref, None, aux)
        torch.cuda.synchronize()
        got = aux.view(-1, 3).cpu().numpy()
        for p0 in range(0, 64, 8):
            want = me_argmin_checker(cur[p0:p0 + 8], ref[p0:p0 + 8], blk, 32)
            nb = want.shape[0]
            assert np.array_equal(got[p0 * nb // 8:(p0 + 8) * nb // 8], want), (blk, p0)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sad_c2_band_shards_equal_full_frame(cuda, world):
    """bench.py's C2 split: every rank's block-row band with
    its Eq. 6 halo rows only, on the device, concatenates to the full-frame
    SAD map and argmin bit for bit."""
    from paper_1911_03458_b200.shard import shard_band
    w = W.config_workload("C2")
    sad_full, mv_full = Plan(w, FLAG_ARGMIN).run_host(w.src_a, w.src_b)
    sads, mvs = [], []
    for r in range(world):
        s, _ = shard_band(w, world, r)
        plan = Plan(s, FLAG_ARGMIN)
        assert plan.kernel == Kernel.SAD
        sad, mv = plan.run_host(s.src_a, s.src_b)
        sads.append(sad)
        # motion vectors are ref row - cur row in the sliced sources' coordinates
        mv[:, 0] += s.row_origin[1] - s.row_origin[0]
        mvs.append(mv)
    assert np.array_equal(np.concatenate(sads), sad_full)
    assert np.array_equal(np.concatenate(mvs), mv_full)
