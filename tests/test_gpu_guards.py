"""Out-of-bounds write guards (compute-sanitizer is closed on this GPU pool:
the runs under it left GPUs needing a reset).  Every kernel writes into a
buffer carved out of a larger allocation whose margins hold a canary
pattern; after the run the margins must be intact and the result must equal
the oracle, at shapes that exercise ragged tiles, partial waves and the
persistent loops (failure detection)."""
import numpy as np
import pytest

from oracle import binding as O
from paper_1911_03458_b200 import FLAG_ARGMIN, FLAG_NO_MAP, Plan, PlanGroup
from paper_1911_03458_b200 import workloads as W

pytestmark = pytest.mark.gpu

MARGIN = 1 << 16  # bytes of canary on each side
CANARY = 0xA5


def _guarded(cuda, nbytes):
    import torch
    buf = torch.full((nbytes + 2 * MARGIN,), CANARY, dtype=torch.uint8, device=cuda)
    return buf, buf[MARGIN:MARGIN + nbytes]


def _intact(buf, nbytes):
    h = buf.cpu().numpy()
    return bool(np.all(h[:MARGIN] == CANARY) and np.all(h[MARGIN + nbytes:] == CANARY))


def _run_guarded(cuda, plan, a, b):
    import torch
    ta = torch.from_numpy(np.ascontiguousarray(a)).to(cuda)
    tb = torch.from_numpy(np.ascontiguousarray(b)).to(cuda)
    ob, out = _guarded(cuda, max(1, int(plan.info.out_bytes)))
    xb, aux = _guarded(cuda, max(1, int(plan.info.aux_elems) * 4))
    plan.run(ta, tb, out.data_ptr() if plan.info.out_elems else None,
             aux.data_ptr() if plan.info.aux_elems else None)
    torch.cuda.synchronize()
    assert _intact(ob, max(1, int(plan.info.out_bytes))), "write outside the output buffer"
    assert _intact(xb, max(1, int(plan.info.aux_elems) * 4)), "write outside the argmin buffer"
    return out.cpu().numpy(), (aux.cpu().numpy().view(np.int32) if plan.info.aux_elems else None)


@pytest.mark.parametrize("n,c,h,w", [(2, 64, 112, 112), (1, 3, 17, 23), (3, 5, 60, 60)])
def test_maxpool_guarded(cuda, n, c, h, w):
    wl = W.maxpool_nchw_view(n, c, h, w)
    x = W.gen_uniform([n, c, h, w], 400)
    out, _ = _run_guarded(cuda, Plan(wl), x, np.zeros(1, np.float32))
    want = O.maxpool(x, wl.view_a.p_shape[2], wl.view_a.p_shape[3])
    assert np.array_equal(out.view(np.float32), want.ravel())


@pytest.mark.parametrize("h,wd,blk,r", [(1080, 1920, 16, 16), (136, 200, 8, 32), (72, 88, 16, 32), (50, 70, 8, 5)])
def test_sad_guarded(cuda, h, wd, blk, r):
    cur, ref = W.gen_me_pair(h, wd, 401, blk, min(r, 16), 4)
    wl = W.me_view(h, wd, blk, r)
    out, aux = _run_guarded(cuda, Plan(wl, FLAG_ARGMIN), cur, ref)
    want = O.me_sad(cur, ref, blk, r)
    assert np.array_equal(out.view(np.int32), want.ravel())
    assert np.array_equal(aux.reshape(-1, 3), O.me_argmin(want, r))


def test_fused_sad_guarded(cuda):
    cur = np.empty((2, 160, 256), np.uint8)
    ref = np.empty((2, 160, 256), np.uint8)
    for i in range(2):
        cur[i], ref[i] = W.gen_me_pair(160, 256, 402 + i)
    ws = [W.me_view(160, 256, b, 32, pairs=2) for b in (16, 8)]
    g = PlanGroup(ws, FLAG_ARGMIN | FLAG_NO_MAP)
    _, aux = _run_guarded(cuda, g, cur, ref)
    off = g.members[1]["aux_offset"]
    assert np.array_equal(aux[:off].reshape(-1, 3), O.me_argmin(O.me_sad(cur, ref, 16, 32), 32))
    assert np.array_equal(aux[off:].reshape(-1, 3), O.me_argmin(O.me_sad(cur, ref, 8, 32), 32))


@pytest.mark.parametrize("cfg", [
    (3, 64, 56, 56, 64, 1, False),     # C3 kernel (stride 1, taps on N, tail split)
    (5, 128, 56, 56, 256, 2, True),    # C4 kernel (stride 2 pairs), odd M tiles
    (2, 3, 13, 11, 40, 2, False),      # general kernels
])
def test_conv_guarded(cuda, cfg):
    n, cin, h, w, cout, s, bf16 = cfg
    wl = W.conv_nchw_view(n, cin, h, w, cout, 3, s, 1)
    x = W.gen_uniform([n, cin, h, w], 403)
    wt = W.gen_normal([cout, cin, 3, 3], 404, (2.0 / (9 * cin)) ** 0.5)
    a, b = x, wt
    if bf16:
        a, b = W.to_bf16_bits(x), W.to_bf16_bits(wt)
        wl.dtype_a = wl.dtype_b = W.Dtype.BF16
    plan = Plan(wl)
    out, _ = _run_guarded(cuda, plan, a, b)
    want = O.conv2d(W.bf16_bits_to_f32(a) if bf16 else a, W.bf16_bits_to_f32(b) if bf16 else b, s, 1)
    got = out.view(np.float32).reshape(want.shape)
    assert np.max(np.abs(got - want) / (1 + np.abs(want))) <= 1e-4
