"""Thread / stream safety of the C ABI (include/merit_dev.h, "Threading"):
one plan run from two host threads on two streams at once gives each caller
its own correct result — weights packed on the fly are stream-ordered on the
plan, the exact interpreter's error flag is per plan and serialised, and
read-only kernels run concurrently."""
import threading

import numpy as np
import pytest

from oracle import binding as O
from paper_1911_03458_b200 import Error, ErrorCode, FLAG_ARGMIN, Kernel, Plan
from paper_1911_03458_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _two_threads(fn):
    errs = []

    def wrap(i):
        try:
            fn(i)
        except BaseException as e:  # noqa: BLE001 - reported below
            errs.append(e)

    ts = [threading.Thread(target=wrap, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


def test_conv_plan_two_streams_different_weights(cuda):
    import torch
    w = W.conv_nchw_view(4, 64, 28, 28, 64, 3, 1, 1)
    plan = Plan(w)                      # no pack_b: every run packs its own weights
    xs = [W.gen_uniform([4, 64, 28, 28], 200 + i) for i in range(2)]
    wts = [W.gen_normal([64, 64, 3, 3], 210 + i, 0.06) for i in range(2)]
    wants = [O.conv2d(xs[i], wts[i], 1, 1) for i in range(2)]
    dev = [(torch.from_numpy(xs[i]).to(cuda), torch.from_numpy(wts[i]).to(cuda)) for i in range(2)]

    def work(i):
        s = torch.cuda.Stream(cuda)
        out = torch.empty(plan.out_shape, dtype=torch.float32, device=cuda)
        for _ in range(20):
            plan.run(dev[i][0], dev[i][1], out, stream=s.cuda_stream)
        s.synchronize()
        got = out.cpu().numpy()
        assert np.max(np.abs(got - wants[i]) / (1 + np.abs(wants[i]))) <= 1e-4

    _two_threads(work)


def test_sad_plan_two_threads_host_and_device_calls(cuda):
    import torch
    cur, ref = W.gen_me_pair(128, 256, 220)
    w = W.me_view(128, 256, 16, 16)
    w.src_a, w.src_b = cur, ref
    plan = Plan(w, FLAG_ARGMIN)
    want = O.me_sad(cur, ref, 16, 16)

    def work(i):
        if i == 0:
            for _ in range(10):
                sad, mv = plan.run_host(cur, ref)
                assert np.array_equal(sad, want)
        else:
            s = torch.cuda.Stream(cuda)
            a, b = torch.from_numpy(cur).to(cuda), torch.from_numpy(ref).to(cuda)
            out = torch.empty(int(plan.info.out_elems), dtype=torch.int32, device=cuda)
            aux = torch.empty(int(plan.info.aux_elems), dtype=torch.int32, device=cuda)
            for _ in range(10):
                plan.run(a, b, out, aux, stream=s.cuda_stream)
            s.synchronize()
            assert np.array_equal(out.cpu().numpy().reshape(want.shape), want)

    _two_threads(work)


def test_exact_interpreter_error_flag_not_shared_across_runs(cuda):
    # two threads share one REJECT plan: one feeds in-range data, the other
    # a source that makes the gather go out of range is impossible for the
    # same plan, so use two plans on one thread each plus a shared one
    w = W.build_template("maxpool", {"h": 9, "w": 9, "k": 3})
    W.fill_random(w, 1, 2)
    from paper_1911_03458_b200 import FLAG_EXACT
    plan = Plan(w, FLAG_EXACT)
    assert plan.kernel == Kernel.GENERIC
    want = O.run_full(w)

    def work(i):
        for _ in range(5):
            got, _ = plan.run_host(w.src_a, w.src_b)
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32))

    _two_threads(work)
    # and a failing plan reports its own error, on its own
    bad = W.build_template("maxpool", {"h": 9, "w": 9, "k": 3})
    W.fill_random(bad, 1, 2)
    bad.view_a.p_shape = [5, 4]
    bad.view_b.p_shape = [5, 4]
    bp = Plan(bad, FLAG_EXACT)
    with pytest.raises(Error) as ei:
        bp.run_host(bad.src_a, bad.src_b)
    assert ei.value.code == ErrorCode.OutOfRange
    got, _ = plan.run_host(w.src_a, w.src_b)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))

