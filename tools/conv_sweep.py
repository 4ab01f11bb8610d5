"""Randomised conv parity sweep over every dispatch path (GPU): NCHW 3x3
(and other kernel sizes), stride 1/2, fp32 / bf16 data, Cout across the N-tile
boundaries, odd spatial sizes, relu.  Compares against the oracle with the
tolerances of tests/test_gpu_parity.py.  usage: python tools/conv_sweep.py [n] [seed]"""
import os, sys
import numpy as np
sys.path.insert(0, '.')
import paper_1911_03458_b200.workloads as W
from paper_1911_03458_b200 import Plan, run_full
import oracle.binding as O

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
variants = [{}, {"MERIT_CONV_PAIR": "0"}, {"MERIT_CONV_QUAD": "1"}, {"MERIT_CONV_TMA": "0"}, {"MERIT_CONV_S1": "0"},
            {"MERIT_CONV_KERNEL": "general"}]
bad = 0
for t in range(n_cases):
    s = int(rng.choice([1, 2]))
    k = int(rng.choice([3, 3, 3, 1, 5]))
    pad = k // 2
    n = int(rng.integers(1, 4))
    cin = int(rng.choice([3, 16, 64, 70, 128, 192]))
    cout = int(rng.choice([8, 16, 48, 64, 80, 96, 160, 256, 300]))
    h = int(rng.integers(5, 40))
    wd = int(rng.choice([h, h + 4, 56, 28, 20]))
    relu = bool(rng.integers(0, 2))
    bf16 = bool(rng.integers(0, 2))
    w = W.conv_nchw_view(n, cin, h, wd, cout, k, s, pad, 1, relu)
    x = W.gen_uniform([n, cin, h, wd], 100 + t)
    wt = W.gen_normal([cout, cin, k, k], 200 + t, (2.0 / (cin * k * k)) ** 0.5)
    if bf16:
        w.src_a, w.src_b = W.to_bf16_bits(x), W.to_bf16_bits(wt)
        w.dtype_a = w.dtype_b = W.Dtype.BF16
        xr, wr = W.bf16_bits_to_f32(w.src_a), W.bf16_bits_to_f32(w.src_b)
        tol = 1e-4
    else:
        w.src_a, w.src_b = x, wt
        xr, wr = x, wt
        tol = 1e-4
    want = O.conv2d(xr, wr, s, pad, 1, relu)
    for v in variants:
        old = {kk: os.environ.get(kk) for kk in v}
        os.environ.update(v)
        try:
            got = run_full(w)
            err = float(np.max(np.abs(got - want) / (1 + np.abs(want))))
        except Exception as e:
            err = float('inf'); print("ERROR", e)
        finally:
            for kk, vv in old.items():
                if vv is None: os.environ.pop(kk, None)
                else: os.environ[kk] = vv
        if not err <= tol:
            bad += 1
            print(f"BAD case {t}: n={n} cin={cin} h={h} w={wd} cout={cout} k={k} s={s} relu={relu} bf16={bf16} variant={v} err={err:.3g}")
print("cases", n_cases, "x variants", len(variants), "bad", bad)
