"""One convolution case against the oracle, repeated (GPU).
usage: python tools/conv_case.py n cin h w cout k s relu(0/1) bf16(0/1) [repeats]"""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1911_03458_b200.workloads as W
from paper_1911_03458_b200 import run_full, _capi
import oracle.binding as O

n, cin, h, wd, cout, k, s, relu, bf16 = map(int, sys.argv[1:10])
reps = int(sys.argv[10]) if len(sys.argv) > 10 else 3
pad = k // 2
w = W.conv_nchw_view(n, cin, h, wd, cout, k, s, pad, 1, bool(relu))
x = W.gen_uniform([n, cin, h, wd], 100)
wt = W.gen_normal([cout, cin, k, k], 200, (2.0 / (cin * k * k)) ** 0.5)
if bf16:
    w.src_a, w.src_b = W.to_bf16_bits(x), W.to_bf16_bits(wt)
    w.dtype_a = w.dtype_b = W.Dtype.BF16
    xr, wr = W.bf16_bits_to_f32(w.src_a), W.bf16_bits_to_f32(w.src_b)
else:
    w.src_a, w.src_b = x, wt
    xr, wr = x, wt
want = O.conv2d(xr, wr, s, pad, 1, bool(relu))
poison = None
import os
if os.environ.get("CONV_CASE_POISON"):  # NaN-fill every SM's shared memory before each run (tests/cuda/poison.cu)
    import ctypes
    sys.path.insert(0, "tests/cuda")
    import build_helpers
    poison = ctypes.CDLL(str(build_helpers.build()))
    poison.poison_shared_memory.argtypes = [ctypes.c_uint32, ctypes.c_void_p]
for i in range(reps):
    if poison is not None:
        assert poison.poison_shared_memory(0xFFFFFFFF, None) == 0
    got = run_full(w)
    e = np.abs(got - want) / (1 + np.abs(want))
    bad = np.argwhere(~(e <= 1e-4))
    kern = (_capi.load().merit_dev_last_kernel() or b"").decode()
    print(f"err {float(np.nanmax(e)):.3e} nan {int(np.isnan(got).sum())} bad {len(bad)} first {bad[:3].tolist()} last {bad[-2:].tolist()} | {kern}")
