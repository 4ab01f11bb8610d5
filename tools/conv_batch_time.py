"""Time the C4-shaped convolution at several batch sizes (GPU): exposes the
persistent grid's wave quantisation (units per CTA pair).

  python tools/conv_batch_time.py 256 248 244 ...
Relative experiments only (the bench is bench.py).
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1911_03458_b200 import Plan  # noqa: E402
from paper_1911_03458_b200 import workloads as W  # noqa: E402

for n in map(int, sys.argv[1:] or ["256"]):
    w = W.conv_nchw_view(n, 128, 56, 56, 256, 3, 2, 1)
    w.dtype_a = w.dtype_b = W.Dtype.BF16
    plan = Plan(w)
    g = torch.Generator().manual_seed(1)
    a = (torch.rand(n, 128, 56, 56, generator=g) * 2 - 1).bfloat16().view(torch.uint16).cuda()
    b = (torch.randn(256, 128, 3, 3, generator=g) * 0.04).bfloat16().view(torch.uint16).cuda()
    plan.pack_b(b)
    sets = [(a.clone(), torch.empty(int(plan.info.out_bytes), dtype=torch.uint8, device="cuda")) for _ in range(2)]
    for i in range(3):
        plan.run(sets[i % 2][0], None, sets[i % 2][1])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(40):
        plan.run(sets[i % 2][0], None, sets[i % 2][1])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 40
    print(f"N={n}: {us:8.2f} us  {us / n:6.3f} us/image  {2 * n * 256 * 28 * 28 * 1152 / us / 1e6:7.1f} TFLOP/s  "
          f"[{plan.description}]", flush=True)
