"""Time the correlation kernel (K4) against the exact interpreter (K0) (GPU).

usage: python tools/corr_time.py [c h w d] ...   (default: small + FlowNetC-sized)
CUDA events over back-to-back launches on device buffers.
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1911_03458_b200 import FLAG_EXACT, Plan  # noqa: E402
from paper_1911_03458_b200 import workloads as W  # noqa: E402


def time_plan(plan, a, b, out, iters):
    for _ in range(2):
        plan.run(a, b, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        plan.run(a, b, out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


specs = [tuple(map(int, s.split())) for s in sys.argv[1:]] or [(64, 24, 24, 9), (256, 48, 48, 21)]
for (c, h, w, d) in specs:
    wl = W.build_template("correlation", {"c": c, "h": h, "w": w, "d": d})
    for t in wl.view_b.terms:
        if t.component in (2, 3):
            t.offset = -(d // 2)
    a = torch.rand(c * h * w, device="cuda")
    b = torch.rand(c * h * w, device="cuda")
    flops = 2.0 * c * h * w * d * d
    for flags, name in ((0, "K4"), (FLAG_EXACT, "K0")):
        plan = Plan(wl, flags)
        out = torch.empty(int(plan.info.out_bytes), dtype=torch.uint8, device="cuda")
        us = time_plan(plan, a, b, out, 50 if flags == 0 else 3)
        print(f"c={c} {h}x{w} d={d} {name}: {us:10.2f} us  {flops / us / 1e6:8.3f} TFLOP/s  [{plan.description[:60]}]",
              flush=True)
