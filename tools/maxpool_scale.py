"""K1 (max-pool 3x3/s2/p1, C1 geometry) time vs batch size (GPU).

usage: python tools/maxpool_scale.py [N ...]   (default 8 16 32 64)
Separates the per-launch ramp from the streaming rate: t(N) = t0 + bytes(N) / BW.
Rotating input/output sets keep every launch's working set out of L2.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_03458_b200 import Plan  # noqa: E402
from paper_1911_03458_b200 import workloads as W  # noqa: E402

ns = [int(a) for a in sys.argv[1:]] or [8, 16, 32, 64]
rows = []
for n in ns:
    w = W.maxpool_nchw_view(n, 64, 112, 112, 3, 2, 1)
    plan = Plan(w)
    nsets = max(2, -(-300 // (n * 4)))  # > 2x L2 in total
    sets = [(torch.rand(n * 64 * 112 * 112, device="cuda"),
             torch.empty(int(plan.info.out_bytes), dtype=torch.uint8, device="cuda")) for _ in range(nsets)]
    for i in range(3):
        plan.run(sets[i % nsets][0], None, sets[i % nsets][1])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 60
    e0.record()
    for i in range(iters):
        plan.run(sets[i % nsets][0], None, sets[i % nsets][1])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    byts = n * 64 * (112 * 112 + 56 * 56) * 4
    rows.append((n, us, byts))
    print(f"N={n:3d}: {us:8.2f} us  {byts / us / 1e3:7.1f} GB/s", flush=True)
if len(rows) >= 2:
    x = np.array([r[2] for r in rows], float)
    y = np.array([r[1] for r in rows], float)
    slope, t0 = np.polyfit(x, y, 1)
    print(f"fit: t = {t0:.2f} us + bytes / {1e-3 / slope:.0f} GB/s")
