"""Time the SAD kernel on device-resident frames (GPU).

usage: python tools/sad_time.py [H W blk r pairs nomap] ...
Each spec prints us/launch and us per frame pair; back-to-back launches, CUDA
events, after warm-up.  Relative experiments only (the bench is bench.py).
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_03458_b200 import FLAG_ARGMIN, FLAG_NO_MAP, Plan  # noqa: E402
from paper_1911_03458_b200 import workloads as W  # noqa: E402


def time_spec(h, wd, blk, r, pairs, nomap, iters=50):
    w = W.me_view(h, wd, blk, r, pairs=pairs if pairs > 1 else None)
    flags = FLAG_ARGMIN | (FLAG_NO_MAP if nomap else 0)
    plan = Plan(w, flags)
    g = torch.Generator().manual_seed(1)
    shape = (pairs, h, wd) if pairs > 1 else (h, wd)
    a = torch.randint(0, 256, shape, dtype=torch.uint8, generator=g).cuda()
    b = torch.randint(0, 256, shape, dtype=torch.uint8, generator=g).cuda()
    out = torch.empty(max(1, int(plan.info.out_bytes)), dtype=torch.uint8, device="cuda")
    aux = torch.empty(max(1, int(plan.info.aux_elems)), dtype=torch.int32, device="cuda")
    run = lambda: plan.run(a, b, out if plan.info.out_elems else None, aux)  # noqa: E731
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    print(f"H={h} W={wd} blk={blk} r={r} pairs={pairs} nomap={nomap}: {us:9.2f} us/launch "
          f"{us / pairs:9.2f} us/pair  [{plan.description}]", flush=True)
    return us


if __name__ == "__main__":
    specs = sys.argv[1:] or ["1080 1920 16 16 1 0", "1080 1920 16 16 4 0", "1080 1920 16 16 1 1",
                             "1080 1920 16 16 4 1"]
    for s in specs:
        h, wd, blk, r, pairs, nomap = map(int, s.split())
        time_spec(h, wd, blk, r, pairs, bool(nomap))
