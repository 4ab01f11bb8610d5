"""K1 launch-configuration sweep on C1 (GPU): CTAs per SM x ring depth x
L2-prefetch depth, timed like bench.py (K launches over rotating input /
output sets > L2, captured once into a CUDA graph and replayed).

usage: python tools/maxpool_sweep.py [CTAS:STAGES:PF[:RB[:PDL]] ...]
       PF = bands per CTA prefetched into L2 before the PDL wait (-1 = all);
       PDL is read once per process (MERIT_PDL), so give one PDL value per run
"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1911_03458_b200 import Plan  # noqa: E402
from paper_1911_03458_b200 import workloads as W  # noqa: E402

variants = sys.argv[1:] or ["7:4:4", "7:4:-1", "4:4:-1", "3:4:-1", "3:8:-1", "2:8:-1", "4:2:-1", "3:2:-1"]
w = W.maxpool_nchw_view(8, 64, 112, 112, 3, 2, 1)
plan = Plan(w)
nsets = 10
sets = [(torch.rand(8 * 64 * 112 * 112, device="cuda"),
         torch.empty(int(plan.info.out_bytes), dtype=torch.uint8, device="cuda")) for _ in range(nsets)]
byts = 8 * 64 * (112 * 112 + 56 * 56) * 4
K = 200
for v in variants:
    parts = v.split(":")
    c, s, pf, rb, pdl = parts + ["4", "-1", "8", "1"][len(parts) - 1:]
    os.environ["MERIT_MP_CTAS"], os.environ["MERIT_MP_STAGES"], os.environ["MERIT_MP_PF"] = c, s, pf
    os.environ["MERIT_MP_RB"], os.environ["MERIT_PDL"] = rb, pdl
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for i in range(5):
            plan.run(sets[i % nsets][0], None, sets[i % nsets][1], stream=stream.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(K):
            plan.run(sets[i % nsets][0], None, sets[i % nsets][1], stream=torch.cuda.current_stream().cuda_stream)
    best = 1e9
    for rep in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record()
            g.replay()
            e1.record()
        torch.cuda.synchronize()
        if rep:  # the first replay uploads the graph
            best = min(best, e0.elapsed_time(e1) * 1e3 / K)
    print(f"ctas={c} stages={s} pf={pf:>3s} rb={rb:>2s} pdl={pdl}: {best:7.3f} us/step  {byts / best / 1e3:7.1f} GB/s "
          f"({byts / best / 1e3 / 6550.7 * 100:.1f}% of HBM)", flush=True)
