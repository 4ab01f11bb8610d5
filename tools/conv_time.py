"""Time the C3 / C4 convolution on device buffers (GPU).

usage: python tools/conv_time.py [C3|C4] [sets]
`sets` rotating input/output copies (default 1 = L2-warm; 4 for C3 / 2 for
C4 exceed L2 like bench.py).  Relative experiments only (the bench is bench.py).
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1911_03458_b200 import Plan  # noqa: E402
from paper_1911_03458_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
nsets = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = W.config_workload(name)
plan = Plan(w)
b = torch.from_numpy(w.src_b).cuda()
plan.pack_b(b)
sets = []
for i in range(nsets):
    a = torch.from_numpy(w.src_a).cuda()
    out = torch.empty(int(plan.info.out_bytes), dtype=torch.uint8, device="cuda")
    sets.append((a, out))
for i in range(3):
    plan.run(sets[i % nsets][0], None, sets[i % nsets][1])
torch.cuda.synchronize()
iters = 40
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(iters):
    plan.run(sets[i % nsets][0], None, sets[i % nsets][1])
e1.record()
torch.cuda.synchronize()
print("us", e0.elapsed_time(e1) * 1e3 / iters, plan.description)
