"""Time SAD kernel variants on C2 (map+argmin, map only, argmin only)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1911_03458_b200 import Plan, FLAG_ARGMIN, FLAG_NO_MAP
from paper_1911_03458_b200 import workloads as W

w = W.config_workload("C2")
dev = torch.device("cuda:0")
cur = torch.from_numpy(w.src_a).to(dev)
ref = torch.from_numpy(w.src_b).to(dev)
for name, flags in (("map+argmin", FLAG_ARGMIN), ("map", 0), ("argmin-only", FLAG_ARGMIN | FLAG_NO_MAP)):
    p = Plan(w, flags)
    out = torch.empty(max(1, p.info.out_bytes), dtype=torch.uint8, device=dev)
    aux = torch.empty(max(1, p.info.aux_elems), dtype=torch.int32, device=dev)
    for _ in range(5):
        p.run(cur, ref, out if p.info.out_elems else None, aux if p.info.aux_elems else None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        p.run(cur, ref, out if p.info.out_elems else None, aux if p.info.aux_elems else None)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:12s} {e0.elapsed_time(e1) / 100 * 1000:.1f} us")
