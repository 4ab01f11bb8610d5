import sys, torch
sys.path.insert(0,'.')
from paper_1911_03458_b200 import Plan, workloads as W
wl = W.build_template("correlation", {"c": 256, "h": 48, "w": 48, "d": 21})
for t in wl.view_b.terms:
    if t.component in (2, 3): t.offset = -10
a = torch.rand(256*48*48, device="cuda"); b = torch.rand(256*48*48, device="cuda")
plan = Plan(wl); out = torch.empty(int(plan.info.out_bytes), dtype=torch.uint8, device="cuda")
for _ in range(3): plan.run(a, b, out)
torch.cuda.synchronize()
