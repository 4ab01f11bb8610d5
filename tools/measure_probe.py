"""GPU probe of merit_dev_measure_traffic on the C1 / C2 plans (diagnostics)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1911_03458_b200 import Plan, FLAG_ARGMIN, Error  # noqa: E402
from paper_1911_03458_b200 import workloads as W  # noqa: E402

for cfg in ("C1", "C2"):
    w = W.config_workload(cfg, scale=4) if cfg == "C1" else W.config_workload(cfg)
    plan = Plan(w, FLAG_ARGMIN if cfg == "C2" else 0)
    a = torch.from_numpy(np.ascontiguousarray(w.src_a)).cuda()
    b = torch.from_numpy(np.ascontiguousarray(w.src_b)).cuda()
    o = torch.empty(max(1, int(plan.info.out_bytes)), dtype=torch.uint8, device="cuda")
    x = torch.empty(max(1, int(plan.info.aux_elems)), dtype=torch.int32, device="cuda")
    try:
        print(cfg, plan.measure_traffic(a, b, o, x if plan.info.aux_elems else None), flush=True)
    except Error as e:
        print(cfg, "error", e, flush=True)
