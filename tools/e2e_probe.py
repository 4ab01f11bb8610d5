"""Where does the host-buffer (e2e) path spend time?  C2 sizes: 4.1 MB in,
35 MB map out; pinned host buffers; compares raw copies with run_host."""
import sys, time, ctypes as C
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1911_03458_b200 import Plan, FLAG_ARGMIN, workloads as W
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
w = W.config_workload("C2")
plan = Plan(w, FLAG_ARGMIN)
pa = torch.from_numpy(w.src_a).pin_memory(); pb = torch.from_numpy(w.src_b).pin_memory()
po = torch.empty(int(plan.info.out_bytes), dtype=torch.uint8).pin_memory()
px = torch.empty(int(plan.info.aux_elems), dtype=torch.int32).pin_memory()
da, db = pa.to(dev), pb.to(dev)
do = torch.empty(int(plan.info.out_bytes), dtype=torch.uint8, device=dev)
def t(fn, n=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3
with torch.cuda.stream(s):
    print("H2D 4.1MB ms", round(t(lambda: (da.copy_(pa, non_blocking=True), db.copy_(pb, non_blocking=True))), 3))
    print("D2H 35MB ms", round(t(lambda: po.copy_(do, non_blocking=True)), 3))
    print("D2H GB/s", round(35e6 / t(lambda: po.copy_(do, non_blocking=True)) / 1e6, 1))
lib = plan.lib
def rh():
    st = lib.merit_dev_run_host(plan.handle, C.c_void_p(pa.data_ptr()), C.c_void_p(pb.data_ptr()),
                                C.c_void_p(po.data_ptr()), C.c_void_p(px.data_ptr()), C.c_void_p(s.cuda_stream))
    assert st == 0
print("run_host ms", round(t(rh), 3))
