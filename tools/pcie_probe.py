"""PCIe copy rates on the GPU box and run_host time vs slice count (GPU).

usage: python tools/pcie_probe.py [configs...]   (default C2 C3)
Prints H2D / D2H / concurrent GB/s for a few sizes (pinned host memory), then
the merit_dev_run_host wall time per config for MERIT_HOST_CHUNKS in a sweep.
"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_03458_b200 import FLAG_ARGMIN, Plan  # noqa: E402
from paper_1911_03458_b200 import workloads as W  # noqa: E402

dev = torch.device("cuda", 0)


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


def copy_rates():
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for mb in (4, 26, 206):
        n = mb << 20
        h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
        h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
        d_in = torch.empty(n, dtype=torch.uint8, device=dev)
        d_out = torch.empty(n, dtype=torch.uint8, device=dev)

        def h2d():
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)

        def d2h():
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)

        def both():
            h2d()
            d2h()

        t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
        print(f"{mb:4d} MB: H2D {n / t1 / 1e9:6.1f} GB/s  D2H {n / t2 / 1e9:6.1f} GB/s  "
              f"concurrent {2 * n / t3 / 1e9:6.1f} GB/s (sum)", flush=True)


def run_host_sweep(name):
    flags = FLAG_ARGMIN if name == "C2" else 0
    w = W.config_workload(name, scale=8 if name == "C4" else 1)
    a = torch.from_numpy(np.ascontiguousarray(w.src_a)).pin_memory()
    b = torch.from_numpy(np.ascontiguousarray(w.src_b)).pin_memory()
    s = torch.cuda.Stream()
    for chunks in (1, 2, 4, 8, 12, 16, 24, 32):
        os.environ["MERIT_HOST_CHUNKS"] = str(chunks)
        plan = Plan(w, flags)
        o = torch.empty(max(1, int(plan.info.out_bytes)), dtype=torch.uint8).pin_memory()
        x = torch.empty(max(1, int(plan.info.aux_elems)), dtype=torch.int32).pin_memory()

        def rh():
            st = plan.lib.merit_dev_run_host(plan.handle, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                             C.c_void_p(o.data_ptr()) if plan.info.out_elems else None,
                                             C.c_void_p(x.data_ptr()) if plan.info.aux_elems else None,
                                             C.c_void_p(s.cuda_stream))
            assert st == 0

        t = timed(rh, 20)
        mb = (plan.info.src_a_bytes + plan.info.src_b_bytes + plan.info.out_bytes + 4 * plan.info.aux_elems) / 1e6
        print(f"{name} chunks={chunks:2d}: {t * 1e3:7.3f} ms  ({mb / t / 1e3:5.1f} GB/s moved)", flush=True)
    os.environ.pop("MERIT_HOST_CHUNKS", None)


if __name__ == "__main__":
    copy_rates()
    for name in sys.argv[1:] or ["C2", "C3"]:
        run_host_sweep(name)
