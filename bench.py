#!/usr/bin/env python
"""Benchmark of the MERIT device operator (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A "step" is one pass of the hot path over one batch of synthetic input of the
configuration (default C2 = BASELINE.json configs[1]: block-matching motion
estimation on a 1920x1080 uint8 frame pair, 16x16 blocks, +/-16, int32 SAD map
+ argmin with lowest-raster tie-break).  Metric: MERIT-op throughput = ranged
inner products (= elements of the reference operator's output,
prod(p_shape), engine.hpp:24-28) per second, in G/s.

* ``value``: device-resident inputs, the kernel timed with CUDA events over
  exactly K steps between a barrier + synchronize on both sides; input /
  output buffer sets rotate so the working set exceeds the 126 MB L2.
* ``e2e``: the same steps through the C-ABI host-buffer call
  (merit_dev_run_host: pinned H2D of the inputs, kernel, D2H of the SAD map +
  motion vectors) — the reference's run_full calling convention.
* ``roofline``: the dominant kernel's achieved rate vs the measured peak.
* ``cpu_baseline``: the UNMODIFIED reference engine (oracle/_ref) on a
  bounded sample, one process per host core (rank 0, N=1 only).

Multi-GPU (torchrun): one process per GPU, each rank processes its own frame
pair(s) (weak scaling, no collective on the data path); the timed region is
bracketed by barriers and the max over ranks is reported.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MERIT-op throughput (Goutputs/s) and % of HBM/tensor roofline at 1-8 B200"
UNIT = "Goutputs/s"
PROFILES = ROOT / "profiles"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def int_simd_peak():
    """Measured VABSDIFF4.U8.ACC throughput (tools/microbench/int_simd.cu) in
    abs-diff ops/s; falls back to 4 ops x 64 lanes/clk/SM x 148 SMs x 1965 MHz."""
    p = PROFILES / "int_simd_peak.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["vabsdiff4_absdiff_ops_per_s"]), "measured"
    return 4 * 64 * 148 * 1965e6, "analytic"


# --------------------------------------------------------------- clocks ----
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while running."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.005)

    def sample(self):
        if not self.nv:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if mask & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()
        self.sample()

    def summary(self, window):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "window": window}


# ------------------------------------------------------------- workloads ---
class Case:
    """One benchmark configuration bound to a device: rotating buffer sets."""

    def __init__(self, config: str, rank: int, world: int, device):
        import torch
        from paper_1911_03458_b200 import FLAG_ARGMIN, FLAG_NO_MAP, Plan
        from paper_1911_03458_b200 import workloads as W
        self.config = config
        self.torch = torch
        self.device = device
        flags = 0
        self.sets = []
        if config == "C2":
            w = W.config_workload("C2", with_inputs=False)
            flags = FLAG_ARGMIN
            self.plan = Plan(w, flags)
            nsets = 8   # 8 x (4.1 MB in + 35 MB SAD map) = 314 MB > 2 x L2
            for s in range(nsets):
                cur, ref = W.gen_me_pair(1080, 1920, 2 + rank * 1000 + s)
                self.sets.append(self._bufs(cur, ref))
            self.cpu_inputs = (cur, ref)
            self.units = "1 frame pair (1920x1080 u8) per rank per step"
            self.workload = "C2 motion estimation 1080p, 16x16 blocks, +/-16, SAD map + argmin"
            self.rotation = f"{nsets} rotating input/output sets ({nsets * 39.3:.0f} MB > 126 MB L2)"
            self.dtype = "u8 (int32 SAD)"
        elif config == "C1":
            # batch-sharded: 8 / world images per rank
            w = W.config_workload("C1", scale=world, with_inputs=False)
            n_img = w.view_a.p_shape[0]
            self.plan = Plan(w)
            nsets = 6 * max(1, 8 // n_img)
            for s in range(nsets):
                x = W.gen_uniform([n_img, 64, 112, 112], 1 + rank * 1000 + s)
                self.sets.append(self._bufs(x, np.zeros(1, np.float32)))
            self.cpu_inputs = (x, np.zeros(1, np.float32))
            self.units = f"{n_img} of the 8 images (N,64,112,112) per rank per step"
            self.workload = "C1 maxpool 3x3 s2 p1 fp32 NCHW (8,64,112,112)"
            self.rotation = f"{nsets} rotating input/output sets ({nsets * 4.0 * n_img:.0f} MB > 126 MB L2)"
            self.dtype = "f32"
        elif config in ("C3", "C4"):
            # C4 is batch-sharded over the GPUs (BASELINE configs[3]): 256 / world
            # images per rank; C3 runs its 32 images on every rank
            w = W.config_workload(config, scale=world if config == "C4" else 1, with_inputs=True,
                                  seed_offset=rank * 1000)
            n_img = w.view_a.p_shape[0]
            self.plan = Plan(w)
            # rotating device copies so the sets together exceed 2x L2 (C4
            # shards at 8 GPUs are 51 MB)
            nsets = 4 if config == "C3" else max(1, -(-300 // int(1.6 * n_img)))
            a0, b0 = w.src_a, w.src_b
            for s in range(nsets):
                a = a0 if s == 0 else (W.gen_uniform(list(a0.shape), 3 + rank * 1000 + s)
                                       if config == "C3" else a0)
                self.sets.append(self._bufs(a, b0))
            self.plan.pack_b(self.sets[0][1])
            torch.cuda.synchronize()
            self.cpu_inputs = (a0, b0)
            self.units = ("32 images (32,64,56,56) fp32 per rank per step" if config == "C3"
                          else f"{n_img} of the 256 images (N,128,56,56) bf16 per rank per step")
            self.workload = W.CONFIGS[config]
            self.rotation = (f"{nsets} rotating sets ({nsets * 51.5:.0f} MB > 126 MB L2)" if config == "C3"
                             else f"{nsets} rotating set(s) of {1.6 * n_img:.0f} MB (> 126 MB L2 in total)")
            self.dtype = "f32 (3-term bf16 split, fp32 accumulate)" if config == "C3" else "bf16 (fp32 accumulate)"
        elif config == "C5":
            pairs = max(1, 64 // world)
            w = W.config_workload("C5", with_inputs=True, pairs=pairs, seed_offset=rank * pairs)
            flags = FLAG_ARGMIN | FLAG_NO_MAP
            self.plan = Plan(w, flags)
            w8 = W.me_view(2160, 3840, 8, 32, pairs=pairs)
            self.plan8 = Plan(w8, flags)
            self.sets.append(self._bufs(w.src_a, w.src_b))
            self.cpu_inputs = (w.src_a[0], w.src_b[0])
            self.units = f"{pairs} frame pairs (3840x2160 u8) per rank per step, 16x16 and 8x8 blocks"
            self.workload = "C5 motion estimation 4K x64 pairs (sharded), 16x16 + 8x8 blocks, +/-32, argmin"
            self.rotation = "1.06 GB input working set > 126 MB L2"
            self.dtype = "u8 (int32 SAD)"
            self.aux8 = torch.empty(int(self.plan8.info.aux_elems), dtype=torch.int32, device=device)
        else:
            raise SystemExit(f"unknown config {config}")
        self.info = self.plan.info
        self.outputs_per_step = int(self.info.n_outputs) + (int(self.plan8.info.n_outputs) if config == "C5" else 0)

    def _bufs(self, a, b):
        torch = self.torch
        ta = torch.from_numpy(np.ascontiguousarray(a)).to(self.device)
        tb = torch.from_numpy(np.ascontiguousarray(b)).to(self.device)
        out = torch.empty(max(1, int(self.plan.info.out_bytes)), dtype=torch.uint8, device=self.device) \
            if hasattr(self, "plan") else None
        aux = torch.empty(max(1, int(self.plan.info.aux_elems)), dtype=torch.int32, device=self.device) \
            if hasattr(self, "plan") else None
        return ta, tb, out, aux

    def step(self, i, stream):
        a, b, out, aux = self.sets[i % len(self.sets)]
        self.plan.run(a, b, out if self.info.out_elems else None, aux if self.info.aux_elems else None,
                      stream=stream)
        if self.config == "C5":
            self.plan8.run(a, b, None, self.aux8, stream=stream)

    # e2e: host buffers through the C ABI (merit_dev_run_host)
    def e2e_setup(self):
        torch = self.torch
        a, b = self.cpu_inputs if self.config != "C5" else (None, None)
        if self.config == "C5":
            a = self.sets[0][0].cpu().numpy()
            b = self.sets[0][1].cpu().numpy()
        pa = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        pb = torch.from_numpy(np.ascontiguousarray(b)).pin_memory()
        po = torch.empty(max(1, int(self.info.out_bytes)), dtype=torch.uint8).pin_memory()
        px = torch.empty(max(1, int(self.info.aux_elems)), dtype=torch.int32).pin_memory()
        self.host = (pa, pb, po, px)
        self.h2d = pa.numel() * pa.element_size() + pb.numel() * pb.element_size()
        self.d2h = int(self.info.out_bytes) + int(self.info.aux_elems) * 4
        if self.config == "C5":
            self.host8 = torch.empty(max(1, int(self.plan8.info.aux_elems)), dtype=torch.int32).pin_memory()
            self.d2h += int(self.plan8.info.aux_elems) * 4

    def e2e_step(self, stream):
        import ctypes as C
        pa, pb, po, px = self.host
        lib = self.plan.lib
        st = lib.merit_dev_run_host(self.plan.handle, C.c_void_p(pa.data_ptr()), C.c_void_p(pb.data_ptr()),
                                    C.c_void_p(po.data_ptr()) if self.info.out_elems else None,
                                    C.c_void_p(px.data_ptr()) if self.info.aux_elems else None,
                                    C.c_void_p(stream))
        if st:
            raise RuntimeError(lib.merit_dev_last_error().decode())
        if self.config == "C5":
            st = lib.merit_dev_run_host(self.plan8.handle, C.c_void_p(pa.data_ptr()), C.c_void_p(pb.data_ptr()),
                                        None, C.c_void_p(self.host8.data_ptr()), C.c_void_p(stream))
            if st:
                raise RuntimeError(lib.merit_dev_last_error().decode())


def roofline(case: "Case", ms_per_launch: float, peaks, peaks_kind, kern: str, clk: dict):
    """Roofline object for the dominant kernel of the step.

    Tensor peak: the burst figure, unless the timed region ran power-capped
    (median SM clock below 97% of max with sw_power_cap reported), in which
    case the sustained figure of MEASURED_PEAKS.json applies (the profiling
    recipe's rule for a kernel timed inside a long run); frac_vs_burst is
    reported either way."""
    info = case.info
    traffic = None
    tf = PROFILES / "ncu_traffic.json"
    if tf.exists():
        try:
            d = json.loads(tf.read_text())
            traffic = d.get(case.config, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    sec = ms_per_launch * 1e-3
    hbm_peak = float(peaks["hbm_gbs"])
    bytes_alg = float(info.algorithmic_bytes)
    hbm = {"bound": "hbm", "achieved": round(bytes_alg / sec / 1e9, 1), "peak": hbm_peak,
           "unit": "GB/s", "frac": round(bytes_alg / sec / 1e9 / hbm_peak, 4),
           "traffic": traffic, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peaks_kind})",
           "algorithmic_bytes_per_launch": bytes_alg, "kernel": kern}
    if info.kernel == 3:  # tensor-core conv
        flops = 2.0 * float(info.algorithmic_ops)
        split = case.plan.description.split("split=")[1].split()[0]
        burst = float(peaks["bf16_tflops"])
        capped = ("sw_power_cap" in clk.get("reasons", []) and
                  float(clk.get("sm_mhz", 0)) < 0.97 * float(clk.get("sm_max_mhz", 1)))
        peak = float(peaks.get("bf16_tflops_sustained", burst)) if capped else burst
        achieved = flops / sec / 1e12
        r = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
             "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": kern,
             "peak_source": (f"MEASURED_PEAKS.json bf16_tflops_{'sustained' if capped else 'burst'} "
                             f"({peaks_kind}; timed region {'power-capped' if capped else 'at full clock'})"),
             "frac_vs_burst": round(achieved / burst, 4),
             "algorithmic_flops_per_launch": flops, "bf16_products_per_mac": int(split),
             "tensor_issue_frac": round(achieved * int(split) / peak, 4)}
        return r, hbm
    if info.kernel == 2:  # byte-SIMD SAD
        peak, pk = int_simd_peak()
        ops = float(info.algorithmic_ops) + (float(case.plan8.info.algorithmic_ops) if case.config == "C5" else 0.0)
        achieved = ops / sec
        r = {"bound": "alu", "achieved": round(achieved / 1e12, 2), "peak": round(peak / 1e12, 2),
             "unit": "Tabsdiff/s", "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": kern,
             "peak_source": f"VABSDIFF4.U8.ACC microbenchmark, profiles/int_simd_peak.json ({pk})",
             "algorithmic_ops_per_launch": ops}
        return r, hbm
    return hbm, None


def run_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback exists)")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    from paper_1911_03458_b200 import _capi
    lib = _capi.load()
    case = Case(args.config, rank, world, device)
    stream = torch.cuda.Stream(device)
    sp = stream.cuda_stream

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up (untimed)
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            case.step(i, sp)
    torch.cuda.synchronize()
    # clock soak: the same step, untimed, so the sampler sees the loaded clock
    clocks = ClockSampler(local)
    clocks.start()
    t_soak = time.perf_counter()
    i = 0
    with torch.cuda.stream(stream):
        while time.perf_counter() - t_soak < args.soak:
            for _ in range(8):
                case.step(i, sp)
                i += 1
            stream.synchronize()
    # timed region: exactly K steps.  By default the K launches are captured
    # once into a CUDA graph and the graph is replayed inside the timed region
    # (microsecond-scale kernels are otherwise bound by the host launch path).
    l0 = lib.merit_dev_launch_count()
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for i in range(args.steps):
                case.step(i, sp)
        torch.cuda.synchronize()
        # one untimed replay: the first launch of an instantiated graph also
        # uploads it (~1 us per captured node), which is not a step's cost
        with torch.cuda.stream(stream):
            graph.replay()
        torch.cuda.synchronize()
    launches = lib.merit_dev_launch_count() - l0
    kern_name = (lib.merit_dev_last_kernel() or b"").decode()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    if graph is not None:
        with torch.cuda.stream(stream):
            graph.replay()
    else:
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                case.step(i, sp)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks.stop()
    if graph is None:
        launches = lib.merit_dev_launch_count() - l0
        kern_name = (lib.merit_dev_last_kernel() or b"").decode()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    # e2e through the host-buffer C-ABI call
    case.e2e_setup()
    for i in range(max(1, min(args.warmup, 3))):
        case.e2e_step(sp)
    torch.cuda.synchronize()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        case.e2e_step(sp)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    barrier()
    te = torch.tensor([e2e_s], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())

    peaks, peaks_kind = load_peaks()
    total_outputs = case.outputs_per_step * args.steps * world
    value = total_outputs / (ms_max * 1e-3) / 1e9
    ms_per_launch = ms_max / args.steps / (2 if args.config == "C5" else 1)
    clk = clocks.summary(f"timed region + {args.soak:.1f} s soak of the same step just before")
    rf, rf2 = roofline(case, ms_per_launch if args.config != "C5" else ms_max / args.steps, peaks, peaks_kind,
                       kern_name, clk)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 5), "higher_is_better": True,
        "scaling": "strong" if args.config in ("C1", "C4", "C5") else "weak", "vs_baseline": None,
        "dtype": case.dtype, "data": "synthetic (seeded SplitMix64 generators, SURVEY §8(d))",
        "config": {"workload": case.workload, "units": case.units,
                   "outputs_per_step_per_rank": case.outputs_per_step,
                   "l2": case.rotation, "kernel": case.plan.description,
                   "parallelism": f"dp{world} (independent shards, no collective)",
                   "timing": ("CUDA events around one CUDA-graph replay of the K captured steps"
                              if not args.no_graph else "CUDA events around K eager launches")},
        "roofline": rf,
        "e2e": {"value": round(case.outputs_per_step * e2e_steps * world / e2e_s / 1e9, 4), "unit": UNIT,
                "h2d_bytes_per_step": int(case.h2d), "d2h_bytes_per_step": int(case.d2h),
                "steps": e2e_steps, "path": "merit_dev_run_host (pinned host buffers in, host results out)"},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if rf2 is not None:
        line["roofline_hbm"] = rf2
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(config, budget_s=20.0, steps=1, warmup=0):
    from oracle.cpu_baseline import CpuBaseline, unit_cost_s
    cfg = config
    cb = CpuBaseline(cfg)
    try:
        per_proc = max(1, int(budget_s / max(steps + warmup, 1) / unit_cost_s(cfg, cb.kind)))
        if cfg == "C1":
            per_proc = 1
        for i in range(warmup):
            cb.step(per_proc, first_shard=i * cb.procs)
        n = 0
        wall = 0.0
        for i in range(steps):
            dn, dt = cb.step(per_proc, first_shard=(warmup + i) * cb.procs)
            n += dn
            wall += dt
    finally:
        cb.close()
    unit_name = {"C2": "16x16 blocks of the 1080p pair", "C5": "16x16 blocks of a 4K pair",
                 "C1": "images (64 channels)", "C3": "output channels of one 56x56 image (fp32)",
                 "C4": "output channels of one image (bf16-rounded values in REAL32)"}[cfg]
    return {"value": round(n / wall / 1e9, 9), "unit": UNIT, "cores": cb.procs, "kind": cb.kind,
            "sample": f"{cfg}: {cb.procs} processes x {per_proc} {unit_name} per step, {steps} step(s), "
                      f"{n} outputs in {wall:.2f} s through merit::run_full"
                      + ("" if cfg == config else f" (CPU sample taken on {cfg})")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    budget = args.cpu_budget_ref
    cb = cpu_baseline(args.config, budget_s=budget, steps=args.steps, warmup=args.warmup)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "impl": "reference",
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (REAL32 engine)",
            "data": "synthetic (seeded SplitMix64 generators, SURVEY §8(d))",
            "config": {"workload": args.config, "parallelism": f"{cb['cores']} host processes"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--soak", type=float, default=0.5)
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--cpu-budget-ref", type=float, default=90.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA graph")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
