#!/usr/bin/env python
"""Benchmark of the MERIT device operator (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

Metric: MERIT-op throughput = ranged inner products (= elements of the
reference operator's output, prod(p_shape), engine.hpp:24-28) per second, in
G/s, plus the binding roofline fraction of the dominant kernel.

A "step" is one pass of the hot path over one batch of the configuration.
Default config C5 (BASELINE.json configs[4], the largest configuration that
fits one GPU): motion estimation over 64 pairs of 3840x2160 uint8 frames,
16x16 and 8x8 blocks (the reference runs them as two Workloads), +/-32,
argmin with the lowest-raster tie-break.  --config C1..C4 selects the others.

* ``value``: device-resident inputs, the K steps timed with CUDA events on the
  launching stream between a barrier + synchronize on both sides, the max
  over ranks; input sets rotate / exceed the 126 MB L2.
* ``e2e``: the same steps through the C-ABI host-buffer call
  (merit_dev_run_host: pinned H2D of the inputs, kernels, D2H of the
  results) — the reference's run_full calling convention.
* ``roofline``: the dominant kernel's achieved rate vs the measured peak.
* ``cpu_baseline``: the UNMODIFIED reference (oracle/_ref) on a bounded
  sample, one process per host core (rank 0, N=1 only): merit::run_full, and
  the reference's brute-force oracle loop as a second, labelled figure.

Multi-GPU: ``--gpus N`` without a torchrun environment re-launches itself
under torch.distributed.run with N ranks (one process per GPU).  Every rank
runs its own shard with no collective on the data path: C1 /
C3 / C4 / C5 split their batch of images / frame pairs, C2 splits its one
frame pair into block-row bands, each with the Eq. 6 footprint of its band
(its rows plus the 16-row search halo, paper_1911_03458_b200/shard.py).
NCCL carries only the barriers and the max-over-ranks timing.  ``--dry-run``
runs the rank logic on CPU (gloo) and prints each rank's shard.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
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
DATA = "synthetic (seeded SplitMix64 generators, SURVEY §8(d))"

# config.workload: the same string in both arms
WORKLOAD = {
    "C1": "C1 max-pool 3x3 s2 p1 (-inf pad) fp32 NCHW (8,64,112,112)",
    "C2": "C2 motion estimation 1920x1080 u8 pair, 16x16 blocks, +/-16, int32 SAD map + argmin",
    "C3": "C3 conv fp32 NCHW (32,64,56,56) * (64,64,3,3) s1 p1",
    "C4": "C4 conv bf16 NCHW (256,128,56,56) * (256,128,3,3) s2 p1, fp32 accumulate",
    "C5": "C5 motion estimation 64 x 3840x2160 u8 pairs, 16x16 + 8x8 blocks, +/-32, argmin",
}
BATCH = {"C1": 8, "C2": 67, "C3": 32, "C4": 256, "C5": 64}   # units split over ranks (C2: block rows)


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


# --------------------------------------------------------------- shards ----
def shard_for(config: str, rank: int, world: int, with_inputs: bool = True, seed_offset: int = 0):
    """This rank's part of the config: (workloads, meta).

    workloads: the Workload(s) one step runs (C5: the 16x16 and the 8x8
    blocks, two Workloads over the same frames, as the reference runs them).
    meta: the shard range and a description.  The same function serves the
    GPU run and the --dry-run rank check."""
    from paper_1911_03458_b200 import workloads as W
    from paper_1911_03458_b200.shard import shard_band, shard_range, shard_workload
    total = BATCH[config]
    lo, hi = shard_range(total, world, rank)
    if config == "C2":
        w = W.config_workload("C2", with_inputs=with_inputs, seed_offset=seed_offset)
        s, (lo, hi) = shard_band(w, world, rank) if world > 1 else (w, (0, total))
        return [s], {"range": [lo, hi], "what": f"block rows [{lo}, {hi}) of the 67 (+ the Eq. 6 halo rows)"}
    if config == "C5":
        n = hi - lo
        w16 = W.config_workload("C5", with_inputs=with_inputs, pairs=n, seed_offset=lo + seed_offset)
        w8 = W.me_view(2160, 3840, 8, 32, pairs=n)
        w8.src_a, w8.src_b = w16.src_a, w16.src_b
        return [w16, w8], {"range": [lo, hi], "what": f"frame pairs [{lo}, {hi}) of the 64"}
    # C1 / C3 / C4: the batch axis
    w = W.config_workload(config, with_inputs=with_inputs, seed_offset=seed_offset)
    if world > 1:
        fp32 = getattr(w, "fp32_inputs", None)
        w, (lo, hi) = shard_workload(w, world, rank)
        if fp32 is not None:
            w.fp32_inputs = (fp32[0][lo:hi], fp32[1])
    name = {"C1": "images", "C3": "images", "C4": "images"}[config]
    return [w], {"range": [lo, hi], "what": f"{name} [{lo}, {hi}) of the {total}"}


# ------------------------------------------------------------- workloads ---
class Case:
    """One benchmark configuration bound to a device: plans + rotating buffers."""

    def __init__(self, config: str, rank: int, world: int, device, fuse: bool = True, sad_map: str = "i32"):
        import torch
        from paper_1911_03458_b200 import FLAG_ARGMIN, FLAG_NO_MAP, Plan, PlanGroup
        self.config = config
        self.torch = torch
        self.device = device
        ws, self.meta = shard_for(config, rank, world)
        if config == "C2" and sad_map == "u16":
            from paper_1911_03458_b200 import Dtype
            for w in ws:
                w.dtype_out = Dtype.U16  # exact (every 16x16 SAD <= 65,280): half the map bytes
        flags = {"C2": FLAG_ARGMIN, "C5": FLAG_ARGMIN | FLAG_NO_MAP}.get(config, 0)
        if len(ws) > 1 and fuse:
            # C5: the two Workloads over the same frames as one plan (one fused
            # launch: the 16x16 SADs are sums of 2 x 2 of the 8x8 ones)
            self.plans = [PlanGroup(ws, flags)]
        else:
            self.plans = [Plan(w, flags) for w in ws]
        self.workloads = ws
        w0 = ws[0]
        a_bytes = int(self.plans[0].info.src_a_bytes) + int(self.plans[0].info.src_b_bytes)
        out_bytes = sum(int(p.info.out_bytes) + 4 * int(p.info.aux_elems) for p in self.plans)
        # rotating input / output sets: together > 2 x the 126 MB L2
        per_set = a_bytes + out_bytes
        nsets = max(1, min(8, -(-300_000_000 // max(1, per_set))))
        self.sets = []
        for s in range(nsets):
            if s == 0:
                a, b = w0.src_a, w0.src_b
            elif config in ("C1", "C3"):
                a, b = (np.ascontiguousarray(np.roll(w0.src_a, s, axis=-1)), w0.src_b)
            elif config == "C2":
                a, b = np.roll(w0.src_a, s, axis=-1), np.roll(w0.src_b, s, axis=-1)
            else:  # C4 / C5 sets exceed L2 on their own; C4 at 8 GPUs: 51 MB per rank -> copies
                a, b = w0.src_a, w0.src_b
            self.sets.append(self._bufs(a, b))
        if config in ("C3", "C4"):
            self.plans[0].pack_b(self.sets[0][1])
            torch.cuda.synchronize()
        self.rotation = f"{nsets} rotating input/output set(s) of {per_set / 1e6:.0f} MB ({nsets * per_set / 1e6:.0f} MB; L2 126 MB)"
        self.outputs_per_step = sum(int(p.info.n_outputs) for p in self.plans)
        self.dtype = {"C1": "f32", "C2": "u8 (int32 SAD)" if sad_map == "i32" else "u8 (int32 SAD, uint16 map)", "C3": "f32 (3-term bf16 split, fp32 accumulate)",
                      "C4": "bf16 (fp32 accumulate)", "C5": "u8 (int32 SAD)"}[config]
        self.info = self.plans[0].info

    def _bufs(self, a, b):
        torch = self.torch
        ta = torch.from_numpy(np.ascontiguousarray(a)).to(self.device)
        tb = torch.from_numpy(np.ascontiguousarray(b)).to(self.device)
        outs = [torch.empty(max(1, int(p.info.out_bytes)), dtype=torch.uint8, device=self.device)
                if p.info.out_elems else None for p in self.plans]
        auxs = [torch.empty(max(1, int(p.info.aux_elems)), dtype=torch.int32, device=self.device)
                if p.info.aux_elems else None for p in self.plans]
        return ta, tb, outs, auxs

    def step(self, i, stream):
        a, b, outs, auxs = self.sets[i % len(self.sets)]
        for p, o, x in zip(self.plans, outs, auxs):
            p.run(a, None if p.packed else b, o, x, stream=stream)

    # e2e: host buffers through the C ABI (merit_dev_run_host)
    def e2e_setup(self):
        torch = self.torch
        w0 = self.workloads[0]
        pa = torch.from_numpy(np.ascontiguousarray(w0.src_a)).pin_memory()
        pb = torch.from_numpy(np.ascontiguousarray(w0.src_b)).pin_memory()
        self.host = (pa, pb)
        self.host_out = [(torch.empty(max(1, int(p.info.out_bytes)), dtype=torch.uint8).pin_memory(),
                          torch.empty(max(1, int(p.info.aux_elems)), dtype=torch.int32).pin_memory())
                         for p in self.plans]
        # every plan's run_host copies its sources (C5 unfused: twice)
        self.h2d = len(self.plans) * (pa.numel() * pa.element_size() + pb.numel() * pb.element_size())
        if self.config in ("C3", "C4"):
            self.h2d = pa.numel() * pa.element_size() + pb.numel() * pb.element_size()
        self.d2h = sum(int(p.info.out_bytes) + int(p.info.aux_elems) * 4 for p in self.plans)

    def e2e_step(self, stream):
        import ctypes as C
        pa, pb = self.host
        for p, (po, px) in zip(self.plans, self.host_out):
            st = p.lib.merit_dev_run_host(p.handle, C.c_void_p(pa.data_ptr()), C.c_void_p(pb.data_ptr()),
                                          C.c_void_p(po.data_ptr()) if p.info.out_elems else None,
                                          C.c_void_p(px.data_ptr()) if p.info.aux_elems else None,
                                          C.c_void_p(stream))
            if st:
                raise RuntimeError(p.lib.merit_dev_last_error().decode())


def roofline(case: "Case", ms_per_step: float, peaks, peaks_kind, kern: str, clk: dict):
    """Roofline object for the dominant kernel of the step.

    Tensor peak: the burst figure of MEASURED_PEAKS.json (the profiling
    recipe's figure for a kernel timed alone; a C3/C4 step is 25-120 us);
    the sustained figure is reported beside it.  SAD: the measured
    VABSDIFF4.U8.ACC rate."""
    info = case.info
    traffic = None
    tf = PROFILES / "ncu_traffic.json"
    if tf.exists():
        try:
            d = json.loads(tf.read_text())
            traffic = d.get(case.config, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    sec = ms_per_step * 1e-3
    hbm_peak = float(peaks["hbm_gbs"])
    bytes_alg = sum(float(p.info.algorithmic_bytes) for p in case.plans)
    hbm = {"bound": "hbm", "achieved": round(bytes_alg / sec / 1e9, 1), "peak": hbm_peak,
           "unit": "GB/s", "frac": round(bytes_alg / sec / 1e9 / hbm_peak, 4),
           "traffic": traffic, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peaks_kind})",
           "algorithmic_bytes_per_step": bytes_alg, "kernel": kern}
    if info.kernel == 3:  # tensor-core conv
        flops = 2.0 * float(info.algorithmic_ops)
        split = case.plans[0].description.split("split=")[1].split()[0]
        burst = float(peaks["bf16_tflops"])
        sustained = float(peaks.get("bf16_tflops_sustained", burst))
        achieved = flops / sec / 1e12
        r = {"bound": "tensor", "achieved": round(achieved, 1), "peak": burst, "unit": "TFLOP/s",
             "frac": round(achieved / burst, 4), "traffic": traffic, "kernel": kern,
             "peak_source": f"MEASURED_PEAKS.json bf16_tflops (burst, {peaks_kind})",
             "frac_vs_sustained": round(achieved / sustained, 4),
             "algorithmic_flops_per_launch": flops, "bf16_products_per_mac": int(split),
             "tensor_issue_frac": round(achieved * int(split) / burst, 4)}
        return r, hbm
    if info.kernel == 2:  # byte-SIMD SAD
        peak, pk = int_simd_peak()
        ops = sum(float(p.info.algorithmic_ops) for p in case.plans)
        exe = sum(float(p.info.executed_ops) for p in case.plans)
        # the fraction is of the abs-diffs the kernel executes: a fused plan's
        # shared work (C5: 16x16 SADs as sums of 8x8 ones) is not counted twice
        achieved = exe / sec
        r = {"bound": "alu", "achieved": round(achieved / 1e12, 2), "peak": round(peak / 1e12, 2),
             "unit": "Tabsdiff/s", "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": kern,
             "peak_source": f"VABSDIFF4.U8.ACC microbenchmark, profiles/int_simd_peak.json ({pk})",
             "executed_ops_per_step": exe, "algorithmic_ops_per_step": ops,
             "reference_equivalent_rate": round(ops / sec / 1e12, 2)}
        return r, hbm
    return hbm, None


def _dist_init(backend, device=None):
    import torch.distributed as dist
    kw = {"device_id": device} if device is not None else {}
    dist.init_process_group(backend, **kw)
    return dist


def time_device(case, steps, warmup, soak, stream, lib, barrier, local, graph=True):
    """W untimed warm-up steps, a clock soak of the same step, then exactly K
    steps between barrier + synchronize on both sides, CUDA events on the
    launching stream.  The K steps are captured once into a CUDA graph that is
    replayed inside the timed region (microsecond-scale kernels are otherwise
    bound by the host launch path).  Returns (ms, launches, last kernel, clocks)."""
    import torch
    sp = stream.cuda_stream
    with torch.cuda.stream(stream):
        for i in range(warmup):
            case.step(i, sp)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t_soak = time.perf_counter()
    i = 0
    with torch.cuda.stream(stream):
        while time.perf_counter() - t_soak < soak:
            for _ in range(4):
                case.step(i, sp)
                i += 1
            stream.synchronize()
    l0 = lib.merit_dev_launch_count()
    g = None
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i in range(steps):
                case.step(i, sp)
        torch.cuda.synchronize()
        # one untimed replay: the first launch of an instantiated graph also
        # uploads it (~1 us per captured node), which is not a step's cost
        with torch.cuda.stream(stream):
            g.replay()
        torch.cuda.synchronize()
    launches = lib.merit_dev_launch_count() - l0
    kern_name = (lib.merit_dev_last_kernel() or b"").decode()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    with torch.cuda.stream(stream):
        if g is not None:
            g.replay()
        else:
            for i in range(steps):
                case.step(i, sp)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks.stop()
    if g is None:
        launches = lib.merit_dev_launch_count() - l0
        kern_name = (lib.merit_dev_last_kernel() or b"").decode()
    return e0.elapsed_time(e1), launches, kern_name, clocks


# steps for the other configurations' per_config entries (microsecond-scale steps)
PER_CONFIG_STEPS = {"C1": 200, "C2": 200, "C3": 200, "C4": 100}


def time_e2e(case, steps, warm, sp, barrier=lambda: None):
    """The host-buffer C-ABI call (merit_dev_run_host: pinned host sources in,
    host results out, both copies inside the timed region): wall seconds for
    `steps` calls after `warm` untimed ones."""
    import torch
    case.e2e_setup()
    for _ in range(max(1, warm)):
        case.e2e_step(sp)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        case.e2e_step(sp)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    barrier()
    return dt


E2E_PATH = "merit_dev_run_host per plan (pinned host buffers in, host results out)"


def per_config_entries(args, device, stream, lib, local, peaks, peaks_kind):
    """The other configurations on the same GPU (N = 1 only), device-resident
    inputs, the same timing protocol as the headline (own K, W = 5, clock
    soak, CUDA-graph replay, rotating sets > L2): value, ms/step, the dominant
    kernel's roofline fraction and the clocks seen; the host-buffer call
    (e2e) and a short reference-engine sample on the host cores beside it."""
    import torch
    out = {}
    for c in ("C1", "C2", "C3", "C4"):
        if c == args.config:
            continue
        case = Case(c, 0, 1, device)
        k = PER_CONFIG_STEPS[c]
        ms, launches, kern, clk = time_device(case, k, 5, 0.3, stream, lib, lambda: None, local)
        step_ms = ms / k
        rf, _ = roofline(case, step_ms, peaks, peaks_kind, kern, None)
        out[c] = {"workload": WORKLOAD[c], "value": round(case.outputs_per_step / (step_ms * 1e-3) / 1e9, 4),
                  "unit": UNIT, "ms_per_step": round(step_ms, 6), "steps": k, "warmup": 5,
                  "dtype": case.dtype, "gpu_launches": int(launches), "l2": case.rotation,
                  "roofline": {kk: rf[kk] for kk in ("bound", "achieved", "peak", "unit", "frac", "kernel")
                               if kk in rf},
                  "clocks": clk.summary("timed region + 0.3 s soak")}
        n_e2e = max(1, min(args.e2e_steps, 10))
        e2e_s = time_e2e(case, n_e2e, 2, stream.cuda_stream)
        out[c]["e2e"] = {"value": round(case.outputs_per_step * n_e2e / e2e_s / 1e9, 4), "unit": UNIT,
                         "h2d_bytes_per_step": int(case.h2d), "d2h_bytes_per_step": int(case.d2h),
                         "steps": n_e2e, "path": E2E_PATH}
        if not args.no_cpu_baseline:
            out[c]["cpu_baseline"] = cpu_baseline(c, budget_s=args.cpu_budget / 3)
        del case
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback exists; --dry-run checks the rank logic)")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = _dist_init("nccl", device) if world > 1 else None
    from paper_1911_03458_b200 import _capi
    lib = _capi.load()
    case = Case(args.config, rank, world, device, fuse=not args.no_fuse, sad_map=args.sad_map)
    stream = torch.cuda.Stream(device)
    sp = stream.cuda_stream

    def barrier():
        if dist is not None:
            dist.barrier()

    ms, launches, kern_name, clocks = time_device(case, args.steps, args.warmup, args.soak, stream, lib, barrier,
                                                  local, graph=not args.no_graph)
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_per_step = torch.tensor([case.outputs_per_step], dtype=torch.float64, device=device)
    if dist is not None:
        dist.all_reduce(total_per_step)
    outputs_all = float(total_per_step.item())

    # e2e through the host-buffer C-ABI call
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    e2e_s = time_e2e(case, e2e_steps, min(args.warmup, 3), sp, barrier)
    te = torch.tensor([e2e_s], dtype=torch.float64, device=device)
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())

    peaks, peaks_kind = load_peaks()
    value = outputs_all * args.steps / (ms_max * 1e-3) / 1e9
    clk = clocks.summary(f"timed region + {args.soak:.1f} s soak of the same step just before")
    rf, rf2 = roofline(case, ms_max / args.steps, peaks, peaks_kind, kern_name, clk)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": case.dtype, "data": DATA,
        "config": {"workload": WORKLOAD[args.config],
                   "shard": f"rank 0: {case.meta['what']}" + (f" (one of {world} ranks)" if world > 1 else ""),
                   "outputs_per_step": int(outputs_all),
                   "l2": case.rotation, "kernel": " | ".join(p.description for p in case.plans),
                   "parallelism": f"dp{world} (independent shards, no collective on the data path)",
                   "timing": ("CUDA events around one CUDA-graph replay of the K captured steps"
                              if not args.no_graph else "CUDA events around K eager launches")},
        "roofline": rf,
        "e2e": {"value": round(outputs_all * e2e_steps / e2e_s / 1e9, 4), "unit": UNIT,
                "h2d_bytes_per_step": int(case.h2d), "d2h_bytes_per_step": int(case.d2h),
                "steps": e2e_steps, "path": E2E_PATH},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if rf2 is not None:
        line["roofline_hbm"] = rf2
    if world == 1 and args.config == "C5" and not args.no_per_config:
        line["per_config"] = per_config_entries(args, device, stream, lib, local, peaks, peaks_kind)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_budget)
        line["cpu_baseline_oracle_loop"] = cpu_baseline(args.config, budget_s=args.cpu_budget / 3,
                                                        leg="oracle_loop")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def cpu_baseline(config, budget_s=20.0, steps=1, warmup=0, leg="engine"):
    from oracle.cpu_baseline import CpuBaseline, cpu_model
    cb = CpuBaseline(config)
    try:
        # calibrate: one unit per process, then size the sample to the budget
        _, t1 = cb.step(1, first_shard=0, leg=leg)
        per_proc = max(1, int(budget_s / max(steps + warmup, 1) / max(t1, 1e-3)))
        if config == "C1":
            per_proc = 1
        elif config in ("C3", "C4"):
            per_proc = min(per_proc, 64)
        elif config == "C2":
            per_proc = min(per_proc, 120)
        elif config == "C5":
            per_proc = min(per_proc, 240)
        for i in range(warmup):
            cb.step(per_proc, first_shard=i * cb.procs, leg=leg)
        n = 0
        wall = 0.0
        for i in range(steps):
            dn, dt = cb.step(per_proc, first_shard=(warmup + i) * cb.procs, leg=leg)
            n += dn
            wall += dt
    finally:
        cb.close()
    unit_name = {"C2": "16x16 blocks of the 1080p pair", "C5": "(16x16 block + four 8x8 blocks) of a 4K pair",
                 "C1": "image(s) (64 channels)", "C3": "output channels of one 56x56 image (fp32)",
                 "C4": "output channels of one image (bf16-rounded values in REAL32)"}[config]
    path = ("merit::run_full (engine.hpp:282-287)" if leg == "engine" else
            "the reference's brute-force oracle loop (workloads.hpp oracle_*)")
    return {"value": round(n / wall / 1e9, 9), "unit": UNIT, "cores": cb.procs, "kind": cb.kind,
            "leg": leg, "cpu": cpu_model(),
            "sample": f"{config}: {cb.procs} processes x {per_proc} {unit_name} per step, {steps} step(s), "
                      f"{n} outputs in {wall:.2f} s through {path}"}


def run_reference(args):
    """The reference's own CPU implementation of the path (merit::run_full of
    the unmodified reference, oracle/_ref) on the host cores.  Under torchrun
    only rank 0 runs it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_baseline(args.config, budget_s=args.cpu_budget_ref, steps=args.steps, warmup=args.warmup)
    ol = cpu_baseline(args.config, budget_s=args.cpu_budget_ref / 4, steps=1, leg="oracle_loop")
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "impl": "reference",
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (REAL32 engine)", "data": DATA,
            "config": {"workload": WORKLOAD[args.config],
                       "parallelism": f"{cb['cores']} host processes ({cb['cpu']})"},
            "cpu_baseline": cb, "cpu_baseline_oracle_loop": ol,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_dry(args):
    """The N>1 rank logic on CPU (gloo): every rank builds its shard exactly
    as the GPU run does (shard_for, without generating inputs) and rank 0
    prints all ranks' shards."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = _dist_init("gloo") if world > 1 else None
    ws, meta = shard_for(args.config, rank, world, with_inputs=False)
    from paper_1911_03458_b200 import Plan
    from paper_1911_03458_b200 import FLAG_ARGMIN, FLAG_NO_MAP
    flags = {"C2": FLAG_ARGMIN, "C5": FLAG_ARGMIN | FLAG_NO_MAP}.get(args.config, 0)
    mine = {"rank": rank, "range": meta["range"], "what": meta["what"],
            "src_a_shape": list(ws[0].view_a.source_shape), "src_b_shape": list(ws[0].view_b.source_shape),
            "outputs": sum(int(Plan(w, flags).info.n_outputs) for w in ws),
            "kernels": [int(Plan(w, flags).kernel) for w in ws]}
    shards = [None] * world
    if dist is not None:
        dist.all_gather_object(shards, mine)
    else:
        shards = [mine]
    if rank == 0:
        print(json.dumps({"dry_run": True, "config": args.config, "n_gpus": world,
                          "workload": WORKLOAD[args.config], "shards": shards}), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_distributed(args) -> int:
    """--gpus N without a torchrun environment: run this script under
    torch.distributed.run with N ranks on this node."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 20 for C5; 200 / 200 / 200 / 100 for the microsecond-scale C1-C4, "
                         "whose K-step CUDA graph would otherwise be shorter than its own launch cost)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--soak", type=float, default=0.5)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--cpu-budget-ref", type=float, default=60.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA graph")
    ap.add_argument("--dry-run", action="store_true", help="CPU check of the multi-rank shard logic (gloo)")
    ap.add_argument("--no-per-config", action="store_true",
                    help="C5 at N=1: skip the per_config entries (C1-C4 on the same GPU, device-resident)")
    ap.add_argument("--no-fuse", action="store_true", help="C5: run the two Workloads as separate plans")
    ap.add_argument("--sad-map", default="i32", choices=["i32", "u16"],
                    help="C2: SAD map element type (u16 is exact and halves the map's bytes)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 20 if args.impl == "reference" else {"C5": 20, **PER_CONFIG_STEPS}[args.config]
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(relaunch_distributed(args))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
