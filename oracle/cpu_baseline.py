"""CPU baseline: the UNMODIFIED reference engine (merit::run_full, compiled
into oracle/_ref/libmerit_ref.so) timed on the host cores, on a bounded
sample of a BASELINE config.  BASELINE / TEST INFRASTRUCTURE ONLY (bench.py's
cpu_baseline leg and --impl reference arm).

One process per core (processes, not threads: the engine's per-step heap
allocations make threads scale poorly); each process runs an
independent shard Workload through the reference API.  If the reference
library is unavailable the C restatement (oracle.c, kind "port") is timed
instead, with the same sharding.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

_state = {}


def _kind():
    from oracle import binding as O
    try:
        O.ref()
        return "reference"
    except Exception:
        return "port"


def _init(config, seed):
    from paper_1911_03458_b200 import workloads as W
    from oracle import binding as O
    _state["kind"] = _kind()
    _state["O"] = O
    if config == "C2":
        cur, ref = W.gen_me_pair(1080, 1920, 2 + seed)
        _state["frames"] = (cur, ref)
    elif config == "C5":
        cur, ref = W.gen_me_pair(2160, 3840, 5 + seed)
        _state["frames"] = (cur, ref)
    elif config == "C1":
        _state["x"] = W.gen_uniform([1, 64, 112, 112], 1 + seed)
    elif config in ("C3", "C4"):
        cin, h, cout = CONV_GEOM[config][1:4]
        x = W.gen_uniform([1, cin, h, h], 3 + seed)
        wt = W.gen_normal([cout, cin, 3, 3], 4 + seed, (2.0 / (9 * cin)) ** 0.5)
        if config == "C4":  # the engine has no bf16: bf16-rounded values in REAL32
            x = W.bf16_bits_to_f32(W.to_bf16_bits(x))
            wt = W.bf16_bits_to_f32(W.to_bf16_bits(wt))
        _state["x"], _state["wt"] = x, wt


# (N, Cin, H=W, Cout, stride) of the conv configs
CONV_GEOM = {"C3": (32, 64, 56, 64, 1), "C4": (256, 128, 56, 256, 2)}


def strip_workload(config, shard, units):
    """A shard of `units` ranged-inner-product rows of the config, as a custom
    ViewSpec over the full source tensors (offsets select the shard)."""
    from paper_1911_03458_b200 import workloads as W
    from paper_1911_03458_b200.merit import ViewTerm
    if config in ("C2", "C5"):
        H, Wd, blk, r = (1080, 1920, 16, 16) if config == "C2" else (2160, 3840, 16, 32)
        BX = Wd // blk
        BY = H // blk
        by = shard % BY
        bx0 = (shard // BY * units) % BX
        nbx = min(units, BX - bx0)
        w = W.me_view(H, Wd, blk, r)
        w.view_a.p_shape[1] = nbx
        w.view_b.p_shape[1] = nbx
        for v in (w.view_a, w.view_b):
            v.p_shape[0] = 1
            v.terms.append(ViewTerm(0, 0, 0, by * blk))    # block row offset
            v.terms.append(ViewTerm(1, 1, 0, bx0 * blk))   # block column offset
        cur, ref = _state["frames"]
        w.src_a, w.src_b = cur, ref
        return w, nbx * (2 * r + 1) ** 2
    if config == "C1":
        w = W.maxpool_nchw_view(1, 64, 112, 112)
        w.src_a = _state["x"]
        return w, 64 * 56 * 56
    if config in ("C3", "C4"):
        # `units` output channels of one image (all output pixels)
        _, cin, h, cout, s = CONV_GEOM[config]
        co0 = (shard * units) % cout
        units = min(units, cout - co0)
        w = W.conv_nchw_view(1, cin, h, h, units, 3, s, 1)
        w.src_a = _state["x"]
        w.src_b = np.ascontiguousarray(_state["wt"][co0:co0 + units])
        ho = (h + 2 - 3) // s + 1
        return w, units * ho * ho
    raise ValueError(config)


def _work(args):
    config, shard, units = args
    w, outputs = strip_workload(config, shard, units)
    O = _state["O"]
    t0 = time.perf_counter()
    if _state["kind"] == "reference":
        O.ref_run_full(w)
    else:
        O.run_full(w)
    return outputs, time.perf_counter() - t0


class CpuBaseline:
    """Pool of P worker processes, each timing reference-engine shards."""

    def __init__(self, config="C2", procs=None, seed=0):
        self.config = config
        self.procs = procs or os.cpu_count() or 1
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(self.procs, initializer=_init, initargs=(config, seed))
        self.kind = self.pool.apply(_kind)

    def step(self, units_per_proc, first_shard=0):
        jobs = [(self.config, first_shard + i, units_per_proc) for i in range(self.procs)]
        t0 = time.perf_counter()
        res = self.pool.map(_work, jobs, chunksize=1)
        wall = time.perf_counter() - t0
        return sum(r[0] for r in res), wall

    def close(self):
        self.pool.close()
        self.pool.join()


def unit_cost_s(config, kind):
    """Rough seconds per unit (block / image) for sizing a bounded sample:
    ~5.8 M abs-diff/s/core for the reference engine."""
    if config == "C2":
        per = 1089 * 256
    elif config == "C5":
        per = 4225 * 256
    elif config in ("C3", "C4"):
        _, cin, h, _, s = CONV_GEOM[config]
        ho = (h + 2 - 3) // s + 1
        per = ho * ho * cin * 9  # MACs per output channel of one image
    else:
        per = 64 * 56 * 56 * 9
    rate = 1.1e6 if kind == "reference" else 3.0e8  # measured: 4 blocks/proc in 5.5 s
    if config in ("C3", "C4") and kind == "reference":
        rate = 6.0e6  # measured: one C4 output channel (0.9 M MAC) in 0.13 s, warm
    return per / rate


if __name__ == "__main__":
    cb = CpuBaseline(sys.argv[1] if len(sys.argv) > 1 else "C2")
    n, t = cb.step(4)
    print(cb.kind, cb.procs, n, t, n / t)
    cb.close()
