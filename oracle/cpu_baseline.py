"""CPU baselines of bench.py: the reference's own CPU path timed on the host
cores on a bounded sample of a BASELINE config.  BASELINE / TEST
INFRASTRUCTURE ONLY (bench.py's cpu_baseline leg and --impl reference arm).

Two legs, both through the UNMODIFIED reference compiled from its headers
(oracle/_ref/libmerit_ref.so, oracle/ref_shim.cpp `ref_sample_*`):

* ``engine`` — ``merit::run_full`` (engine.hpp:282-287), the operator the
  device library replaces, on the config's batched custom view restricted to
  the sample;
* ``oracle_loop`` — the reference's brute-force oracle loops
  (workloads.hpp:458-499 conv, :548-585 motion estimation, :642-671
  max-pool) on the same amount of work: the fastest CPU code the reference
  ships for these operators.

One process per core (processes, not threads: the engine's per-step heap
allocations make threads scale poorly); each runs independent
shards.  Inputs are generated with liboracle (oracle.c's restatement of the
SURVEY §8(d) generators, byte-identical to the GPU arm's), so these worker
processes never import the product package or map libmerit_dev.so.  If the
reference library is unavailable the C restatement's brute-force loops are
timed instead (kind "port").
"""
from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

_state = {}

# (N, Cin, H=W, Cout, stride) of the conv configs
CONV_GEOM = {"C3": (32, 64, 56, 64, 1), "C4": (256, 128, 56, 256, 2)}
# (H, W, radius) of the motion-estimation configs; C5 runs 16x16 and 8x8 blocks
ME_GEOM = {"C2": (1080, 1920, 16), "C5": (2160, 3840, 32)}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _kind():
    from oracle import binding as O
    try:
        O.ref()
        return "reference"
    except Exception:
        return "port"


def _init(config, seed):
    import numpy as np
    from oracle import binding as O
    _state["kind"] = _kind()
    _state["config"] = config
    ref = O.ref() if _state["kind"] == "reference" else None
    if config in ME_GEOM:
        H, W, _ = ME_GEOM[config]
        cur, refr = O.gen_me_pair(H, W, (2 if config == "C2" else 5) + seed)
        _state["frames"] = (cur, refr)
        if ref is not None:
            ref.ref_bench_load_frames(O._p(cur), O._p(refr), H, W)
    elif config == "C1":
        x = O.gen_uniform([1, 64, 112, 112], 1 + seed)
        _state["x"] = x
        if ref is not None:
            ref.ref_bench_load_images(O._p(x), 64, 112, None, 0)
    elif config in CONV_GEOM:
        _, cin, h, cout, _ = CONV_GEOM[config]
        x = O.gen_uniform([1, cin, h, h], (3 if config == "C3" else 4) + seed)
        wt = O.gen_normal([cout, cin, 3, 3], (1003 if config == "C3" else 1004) + seed, (2.0 / (9 * cin)) ** 0.5)
        if config == "C4":  # the engine has no bf16: bf16-rounded values in REAL32
            x = (O.to_bf16_bits(x).astype(np.uint32) << 16).view(np.float32)
            wt = (O.to_bf16_bits(wt).astype(np.uint32) << 16).view(np.float32)
        x = np.ascontiguousarray(x, np.float32)
        wt = np.ascontiguousarray(wt, np.float32)
        _state["x"], _state["wt"] = x, wt
        if ref is not None:
            ref.ref_bench_load_images(O._p(x), cin, h, O._p(wt), cout)


def _me_sample(blk, radius, shard, units, leg):
    """`units` blocks of one block row of the loaded frame pair."""
    from oracle import binding as O
    H, W, _ = ME_GEOM[_state["config"]]
    BX, BY = W // blk, H // blk
    by = shard % BY
    bx0 = (shard // BY * units) % BX
    nbx = min(units, BX - bx0)
    if _state["kind"] == "reference":
        n = O.ref().ref_sample_me(blk, radius, by, bx0, nbx, 0 if leg == "engine" else 1)
        if n < 0:
            raise RuntimeError(O.ref().ref_last_error().decode())
        return n
    # port: the C restatement's brute-force loop on the same blk x (nbx*blk) crop
    cur, ref = _state["frames"]
    rows, cols = slice(by * blk, by * blk + blk), slice(bx0 * blk, (bx0 + nbx) * blk)
    return O.me_sad(cur[rows, cols].copy(), ref[rows, cols].copy(), blk, radius).size


def _work(args):
    config, shard, units, leg = args
    from oracle import binding as O
    t0 = time.perf_counter()
    if config == "C2":
        n = _me_sample(16, 16, shard, units, leg)
    elif config == "C5":
        # the C5 mix: per 16x16 block also four 8x8 blocks (both block sizes
        # do the same abs-diff work per frame, BASELINE configs[4])
        n = _me_sample(16, 32, shard, units, leg) + _me_sample(8, 32, shard, 4 * units, leg)
    elif config == "C1":
        if _state["kind"] == "reference":
            n = O.ref().ref_sample_maxpool(0 if leg == "engine" else 1)
        else:
            n = O.maxpool(_state["x"], 56, 56).size
    else:
        _, cin, h, cout, s = CONV_GEOM[config]
        co0 = (shard * units) % cout
        u = min(units, cout - co0)
        if _state["kind"] == "reference":
            n = O.ref().ref_sample_conv(s, co0, u, 0 if leg == "engine" else 1)
        else:
            n = O.conv2d(_state["x"], _state["wt"][co0:co0 + u], s, 1).size
    if n < 0:
        raise RuntimeError(O.ref().ref_last_error().decode())
    return n, time.perf_counter() - t0


class CpuBaseline:
    """Pool of P worker processes, each timing reference shards."""

    def __init__(self, config="C5", procs=None, seed=0):
        self.config = config
        self.procs = procs or os.cpu_count() or 1
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(self.procs, initializer=_init, initargs=(config, seed))
        self.kind = self.pool.apply(_kind)

    def step(self, units_per_proc, first_shard=0, leg="engine"):
        jobs = [(self.config, first_shard + i, units_per_proc, leg) for i in range(self.procs)]
        t0 = time.perf_counter()
        res = self.pool.map(_work, jobs, chunksize=1)
        wall = time.perf_counter() - t0
        return sum(r[0] for r in res), wall

    def close(self):
        self.pool.close()
        self.pool.join()


def unit_cost_s(config, kind, leg="engine"):
    """Rough seconds per unit (block / output channel / image) for sizing a
    bounded sample (measured on the 16-core GPU hosts: the engine at ~1.1 M
    abs-diff/s and ~6 M MAC/s per process, the oracle loops ~50-100x faster)."""
    if config == "C2":
        per = 1089 * 256
    elif config == "C5":
        per = 2 * 4225 * 256   # one 16x16 block + four 8x8 blocks
    elif config in CONV_GEOM:
        _, cin, h, _, s = CONV_GEOM[config]
        ho = (h + 2 - 3) // s + 1
        per = ho * ho * cin * 9  # MACs per output channel of one image
    else:
        per = 64 * 56 * 56 * 9
    if kind != "reference":
        return per / 3.0e8
    if leg == "engine":
        rate = 6.0e6 if config in CONV_GEOM else 1.1e6
    else:
        rate = 2.0e8 if config in CONV_GEOM else 3.0e8
    return per / rate


if __name__ == "__main__":
    cb = CpuBaseline(sys.argv[1] if len(sys.argv) > 1 else "C5")
    for leg in ("engine", "oracle_loop"):
        n, t = cb.step(2, leg=leg)
        print(cb.kind, leg, cb.procs, n, t, n / t)
    cb.close()
