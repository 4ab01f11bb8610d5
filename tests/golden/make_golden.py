"""Generate golden fixtures FROM THE REFERENCE ITSELF.

Runs in the build container, where /root/reference exists: every vector here
is produced by oracle/_ref/libmerit_ref.so, i.e. the unmodified reference
headers (merit::build_template, merit::fill_random, merit::run_full,
merit::oracle) compiled by oracle/build.py.  Output: tests/golden/*.npz.

  python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import binding as O  # noqa: E402
from tests.golden_io import case_key  # noqa: E402
from tests.test_gpu_parity import TEMPLATE_CASES  # noqa: E402


class SplitMix64:  # workloads.hpp:74-94, to replay the reference tests' parameter draws
    def __init__(self, seed):
        self.state = seed & (2**64 - 1)

    def next(self):
        self.state = (self.state + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        return z ^ (z >> 31)

    def range(self, lo, hi):
        return lo + self.next() % (hi - lo + 1)

    def uniform(self, lo, hi):
        return lo + (hi - lo) * ((self.next() >> 11) * 2.0**-53)


def reference_random_cases():
    """The parameter draws of the reference's tests/test_workloads.cpp:123-216."""
    cases = []
    rng = SplitMix64(11)
    for t in range(30):
        prm = {"m": rng.range(1, 12), "n": rng.range(1, 12), "k": rng.range(1, 12)}
        if t % 2:
            prm["fix"] = 1
            prm["frac"] = rng.range(4, 10)
        cases.append(("gemm", prm, 1000 + t))
    rng = SplitMix64(12)
    for t in range(24):
        prm = {"h": rng.range(5, 12), "w": rng.range(5, 12), "k": rng.range(1, 3),
               "stride": rng.range(1, 2), "cin": rng.range(1, 2), "cout": rng.range(1, 3)}
        if t % 3 == 1:
            prm["fix"] = 1
            prm["frac"] = rng.range(4, 10)
        cases.append(("relu_fused_conv" if t % 3 == 2 else "conv2d", prm, 2000 + t))
    rng = SplitMix64(13)
    for t in range(12):
        prm = {"h": rng.range(6, 12), "w": rng.range(6, 12), "k": rng.range(1, 3)}
        if t % 2:
            prm["fix"] = 1
            prm["frac"] = 8
        cases.append(("dilated", prm, 3000 + t))
    rng = SplitMix64(14)
    for t in range(12):
        prm = {"c": rng.range(1, 4), "h": rng.range(3, 9), "w": rng.range(3, 9), "d": rng.range(1, 4)}
        cases.append(("correlation", prm, 4000 + t))
    rng = SplitMix64(15)
    for t in range(12):
        blk = 2 * rng.range(1, 2)
        prm = {"blk": blk, "h": blk * rng.range(1, 3), "w": blk * rng.range(1, 3),
               "win": 2 * rng.range(0, 2) + 1}
        if t % 2:
            prm["fix"] = 1
        cases.append(("motion_estimation", prm, 5000 + t))
    rng = SplitMix64(16)
    for t in range(8):
        prm = {"h": rng.range(4, 10), "w": rng.range(4, 10), "k": 2 * rng.range(0, 2) + 1,
               "sigma_r": rng.uniform(0.2, 1.5), "sigma_s": rng.uniform(0.5, 3.0)}
        cases.append(("bilateral", prm, 6000 + t))
    rng = SplitMix64(17)
    for t in range(12):
        k = rng.range(1, 3)
        prm = {"h": rng.range(k, 9), "w": rng.range(k, 9), "k": k, "stride": rng.range(1, k)}
        if t % 2:
            prm["fix"] = 1
        cases.append(("maxpool", prm, 7000 + t))
    return cases


def main():
    out = {}
    index = []
    for i, (name, prm) in enumerate(TEMPLATE_CASES):
        r = O.ref_template_case(name, prm, 9000 + i)
        k = case_key(name, prm)
        for f in ("src_a", "src_b", "engine", "oracle"):
            out[k + "::" + f] = r[f]
        out[k + "::fix"] = np.array(r["fix"])
    for name, prm, seed in reference_random_cases():
        r = O.ref_template_case(name, prm, seed)
        k = "random/" + case_key(name, prm) + f"|seed={seed}"
        for f in ("src_a", "src_b", "engine", "oracle"):
            out[k + "::" + f] = r[f]
        out[k + "::fix"] = np.array(r["fix"])
        index.append(k)
    out["random_index"] = np.array(index)
    # fill_random vectors (workloads.hpp:96-105) for seeds 1..5 and 2s+1/2s+2 style seeds
    import ctypes as C
    ref = O.ref()
    for seed in (1, 2, 3, 4, 5, 2001, 2002):
        v = np.empty(256, np.float32)
        ref.ref_fill_random_f32(v.ctypes.data_as(C.c_void_p), 256, seed, -1.0, 1.0)
        out[f"fill_f32/{seed}"] = v
        q = np.empty(256, np.int16)
        ref.ref_fill_random_i16(q.ctypes.data_as(C.c_void_p), 256, seed)
        out[f"fill_i16/{seed}"] = q
    np.savez_compressed(Path(__file__).parent / "templates.npz", **out)
    print("wrote", len(out), "arrays")

    # Config slices through the reference engine with the batched custom views.
    from paper_1911_03458_b200 import workloads as W
    cfg = {}
    w = W.maxpool_nchw_view(1, 3, 112, 112)  # C1 slice: 1 image, 3 channels
    w.src_a = W.gen_uniform([1, 3, 112, 112], 1)
    cfg["C1::src_a"], cfg["C1::engine"] = w.src_a, O.ref_run_full(w)
    cur, ref_ = W.gen_me_pair(64, 96, 2)      # C2-style crop: 16x16 blocks, +/-16
    w = W.me_view(64, 96, 16, 16)
    w.src_a, w.src_b = cur, ref_
    cfg["C2::src_a"], cfg["C2::src_b"], cfg["C2::engine"] = cur, ref_, O.ref_run_full(w)
    w = W.conv_nchw_view(1, 64, 12, 12, 8, 3, 1, 1)  # C3-style slice
    w.src_a = W.gen_uniform([1, 64, 12, 12], 3)
    w.src_b = W.gen_normal([8, 64, 3, 3], 1003, (2.0 / 576) ** 0.5)
    cfg["C3::src_a"], cfg["C3::src_b"], cfg["C3::engine"] = w.src_a, w.src_b, O.ref_run_full(w)
    w = W.conv_nchw_view(1, 128, 14, 14, 8, 3, 2, 1)  # C4-style slice (bf16 data as REAL32)
    x = W.bf16_bits_to_f32(W.to_bf16_bits(W.gen_uniform([1, 128, 14, 14], 4)))
    wt = W.bf16_bits_to_f32(W.to_bf16_bits(W.gen_normal([8, 128, 3, 3], 1004, (2.0 / 1152) ** 0.5)))
    w.src_a, w.src_b = x, wt
    cfg["C4::src_a"], cfg["C4::src_b"], cfg["C4::engine"] = x, wt, O.ref_run_full(w)
    np.savez_compressed(Path(__file__).parent / "configs.npz", **cfg)
    print("wrote configs.npz")


if __name__ == "__main__":
    main()
