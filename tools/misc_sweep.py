"""Randomised bit-exact sweep of the non-conv kernels against the oracle (GPU):
max-pool views (K1), SAD maps + argmin for single and batched frame pairs, the
fused 16x16 + 8x8 search (K2), and displacement correlation (K4) against the
reference engine where oracle/_ref is built.  usage: python tools/misc_sweep.py [n] [seed]"""
import sys

import numpy as np

sys.path.insert(0, '.')
import oracle.binding as O
import paper_1911_03458_b200.workloads as W
from paper_1911_03458_b200 import FLAG_ARGMIN, FLAG_NO_MAP, Boundary, Plan, PlanGroup, run_full, run_full_argmin

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = {"maxpool": 0, "sad": 0, "fused": 0, "corr": 0}

for t in range(n_cases):
    # ---- max-pool
    n, c = int(rng.integers(1, 5)), int(rng.integers(1, 70))
    h, wd = int(rng.integers(5, 130)), int(rng.choice([int(rng.integers(5, 300)), 112, 56, 64, 16]))
    k, s, pad = [(3, 2, 1), (3, 2, 1), (2, 2, 0), (3, 1, 1), (2, 1, 0), (3, 3, 1), (5, 1, 2)][int(rng.integers(0, 7))]
    if h + 2 * pad >= k and wd + 2 * pad >= k:
        w = W.maxpool_nchw_view(n, c, h, wd, k, s, pad)
        w.src_a = W.gen_uniform([n, c, h, wd], 300 + t)
        ho, wo = w.view_a.p_shape[2:]
        try:
            got = run_full(w)
            ok = np.array_equal(got.view(np.uint32), O.maxpool(w.src_a, ho, wo, k, s, pad).view(np.uint32))
        except Exception as e:  # noqa: BLE001
            ok = False
            print("ERROR", e)
        if not ok:
            bad["maxpool"] += 1
            print(f"BAD maxpool case {t}: {n}x{c}x{h}x{wd} k{k} s{s} p{pad}")
    # ---- SAD map + argmin, single pair or a pair axis
    blk = int(rng.choice([8, 16]))
    r = int(rng.choice([4, 7, 8, 16, 16, 32, 32]))
    h = int(rng.integers(blk, 200))
    wd = int(rng.choice([int(rng.integers(blk, 400)), 256, 128, 16 * int(rng.integers(1, 20))]))
    pairs = None if rng.integers(0, 2) else int(rng.integers(1, 4))
    frames = [W.gen_me_pair(h, wd, 400 + 7 * t + i, blk, min(r, 16), 4) for i in range(pairs or 1)]
    cur = np.stack([f[0] for f in frames]) if pairs else frames[0][0]
    ref = np.stack([f[1] for f in frames]) if pairs else frames[0][1]
    w = W.me_view(h, wd, blk, r, pairs=pairs)
    w.src_a, w.src_b = cur, ref
    try:
        sad, mv = run_full_argmin(w)
        want = O.me_sad(cur, ref, blk, r)
        ok = np.array_equal(sad, want.reshape(sad.shape)) and np.array_equal(mv, O.me_argmin(want, r))
    except Exception as e:  # noqa: BLE001
        ok = False
        print("ERROR", e)
    if not ok:
        bad["sad"] += 1
        print(f"BAD sad case {t}: {h}x{wd} blk{blk} r{r} pairs{pairs}")
    # ---- fused 16x16 + 8x8, +/-32 (argmin only), on the same frames when they allow it
    if h >= 16 and wd >= 16:
        ws = [W.me_view(h, wd, b, 32, pairs=pairs) for b in (16, 8)]
        try:
            g = PlanGroup(ws, FLAG_ARGMIN | FLAG_NO_MAP)
            res = g.run_host(cur, ref)
            ok = all(np.array_equal(mv, O.me_argmin(O.me_sad(cur, ref, b, 32), 32)) for (_, mv), b in zip(res, (16, 8)))
        except Exception as e:  # noqa: BLE001
            ok = False
            print("ERROR", e)
        if not ok:
            bad["fused"] += 1
            print(f"BAD fused case {t}: {h}x{wd} pairs{pairs} | {g.description}")
    # ---- correlation against the reference engine
    if O.ref_available():
        prm = {"c": int(rng.choice([1, 3, 16, 32, 64])), "h": int(rng.integers(2, 30)), "w": int(rng.integers(2, 40)),
               "d": int(rng.choice([1, 3, 5, 9]))}
        w = W.build_template("correlation", prm)
        W.fill_random(w, 900 + 2 * t, 901 + 2 * t)
        try:
            ok = np.array_equal(run_full(w).view(np.uint32), O.ref_run_full(w).view(np.uint32))
        except Exception as e:  # noqa: BLE001
            ok = False
            print("ERROR", e)
        if not ok:
            bad["corr"] += 1
            print(f"BAD corr case {t}: {prm}")
print("cases", n_cases, "bad", bad)
