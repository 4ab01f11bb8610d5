"""Bit-exact sweep of the SAD kernel over frame sizes / radii (GPU)."""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1911_03458_b200.workloads as W
from paper_1911_03458_b200.merit import run_full_argmin
import oracle.binding as O
blk = int(sys.argv[1])
bad = 0
for (h, wd) in [(48, 64), (64, 96), (72, 96), (80, 160), (88, 128), (96, 112), (112, 192), (128, 256), (144, 80)]:
    for r in [2, 4, 7, 8, 12, 16, 20, 24, 32]:
        cur, ref = W.gen_me_pair(h, wd, 9, blk, min(r, 16), 4)
        w = W.me_view(h, wd, blk, r)
        w.src_a, w.src_b = cur, ref
        try:
            sad, mv = run_full_argmin(w)
            ok = np.array_equal(sad, O.me_sad(cur, ref, blk, r))
        except Exception as e:
            print("ERROR", h, wd, r, e); sys.exit(1)
        if not ok:
            bad += 1; print("MISMATCH", h, wd, r)
print("blk", blk, "mismatches", bad)
