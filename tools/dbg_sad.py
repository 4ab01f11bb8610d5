import sys, numpy as np
sys.path.insert(0, '.')
import paper_1911_03458_b200.workloads as W
from paper_1911_03458_b200.merit import run_full_argmin
import oracle.binding as O
h, wd, r = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (32, 128, 32)
cur, ref = W.gen_me_pair(h, wd, 9, 16, 16, 4)
w = W.me_view(h, wd, 16, r)
w.src_a, w.src_b = cur, ref
sad, mv = run_full_argmin(w)
want = O.me_sad(cur, ref, 16, r)
bad = np.argwhere(sad != want)
print("shape", sad.shape, "bad", len(bad))
if len(bad):
    by, bx = bad[:, 0], bad[:, 1]
    print("blocks", sorted(set(zip(by.tolist(), bx.tolist())))[:20])
    print("dy set", sorted(set(bad[:, 2].tolist()))[:70])
    print("dx set", sorted(set(bad[:, 3].tolist()))[:70])
    i = tuple(bad[0]); print("first", i, sad[i], want[i])
    i = tuple(bad[0]); print("row of sad at first bad", sad[i[0], i[1], i[2], 50:], want[i[0], i[1], i[2], 50:])
    print("mv", mv.reshape(-1,3)[:16].tolist())
