"""Time the fused C5 block search (16x16 + 8x8, +/-32, argmin only) on
device-resident 4K frame pairs, for A/B experiments on kernel variants.

  python tools/c5_time.py [pairs] [iters]            # the library in use
  MERIT_DEV_LIB=.../libmerit_dev_X.so python tools/c5_time.py 8

Prints ms per launch and ms per pair (x64 = the C5 step).  Frames are random
bytes (the SAD kernel's cost does not depend on the values).  Relative
experiments only: the measurement of record is bench.py.
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1911_03458_b200 import FLAG_ARGMIN, FLAG_NO_MAP, PlanGroup  # noqa: E402
from paper_1911_03458_b200 import workloads as W  # noqa: E402


def main():
    pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    h, wd = 2160, 3840
    ws = [W.me_view(h, wd, b, 32, pairs=pairs) for b in (16, 8)]
    g = PlanGroup(ws, FLAG_ARGMIN | FLAG_NO_MAP)
    gen = torch.Generator().manual_seed(5)
    a = torch.randint(0, 256, (pairs, h, wd), dtype=torch.uint8, generator=gen).cuda()
    b = torch.randint(0, 256, (pairs, h, wd), dtype=torch.uint8, generator=gen).cuda()
    aux = torch.empty(int(g.info.aux_elems), dtype=torch.int32, device="cuda")
    for _ in range(3):
        g.run(a, b, None, aux)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        g.run(a, b, None, aux)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"C5 fused pairs={pairs}: {ms:8.3f} ms/launch {ms / pairs * 64:8.2f} ms per 64 pairs "
          f"[{g.description}]", flush=True)


if __name__ == "__main__":
    main()
