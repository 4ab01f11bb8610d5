"""Write a reference workload template as a manifest + MRT1 tensors.

    python -m paper_1911_03458_b200.manifest --template conv2d --params h=9,w=8 \\
        --seed 3 --dir out/ [--tile 4x4,3x3]

Same inputs as the reference CLI's `run --template` (tools/merit.cpp:120-138:
build_template, fill_random with seeds 2s+1 / 2s+2, shared-input templates
reuse src_a), so `bin/merit-dev run --manifest out/workload.json` on the
device and the reference CLI on the same files see identical workloads.
"""
import argparse

from . import workloads as W
from .formats import write_manifest


def params(s: str) -> dict:  # tools/merit.cpp:46-58
    out = {}
    for item in filter(None, s.split(",")):
        k, v = item.split("=")
        out[k] = float(v)
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--template", required=True)
    ap.add_argument("--params", default="")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dir", required=True)
    ap.add_argument("--tile", default=None)
    ap.add_argument("--stem", default="workload")
    a = ap.parse_args(argv)
    w = W.build_template(a.template, params(a.params))
    W.fill_random(w, 2 * a.seed + 1, 2 * a.seed + 2)
    if W.template_shares_input(a.template):
        w.src_b = w.src_a
    print(write_manifest(a.dir, w, a.tile, a.stem))


if __name__ == "__main__":
    main()
