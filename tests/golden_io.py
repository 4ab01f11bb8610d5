"""Load the golden fixtures produced by the reference (tests/golden/make_golden.py)."""
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
_cache = {}


def case_key(name, prm):
    return name + "|" + ",".join(f"{k}={prm[k]}" for k in sorted(prm))


def load(file="templates.npz"):
    if file not in _cache:
        with np.load(GOLDEN / file, allow_pickle=False) as z:
            _cache[file] = {k: z[k] for k in z.files}
    return _cache[file]


def keys(file="templates.npz"):
    d = load(file)
    return sorted({k.rsplit("::", 1)[0] for k in d})


def load_case(name, prm=None, file="templates.npz", key=None):
    d = load(file)
    k = key if key is not None else case_key(name, prm)
    out = {f: d[k + "::" + f] for f in ("src_a", "src_b", "engine", "oracle") if k + "::" + f in d}
    out["fix"] = bool(d[k + "::fix"])
    return out
