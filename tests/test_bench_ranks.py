"""bench.py's multi-GPU rank logic, run on CPU: `bench.py --gpus 2 --dry-run`
re-launches itself under torch.distributed.run with two gloo ranks, each
builds its shard through the same shard_for() the GPU run uses, and rank 0
prints every rank's shard (disjoint shards covering the whole
config, no exchange)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

FULL_OUTPUTS = {"C1": 8 * 64 * 56 * 56, "C2": 67 * 120 * 33 * 33, "C3": 32 * 64 * 56 * 56,
                "C4": 256 * 256 * 28 * 28, "C5": 64 * (135 * 240 + 270 * 480) * 65 * 65}


@pytest.mark.parametrize("config,world", [("C2", 2), ("C5", 2), ("C3", 2), ("C2", 3), ("C1", 2), ("C4", 2)])
def test_bench_dry_run_shards_disjoint_and_complete(config, world):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(world), "--dry-run",
                        "--config", config], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == world and len(line["shards"]) == world
    shards = sorted(line["shards"], key=lambda s: s["rank"])
    assert [s["rank"] for s in shards] == list(range(world))
    # contiguous, disjoint ranges covering the batch / block rows
    assert shards[0]["range"][0] == 0
    for a, b in zip(shards, shards[1:]):
        assert a["range"][1] == b["range"][0]
    total = {"C1": 8, "C2": 67, "C3": 32, "C4": 256, "C5": 64}[config]
    assert shards[-1]["range"][1] == total
    assert all(s["range"][1] > s["range"][0] for s in shards)
    # every output exactly once, each rank on its device kernel
    assert sum(s["outputs"] for s in shards) == FULL_OUTPUTS[config]
    assert all(k != 0 for s in shards for k in s["kernels"])
    if config == "C2":
        # each band holds only its rows (cur) and its rows + the 16-row halo (ref)
        for s in shards:
            lo, hi = s["range"]
            assert s["src_a_shape"] == [16 * (hi - lo), 1920]
            top = 16 if lo > 0 else 0
            bottom = min(16, 1080 - 16 * hi)
            assert s["src_b_shape"] == [16 * (hi - lo) + top + bottom, 1920]
