"""N>1 host path on CPU: world_size-2 gloo processes shard the batch /
frame-pair axis (paper_1911_03458_b200/shard.py), compute their shard with the
CPU checker, and the gathered shards equal the unsharded result — the same
partitioning bench.py uses on GPUs, with no collective on the data path."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1911_03458_b200.shard import shard_band, shard_range, shard_workload
from paper_1911_03458_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frames():
    pairs = [W.gen_me_pair(32, 48, 10 + i) for i in range(3)]
    return np.stack([p[0] for p in pairs]), np.stack([p[1] for p in pairs])


def _worker(rank, world, port, q):
    from oracle import binding as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # conv batch shard (C4 shape, scaled down): weights replicated
    w = W.conv_nchw_view(5, 3, 9, 9, 4, 3, 2, 1)
    w.src_a = W.gen_uniform([5, 3, 9, 9], 1)
    w.src_b = W.gen_uniform([4, 3, 3, 3], 2)
    s, (a, b) = shard_workload(w, world, rank)
    assert s.src_b is w.src_b
    out = O.conv2d(s.src_a, s.src_b, 2, 1)
    parts = [None] * world
    dist.all_gather_object(parts, (a, b, out))
    # frame-pair shard (C5 shape, scaled down)
    cur, ref = _frames()
    m = W.me_view(32, 48, 8, 4, pairs=3)
    m.src_a, m.src_b = cur, ref
    sm, (c0, c1) = shard_workload(m, world, rank)
    mv = O.me_argmin(O.me_sad(sm.src_a, sm.src_b, 8, 4), 4)
    mparts = [None] * world
    dist.all_gather_object(mparts, (c0, c1, mv))
    # block-row band of ONE frame pair (C2 split): rows + Eq. 6 halo only
    bc, br = W.gen_me_pair(120, 64, 33)
    b = W.me_view(120, 64, 16, 16)
    b.src_a, b.src_b = bc, br
    sb, (r0, r1) = shard_band(b, world, rank)
    assert sb.src_a.shape[0] == 16 * (r1 - r0) and sb.src_b.shape[0] < 120
    bparts = [None] * world
    dist.all_gather_object(bparts, (r0, r1, O.run_full(sb)))
    if rank == 0:
        q.put((parts, mparts, bparts))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_balanced():
    assert [shard_range(10, 4, r) for r in range(4)] == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert sum(b - a for a, b in (shard_range(64, 8, r) for r in range(8))) == 64


def test_two_rank_gloo_sharding_equals_unsharded():
    from oracle import binding as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts, mparts, bparts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = O.conv2d(W.gen_uniform([5, 3, 9, 9], 1), W.gen_uniform([4, 3, 3, 3], 2), 2, 1)
    got = np.concatenate([p[2] for p in sorted(parts, key=lambda t: t[0])])
    assert np.array_equal(got, full)
    cur, ref = _frames()
    full_mv = O.me_argmin(O.me_sad(cur, ref, 8, 4), 4)
    got_mv = np.concatenate([p[2] for p in sorted(mparts, key=lambda t: t[0])])
    assert np.array_equal(got_mv, full_mv)
    bc, br = W.gen_me_pair(120, 64, 33)
    b = W.me_view(120, 64, 16, 16)
    b.src_a, b.src_b = bc, br
    got_b = np.concatenate([p[2] for p in sorted(bparts, key=lambda t: t[0])])
    assert np.array_equal(got_b, O.run_full(b))
