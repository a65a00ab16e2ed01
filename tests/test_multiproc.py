"""The N>1 path on CPU: world_size-2 gloo ranks run bench.py's sharding and
max-over-ranks timing reduction (no data-path collective exists)."""

import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench
    d = bench.Dist(backend_gpu=False)
    seeds = [bench.shard_seeds(d.rank, k, 4, 8) for k in range(3)]
    mx = d.max(float(10 + rank))
    sm = d.sum(float(rank + 1))
    d.barrier()
    q.put((rank, seeds, mx, sm))
    d.close()


def test_two_rank_sharding_and_reductions():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    (r0, s0, mx0, sm0), (r1, s1, mx1, sm1) = out
    assert mx0 == mx1 == 11.0                  # max over ranks (bench timing rule)
    assert sm0 == sm1 == 3.0
    flat0 = {x for step in s0 for x in step}
    flat1 = {x for step in s1 for x in step}
    assert not flat0 & flat1                  # ranks decode disjoint utterances
    assert all(len(set(step)) == 4 for step in s0 + s1)


def test_shard_pool_cycles():
    sys.path.insert(0, ROOT)
    import bench
    a = bench.shard_seeds(0, 0, 4, 8)
    b = bench.shard_seeds(0, 2, 4, 8)
    assert a == b and len(set(a + bench.shard_seeds(0, 1, 4, 8))) == 8
