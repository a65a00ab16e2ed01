"""The N>1 path on CPU: world_size-2 gloo ranks run the multi-device split
(shard_lpt, the same LPT assignment lb_decode_batch_multi uses), decode their
shards (the CPU oracle stands in for a device here), gather to rank 0 and merge
back into input order; plus bench.py's max-over-ranks timing reduction.  No
data-path collective exists in the product; the gather is the
test's way of checking the merge."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch():
    from paper_1804_03243_b200 import synthetic
    w = synthetic.uniform_bench_graph(2, num_states=800, arcs_per_state=4, num_labels=40)
    mats = [synthetic.bench_matrix(50 + i, num_frames=6 + (7 * i) % 23, num_labels=40) for i in range(11)]
    return w, mats


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench
    from oracle import oracle as O
    from paper_1804_03243_b200.decoder import merge_in_order, split_batch
    d = bench.Dist(backend_gpu=False)
    w, mats = _batch()
    shards = split_batch([m.costs.shape[0] for m in mats], d.world)
    mine = [O.decode(w, mats[i], 9.0, want_lattice=False, collect_frames=False) for i in shards[d.rank]]
    mine = [(r.total_cost, r.words) for r in mine]
    gathered = [None] * d.world
    d.pg.all_gather_object(gathered, mine)
    merged = merge_in_order(len(mats), shards, gathered)
    mx = d.max(float(10 + rank))
    sm = d.sum(float(rank + 1))
    d.barrier()
    q.put((rank, shards, merged, mx, sm))
    d.close()


def test_two_rank_split_decode_merge():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda x: x[0])
    (_, sh0, m0, mx0, sm0), (_, sh1, m1, mx1, sm1) = out
    assert mx0 == mx1 == 11.0                  # max over ranks (bench timing rule)
    assert sm0 == sm1 == 3.0
    assert sh0 == sh1 and not set(sh0[0]) & set(sh0[1])
    assert sorted(sh0[0] + sh0[1]) == list(range(11))
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    w, mats = _batch()
    want = [O.decode(w, m, 9.0, want_lattice=False, collect_frames=False) for m in mats]
    assert m0 == m1 == [(r.total_cost, r.words) for r in want]   # input order restored


def test_shard_lpt_balance_and_determinism():
    sys.path.insert(0, ROOT)
    from paper_1804_03243_b200.decoder import merge_in_order, shard_lpt, split_batch
    rng = np.random.default_rng(3)
    for n_shards in (1, 2, 3, 8):
        T = rng.integers(100, 501, size=4096)
        sh = shard_lpt(T, n_shards)
        assert np.array_equal(sh, shard_lpt(T, n_shards))
        loads = np.bincount(sh, weights=T, minlength=n_shards)
        assert loads.max() - loads.min() <= T.max()       # LPT bound
        parts = split_batch(T, n_shards)
        back = merge_in_order(len(T), parts, [[int(T[i]) for i in p] for p in parts])
        assert back == T.tolist()
    # longest first, ties by input order, to the least-loaded (lowest) shard
    assert shard_lpt([5, 3, 8, 1, 9, 2], 2).tolist() == [1, 0, 1, 1, 0, 0]
    assert shard_lpt([], 4).tolist() == []


def test_bench_rank_shards_are_disjoint():
    sys.path.insert(0, ROOT)
    import bench
    a = [bench.rank_utterances(r, 4, 4096) for r in range(4)]
    flat = [i for x in a for i in x]
    assert sorted(flat) == list(range(4096))
