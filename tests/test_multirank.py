"""CPU: the N>1 path with world_size 2 on gloo — shard coverage and the
max-over-ranks timing used by bench.py (no collective on the data path)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1902_08115_b200.shard import chain_cost, contiguous_shard, cost_balanced_shard


def test_contiguous_shards_cover_once():
    for batch in (0, 1, 7, 16384):
        for world in (1, 2, 4, 8):
            seen = []
            for r in range(world):
                lo, hi = contiguous_shard(batch, world, r)
                seen.extend(range(lo, hi))
            assert seen == list(range(batch))


def test_cost_balanced_shards():
    import random
    rng = random.Random(5)
    ns = [4 * rng.randint(1, 64) for _ in range(32768)]
    costs = [chain_cost(n) for n in ns]
    for world in (1, 2, 4, 8):
        parts = [cost_balanced_shard(costs, world, r) for r in range(world)]
        assert parts[0][0] == 0 and parts[-1][1] == len(costs)
        for a, b in zip(parts, parts[1:]):
            assert a[1] == b[0]
        loads = [sum(costs[lo:hi]) for lo, hi in parts]
        assert max(loads) <= sum(costs) / world * 1.01


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import torch.distributed as dist
    ws, rk, _ = bench.dist_init()
    try:
        lo, hi = contiguous_shard(16384, ws, rk)
        t = bench.max_over_ranks(float(rk + 1) * 1.5, ws)  # each rank's "elapsed"
        bench.barrier(ws)
        q.put((rk, lo, hi, t))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_timing_and_shards():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = sorted(q.get(timeout=10) for _ in range(2))
    assert [g[3] for g in got] == [3.0, 3.0]  # max over ranks
    assert got[0][1:3] == (0, 8192) and got[1][1:3] == (8192, 16384)
