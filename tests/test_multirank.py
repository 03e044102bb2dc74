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


# --------------------------------------------------------------- split + gather == unsplit
def _split_worker(rank, world, port, use_gpu, q):
    """Each rank computes its shard of ONE seeded batch (cfg1 dgemm and a cfg5-style chain with
    the cost-balanced cut), results gathered on rank 0."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import numpy as np
    import torch.distributed as dist
    from oracle import binding as ob
    from paper_1902_08115_b200.shard import gather_slices, shard_of
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(9)
        m = 32
        batch = 37
        A = rng.uniform(-1, 1, (batch, m * m)); B = rng.uniform(-1, 1, (batch, m * m))
        C = rng.uniform(-1, 1, (batch, m * m))
        lo, hi = shard_of(batch, world, rank)
        c = C[lo:hi].copy()
        if use_gpu:
            import torch
            import paper_1902_08115_b200 as pb
            dc = torch.from_numpy(c).cuda()
            assert pb.dgemm_batched("n", "n", m, m, m, 1.0, torch.from_numpy(A[lo:hi].copy()).cuda(), m, m * m,
                                    torch.from_numpy(B[lo:hi].copy()).cuda(), m, m * m, 1.0, dc, m, m * m,
                                    hi - lo).ok()
            c = dc.cpu().numpy()
        else:  # no device here: the oracle stands in for the per-rank compute (test only)
            a, b = A[lo:hi].copy(), B[lo:hi].copy()
            ob.oracle().dgemm_batch(b"n", b"n", m, m, m, 1.0, a.ctypes.data, m, m * m, b.ctypes.data, m, m * m,
                                    1.0, c.ctypes.data, m, m * m, hi - lo, 1)
        full = gather_slices(c, lo, hi, world, rank)
        # cfg5-style variable batch: cost-balanced cut of the chain flop model
        ns = (rng.integers(1, 17, 50) * 4).astype(np.int32)
        from paper_1902_08115_b200.shard import chain_cost
        clo, chi = shard_of(len(ns), world, rank, costs=[chain_cost(int(n)) for n in ns])
        part = np.array([[p, int(ns[p])] for p in range(clo, chi)], dtype=np.int64).reshape(-1, 2)
        owners = gather_slices(part, clo, chi, world, rank)
        if rank == 0:
            want = C.copy()
            ob.oracle().dgemm_batch(b"n", b"n", m, m, m, 1.0, A.ctypes.data, m, m * m, B.ctypes.data, m, m * m,
                                    1.0, want.ctypes.data, m, m * m, batch, 1)
            q.put(("ok", full.tobytes() == want.tobytes() if not use_gpu else
                   float(np.abs(full - want).max()), owners[:, 0].tolist(), chi))
        else:
            q.put(("rank", rank, clo, chi))
    finally:
        dist.destroy_process_group()


def _run_split(use_gpu):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_split_worker, args=(r, 2, port, use_gpu, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return [q.get(timeout=10) for _ in range(2)]


def test_split_gather_equals_unsplit_oracle():
    """world_size 2 on gloo: the two shards of one batch, gathered, equal the unsplit result
    bit for bit; the cost-balanced cut covers every problem exactly once, in order."""
    res = _run_split(False)
    ok = [r for r in res if r[0] == "ok"][0]
    assert ok[1] is True
    assert ok[2] == list(range(50))


@pytest.mark.gpu
def test_split_gather_two_ranks_on_gpu0():
    """Two ranks sharing GPU 0 (independent kernels, no inter-rank waits): gathered shards
    equal the unsplit oracle within the north star's tolerance."""
    res = _run_split(True)
    ok = [r for r in res if r[0] == "ok"][0]
    assert ok[1] <= 1e-13 * 32 * 8
    assert ok[2] == list(range(50))
