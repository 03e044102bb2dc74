"""Batch sharding across GPUs: problems are independent, so the
batch is split by problem index with no collective on the data path.

* contiguous_shard(batch, world, rank): equal contiguous slices (configs 1-4);
* cost_balanced_shard(costs, world, rank): cut the prefix sum of per-problem
  cost into equal slices (config 5: cost ~ 7 n^3 / 3 per problem).
"""
from __future__ import annotations

from typing import Sequence


def contiguous_shard(batch: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of problems owned by `rank`; sizes differ by at most one."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def chain_cost(n: int) -> float:
    """Flop model of one config-5 problem: syrk n^3 + potrf n^3/3 + trsm n^3 (bench.hpp:119-138)."""
    return n ** 3 + (n ** 3) // 3 + n ** 3


def cost_balanced_shard(costs: Sequence[float], world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) such that every rank's slice carries ~1/world of the total cost."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    total = float(sum(costs))
    cuts = [0]
    acc, target_i = 0.0, 1
    for i, c in enumerate(costs):
        acc += c
        while target_i < world and acc >= total * target_i / world:
            cuts.append(i + 1)
            target_i += 1
    while len(cuts) < world:
        cuts.append(len(costs))
    cuts.append(len(costs))
    return cuts[rank], cuts[rank + 1]


def shard_of(batch: int, world: int, rank: int, costs: Sequence[float] | None = None) -> tuple[int, int]:
    """The slice of one host-generated batch that `rank` computes: contiguous equal slices,
    or equal-cost slices when per-problem `costs` are given."""
    if costs is not None:
        if len(costs) != batch:
            raise ValueError("costs must have one entry per problem")
        return cost_balanced_shard(costs, world, rank)
    return contiguous_shard(batch, world, rank)


def gather_slices(local, lo: int, hi: int, world: int, rank: int, root: int = 0):
    """Collects every rank's [lo, hi) result slice (numpy, problem-major) on `root` in problem
    order and returns the concatenation there (None elsewhere).  Host-side only: the data path
    itself has no collective; this is the optional D2H gather of §8e for parity checks."""
    import numpy as np
    if world == 1:
        return local
    import torch.distributed as dist
    objs = [None] * world if rank == root else None
    dist.gather_object((lo, hi, local), objs, dst=root)
    if rank != root:
        return None
    objs.sort(key=lambda o: o[0])
    for a, b in zip(objs, objs[1:]):
        if a[1] != b[0]:
            raise RuntimeError("shards do not tile the batch")
    return np.concatenate([o[2] for o in objs])
