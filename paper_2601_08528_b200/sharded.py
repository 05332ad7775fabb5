"""Dataset-sharded search across GPUs.

One process per GPU (torchrun); rank r owns shard r: its own graph, vectors and tombstones in its HBM.
Global ids interleave the shards: g = local * G + r.  The map is monotone inside a shard, so a shard's local
(dist, id) order equals the global order and the merged top-k is identical for every G; inserts grow each shard
at its end without colliding with other ranks' ids.

Search: queries are broadcast -> each rank searches its shard (K-S) -> local ids -> global ids ->
all-gather (NCCL over NVLink / NVSwitch) of the [nq, k] id and distance blocks -> K-M merge (svf_merge_topk).
Inserts and deletes route to the owning shard; there is no exchange on those paths.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np

SENT32 = -1  # 0xFFFFFFFF viewed as int32


def to_global(ids, rank: int, world: int):
    """local -> global ids (g = local*G + r); sentinels stay sentinels.  Works on torch int32 tensors."""
    import torch

    g = ids.to(torch.int64) * world + rank
    return torch.where(ids == SENT32, torch.full_like(g, SENT32), g).to(torch.int32)


def owner_and_local(global_ids: np.ndarray, world: int):
    g = np.asarray(global_ids, dtype=np.int64)
    return (g % world).astype(np.int64), (g // world).astype(np.uint32)


def gather_topk(ids, dists, group=None):
    """All-gather each rank's [nq, k] block -> [G, nq, k] on every rank (NCCL on GPU, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out_i = [torch.empty_like(ids) for _ in range(world)]
    out_d = [torch.empty_like(dists) for _ in range(world)]
    dist.all_gather(out_i, ids.contiguous(), group=group)
    dist.all_gather(out_d, dists.contiguous(), group=group)
    return torch.stack(out_i), torch.stack(out_d)


class ShardedIndex:
    """A rank's shard plus the exchange that turns per-shard top-k lists into the global top-k."""

    def __init__(self, local, rank: int, world: int, group=None, merge_fn: Optional[Callable] = None):
        self.local, self.rank, self.world, self.group = local, rank, world, group
        if merge_fn is None:
            from . import merge_topk as merge_fn  # K-M on the GPU
        self.merge_fn = merge_fn

    @classmethod
    def build(cls, X_local, degree: int, group=None, **kw) -> "ShardedIndex":
        import torch.distributed as dist

        from . import Index

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        return cls(Index.build(X_local, degree, **kw), rank, world, group)

    def search(self, Q, k: int, itopk: int):
        ids, d = self.local.search(Q, k, itopk)
        gids = to_global(ids, self.rank, self.world)
        if self.world == 1:
            return gids, d
        ai, ad = gather_topk(gids, d, self.group)
        return self.merge_fn(ai, ad)

    def knn_exact(self, Q, k: int):
        ids, d = self.local.knn_exact(Q, k)
        gids = to_global(ids, self.rank, self.world)
        if self.world == 1:
            return gids, d
        ai, ad = gather_topk(gids, d, self.group)
        return self.merge_fn(ai, ad)

    def insert(self, X_local) -> np.ndarray:
        """Insert this rank's share of a batch; returns the new global ids."""
        lid = self.local.insert(X_local).astype(np.int64)
        return (lid * self.world + self.rank).astype(np.uint32)

    def delete(self, global_ids) -> int:
        """Every rank receives the same id list and deletes the ids it owns."""
        own, loc = owner_and_local(global_ids, self.world)
        mine = loc[own == self.rank]
        return self.local.delete(mine) if len(mine) else 0
