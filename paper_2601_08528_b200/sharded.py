"""Dataset-sharded search across GPUs.

The dataset is split into S logical shards (default 8): global id g lives in shard g mod S as local id g div S.
The map is monotone inside a shard, so a shard's local (dist, id) order equals the global order.  One process per
GPU (torchrun); rank r of G holds every shard s with s mod G = r, each an svf index (its own graph, vectors and
tombstones) in that GPU's HBM, so G in {1, 2, 4, 8} regroups the same 8 graphs.

Search (north star: "queries are broadcast to every shard, each shard returns a local top-k, and a NCCL allgather
over NVLink feeds a final top-k merge"):
  1. every rank has the query batch (generated or copied on each rank: no collective);
  2. the rank searches each of its shards (K-S) and pre-merges them into its top-k with global ids, packed as u64
     pairs (svf_shard_premerge, K-M);
  3. ONE all_gather_into_tensor of the [nq, k] pair block (nq * k * 8 bytes per rank; NCCL over NVLink/NVSwitch);
  4. K-M merges the G gathered lists (svf_merge_pairs).
The merge is associative over the (dist, id) total order, so the output is bit-identical for every G.
Inserts route row i of a batch with global ids first..first+n-1 to shard (first+i) mod S; deletes route g to
(g mod S, g div S).  Neither path exchanges data.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional

import numpy as np

SENT32 = -1  # 0xFFFFFFFF viewed as int32


def owned_shards(S: int, rank: int, world: int) -> List[int]:
    """The logical shards rank r of G holds: s mod G = r."""
    return [s for s in range(S) if s % world == rank]


def owner_and_local(global_ids, S: int):
    """global id -> (shard, local id)."""
    g = np.asarray(global_ids, dtype=np.int64)
    return (g % S).astype(np.int64), (g // S).astype(np.uint32)


def to_global(ids, shard: int, S: int):
    """local -> global ids (g = local*S + shard); sentinels stay sentinels.  Works on torch int32 tensors."""
    import torch

    g = ids.to(torch.int64) * S + shard
    return torch.where(ids == SENT32, torch.full_like(g, SENT32), g).to(torch.int32)


def shard_rows(n_global: int, s: int, S: int) -> int:
    """How many of the global ids 0..n_global-1 fall in shard s."""
    return max(0, (n_global - s + S - 1) // S)


class ShardedIndex:
    """The shards a rank holds plus the exchange that turns their top-k lists into the global top-k."""

    def __init__(self, shards: Dict[int, object], S: int, rank: int = 0, world: int = 1, group=None,
                 premerge_fn: Optional[Callable] = None, merge_pairs_fn: Optional[Callable] = None):
        if sorted(shards) != owned_shards(S, rank, world):
            raise ValueError(f"rank {rank} of {world} must hold shards {owned_shards(S, rank, world)}")
        self.shards, self.S, self.rank, self.world, self.group = shards, S, rank, world, group
        if premerge_fn is None or merge_pairs_fn is None:
            from . import merge_pairs, shard_premerge

            premerge_fn, merge_pairs_fn = shard_premerge, merge_pairs
        self.premerge_fn, self.merge_pairs_fn = premerge_fn, merge_pairs_fn
        self._bufs: dict = {}

    @property
    def local(self) -> List[int]:
        return sorted(self.shards)

    # ---- construction -------------------------------------------------------------------------------------------
    @classmethod
    def build(cls, X, S: int = 8, rank: int = 0, world: int = 1, group=None, degree: int = 64, **kw) -> "ShardedIndex":
        """Build the rank's shards from the GLOBAL rows X (row g is global id g): shard s gets X[s::S]."""
        from . import Index

        shards = {s: Index.build(X[s::S], degree, **kw) for s in owned_shards(S, rank, world)}
        return cls(shards, S, rank, world, group)

    # ---- search -------------------------------------------------------------------------------------------------
    def _buffers(self, like, nq: int, k: int):
        import torch

        key = (nq, k, str(getattr(like, "device", "cpu")))
        if key not in self._bufs:
            dev = like.device if hasattr(like, "device") else "cpu"
            n = len(self.shards)
            self._bufs[key] = (torch.empty((n, nq, k), dtype=torch.int32, device=dev),
                               torch.empty((n, nq, k), dtype=torch.float32, device=dev),
                               torch.empty((self.world * nq, k), dtype=torch.int64, device=dev))
        return self._bufs[key]

    def _exchange(self, per_shard: Callable, Q, k: int):
        """per_shard(index, Q, k, out_ids, out_d) for every local shard -> pre-merge -> all-gather -> merge."""
        nq = int(Q.shape[0])
        ids_l, d_l, gathered = self._buffers(Q, nq, k)
        for i, s in enumerate(self.local):
            per_shard(self.shards[s], Q, k, ids_l[i], d_l[i])
        pairs = self.premerge_fn(ids_l, d_l, self.S, self.local)         # [nq, k] int64 pairs, global ids
        if self.world == 1:
            gathered = pairs.unsqueeze(0)
        else:
            import torch.distributed as dist

            if pairs.is_cuda and dist.get_backend(self.group) == "gloo":   # gloo gathers host tensors (tests)
                host = gathered.cpu()
                dist.all_gather_into_tensor(host, pairs.cpu(), group=self.group)
                gathered.copy_(host)
            else:
                dist.all_gather_into_tensor(gathered, pairs.contiguous(), group=self.group)  # rank-major blocks
            gathered = gathered.view(self.world, nq, k)
        return self.merge_pairs_fn(gathered)

    def search(self, Q, k: int, itopk: int):
        """Search(q, k) over the whole sharded dataset: (ids int32 [nq, k] global, dists f32 [nq, k])."""
        return self._exchange(lambda idx, q, kk, oi, od: idx.search_into(q, kk, itopk, oi, od), Q, k)

    def knn_exact(self, Q, k: int):
        """Exact k-NN over the live union of all shards (the per-shard exact lists merge exactly)."""
        return self._exchange(lambda idx, q, kk, oi, od: idx.knn_exact_into(q, kk, oi, od), Q, k)

    # ---- updates ------------------------------------------------------------------------------------------------
    def insert(self, X_batch, first_gid: int) -> np.ndarray:
        """Insert the global batch with ids first_gid..first_gid+n-1 (every rank passes the whole batch; each
        inserts the rows of its shards).  Returns the global ids this rank inserted."""
        n = int(X_batch.shape[0])
        gids = np.arange(first_gid, first_gid + n, dtype=np.int64)
        mine = []
        for s in self.local:
            rows = np.flatnonzero(gids % self.S == s)
            if len(rows) == 0:
                continue
            idx = self.shards[s]
            expect = shard_rows(first_gid, s, self.S)
            if idx.info()["n_alloc"] != expect:
                raise ValueError(f"shard {s} holds {idx.info()['n_alloc']} rows, expected {expect} before global "
                                 f"id {first_gid}: inserts must arrive in global id order")
            sel = X_batch[rows] if not hasattr(X_batch, "index_select") else X_batch[rows.tolist()]
            lid = idx.insert(sel).astype(np.int64)
            assert np.array_equal(lid * self.S + s, gids[rows])
            mine.append(gids[rows])
        return np.sort(np.concatenate(mine)).astype(np.uint32) if mine else np.empty(0, np.uint32)

    def delete(self, global_ids) -> int:
        """Every rank receives the same global id list and deletes the ids its shards hold."""
        own, loc = owner_and_local(global_ids, self.S)
        n = 0
        for s in self.local:
            ids = loc[own == s]
            if len(ids):
                n += self.shards[s].delete(ids)
        return n

    def close(self):
        for idx in self.shards.values():
            idx.close()
        self.shards = {}
