"""world_size-2 gloo tests of the sharded layer's host logic on CPU (no GPU): id interleaving, all-gather layout,
routing of deletes/inserts, and that merging the gathered per-shard lists reproduces the unsharded answer.
The per-shard search and the merge are the oracle's here (the GPU kernels are covered by -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import int_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _OracleShard:
    """Stands in for the rank-local svf Index: exact kNN over the shard via the oracle."""

    def __init__(self, X):
        self.X = X
        self.dead = set()

    def _tomb(self):
        from workloads import pack_tomb

        return pack_tomb(sorted(self.dead), len(self.X)) if self.dead else None

    def search(self, Q, k, itopk):
        import oracle

        ids, d = oracle.bf_knn(self.X, Q.numpy(), k, tomb=self._tomb())
        return torch.from_numpy(ids.view(np.int32).copy()), torch.from_numpy(d)

    knn_exact = lambda self, Q, k: self.search(Q, k, k)  # noqa: E731

    def insert(self, X):
        first = len(self.X)
        self.X = np.vstack([self.X, X])
        return np.arange(first, len(self.X), dtype=np.uint32)

    def delete(self, ids):
        before = len(self.dead)
        self.dead |= set(int(i) for i in ids)
        return len(self.dead) - before


def _merge_oracle(ai, ad):
    import oracle

    mi, md = oracle.merge_topk(ai.numpy().view(np.uint32), ad.numpy())
    return torch.from_numpy(mi.view(np.int32).copy()), torch.from_numpy(md)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_08528_b200.sharded import ShardedIndex

        N, D, k = 600, 6, 10
        Xall = int_rows(N, D, seed=11, hi=6)         # many exact ties across shards
        Q = torch.from_numpy(int_rows(25, D, seed=12, hi=6))
        gid = np.arange(rank, N, world)              # global id g = local*G + r
        sh = ShardedIndex(_OracleShard(Xall[gid]), rank, world, merge_fn=_merge_oracle)
        ids, d = sh.search(Q, k, 32)
        # insert a rank-specific batch, delete a broadcast id list
        newX = int_rows(7, D, seed=100 + rank, hi=6)
        new_gids = sh.insert(newX)
        n_del = sh.delete(np.array([0, 1, 2, 3, 5, 8, 13, 21], np.uint32))
        ids2, d2 = sh.search(Q, k, 32)
        q.put((rank, ids.numpy(), d.numpy(), new_gids, n_del, ids2.numpy(), d2.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_sharded_search_world2_gloo():
    import oracle
    from workloads import pack_tomb

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=150)
        res[r[0]] = r
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    N, D, k = 600, 6, 10
    Xall = int_rows(N, D, seed=11, hi=6)
    Q = int_rows(25, D, seed=12, hi=6)
    gi, gd = oracle.bf_knn(Xall, Q, k)
    for r in range(world):
        _, ids, d, new_gids, n_del, ids2, d2 = res[r]
        assert np.array_equal(ids.view(np.uint32), gi) and np.array_equal(d, gd)   # identical on every rank
        assert np.all(new_gids % world == r)                                         # ids owned by the rank
        assert new_gids.tolist() == [(N // world + i) * world + r for i in range(7)]
    assert sum(res[r][4] for r in range(world)) == 8                                 # each id deleted once
    # after: the union of both shards (with their inserts), minus deletions, exact kNN
    rows = {}
    for r in range(world):
        for i, g in enumerate(range(r, N, world)):
            rows[g] = Xall[g]
        newX = int_rows(7, D, seed=100 + r, hi=6)
        for i in range(7):
            rows[(N // world + i) * world + r] = newX[i]
    G = max(rows) + 1
    Xg = np.zeros((G, D), np.float32)
    present = np.zeros(G, bool)
    for g, x in rows.items():
        Xg[g] = x
        present[g] = True
    dead = set([0, 1, 2, 3, 5, 8, 13, 21]) | set(np.flatnonzero(~present).tolist())
    gi2, gd2 = oracle.bf_knn(Xg, Q, k, tomb=pack_tomb(sorted(dead), G))
    assert np.array_equal(res[0][5].view(np.uint32), gi2) and np.array_equal(res[0][6], gd2)
    assert np.array_equal(res[1][5], res[0][5])


def test_id_interleaving_helpers():
    from paper_2601_08528_b200.sharded import owner_and_local, to_global

    ids = torch.tensor([[0, 5, -1], [7, -1, 2]], dtype=torch.int32)
    g = to_global(ids, rank=3, world=8)
    assert g.tolist() == [[3, 43, -1], [59, -1, 19]]
    own, loc = owner_and_local(np.array([3, 43, 59, 19, 8]), 8)
    assert own.tolist() == [3, 3, 3, 3, 0] and loc.tolist() == [0, 5, 7, 2, 1]
