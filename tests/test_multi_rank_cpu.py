"""CPU tests of the sharded layer's host logic (paper_2601_08528_b200/sharded.py), no GPU:
8 logical shards (global id g -> shard g mod 8, local id g div 8), several shards per rank (s mod G = r), the rank
pre-merge, one all_gather_into_tensor of packed (dist bits << 32 | global id) pairs over gloo at world size 2, the
final merge, and insert/delete routing.  The per-shard search and the two merges are the oracle's here (the GPU
kernels svf_shard_premerge / svf_merge_pairs are checked against the same oracle by -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import int_rows, pack_tomb

S = 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleShard:
    """Stands in for one shard's svf Index: exact kNN over the shard's rows via the oracle (local ids)."""

    def __init__(self, X):
        self.X = np.asarray(X, np.float32)
        self.dead = set()

    def _tomb(self):
        return pack_tomb(sorted(self.dead), len(self.X)) if self.dead else None

    def search_into(self, Q, k, itopk, oi, od):
        import oracle

        ids, d = oracle.bf_knn(self.X, Q.numpy(), k, tomb=self._tomb())
        oi.copy_(torch.from_numpy(ids.view(np.int32).copy()))
        od.copy_(torch.from_numpy(d))

    def knn_exact_into(self, Q, k, oi, od):
        self.search_into(Q, k, k, oi, od)

    def info(self):
        return {"n_alloc": len(self.X)}

    def insert(self, X):
        first = len(self.X)
        self.X = np.vstack([self.X, np.asarray(X, np.float32)])
        return np.arange(first, len(self.X), dtype=np.uint32)

    def delete(self, ids):
        before = len(self.dead)
        self.dead |= set(int(i) for i in ids)
        return len(self.dead) - before

    def close(self):
        pass


def pack_pairs(ids_u32, d_f32):
    """(dist bits << 32 | id) as int64, the layout svf_shard_premerge writes (include/svf.h)."""
    hi = np.ascontiguousarray(d_f32, np.float32).view(np.uint32).astype(np.uint64) << np.uint64(32)
    return (hi | np.asarray(ids_u32, np.uint32).astype(np.uint64)).view(np.int64)


def unpack_pairs(p):
    u = np.asarray(p).view(np.uint64)
    return (u & np.uint64(0xFFFFFFFF)).astype(np.uint32), (u >> np.uint64(32)).astype(np.uint32).view(np.float32)


def oracle_premerge(ids_l, d_l, n_logical, shards):
    """Reference of svf_shard_premerge: local -> global ids, then O6's merge."""
    import oracle

    ids = ids_l.numpy().view(np.uint32)
    g = np.where(ids == 0xFFFFFFFF, 0xFFFFFFFF,
                 ids.astype(np.int64) * n_logical + np.asarray(shards, np.int64)[:, None, None]).astype(np.uint32)
    mi, md = oracle.merge_topk(g, d_l.numpy())
    return torch.from_numpy(pack_pairs(mi, md))


def oracle_merge_pairs(gathered):
    import oracle

    ids, d = unpack_pairs(gathered.numpy())
    mi, md = oracle.merge_topk(ids, d)
    return torch.from_numpy(mi.view(np.int32).copy()), torch.from_numpy(md)


def _sharded(X, rank, world):
    from paper_2601_08528_b200.sharded import ShardedIndex, owned_shards

    shards = {s: OracleShard(X[s::S]) for s in owned_shards(S, rank, world)}
    return ShardedIndex(shards, S, rank, world, premerge_fn=oracle_premerge, merge_pairs_fn=oracle_merge_pairs)


N, D, K = 600, 6, 10


def _data():
    return int_rows(N, D, seed=11, hi=6), int_rows(25, D, seed=12, hi=6)   # many exact ties across shards


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, Qn = _data()
        Q = torch.from_numpy(Qn)
        sh = _sharded(X, rank, world)
        ids, d = sh.search(Q, K, 32)
        newX = int_rows(13, D, seed=100, hi=6)                 # one global batch, ids N..N+12, routed by g mod 8
        mine = sh.insert(newX, N)
        n_del = sh.delete(np.array([0, 1, 2, 3, 5, 8, 13, 21, N + 4], np.uint32))
        ids2, d2 = sh.search(Q, K, 32)
        q.put((rank, ids.numpy(), d.numpy(), mine, n_del, ids2.numpy(), d2.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_sharded_search_world2_gloo():
    """Two ranks (4 shards each) return the exact global answer (ties by lower global id) on every rank, before and
    after a routed insert and delete; each new id lands on the rank owning g mod 8, each deletion happens once."""
    import oracle

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
    X, Q = _data()
    gi, gd = oracle.bf_knn(X, Q, K)
    for r in range(world):
        _, ids, d, mine, n_del, ids2, d2 = res[r]
        assert np.array_equal(ids.view(np.uint32), gi) and np.array_equal(d, gd)
        assert np.all((mine.astype(np.int64) % S) % world == r)
    assert sorted(np.concatenate([res[r][3] for r in range(world)]).tolist()) == list(range(N, N + 13))
    assert sum(res[r][4] for r in range(world)) == 9
    Xg = np.vstack([X, int_rows(13, D, seed=100, hi=6)])
    tomb = pack_tomb(np.array([0, 1, 2, 3, 5, 8, 13, 21, N + 4]), N + 13)
    gi2, gd2 = oracle.bf_knn(Xg, Q, K, tomb=tomb)
    for r in range(world):
        assert np.array_equal(res[r][5].view(np.uint32), gi2) and np.array_equal(res[r][6], gd2)


def test_regrouping_the_8_shards_is_invariant():
    """O6: the same 8 shards grouped into G = 1, 2, 4, 8 ranks (rank pre-merge, then the merge of the G
    rank lists, i.e. what the all-gather feeds) give one identical answer, equal to the unsharded exact kNN."""
    import oracle
    from paper_2601_08528_b200.sharded import owned_shards

    X, Qn = _data()
    Q = torch.from_numpy(Qn)
    gi, gd = oracle.bf_knn(X, Qn, K)
    for G in (1, 2, 4, 8):
        blocks = []
        for r in range(G):
            sh = _sharded(X, r, G)
            assert sh.local == owned_shards(S, r, G) == [s for s in range(S) if s % G == r]
            ids_l = torch.empty((len(sh.local), len(Qn), K), dtype=torch.int32)
            d_l = torch.empty((len(sh.local), len(Qn), K), dtype=torch.float32)
            for i, s in enumerate(sh.local):
                sh.shards[s].search_into(Q, K, 32, ids_l[i], d_l[i])
            blocks.append(oracle_premerge(ids_l, d_l, S, sh.local))
        mi, md = oracle_merge_pairs(torch.stack(blocks))
        assert np.array_equal(mi.numpy().view(np.uint32), gi) and np.array_equal(md.numpy(), gd)


def test_id_routing_helpers():
    from paper_2601_08528_b200.sharded import owned_shards, owner_and_local, shard_rows, to_global

    ids = torch.tensor([[0, 5, -1], [7, -1, 2]], dtype=torch.int32)
    assert to_global(ids, shard=3, S=8).tolist() == [[3, 43, -1], [59, -1, 19]]
    own, loc = owner_and_local(np.array([3, 43, 59, 19, 8]), 8)
    assert own.tolist() == [3, 3, 3, 3, 0] and loc.tolist() == [0, 5, 7, 2, 1]
    assert owned_shards(8, 1, 4) == [1, 5] and owned_shards(8, 0, 1) == list(range(8))
    assert [shard_rows(19, s, 8) for s in range(8)] == [3, 3, 3, 2, 2, 2, 2, 2]
    p = pack_pairs(np.array([7, 0xFFFFFFFF], np.uint32), np.array([2.5, np.inf], np.float32))
    i, d = unpack_pairs(p)
    assert i.tolist() == [7, 0xFFFFFFFF] and d.tolist() == [2.5, np.inf]
    assert int(p[0]) == (0x40200000 << 32) | 7        # float bits of 2.5 in the high word


def test_insert_out_of_order_is_refused():
    X, _ = _data()
    sh = _sharded(X, 0, 1)
    with pytest.raises(ValueError):
        sh.insert(int_rows(3, D, seed=5, hi=6), N + 8)   # ids N..N+7 never arrived
