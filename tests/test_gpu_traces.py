"""NEXT-3 on the GPU: the paper's streaming workloads (SlidingWindow and Clustered) replayed step by step
through the C ABI and through the oracle on the same integer-valued C1-sized data.  Every search step must equal
the oracle's O2 on the oracle's own state bit for bit (ids and distances), never return a deleted id, and the final
adjacency (with the automatic global consolidation at 20%, reading C2) must equal the oracle's."""
import numpy as np
import pytest

import oracle
from workloads import GLM, pack_tomb, traces

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
SENT = 0xFFFFFFFF
R, P, L_INS, B_INS, L, K = 32, 16, 64, 512, 32, 10


@pytest.fixture(scope="module")
def svf():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2601_08528_b200 as m

    return m


def replay(svf, X, Q, steps, consolidate_ratio=0.0):
    """Apply `steps` to a GPU index and to the oracle's state side by side; compare at every search step."""
    n = len(X)
    row_of_id = np.empty(n, np.int64)          # ids are assigned in insertion order (I14)
    id_of_row = np.full(n, -1, np.int64)
    G = np.full((n, R), SENT, np.uint32)
    E = np.full((n, R), np.inf, np.float32)
    Xid = np.zeros_like(X)
    tomb = np.zeros((n + 31) // 32, np.uint32)
    n_alloc, n_dead, dead_at_cons, n_cons = 0, 0, 0, 0
    idx = None
    Qd = torch.from_numpy(Q).cuda()
    searches = 0
    for t, s in enumerate(steps):
        ins, dele = np.asarray(s["insert"], np.int64), np.asarray(s["delete"], np.int64)
        if len(ins):
            ids = np.arange(n_alloc, n_alloc + len(ins))
            row_of_id[ids] = ins
            id_of_row[ins] = ids
            Xid[ids] = X[ins]
            if idx is None:
                idx = svf.Index.build(torch.from_numpy(X[ins]).cuda(), degree=R, capacity=n, seed_size=256,
                                      insert_batch=B_INS, insert_itopk=L_INS)
                idx.set_consolidation(consolidate_ratio)
                g0, e0 = oracle.build(X[ins], R=R, P=P, L_ins=L_INS, B_ins=B_INS, seed_size=256)
                G[:len(ins)], E[:len(ins)] = g0, e0
            else:
                got = idx.insert(torch.from_numpy(X[ins]).cuda())
                assert got.tolist() == ids.tolist()
                G, E = oracle.insert(Xid, G, E, n_alloc=n_alloc, n_new=len(ins), P=P, L_ins=L_INS, B_ins=B_INS,
                                     tomb=tomb)
            n_alloc += len(ins)
        if len(dele):
            dids = id_of_row[dele]
            assert (dids >= 0).all()
            newly = idx.delete(torch.from_numpy(dids.astype(np.int32)).cuda())
            tomb, newly_o = oracle.delete(tomb, dids, n_alloc)
            assert newly == newly_o == len(dids)
            n_dead += newly
            # the automatic consolidation trigger (include/svf.h svf_set_consolidation), mirrored on the oracle
            if consolidate_ratio > 0 and n_dead - dead_at_cons > consolidate_ratio * (n_alloc - dead_at_cons):
                G, E, _ = oracle.consolidate(Xid, G, E, tomb, n_alloc=n_alloc, P=P)
                dead_at_cons = n_dead
                n_cons += 1
        if s["search"]:
            ids, d = idx.search(Qd, K, L)
            ri, rd, _ = oracle.graph_search(Xid[:n_alloc], G[:n_alloc], Q, K, L, tomb=tomb, n_alloc=n_alloc)
            assert np.array_equal(ids.cpu().numpy().view(np.uint32), ri), t
            assert np.array_equal(d.cpu().numpy(), rd), t
            dead_ids = np.flatnonzero(np.unpackbits(tomb.view(np.uint8), bitorder="little")[:n_alloc])
            assert not np.isin(ri, dead_ids).any()
            searches += 1
    st = idx.export()
    assert st["n_alloc"] == n_alloc
    assert np.array_equal(st["graph"], G[:n_alloc]) and np.array_equal(st["edge_dist"], E[:n_alloc])
    assert idx.consolidation_stats()["consolidations"] == n_cons
    idx.close()
    return searches, n_cons


def test_sliding_window_trace_step_by_step(svf):
    """SlidingWindow: 24 segments, step t inserts segment t and from t >= 12 deletes segment t - 12;
    search at every step >= 12; automatic consolidation at a 20% deletion ratio."""
    gen = GLM(dim=32, ell=8, integer=True)
    X = gen.rows(21, 21, 0, 7200)
    Q = gen.rows(21, 22, 0, 200)
    searches, n_cons = replay(svf, X, Q, traces.sliding_window(len(X), 24), consolidate_ratio=0.2)
    assert searches == 12 and n_cons >= 1


def test_clustered_trace_step_by_step(svf):
    """Clustered: 8 k-means clusters, 3 rounds of inserting one slice of every cluster (cluster by
    cluster) and deleting half of what is live in every cluster; searches after each phase."""
    gen = GLM(dim=32, ell=8, integer=True)
    X = gen.rows(23, 23, 0, 6000)
    Q = gen.rows(23, 24, 0, 200)
    labels = traces.kmeans_labels(X, k=8, iters=3, sample=6000)
    searches, _ = replay(svf, X, Q, traces.clustered(labels, rounds=3))
    assert searches == 6
