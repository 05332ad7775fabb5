"""Pins for the CPU oracle (oracle/): values the paper/SPEC print, closed forms, exhaustive enumeration on tiny
inputs, hand-traced searches and invariants — chosen so that a dropped term, a wrong sign or index, or a
transposed operand anywhere in the oracle fails at least one of them.  No GPU needed."""
from fractions import Fraction
from math import gcd

import numpy as np
import pytest

from conftest import golden
from workloads import int_rows, pack_tomb, random_graph, random_tombstones, GLM

SENT = 0xFFFFFFFF


# ---- exact enumerators (Python integers / Fractions; no floating point in the decision) -----------------------
def enum_knn(X, Q, k, metric=0, deleted=()):
    """Exhaustive enumeration with exact rational arithmetic; ties by lower id."""
    dead = set(int(i) for i in deleted)
    out = []
    for q in Q:
        qf = [Fraction(float(v)) for v in q]
        rows = []
        for i, x in enumerate(X):
            if i in dead:
                continue
            xf = [Fraction(float(v)) for v in x]
            if metric == 0:
                d = sum((a - b) * (a - b) for a, b in zip(qf, xf))
            else:
                d = -sum(a * b for a, b in zip(qf, xf))
            rows.append((d, i))
        rows.sort()
        out.append(rows[:k])
    return out


# ---- splitmix64 / entry-point law (I2) --------------------------------------------------------------------------
def test_splitmix64_reference_sequence(orc):
    g = golden("splitmix64.json")
    golden_inc = int(g["golden"], 16)
    for n, want in enumerate(g["outputs"]):
        assert orc.splitmix64((n * golden_inc) % (1 << 64)) == int(want, 16)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 12, 30, 97, 210, 1024, 9973])
def test_affine_permutation_is_bijection(orc, n):
    for seed in (0, 1, 42):
        for qidx in (0, 1, 7, 12345):
            a, b = orc.affine_params(seed, qidx, n)
            assert 1 <= a < max(n, 2) and 0 <= b < n and gcd(a, n) == 1
            ids = {(a * j + b) % n for j in range(n)}
            assert len(ids) == n


def test_entry_point_is_first_live_along_permutation(orc):
    """No edges, n_init=1: the pool holds exactly id_0 = b; with b deleted it is the next live id_1 = (a+b) mod n."""
    n, D = 50, 4
    X = int_rows(n, D, seed=3)
    graph = np.full((n, 2), SENT, np.uint32)
    for seed in (1, 2, 3, 42):
        for qi in range(5):
            a, b = orc.affine_params(seed, qi, n)
            ids, _, cnt = orc.graph_search(X, graph, X[:1], k=1, L=1, n_init=1, seed=seed, qidx=[qi])
            assert ids[0, 0] == b and cnt[0, 0] == 1
            tomb = pack_tomb([b], n)
            ids, _, _ = orc.graph_search(X, graph, X[:1], k=1, L=1, n_init=1, seed=seed, qidx=[qi], tomb=tomb)
            assert ids[0, 0] == (a + b) % n


# ---- O1 exact kNN -----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("metric", [0, 1])
def test_bf_knn_matches_exhaustive_enumeration_with_ties(orc, metric):
    X = int_rows(60, 3, seed=5, lo=-2 if metric else 0, hi=3)   # tiny value range => many exact ties
    Q = int_rows(12, 3, seed=6, lo=-2 if metric else 0, hi=3)
    deleted = [3, 17, 40]
    tomb = pack_tomb(deleted, 60)
    for k in (1, 5, 20, 57, 60):
        ids, d = orc.bf_knn(X, Q, k, metric=metric, tomb=tomb)
        ref = enum_knn(X, Q, k, metric, deleted)
        for qi in range(len(Q)):
            for j in range(k):
                if j < len(ref[qi]):
                    assert ids[qi, j] == ref[qi][j][1]
                    assert d[qi, j] == np.float32(float(ref[qi][j][0]))
                else:
                    assert ids[qi, j] == SENT and np.isinf(d[qi, j])


def test_bf_knn_float_data_against_exact_rationals(orc):
    g = GLM(dim=8, ell=4, s=1.0, m=0.0, sigma=0.1)
    X = g.rows(7, 7, 0, 40)
    Q = g.rows(7, 8, 0, 5)
    ids, d = orc.bf_knn(X, Q, 10)
    ref = enum_knn(X, Q, 10)
    for qi in range(5):
        assert [i for _, i in ref[qi]] == ids[qi].tolist()
        np.testing.assert_allclose(d[qi], [float(v) for v, _ in ref[qi]], rtol=1e-7)


def test_spec_ground_truth_example(orc):
    g = golden("spec_examples.json")["ground_truth_1d"]
    X = np.array(g["points"], np.float32)[:, None]
    ids, _ = orc.bf_knn(X, np.array([[g["q"]]], np.float32), g["k"])
    assert ids[0].tolist() == g["expect_ids"]


def test_bf_knn_sorted_prefix_and_deleted_excluded(orc):
    X = int_rows(300, 16, seed=9)
    Q = int_rows(20, 16, seed=10)
    dead = random_tombstones(300, 0.2, seed=11)
    tomb = pack_tomb(dead, 300)
    i10, d10 = orc.bf_knn(X, Q, 10, tomb=tomb)
    i11, _ = orc.bf_knn(X, Q, 11, tomb=tomb)
    assert np.all(np.diff(d10, axis=1) >= 0)                  # non-decreasing (north star invariant)
    assert np.array_equal(i11[:, :10], i10)                   # k-prefix monotonicity
    assert not np.isin(i10, dead).any()                       # deleted never returned
    all_dead = pack_tomb(np.arange(300), 300)
    i0, d0 = orc.bf_knn(X, Q, 3, tomb=all_dead)
    assert np.all(i0 == SENT) and np.all(np.isinf(d0))        # empty live set -> empty


def test_distance_closed_forms(orc):
    q = np.array([1, 2, 3, 4], np.float32)
    x = np.array([-1, 0, 5, 4], np.float32)
    assert orc.dist(q, x, 0) == 4 + 4 + 4 + 0
    assert orc.dist(q, x, 1) == -(-1 + 0 + 15 + 16)
    z = np.zeros(4, np.float32)
    assert np.signbit(orc.dist(z, x, 1)) == False  # -0.0 canonicalised to +0.0


# ---- O2 greedy graph search ---------------------------------------------------------------------------------------
def _trace_graph(g):
    return np.array([[SENT if v is None else v for v in row] for row in g["graph"]], np.uint32)


@pytest.mark.parametrize("case", [c["name"] for c in golden("hand_traces.json")["cases"]])
def test_hand_traced_search(orc, case):
    g = golden("hand_traces.json")
    c = next(c for c in g["cases"] if c["name"] == case)
    X = np.array(g["points"], np.float32)[:, None]
    graph = _trace_graph(g)
    tomb = pack_tomb(c["deleted"], len(X)) if c["deleted"] else None
    ids, d, cnt = orc.graph_search_from(X, graph, np.array([c["q"]], np.float32), c["init"], c["k"], c["L"],
                                        p=c["p"], max_iter=c.get("max_iter", 0), tomb=tomb)
    assert ids.tolist() == c["expect_ids"]
    assert d.tolist() == c["expect_d"]
    assert cnt.tolist() == [c["n_dist"], c["n_exp"], c["iters"]]


def test_spec_search_example(orc):
    g = golden("spec_examples.json")["search_1d"]
    X = np.array(g["points"], np.float32)[:, None]
    graph, _ = orc.build(X, R=g["R"])
    q = np.array([[g["q"]]], np.float32)
    ids, d, _ = orc.graph_search(X, graph, q, k=g["k"], L=g["L"])
    assert ids[0, 0] == g["expect"]["id"] and abs(d[0, 0] - g["expect"]["dist"]) < g["expect"]["tol"]
    a = g["after_delete"]
    ids, d, _ = orc.graph_search(X, graph, q, k=g["k"], L=g["L"], tomb=pack_tomb(a["deleted"], 4))
    assert ids[0, 0] == a["id"] and abs(d[0, 0] - a["dist"]) < a["tol"]


@pytest.mark.parametrize("p", [1, 2, 4])
def test_search_with_full_pool_equals_exact_knn(orc, p):
    """L >= live N and n_init >= live N => the pool holds every live vertex => O2 == O1 exactly."""
    n = 200
    X = int_rows(n, 8, seed=21, hi=4)
    Q = int_rows(15, 8, seed=22, hi=4)
    graph = random_graph(n, 6, seed=23)
    dead = random_tombstones(n, 0.1, seed=24)
    tomb = pack_tomb(dead, n)
    ids, d, _ = orc.graph_search(X, graph, Q, k=10, L=n, n_init=n, p=p, tomb=tomb)
    gi, gd = orc.bf_knn(X, Q, 10, tomb=tomb)
    assert np.array_equal(ids, gi) and np.array_equal(d, gd)


def test_complete_graph_is_exact_after_one_expansion(orc):
    n = 64
    X = int_rows(n, 5, seed=31)
    Q = int_rows(10, 5, seed=32)
    graph = np.array([[u for u in range(n) if u != v] for v in range(n)], np.uint32)
    ids, d, cnt = orc.graph_search(X, graph, Q, k=5, L=5, n_init=1)
    gi, gd = orc.bf_knn(X, Q, 5)
    assert np.array_equal(ids, gi)
    assert np.all(cnt[:, 0] == n)   # every vertex scored exactly once


def test_spec_recall_band_small_dataset(orc):
    """N=2000 random D=16 vectors, R=16, L=512 => recall@10 >= 0.99 over 100 queries."""
    g = GLM(dim=16, ell=8, s=3.0, m=0.0, sigma=0.3)
    X = g.rows(1, 1, 0, 2000)
    Q = g.rows(1, 2, 0, 100)
    graph, _ = orc.build(X, R=16, seed_size=256, B_ins=256)
    ids, _, _ = orc.graph_search(X, graph, Q, k=10, L=512)
    gi, _ = orc.bf_knn(X, Q, 10)
    assert orc.recall_ids(ids, gi, 10) >= 0.99


def test_search_invariants(orc):
    n = 3000
    X = int_rows(n, 16, seed=41)
    Q = int_rows(40, 16, seed=42)
    graph = random_graph(n, 12, seed=43)
    dead = random_tombstones(n, 0.15, seed=44)
    tomb = pack_tomb(dead, n)
    for p in (1, 3):
        ids, d, cnt = orc.graph_search(X, graph, Q, k=10, L=32, p=p, tomb=tomb)
        assert not np.isin(ids, dead).any()
        assert np.all(np.diff(d, axis=1) >= 0)
        assert np.all(cnt[:, 2] <= cnt[:, 0])            # termination: iterations <= distance computations
        assert np.all(cnt[:, 1] <= p * cnt[:, 2]) and np.all(cnt[:, 1] >= cnt[:, 2])
        pool, pd, _ = orc.graph_search(X, graph, Q, k=10, L=32, p=p, tomb=tomb, insert_mode=True)
        assert np.array_equal(pool[:, :10], ids)         # insert mode returns the whole pool
        assert np.all(np.diff(pd, axis=1) >= 0)
        capped, _, cc = orc.graph_search(X, graph, Q, k=10, L=32, p=p, tomb=tomb, max_iter=3)
        assert np.all(cc[:, 2] <= 3)
        # determinism and per-query independence
        ids2, _, _ = orc.graph_search(X, graph, Q[::-1], k=10, L=32, p=p, tomb=tomb, qidx=np.arange(40)[::-1])
        assert np.array_equal(ids2[::-1], ids)


# ---- O3 insert / O5 build -------------------------------------------------------------------------------------------
def test_spec_detour_example(orc):
    g = golden("spec_examples.json")["detour"]
    name = {c: i for i, c in enumerate(g["C"])}          # c1,c2,c3 -> ids 0,1,2
    R = 3
    graph = np.full((4, R), SENT, np.uint32)
    for c, lst in g["lists"].items():
        for s, v in enumerate(lst):
            graph[name[c], s] = name[v]
    ed = np.full((4, R), np.inf, np.float32)
    cand = np.array([[name[c] for c in g["C"]]], np.uint32)
    cd = np.array([[1.0, 2.0, 3.0]], np.float32)
    out, _ = orc.link_candidates(graph, ed, 3, cand, cd, P=R)     # P = R: the whole row is detour order
    assert out[3].tolist() == [name[c] for c in g["expect"]]
    # lists all empty -> output equals input;  single candidate -> itself
    out, _ = orc.link_candidates(np.full((4, R), SENT, np.uint32), ed, 3, cand, cd, P=R)
    assert out[3].tolist() == [0, 1, 2]
    one = np.array([[2, SENT, SENT]], np.uint32)
    out, _ = orc.link_candidates(np.full((4, R), SENT, np.uint32), ed, 3, one, cd, P=R)
    assert out[3].tolist() == [2, SENT, SENT]


def test_spec_exact_rnn_and_padding(orc):
    g = golden("spec_examples.json")
    e = g["exact_rnn"]
    X = np.array(e["points"], np.float32)[:, None]
    graph, _ = orc.build(X, R=e["R"])
    assert set(graph[e["vertex"]].tolist()) == set(e["expect_set"])
    p = g["padding"]
    graph, ed = orc.build(int_rows(p["N"], 4, seed=1), R=p["R"])
    assert np.all((graph != SENT).sum(1) == p["expect_real"])
    assert np.all(np.isinf(ed[graph == SENT]))


def test_spec_insert_example(orc):
    g = golden("spec_examples.json")["insert_1d"]
    pts = g["points"] + [g["new_point"]]
    X = np.array(pts, np.float32)[:, None]
    R, P = g["R"], g["P"]
    graph0, ed0 = orc.build(X[:4], R=R, P=P)
    cap_g = np.vstack([graph0, np.full((1, R), SENT, np.uint32)])
    cap_d = np.vstack([ed0, np.full((1, R), np.inf, np.float32)])
    graph, ed = orc.insert(X, cap_g, cap_d, n_alloc=4, n_new=1, P=P)
    by_val = {str(int(v)): i for i, v in enumerate(pts)}
    for val, row in g["expect_rows_by_value"].items():
        assert [pts[i] for i in graph[by_val[val]]] == row, val
    for val, dd in g["expect_dists_by_value"].items():
        assert ed[by_val[val]].tolist() == dd


def _check_row_layout(orc, X, graph, ed, R, P, tomb=None, metric=0, first=0):
    n = graph.shape[0]
    for v in range(first, n):
        row = graph[v]
        real = row[row != SENT]
        assert v not in real                                  # no self loops
        assert len(set(real.tolist())) == len(real)           # no duplicates
        for s in range(R):
            if row[s] != SENT:                                # stored edge distance is the true distance
                ref = np.float64(((X[v].astype(np.float64) - X[row[s]]) ** 2).sum()) if metric == 0 else \
                    -np.float64((X[v].astype(np.float64) * X[row[s]]).sum())
                assert abs(ed[v, s] - ref) <= 1e-5 * max(1.0, abs(ref))
        tail = [(np.inf if (i == SENT or (tomb is not None and (tomb[i >> 5] >> (i & 31)) & 1)) else ed[v, s], i)
                for s, i in enumerate(row) if s >= P]
        assert tail == sorted(tail)                           # tail sorted by effective key


def test_build_invariants_and_determinism(orc):
    X = GLM(dim=32, ell=8, integer=True).rows(3, 3, 0, 3000)
    R, P = 16, 8
    g1, e1 = orc.build(X, R=R, P=P, seed_size=500, B_ins=400, L_ins=48)
    g2, e2 = orc.build(X, R=R, P=P, seed_size=500, B_ins=400, L_ins=48, threads=1)
    assert np.array_equal(g1, g2) and np.array_equal(e1, e2)   # build determinism
    assert np.all(g1 != SENT)                                  # N > R: every slot filled
    _check_row_layout(orc, X, g1, e1, R, P)
    # seed rows are the exact R-NN of the seed set (self excluded), O1 rules; growth only rewrites their tails
    gs, _ = orc.build(X[:500], R=R, P=P, seed_size=500)
    gi, gd = orc.bf_knn(X[:500], X[:500], R + 1)
    for v in range(0, 500, 37):
        want = [i for i in gi[v] if i != v][:R]
        assert gs[v].tolist() == want
        assert g1[v, :P].tolist() == want[:P]


def test_reverse_edges_keep_the_smallest_tail(orc):
    """(iii) as a set property: new tail(u) is sorted, drawn from tail(u) ∪ requests(u), and no excluded element
    has a smaller effective key than an included one; prefixes never change (reading I12)."""
    X = GLM(dim=16, ell=6, integer=True).rows(4, 4, 0, 1200)
    R, P = 12, 6
    g0, e0 = orc.build(X[:1000], R=R, P=P, seed_size=300, B_ins=200, L_ins=32)
    dead = random_tombstones(1000, 0.1, seed=5)
    tomb = pack_tomb(dead, 1200)
    G = np.vstack([g0, np.full((200, R), SENT, np.uint32)])
    E = np.vstack([e0, np.full((200, R), np.inf, np.float32)])
    # candidate lists from the insert-mode search over the snapshot, then link
    Q = X[1000:1200]
    cid, cd, _ = orc.graph_search(X, G, Q, k=1, L=32, tomb=tomb, n_alloc=1000, qidx=np.arange(1000, 1200),
                                  insert_mode=True)
    G1, E1 = orc.link_candidates(G, E, 1000, cid, cd, P=P, tomb=tomb)
    assert np.array_equal(G1[:1000, :P], G[:1000, :P])          # prefixes untouched
    assert not np.isin(G1[1000:], dead).any()                    # no tombstoned id in a new forward row
    reqs = {}
    for b in range(200):
        v = 1000 + b
        for s in range(R):
            u = G1[v, s]
            if u != SENT:
                reqs.setdefault(int(u), []).append((float(E1[v, s]), v))

    def eff(i, d):
        return (np.inf if i == SENT or ((tomb[i >> 5] >> (i & 31)) & 1) else d, i)

    for u in range(1000):
        old = [eff(int(G[u, s]), float(E[u, s])) for s in range(P, R)]
        new = [eff(int(G1[u, s]), float(E1[u, s])) for s in range(P, R)]
        if u in set(dead.tolist()) or u not in reqs:   # frozen / untouched rows are not rewritten
            assert new == old
            continue
        union = sorted(old + [(d, v) for d, v in reqs.get(u, [])])
        assert new == sorted(new)
        assert sorted(new) == union[:R - P]
    # in-degree recount: every accepted request appears exactly once
    indeg = np.bincount(G1[G1 != SENT].astype(np.int64), minlength=1200)
    assert indeg.sum() == (G1 != SENT).sum()


def test_read_after_write(orc):
    """P:L1035-1036 / S:L432: insert x, then search x with k=1 returns x (paper reports Recall@1 0.96)."""
    X = GLM(dim=32, ell=8).rows(5, 5, 0, 4000)
    g0, e0 = orc.build(X[:3000], R=16, seed_size=1000, B_ins=500, L_ins=64)
    G = np.vstack([g0, np.full((1000, 16), SENT, np.uint32)])
    E = np.vstack([e0, np.full((1000, 16), np.inf, np.float32)])
    G1, E1 = orc.insert(X, G, E, n_alloc=3000, n_new=1000, P=8, L_ins=64, B_ins=10)
    ids, _, _ = orc.graph_search(X, G1, X[3000:], k=1, L=32)
    assert np.mean(ids[:, 0] == np.arange(3000, 4000)) >= 0.95


def test_insert_matches_build_growth(orc):
    """O5 = seed + O3: building n rows equals building the seed then inserting the rest in the same sub-batches."""
    X = GLM(dim=16, ell=6, integer=True).rows(6, 6, 0, 900)
    R = 8
    gb, eb = orc.build(X, R=R, seed_size=200, B_ins=150, L_ins=24)
    g0, e0 = orc.build(X[:200], R=R, seed_size=200, B_ins=150, L_ins=24)
    G = np.vstack([g0, np.full((700, R), SENT, np.uint32)])
    E = np.vstack([e0, np.full((700, R), np.inf, np.float32)])
    gi, ei = orc.insert(X, G, E, n_alloc=200, n_new=700, P=R // 2, L_ins=24, B_ins=150)
    assert np.array_equal(gi, gb) and np.array_equal(ei, eb)


TWO_NEW = {  # hand-derived (docstring of test_two_new_vertices_in_one_sub_batch)
    "xs": [0, 10, 30, 40, 20, 21],
    "base_g": [[1, 2], [0, 2], [3, 1], [2, 1]],
    "graph": [[1, 2], [0, 4], [3, 5], [2, 1], [1, 2], [2, 1]],
    "edge_dist": [[100, 900], [100, 100], [100, 81], [100, 900], [100, 100], [81, 121]],
}


def two_new_inputs():
    """Base points x = 0, 10, 30, 40 (ids 0..3, D = 4 zero-padded), R = 2, P = 1, rows = the exact 2-NN (seed
    layout), then ids 4 (x = 20) and 5 (x = 21) inserted together."""
    xs = TWO_NEW["xs"]
    X = np.zeros((6, 4), np.float32)
    X[:, 0] = xs
    G = np.full((6, 2), SENT, np.uint32)
    E = np.full((6, 2), np.inf, np.float32)
    G[:4] = TWO_NEW["base_g"]
    E[:4] = [[(xs[v] - xs[u]) ** 2 for u in G[v]] for v in range(4)]
    return X, G, E


def test_two_new_vertices_in_one_sub_batch(orc):
    """Sub-batch snapshot semantics (I13, "delayed graph updates"): vertices inserted in one sub-batch
    neither reach nor sample each other.  By hand (L_insert = 4 covers every live id, squared distances):
      v=4 (x=20): C = [1:100, 2:100, 0:400, 3:400]; detour counts 0,1 (2 in row 1),1 (0 in row 1),1 (3 in row 2)
                  -> selected 1, 2 -> row [1 | 2] (100 | 100);
      v=5 (x=21): its nearest vertex is 4 (d 1) but 4 is not in the snapshot: C = [2:81, 1:121, 3:361, 0:441];
                  counts 0,1,1,1 -> row [2 | 1] (81 | 121);
      reverse: row 1 tail {2:900} u {4:100, 5:121} -> 4; row 2 tail {1:900} u {4:100, 5:81} -> 5.
    With sub-batches of one vertex, 5 does see 4 (its first candidate, d 1)."""
    X, G, E = two_new_inputs()
    g2, e2 = orc.insert(X, G, E, n_alloc=4, n_new=2, P=1, L_ins=4, B_ins=4096)
    assert g2.tolist() == TWO_NEW["graph"] and e2.tolist() == TWO_NEW["edge_dist"]
    g1, _ = orc.insert(X, G, E, n_alloc=4, n_new=2, P=1, L_ins=4, B_ins=1)
    assert 4 in g1[5].tolist() and 4 not in g2[5].tolist()


# ---- O6 shard merge / O7 recall -------------------------------------------------------------------------------------
def test_shard_merge_identical_for_any_gpu_count(orc):
    S, nq, k = 8, 30, 10
    n = 800
    X = int_rows(n, 8, seed=51, hi=5)
    Q = int_rows(nq, 8, seed=52, hi=5)
    per = []
    for s in range(S):
        gid = np.arange(s, n, S)                              # shard s holds global ids g with g mod S = s
        ids, d = orc.bf_knn(X[gid], Q, k)
        ids = np.where(ids == SENT, SENT, gid[np.minimum(ids, len(gid) - 1)]).astype(np.uint32)
        per.append((ids, d))
    full, fd = orc.bf_knn(X, Q, k)
    for G in (1, 2, 4, 8):
        # rank r pre-merges shards {s : s mod G = r}, then the G rank lists are merged
        ranks = []
        for r in range(G):
            mine = [per[s] for s in range(S) if s % G == r]
            ranks.append(orc.merge_topk(np.stack([m[0] for m in mine]), np.stack([m[1] for m in mine])))
        mi, md = orc.merge_topk(np.stack([x[0] for x in ranks]), np.stack([x[1] for x in ranks]))
        assert np.array_equal(mi, full) and np.array_equal(md, fd)


def test_spec_recall_examples(orc):
    for res, gt, want in golden("spec_examples.json")["recall"]["cases"]:
        assert abs(orc.recall_ids([res], [gt], 3) - want) < 1e-12


def test_recall_tie_aware_hand_cases(orc):
    """O7 tie-aware recall (P:L736 Recall@k): result i counts when its exact distance is <= the
    k-th true distance (relative slack 1e-5).  Hand cases: an exact tie at the k-th distance counts even with a
    different id (id recall 2/3, tie-aware 1); a result just beyond the slack does not; negative inner-product
    distances loosen toward zero (-8 -> -7.99992), never away from it; padded (+inf) results never count; a k-th
    distance of 0 admits only 0."""
    ids_gt, d_gt = [[7, 8, 9]], [[1.0, 2.0, 3.0]]
    assert orc.recall_ids([[7, 8, 4]], ids_gt, 3) == pytest.approx(2 / 3)
    assert orc.recall_tie_aware([[1.0, 2.0, 3.0]], d_gt, 3) == 1.0
    assert orc.recall_tie_aware([[1.0, 2.0, 3.0001]], d_gt, 3) == pytest.approx(2 / 3)
    assert orc.recall_tie_aware([[1.0, 2.0, 3.00002]], d_gt, 3) == 1.0
    neg = [[-10.0, -9.0, -8.0]]
    assert orc.recall_tie_aware([[-10.0, -8.0, -7.99995]], neg, 3) == 1.0
    assert orc.recall_tie_aware([[-10.0, -8.0, -7.9999]], neg, 3) == pytest.approx(2 / 3)
    assert orc.recall_tie_aware([[1.0, np.inf, np.inf]], d_gt, 3) == pytest.approx(1 / 3)
    assert orc.recall_tie_aware([[0.0, 0.0, 1e-6]], [[0.0, 0.0, 0.0]], 3) == pytest.approx(2 / 3)
    # two queries average; only the first k columns are read
    assert orc.recall_tie_aware([[1.0, 5.0, 0.0], [2.0, 2.0, 9.0]], [[1.0, 2.0, 0.0], [2.0, 3.0, 0.0]],
                                2) == pytest.approx(3 / 4)


# ---- NEXT-1 localized repair ----------------------------------------------------------------------------------------
def _repair_golden():
    g = golden("spec_examples.json")["repair"]
    X = np.array(g["points"], np.float32)[:, None]
    R = g["R"]
    G = np.array([[SENT if v is None else v for v in row] for row in g["rows"]], np.uint32)
    E = np.full(G.shape, np.inf, np.float32)
    for v in range(len(G)):
        for s in range(R):
            if G[v, s] != SENT:
                E[v, s] = (X[v, 0] - X[G[v, s], 0]) ** 2
    return g, X, G, E


def test_spec_repair_example(orc):
    g, X, G, E = _repair_golden()
    tomb = pack_tomb(g["deleted"], len(X))
    # (no detours among the union here, so both readings give the distance order)
    gk, _, _, _ = orc.repair(X, G, E, tomb, c=g["c"], threshold=g["threshold"], mode=0)
    assert gk[0].tolist() == g["expect_row0"]
    g2, e2, nrep, hist = orc.repair(X, G, E, tomb, c=g["c"], threshold=g["threshold"])
    assert g2[0].tolist() == g["expect_row0"] and e2[0].tolist() == g["expect_d0"]
    assert nrep == 1 and hist.sum() == len(X) - len(g["deleted"])
    assert np.array_equal(g2[1:], G[1:])                         # only V^L rows change
    # strict threshold: 1/3 deleted is not > 0.5 -> nothing repaired (S:L392-393 boundary)
    g3, _, nrep3, _ = orc.repair(X, G, E, tomb, c=g["c"], threshold=0.5)
    assert nrep3 == 0 and np.array_equal(g3, G)
    # all of N_out(p) deleted -> no candidates from p; v keeps its live neighbours only
    tomb_all = pack_tomb([1, 4, 5, 6], len(X))
    g4, _, _, _ = orc.repair(X, G, E, tomb_all, c=2, threshold=0.3)
    assert g4[0].tolist() == [2, 3, SENT, SENT]
    # detour selection over the union (R1'): make x list y, so y (count 1) ranks after a and b (count 0)
    G5 = G.copy()
    G5[4, 0] = 5
    g5, e5, _, _ = orc.repair(X, G5, E, tomb, c=g["c"], threshold=g["threshold"])
    assert g5[0].tolist() == [4, 2, 5, 3] and e5[0].tolist() == [1, 9, 4, 16]   # prefix [x,a] | tail [y,b]
    gk5, _, _, _ = orc.repair(X, G5, E, tomb, c=g["c"], threshold=g["threshold"], mode=0)
    assert gk5[0].tolist() == [4, 5, 2, 3]                                         # R1: plain distance order


def test_repair_properties_on_a_built_graph(orc):
    X = GLM(dim=16, ell=6, integer=True).rows(8, 8, 0, 3000)
    R, c = 16, 8
    G, E = orc.build(X, R=R, seed_size=500, B_ins=400, L_ins=48)
    dead = random_tombstones(3000, 0.45, seed=9)
    tomb = pack_tomb(dead, 3000)
    deadset = set(dead.tolist())
    g2, e2, nrep, hist = orc.repair(X, G, E, tomb, c=c, threshold=0.5)
    assert hist.sum() == 3000 - len(dead) and hist[4] == nrep > 0
    changed = np.flatnonzero(np.any(g2 != G, axis=1))
    for v in changed:
        old = [int(x) for x in G[v] if x != SENT]
        assert sum(x in deadset for x in old) / len(old) > 0.5       # only severely affected vertices
        new = [int(x) for x in g2[v] if x != SENT]
        assert not (set(new) & deadset) and v not in new and len(set(new)) == len(new)
        tail = [(float(e2[v, s]), int(g2[v, s])) for s in range(R // 2, R) if g2[v, s] != SENT]
        assert tail == sorted(tail)                                   # prefix detour-ranked, tail sorted
        allowed = set(x for x in old if x not in deadset)
        per_p = {p: [int(x) for x in G[p] if x != SENT] for p in old if p in deadset}
        for x in new:
            if x not in allowed:
                assert any(x in lst for lst in per_p.values())       # replacements come from N_out(p)
        assert len(set(new) - allowed) <= c * len(per_p)            # O(cR) added edges


# ---- NEXT-4 global consolidation (reading C2) -------------------------------------------------------
def test_consolidate_hand_example_line(orc):
    """Points 0,1,2,3,4,10 on a line (D=4, zero-padded), R=2, P=1; vertex 2 deleted; N_out(2) = {1, 3}.  By hand:
    row 0 = [1 | 2]: the live prefix 1 stays, the tail vacancy takes the nearest of U = {3} -> [1 | 3] (d 1, 9).
    Row 1 = [2 | 0]: the deleted prefix slot takes the nearest member of N_out(2) other than 1 itself -> 3 (d 4);
    the live tail 0 stays -> [3 | 0].  Row 3 = [2 | 4]: prefix <- 1 (d 4; 3 itself skipped), tail 4 stays ->
    [1 | 4].  Rows 2 (deleted), 4 and 5 (no deleted neighbour) are untouched."""
    xs = [0, 1, 2, 3, 4, 10]
    X = np.zeros((6, 4), np.float32)
    X[:, 0] = xs
    G = np.array([[1, 2], [2, 0], [1, 3], [2, 4], [3, 5], [4, 3]], np.uint32)
    E = np.array([[(xs[v] - xs[u]) ** 2 for u in G[v]] for v in range(6)], np.float32)
    tomb = pack_tomb(np.array([2], np.uint32), 6)
    g2, e2, n = orc.consolidate(X, G, E, tomb, P=1)
    assert n == 3
    exp_g = np.array([[1, 3], [3, 0], [1, 3], [1, 4], [3, 5], [4, 3]], np.uint32)
    exp_e = np.array([[1, 9], [4, 1], E[2], [4, 1], E[4], E[5]], np.float32)
    assert np.array_equal(g2, exp_g) and np.array_equal(e2, exp_e)


def test_consolidate_hand_example_refill_rules(orc):
    """x = 0,1,2,3,5,8,13 (ids 0..6), R=4, P=2, ids 2 and 3 deleted; N_out(2) = [5,1,6,0], N_out(3) = [5,4,2,6].
    Worked by hand (squared distances):
      row 0 [4,2|1,3]: U = {5:64, 6:169}; prefix slot 1 (p=2) <- 5; the tail keeps 1 and its vacancy takes 6
                       -> [4,5|1,6] (25,64 | 1,169);
      row 1 [3,0|2,-]: U = {5:49, 4:16, 6:144}; prefix slot 0 (p=3) <- 4; both tail slots vacant <- 5, 6
                       -> [4,0|5,6] (16,1 | 49,144);
      row 4 [3,5|-,-]: U = {6:64}; prefix slot 0 <- 6; nothing left for the tail -> [6,5|-,-];
      row 5 [2,3|4,-]: U = {1:49, 6:25, 0:64}; slot 0 (p=2) <- 6; slot 1 (p=3): N_out(3) has only 6 (taken)
                       -> empty; tail keeps 4 and its empty slot takes 1 -> [6,-|4,1] (25,inf | 9,49);
      row 6 has no deleted neighbour; rows 2, 3 are deleted: all three untouched."""
    xs = [0, 1, 2, 3, 5, 8, 13]
    X = np.zeros((7, 4), np.float32)
    X[:, 0] = xs
    S, inf = SENT, np.inf
    G = np.array([[4, 2, 1, 3], [3, 0, 2, S], [5, 1, 6, 0], [5, 4, 2, 6], [3, 5, S, S], [2, 3, 4, S],
                  [5, 4, S, S]], np.uint32)
    E = np.array([[(xs[v] - xs[u]) ** 2 if u != S else inf for u in G[v]] for v in range(7)], np.float32)
    tomb = pack_tomb(np.array([2, 3], np.uint32), 7)
    g2, e2, n = orc.consolidate(X, G, E, tomb, P=2)
    assert n == 4
    exp_g = G.copy()
    exp_e = E.copy()
    exp_g[0], exp_e[0] = [4, 5, 1, 6], [25, 64, 1, 169]
    exp_g[1], exp_e[1] = [4, 0, 5, 6], [16, 1, 49, 144]
    exp_g[4], exp_e[4] = [6, 5, S, S], [64, 9, inf, inf]
    exp_g[5], exp_e[5] = [6, S, 4, 1], [25, inf, 9, 49]
    assert np.array_equal(g2, exp_g) and np.array_equal(e2, exp_e)


def test_consolidate_properties_on_a_built_graph(orc):
    """After consolidation no live row references a deleted vertex (the defining effect: all affected
    neighbourhoods); only rows that held a deleted id change, and they keep every live entry (prefix entries in
    their slots); a refilled prefix slot holds a member of its own deleted neighbour's list; tail refills come from
    the deleted neighbours' lists and are the nearest such candidates not used elsewhere; deleted rows are frozen."""
    X = GLM(dim=16, ell=6, integer=True).rows(8, 8, 0, 3000)
    R, P = 16, 8
    G, E = orc.build(X, R=R, seed_size=500, B_ins=400, L_ins=48)
    dead = random_tombstones(3000, 0.25, seed=11)
    tomb = pack_tomb(dead, 3000)
    deadset = set(dead.tolist())
    g2, e2, n = orc.consolidate(X, G, E, tomb)
    live = np.setdiff1d(np.arange(3000), dead)
    assert not np.isin(g2[live], dead).any()
    affected = [v for v in live if any(int(x) in deadset for x in G[v] if x != SENT)]
    assert n == len(affected) > 0
    assert np.array_equal(g2[dead], G[dead])
    unaff = np.setdiff1d(live, affected)
    assert np.array_equal(g2[unaff], G[unaff])
    for v in affected[:300]:
        old = [int(x) for x in G[v]]
        lists = {p: set(int(x) for x in G[p] if x != SENT) for p in old if p in deadset}
        cand = set().union(*lists.values()) - deadset - {v} - set(old)
        for s in range(P):
            if old[s] == SENT or old[s] not in deadset:
                assert g2[v, s] == G[v, s] and e2[v, s] == E[v, s]          # live prefix entries stay in place
            elif g2[v, s] != SENT:
                assert int(g2[v, s]) in lists[old[s]] and int(g2[v, s]) in cand
        kept = {(float(E[v, s]), old[s]) for s in range(P, R) if old[s] != SENT and old[s] not in deadset}
        tail = [(float(e2[v, s]), int(g2[v, s])) for s in range(P, R) if g2[v, s] != SENT]
        assert tail == sorted(tail) and kept <= set(tail)                  # live tail entries kept, tail sorted
        refills = [t for t in tail if t not in kept]
        assert all(x in cand for _, x in refills)
        used = set(int(x) for x in g2[v] if x != SENT)
        others = [(float(orc.dist(X[v], X[x])), x) for x in cand - used]
        if refills and others:
            assert max(refills) < min(others)                               # the nearest unused candidates
        if len(tail) < R - P:
            assert not others                                               # vacancies stay only when U ran out
        assert v not in used and len(used) == len([x for x in g2[v] if x != SENT])


# ---- O4 lazy deletion -------------------------------------------------------------------------------
def test_delete_sets_bits_idempotently(orc):
    """Bits are set per id (bit id%32 of word id/32, the layout include/svf.h states), a repeated id or an already
    deleted id is not counted again (S:L389 idempotent no-op), an id >= n_alloc deletes nothing."""
    t0 = np.zeros(3, np.uint32)
    t1, newly = orc.delete(t0, [0, 31, 32, 70, 31], n_alloc=80)
    assert newly == 4 and t1.tolist() == [1 | (1 << 31), 1, 1 << 6]
    t2, newly2 = orc.delete(t1, [70, 5], n_alloc=80)
    assert newly2 == 1 and t2.tolist() == [1 | (1 << 31) | (1 << 5), 1, 1 << 6]
    with pytest.raises(KeyError):
        orc.delete(t2, [3, 80], n_alloc=80)
    assert t2.tolist() == [1 | (1 << 31) | (1 << 5), 1, 1 << 6]
