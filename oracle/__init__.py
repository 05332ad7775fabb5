"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/oracle.cpp header).

ctypes wrapper around liboracle.so, the plain CPU reference of the SVFusion hot path.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this module;
the product package paper_2601_08528_b200 never does (and fails loudly without its CUDA library).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
SENT = 0xFFFFFFFF
_lib = None


def compile_lib(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", src, "-o", _SO])
    return _SO


def lib():
    global _lib
    if _lib is None:
        compile_lib()
        L = ctypes.CDLL(_SO)
        P, I64, I, U64, F = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_float
        L.orc_splitmix64.restype, L.orc_splitmix64.argtypes = U64, [U64]
        L.orc_affine_params.restype, L.orc_affine_params.argtypes = None, [U64, U64, U64, P, P]
        L.orc_dist.restype, L.orc_dist.argtypes = F, [P, P, I, I]
        L.orc_bf_knn.argtypes = [P, I64, I, I, P, P, I64, I, P, P, I]
        L.orc_graph_search.argtypes = [P, I, I, P, I, P, I64, P, I64, P, I, I, I, I, I, U64, I, P, P, P, I]
        L.orc_graph_search_from.argtypes = [P, I, I, P, I, P, I64, P, P, I, I, I, I, I, P, P, P]
        L.orc_link_candidates.argtypes = [P, P, P, I, I, I64, I64, P, P, I, I]
        L.orc_insert.argtypes = [P, I, I, P, P, P, I, I, I64, I64, I, I, I, I, I, U64, I]
        L.orc_build.argtypes = [P, I64, I, I, I, I, I, I, I, I, I, I, U64, P, P, I]
        L.orc_merge_topk.argtypes = [P, P, I, I64, I, P, P]
        L.orc_consolidate.argtypes = [P, I, I, P, P, P, I, I, I64, P]
        L.orc_repair.argtypes = [P, I, I, P, P, P, I, I, I64, I, ctypes.c_double, I, P, P]
        L.orc_repair_mode.argtypes = [P, I, I, P, P, P, I, I, I64, I, ctypes.c_double, I, I, P, P]
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _u32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.uint32)


def default_threads() -> int:
    return os.cpu_count() or 1


def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(x))


def affine_params(seed: int, qidx: int, n: int):
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    lib().orc_affine_params(seed, qidx, n, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def dist(q, x, metric: int = 0) -> float:
    q, x = _f32(q), _f32(x)
    return float(lib().orc_dist(_p(q), _p(x), q.shape[-1], metric))


def bf_knn(X, Q, k: int, metric: int = 0, tomb=None, threads: Optional[int] = None):
    """O1: exact k-NN over the live rows of X (ids, fp32 distances), ties -> lower id."""
    X, Q, tomb = _f32(X), _f32(Q), _u32(tomb)
    nq = Q.shape[0]
    ids = np.empty((nq, k), np.uint32)
    d = np.empty((nq, k), np.float32)
    rc = lib().orc_bf_knn(_p(X), X.shape[0], X.shape[1], metric, _p(tomb), _p(Q), nq, k, _p(ids), _p(d),
                          threads or default_threads())
    assert rc == 0
    return ids, d


def graph_search(X, graph, Q, k: int, L: int, p: int = 1, n_init: Optional[int] = None, max_iter: int = 0,
                 seed: int = 42, metric: int = 0, tomb=None, n_alloc: Optional[int] = None, qidx=None,
                 insert_mode: bool = False, threads: Optional[int] = None):
    """O2: batched greedy graph search; returns (ids, dists, counters[nq,3] = n_dist, n_exp, iters)."""
    X, Q, graph, tomb = _f32(X), _f32(Q), _u32(graph), _u32(tomb)
    nq, D = Q.shape
    R = graph.shape[1]
    n_alloc = graph.shape[0] if n_alloc is None else n_alloc
    n_out = L if insert_mode else k
    ids = np.empty((nq, n_out), np.uint32)
    d = np.empty((nq, n_out), np.float32)
    cnt = np.empty((nq, 3), np.int64)
    qi = None if qidx is None else np.ascontiguousarray(qidx, dtype=np.int64)
    rc = lib().orc_graph_search(_p(X), D, metric, _p(graph), R, _p(tomb), n_alloc, _p(Q), nq, _p(qi), k, L, p,
                                n_init or L, max_iter, seed, int(insert_mode), _p(ids), _p(d), _p(cnt),
                                threads or default_threads())
    assert rc == 0
    return ids, d, cnt


def graph_search_from(X, graph, q, init_ids, k: int, L: int, p: int = 1, max_iter: int = 0, metric: int = 0,
                      tomb=None, n_alloc: Optional[int] = None):
    X, q, graph, tomb = _f32(X), _f32(q), _u32(graph), _u32(tomb)
    init = _u32(init_ids)
    ids = np.empty(k, np.uint32)
    d = np.empty(k, np.float32)
    cnt = np.empty(3, np.int64)
    n_alloc = graph.shape[0] if n_alloc is None else n_alloc
    lib().orc_graph_search_from(_p(X), X.shape[1], metric, _p(graph), graph.shape[1], _p(tomb), n_alloc, _p(q),
                                _p(init), len(init), k, L, p, max_iter, _p(ids), _p(d), _p(cnt))
    return ids, d, cnt


def link_candidates(graph, edge_dist, first: int, cand_ids, cand_d, P: int, tomb=None,
                    threads: Optional[int] = None):
    """O3 (ii)+(iii) in place on copies; returns (graph, edge_dist)."""
    graph = np.array(graph, dtype=np.uint32, copy=True, order="C")
    edge_dist = np.array(edge_dist, dtype=np.float32, copy=True, order="C")
    cid, cd, tomb = _u32(cand_ids), _f32(cand_d), _u32(tomb)
    rc = lib().orc_link_candidates(_p(graph), _p(edge_dist), _p(tomb), graph.shape[1], P, first, cid.shape[0],
                                   _p(cid), _p(cd), cid.shape[1], threads or default_threads())
    if rc != 0:
        raise ValueError("orc_link_candidates rejected its input")
    return graph, edge_dist


def insert(X, graph, edge_dist, n_alloc: int, n_new: int, P: int, L_ins: int = 128, B_ins: int = 4096,
           p: int = 1, n_init: Optional[int] = None, max_iter: int = 0, seed: int = 42, metric: int = 0,
           tomb=None, threads: Optional[int] = None):
    """O3 on copies of (graph, edge_dist) sized to the capacity; X holds rows for ids < n_alloc + n_new."""
    X, tomb = _f32(X), _u32(tomb)
    graph = np.array(graph, dtype=np.uint32, copy=True, order="C")
    edge_dist = np.array(edge_dist, dtype=np.float32, copy=True, order="C")
    rc = lib().orc_insert(_p(X), X.shape[1], metric, _p(graph), _p(edge_dist), _p(tomb), graph.shape[1], P,
                          n_alloc, n_new, L_ins, B_ins, p, n_init or L_ins, max_iter, seed,
                          threads or default_threads())
    assert rc == 0
    return graph, edge_dist


def build(X, R: int, P: Optional[int] = None, L_ins: int = 128, B_ins: int = 4096, seed_size: int = 4096,
          p: int = 1, n_init: Optional[int] = None, max_iter: int = 0, seed: int = 42, metric: int = 0,
          threads: Optional[int] = None):
    """O5: exact R-NN seed + O3 growth; returns (graph uint32[n][R], edge_dist f32[n][R])."""
    X = _f32(X)
    n, D = X.shape
    P = R // 2 if P is None else P
    graph = np.empty((n, R), np.uint32)
    edge_dist = np.empty((n, R), np.float32)
    rc = lib().orc_build(_p(X), n, D, metric, R, P, L_ins, B_ins, seed_size, p, n_init or L_ins, max_iter, seed,
                         _p(graph), _p(edge_dist), threads or default_threads())
    assert rc == 0
    return graph, edge_dist


def repair(X, graph, edge_dist, tomb, c: int = 8, threshold: float = 0.5, metric: int = 0,
           n_alloc: Optional[int] = None, mode: int = 1, P: Optional[int] = None, cap: int = 128):
    """NEXT-1 localized repair on copies; returns (graph, edge_dist, n_repaired, hist[5]).
    mode 1 = reading R1' (insertion's detour selection over the union's `cap` nearest; the product's rule),
    mode 0 = R1 (the R nearest of the union; experiment hook)."""
    X, tomb = _f32(X), _u32(tomb)
    graph = np.array(graph, dtype=np.uint32, copy=True, order="C")
    edge_dist = np.array(edge_dist, dtype=np.float32, copy=True, order="C")
    n_alloc = graph.shape[0] if n_alloc is None else n_alloc
    R = graph.shape[1]
    nrep = ctypes.c_int64()
    hist = np.zeros(5, np.int64)
    lib().orc_repair_mode(_p(X), X.shape[1], metric, _p(graph), _p(edge_dist), _p(tomb), R,
                          R // 2 if P is None else P, n_alloc, c, threshold, mode, cap, ctypes.byref(nrep), _p(hist))
    return graph, edge_dist, nrep.value, hist


def consolidate(X, graph, edge_dist, tomb, metric: int = 0, n_alloc: Optional[int] = None, P: Optional[int] = None):
    """NEXT-4 global consolidation ("aggregating candidates from the outgoing neighbors of deleted
    vertices"; reading C2): every live row with a tombstoned entry keeps its live entries in place and refills its
    vacancies from the live members of the deleted neighbours' lists (a deleted prefix slot from its own deleted
    neighbour's list, the tail vacancies by the nearest of the rest).  Returns (graph, edge_dist, n_rewritten)."""
    X, tomb = _f32(X), _u32(tomb)
    graph = np.array(graph, dtype=np.uint32, copy=True, order="C")
    edge_dist = np.array(edge_dist, dtype=np.float32, copy=True, order="C")
    n_alloc = graph.shape[0] if n_alloc is None else n_alloc
    R = graph.shape[1]
    n = ctypes.c_int64()
    rc = lib().orc_consolidate(_p(X), X.shape[1], metric, _p(graph), _p(edge_dist), _p(tomb), R,
                               R // 2 if P is None else P, n_alloc, ctypes.byref(n))
    assert rc == 0
    return graph, edge_dist, n.value


def delete(tomb, ids, n_alloc: int):
    """O4 lazy deletion: set the tombstone bit of each id on a copy of the bitset.  Idempotent.
    Returns (tomb, n_newly_deleted); raises KeyError (nothing deleted) if any id >= n_alloc."""
    t = np.array(tomb, dtype=np.uint32, copy=True)
    ids = [int(i) for i in np.asarray(ids).ravel()]
    if any(i < 0 or i >= n_alloc for i in ids):
        raise KeyError("delete of an id >= n_alloc")
    newly = 0
    for i in ids:
        w, b = i >> 5, i & 31
        if not (int(t[w]) >> b) & 1:
            t[w] = np.uint32(int(t[w]) | (1 << b))
            newly += 1
    return t, newly


def merge_topk(ids, d):
    """O6: ids/d of shape [G][nq][k] (global ids) -> first k by key per query."""
    ids, d = _u32(ids), _f32(d)
    G, nq, k = ids.shape
    oi = np.empty((nq, k), np.uint32)
    od = np.empty((nq, k), np.float32)
    lib().orc_merge_topk(_p(ids), _p(d), G, nq, k, _p(oi), _p(od))
    return oi, od


# ---- O7: recall@k ---------------------------------------------------------------------
def recall_ids(res, gt, k: int) -> float:
    """id-based: |res[:k] ∩ gt[:k]| / k averaged over queries."""
    res, gt = np.asarray(res)[:, :k], np.asarray(gt)[:, :k]
    hits = sum(len(set(r.tolist()) & set(g.tolist()) - {SENT}) for r, g in zip(res, gt))
    return hits / (k * res.shape[0])


def recall_tie_aware(res_d, gt_d, k: int, rel: float = 1e-5) -> float:
    """tie-aware: count result i if its exact distance <= the k-th true distance * (1 + rel) (+abs slack)."""
    res_d, gt_d = np.asarray(res_d, np.float64)[:, :k], np.asarray(gt_d, np.float64)[:, :k]
    kth = gt_d[:, k - 1:k]
    thr = kth + np.abs(kth) * rel + 1e-30
    return float(np.mean(res_d <= thr))
