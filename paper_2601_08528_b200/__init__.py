"""B200-native hot path of SVFusion (arXiv 2601.08528): batched graph ANNS search / insert / delete on sm_100a.

Thin Python binding over libsvf.so (include/svf.h): argument marshalling only.  PyTorch supplies device memory
and streams; every step of the method runs in the CUDA kernels under csrc/.  Inputs may be torch tensors (CUDA
or CPU) or numpy arrays; outputs follow the query's placement (CUDA tensor in -> CUDA tensor out, else numpy).
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from ._lib import SENTINEL, SvfError, SvfParams, check, lib  # noqa: F401

try:  # torch is plumbing only (device memory, streams, process groups)
    import torch
except Exception:  # pragma: no cover
    torch = None

__all__ = ["Index", "merge_topk", "shard_premerge", "merge_pairs", "SvfError", "SENTINEL", "default_params"]


def _is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def _pinned(t) -> bool:
    try:
        return bool(t.is_pinned())
    except Exception:
        return False


def _prep(x, np_dtype, torch_dtype):
    """-> (pointer, keepalive, device or None or "pinned")"""
    if _is_torch(x):
        t = x.detach()
        if t.dtype != torch_dtype:
            t = t.to(torch_dtype)
        t = t.contiguous()
        where = t.device if t.is_cuda else ("pinned" if _pinned(t) else None)
        return t.data_ptr(), t, where
    a = np.ascontiguousarray(x, dtype=np_dtype)
    return a.ctypes.data, a, None


def _stream(device) -> Optional[int]:
    if device is None or torch is None:
        return None
    if device == "pinned":
        return torch.cuda.current_stream().cuda_stream
    return torch.cuda.current_stream(device).cuda_stream


def _cur_stream() -> Optional[int]:
    """The current CUDA stream (for calls without a tensor argument), or the default stream without torch."""
    if torch is None or not torch.cuda.is_available():
        return None
    return torch.cuda.current_stream().cuda_stream


def _empty(shape, np_dtype, torch_dtype, device):
    if device == "pinned":  # pinned host in -> pinned host out (the end-to-end path)
        t = torch.empty(shape, dtype=torch_dtype, pin_memory=True)
        return t.data_ptr(), t
    if device is not None:
        t = torch.empty(shape, dtype=torch_dtype, device=device)
        return t.data_ptr(), t
    a = np.empty(shape, dtype=np_dtype)
    return a.ctypes.data, a


def default_params(dim: int, degree: int, **kw) -> SvfParams:
    p = SvfParams()
    lib().svf_default_params(ctypes.byref(p), dim, degree)
    metric = kw.pop("metric", 0)
    p.metric = {"l2": 0, "ip": 1}.get(metric, metric) if isinstance(metric, str) else int(metric)
    for k, v in kw.items():
        if not hasattr(p, k):
            raise TypeError(f"unknown svf_params field {k!r}")
        setattr(p, k, v)
    return p


class Index:
    """An SVFusion-style dynamic graph index resident in one GPU's HBM (svf_index*)."""

    def __init__(self, handle: int, params: SvfParams):
        self._h = ctypes.c_void_p(handle)
        self.params = params
        self.device = params.device

    # ---- construction -------------------------------------------------------------------------------------------
    @classmethod
    def build(cls, X, degree: int, capacity: Optional[int] = None, **kw) -> "Index":
        """Build(X_init): exact R-NN seed + batched-insert growth (svf_build)."""
        ptr, keep, dev = _prep(X, np.float32, torch.float32 if torch else None)
        n, dim = int(keep.shape[0]), int(keep.shape[1])
        if dev is not None and dev != "pinned":
            kw.setdefault("device", dev.index or 0)
        p = default_params(dim, degree, capacity=capacity or n, **kw)
        h = ctypes.c_void_p()
        check(lib().svf_build(ctypes.byref(p), ptr, n, _stream(dev), ctypes.byref(h)))
        return cls(h.value, p)

    @classmethod
    def from_state(cls, vec, graph, edge_dist=None, tomb=None, capacity: Optional[int] = None, **kw) -> "Index":
        """svf_import: an index from given (vec, graph, edge_dist, tomb) state (tests / bench)."""
        v = np.ascontiguousarray(vec, dtype=np.float32)
        g = np.ascontiguousarray(graph, dtype=np.uint32)
        e = None if edge_dist is None else np.ascontiguousarray(edge_dist, dtype=np.float32)
        t = None if tomb is None else np.ascontiguousarray(tomb, dtype=np.uint32)
        n = v.shape[0]
        p = default_params(v.shape[1], g.shape[1], capacity=capacity or n, **kw)
        h = ctypes.c_void_p()
        check(lib().svf_import(ctypes.byref(p), v.ctypes.data, g.ctypes.data, None if e is None else e.ctypes.data,
                               None if t is None else t.ctypes.data, n, ctypes.byref(h)))
        return cls(h.value, p)

    # ---- operations ---------------------------------------------------------------------------------------------
    def search(self, Q, k: int, itopk: int):
        """Search(q, k) for a batch (svf_search; Algorithm 1).  Returns (ids uint32 [nq,k], dists f32 [nq,k])."""
        qp, qk, dev = _prep(Q, np.float32, torch.float32 if torch else None)
        nq = int(qk.shape[0])
        ip, ids = _empty((nq, k), np.uint32, torch.int32 if torch else None, dev)
        dp, d = _empty((nq, k), np.float32, torch.float32 if torch else None, dev)
        check(lib().svf_search(self._h, qp, nq, k, itopk, ip, dp, _stream(dev)))
        return ids, d

    def search_into(self, Q, k: int, itopk: int, out_ids, out_dists):
        """svf_search into caller-owned CUDA tensors (no allocation: safe inside CUDA-graph capture)."""
        qp, qk, dev = _prep(Q, np.float32, torch.float32 if torch else None)
        check(lib().svf_search(self._h, qp, int(qk.shape[0]), k, itopk, out_ids.data_ptr(), out_dists.data_ptr(),
                               _stream(dev)))
        return out_ids, out_dists

    def insert(self, X):
        """Insert(x) for a batch (svf_insert).  Returns the assigned ids (numpy uint32)."""
        xp, xk, dev = _prep(X, np.float32, torch.float32 if torch else None)
        n = int(xk.shape[0])
        out = np.empty(n, np.uint32)
        check(lib().svf_insert(self._h, xp, n, out.ctypes.data, _stream(dev)))
        return out

    def insert_async(self, X):
        """svf_insert without the id read-back: returns at once after enqueueing on the current stream, so an
        svf_search issued on another stream overlaps it on the GPU.  The ids are the next n in order
        (ids are library-assigned and monotone, I14), returned as numpy uint32 without synchronising."""
        xp, xk, dev = _prep(X, np.float32, torch.float32 if torch else None)
        n = int(xk.shape[0])
        first = self.info()["n_alloc"]
        check(lib().svf_insert(self._h, xp, n, None, _stream(dev)))
        return np.arange(first, first + n, dtype=np.uint32)

    def delete(self, ids) -> int:
        """Delete(x) for a batch of ids (svf_delete).  Returns the number newly deleted."""
        ptr, keep, dev = _prep(ids, np.uint32, torch.int32 if torch else None)
        n = int(keep.numel()) if _is_torch(keep) else int(keep.size)
        newly = ctypes.c_int64()
        check(lib().svf_delete(self._h, ptr, n, ctypes.byref(newly), _stream(dev)))
        return newly.value

    def repair(self, c: int = 8, threshold: float = 0.5) -> dict:
        """Localized topology-aware repair of severely affected vertices (svf_repair)."""
        n = ctypes.c_int64()
        hist = (ctypes.c_uint64 * 5)()
        check(lib().svf_repair(self._h, c, threshold, ctypes.byref(n), hist, _cur_stream()))
        return {"repaired": n.value, "hist": list(hist)}

    def consolidate(self) -> int:
        """Global consolidation (svf_consolidate): every live row with a deleted neighbour is rebuilt
        from all live members of its deleted neighbours' lists.  Returns the rows rewritten."""
        n = ctypes.c_int64()
        check(lib().svf_consolidate(self._h, ctypes.byref(n), _cur_stream()))
        return n.value

    def set_consolidation(self, ratio: float):
        """Consolidate automatically after a delete once the deletions since the last consolidation exceed
        `ratio` of the vertices live then ("e.g., 20%"); 0 = off."""
        check(lib().svf_set_consolidation(self._h, float(ratio)))

    def consolidation_stats(self) -> dict:
        out = (ctypes.c_int64 * 2)()
        check(lib().svf_consolidation_stats(self._h, out))
        return {"consolidations": out[0], "deleted_at_last": out[1]}

    def knn_exact(self, Q, k: int):
        """Exact k-NN over the live set (svf_knn_exact; ground truth)."""
        qp, qk, dev = _prep(Q, np.float32, torch.float32 if torch else None)
        nq = int(qk.shape[0])
        ip, ids = _empty((nq, k), np.uint32, torch.int32 if torch else None, dev)
        dp, d = _empty((nq, k), np.float32, torch.float32 if torch else None, dev)
        check(lib().svf_knn_exact(self._h, qp, nq, k, ip, dp, _stream(dev)))
        return ids, d

    def knn_exact_into(self, Q, k: int, out_ids, out_dists):
        """svf_knn_exact into caller-owned CUDA tensors."""
        qp, qk, dev = _prep(Q, np.float32, torch.float32 if torch else None)
        check(lib().svf_knn_exact(self._h, qp, int(qk.shape[0]), k, out_ids.data_ptr(), out_dists.data_ptr(),
                                  _stream(dev)))
        return out_ids, out_dists

    def link_candidates(self, cand_ids, cand_d, X=None):
        """TEST ENTRY (svf_link_candidates): steps (ii)+(iii) of insertion from given candidate lists."""
        ci = np.ascontiguousarray(cand_ids, dtype=np.uint32)
        cd = np.ascontiguousarray(cand_d, dtype=np.float32)
        xp = None
        if X is not None:
            xk = np.ascontiguousarray(X, dtype=np.float32)
            xp = xk.ctypes.data
        check(lib().svf_link_candidates(self._h, xp, ci.ctypes.data, cd.ctypes.data, ci.shape[0], ci.shape[1], None))

    def export(self) -> dict:
        n = self.info()["n_alloc"]
        D, R = self.params.dim, self.params.degree
        vec = np.empty((n, D), np.float32)
        graph = np.empty((n, R), np.uint32)
        ed = np.empty((n, R), np.float32)
        tomb = np.empty(((n + 31) // 32,), np.uint32)
        na = ctypes.c_int64()
        check(lib().svf_export(self._h, vec.ctypes.data, graph.ctypes.data, ed.ctypes.data, tomb.ctypes.data,
                               ctypes.byref(na)))
        return {"vec": vec, "graph": graph, "edge_dist": ed, "tomb": tomb, "n_alloc": na.value}

    def set_search_params(self, search_width: int = 1, n_init: int = 0, max_iter: int = 0, hash_bits: int = 0):
        check(lib().svf_set_search_params(self._h, search_width, n_init, max_iter, hash_bits))

    def last_search_counters(self) -> dict:
        out = (ctypes.c_uint64 * 5)()
        check(lib().svf_last_search_counters(self._h, out))
        return {"n_dist": out[0], "iters": out[1], "n_exp": out[2], "queries": out[3], "launches": out[4]}

    def set_warps_per_query(self, wpq: int):
        """1 or 2 warps per query (identical results), 0 = automatic."""
        check(lib().svf_set_warps_per_query(self._h, wpq))

    def set_search_handoff(self, pct: int):
        """Hand a one-warp batch's stragglers to a chained pair-mode grid once fewer than pct% of the warps are
        still searching (identical results); -1 = automatic, 0 = off."""
        check(lib().svf_set_search_handoff(self._h, pct))

    def set_trace(self, enable: bool):
        """Record a per-query timeline (start/end ns, SM, iterations) of later searches (diagnostics)."""
        check(lib().svf_set_trace(self._h, int(enable)))

    def read_trace(self, max_nq: int):
        """(start_ns, end_ns, sm, iterations, phase_cycles[n, 5]) of the last traced search (<= max_nq queries)."""
        buf = np.zeros((max(max_nq, 1), 8), dtype=np.uint64)
        n = ctypes.c_int64(0)
        check(lib().svf_read_trace(self._h, buf.ctypes.data, buf.shape[0], ctypes.byref(n)))
        t = buf[: n.value]
        return (t[:, 0].astype(np.int64), t[:, 1].astype(np.int64), (t[:, 2] >> np.uint64(32)).astype(np.int64),
                (t[:, 2] & np.uint64(0xFFFFFFFF)).astype(np.int64), t[:, 3:8].astype(np.int64))

    def set_knn_mode(self, mode: int):
        """0 = tcgen05 TF32 scoring + exact re-rank (auto), 1 = FFMA tiles only."""
        check(lib().svf_set_knn_mode(self._h, mode))

    def knn_stats(self) -> dict:
        out = (ctypes.c_uint64 * 3)()
        check(lib().svf_knn_stats(self._h, out))
        return {"queries": out[0], "fallbacks": out[1], "tc_calls": out[2]}

    def profile(self, enable: bool = True):
        check(lib().svf_profile(self._h, int(enable)))

    def profile_read(self) -> dict:
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_int64 * 4)()
        check(lib().svf_profile_read(self._h, ms, cnt))
        names = ["search", "insert_search", "detour", "reverse"]
        return {n: (ms[i], cnt[i]) for i, n in enumerate(names)}

    def info(self) -> dict:
        a, d, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(lib().svf_info(self._h, ctypes.byref(a), ctypes.byref(d), ctypes.byref(c)))
        return {"n_alloc": a.value, "n_deleted": d.value, "capacity": c.value}

    def close(self):
        if self._h is not None and self._h.value:
            lib().svf_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def merge_topk(ids, dists):
    """K-M (svf_merge_topk): [G, nq, k] CUDA tensors of global ids / dists -> first k per query by (dist, id)."""
    if not (_is_torch(ids) and ids.is_cuda):
        raise TypeError("merge_topk takes CUDA tensors (the all-gather output)")
    G, nq, kk = ids.shape
    k = kk
    ids = ids.contiguous()
    dists = dists.to(torch.float32).contiguous()
    oi = torch.empty((nq, k), dtype=torch.int32, device=ids.device)
    od = torch.empty((nq, k), dtype=torch.float32, device=ids.device)
    check(lib().svf_merge_topk(ids.data_ptr(), dists.data_ptr(), G, nq, kk, oi.data_ptr(), od.data_ptr(),
                               _stream(ids.device)))
    return oi, od


def shard_premerge(ids, dists, n_logical: int, shards):
    """K-M pre-merge of a rank's shard results (svf_shard_premerge): ids/dists [n, nq, k] CUDA
    tensors of LOCAL ids from shards `shards` -> [nq, k] int64 packed pairs (dist bits << 32 | global id)."""
    n, nq, k = ids.shape
    sh = (ctypes.c_uint32 * n)(*[int(s) for s in shards])
    out = torch.empty((nq, k), dtype=torch.int64, device=ids.device)
    check(lib().svf_shard_premerge(ids.data_ptr(), dists.data_ptr(), n, nq, k, n_logical, sh, out.data_ptr(),
                                   _stream(ids.device)))
    return out


def merge_pairs(pairs):
    """K-M merge of G all-gathered pair lists (svf_merge_pairs): [G, nq, k] int64 CUDA tensor
    -> (ids int32 [nq, k], dists f32 [nq, k]), the first k by (dist, id)."""
    G, nq, k = pairs.shape
    pairs = pairs.contiguous()
    oi = torch.empty((nq, k), dtype=torch.int32, device=pairs.device)
    od = torch.empty((nq, k), dtype=torch.float32, device=pairs.device)
    check(lib().svf_merge_pairs(pairs.data_ptr(), G, nq, k, oi.data_ptr(), od.data_ptr(), _stream(pairs.device)))
    return oi, od
