"""ctypes declarations of include/svf.h.  Loading fails loudly if libsvf.so is missing: there is no CPU path."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SVF_LIB selects a tuning variant built by build_lib.build(out=..., extra=...) (experiments only)
LIB_PATH = os.environ.get("SVF_LIB") or os.path.join(HERE, "libsvf.so")

SVF_OK, SVF_ERR_INVALID, SVF_ERR_CAPACITY, SVF_ERR_NOT_FOUND = 0, 1, 2, 3
SVF_ERR_CUDA, SVF_ERR_OOM, SVF_ERR_NCCL, SVF_ERR_POISONED = 4, 5, 6, 7
STATUS_NAMES = {0: "OK", 1: "INVALID", 2: "CAPACITY", 3: "NOT_FOUND", 4: "CUDA", 5: "OOM", 6: "NCCL", 7: "POISONED"}
SENTINEL = 0xFFFFFFFF

EXPORTED = ["svf_default_params", "svf_build", "svf_search", "svf_insert", "svf_delete", "svf_knn_exact",
            "svf_merge_topk", "svf_shard_premerge", "svf_merge_pairs", "svf_export", "svf_import", "svf_link_candidates", "svf_set_search_params",
            "svf_last_search_counters", "svf_set_knn_mode", "svf_knn_stats", "svf_set_warps_per_query", "svf_set_search_handoff", "svf_set_trace", "svf_read_trace", "svf_repair", "svf_consolidate", "svf_set_consolidation", "svf_consolidation_stats", "svf_profile", "svf_profile_read", "svf_info", "svf_destroy",
            "svf_last_error"]


class SvfParams(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32), ("degree", ctypes.c_int32), ("metric", ctypes.c_int32),
        ("capacity", ctypes.c_int64), ("search_width", ctypes.c_int32), ("n_init", ctypes.c_int32),
        ("max_iter", ctypes.c_int32), ("insert_itopk", ctypes.c_int32), ("protect_prefix", ctypes.c_int32),
        ("insert_batch", ctypes.c_int32), ("seed_size", ctypes.c_int32), ("hash_bits", ctypes.c_int32),
        ("seed", ctypes.c_uint64), ("device", ctypes.c_int32), ("build_itopk", ctypes.c_int32),
    ]


class SvfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"svf status {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (the CUDA library is the only implementation; there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "svf_default_params": (None, [ctypes.POINTER(SvfParams), I32, I32]),
        "svf_build": (ctypes.c_int, [ctypes.POINTER(SvfParams), P, I64, P, PP]),
        "svf_search": (ctypes.c_int, [P, P, I64, I32, I32, P, P, P]),
        "svf_insert": (ctypes.c_int, [P, P, I64, P, P]),
        "svf_delete": (ctypes.c_int, [P, P, I64, ctypes.POINTER(I64), P]),
        "svf_knn_exact": (ctypes.c_int, [P, P, I64, I32, P, P, P]),
        "svf_merge_topk": (ctypes.c_int, [P, P, I32, I64, I32, P, P, P]),
        "svf_shard_premerge": (ctypes.c_int, [P, P, I32, I64, I32, ctypes.c_uint32, P, P, P]),
        "svf_merge_pairs": (ctypes.c_int, [P, I32, I64, I32, P, P, P]),
        "svf_export": (ctypes.c_int, [P, P, P, P, P, ctypes.POINTER(I64)]),
        "svf_import": (ctypes.c_int, [ctypes.POINTER(SvfParams), P, P, P, P, I64, PP]),
        "svf_link_candidates": (ctypes.c_int, [P, P, P, P, I64, I32, P]),
        "svf_set_search_params": (ctypes.c_int, [P, I32, I32, I32, I32]),
        "svf_last_search_counters": (ctypes.c_int, [P, ctypes.POINTER(U64)]),
        "svf_set_knn_mode": (ctypes.c_int, [P, I32]),
        "svf_set_warps_per_query": (ctypes.c_int, [P, I32]),
        "svf_set_search_handoff": (ctypes.c_int, [P, I32]),
        "svf_set_trace": (ctypes.c_int, [P, I32]),
        "svf_read_trace": (ctypes.c_int, [P, P, I64, P]),
        "svf_repair": (ctypes.c_int, [P, I32, ctypes.c_double, ctypes.POINTER(I64), ctypes.POINTER(U64), P]),
        "svf_knn_stats": (ctypes.c_int, [P, ctypes.POINTER(U64)]),
        "svf_consolidate": (ctypes.c_int, [P, ctypes.POINTER(I64), P]),
        "svf_set_consolidation": (ctypes.c_int, [P, ctypes.c_double]),
        "svf_consolidation_stats": (ctypes.c_int, [P, ctypes.POINTER(I64)]),
        "svf_profile": (ctypes.c_int, [P, I32]),
        "svf_profile_read": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64)]),
        "svf_info": (ctypes.c_int, [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "svf_destroy": (ctypes.c_int, [P]),
        "svf_last_error": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    _lib = L
    return L


def check(status: int) -> None:
    if status != SVF_OK:
        raise SvfError(status, lib().svf_last_error().decode(errors="replace"))
