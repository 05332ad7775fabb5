"""Streaming operation traces (paper §6.1 workloads).  Operation sequencing only:
each step lists dataset rows to insert, dataset rows to delete, and whether to evaluate search.

  sliding_window    T_max segments; step t inserts segment t, from t > T_max/2 deletes segment t - T_max/2
  expiration_time   each row gets a lifetime of 10 / 50 / 100 steps in a 10:2:1 ratio; step t inserts 1/T_max of
                    the rows and deletes the rows whose lifetime ended
  clustered         rows grouped into `n_clusters` clusters (k-means on a sample, a few Lloyd rounds); `rounds`
                    rounds, each inserting one more slice of every cluster, then deleting a random half of what is
                    live in every cluster
  insert_heavy      start with `n0` rows, then steps of 90% inserts / 10% searches until all rows are in
"""
from __future__ import annotations

import numpy as np


def _rng(seed):
    return np.random.default_rng(np.random.PCG64(seed))


def sliding_window(n: int, t_max: int = 200):
    seg = np.array_split(np.arange(n), t_max)
    steps = []
    for t in range(t_max):
        dele = seg[t - t_max // 2] if t >= t_max // 2 else np.empty(0, np.int64)
        steps.append({"insert": seg[t], "delete": dele, "search": t >= t_max // 2})
    return steps


def expiration_time(n: int, t_max: int = 200, seed: int = 7):
    g = _rng(seed)
    life = g.choice(np.array([10, 50, 100]), size=n, p=np.array([10, 2, 1]) / 13.0)
    seg = np.array_split(np.arange(n), t_max)
    born = np.empty(n, np.int64)
    for t, s in enumerate(seg):
        born[s] = t
    death = born + life
    steps = []
    for t in range(t_max):
        steps.append({"insert": seg[t], "delete": np.flatnonzero(death == t), "search": t >= 10})
    return steps


def kmeans_labels(X: np.ndarray, k: int = 64, iters: int = 5, sample: int = 100_000, seed: int = 3) -> np.ndarray:
    """Plain Lloyd iterations on a sample (workload partitioning only), then nearest-centroid labels for all rows."""
    g = _rng(seed)
    S = X[g.choice(len(X), size=min(sample, len(X)), replace=False)].astype(np.float32)
    C = S[g.choice(len(S), size=k, replace=False)].copy()
    for _ in range(iters):
        lab = np.argmin(-2 * S @ C.T + (C * C).sum(1)[None, :], axis=1)
        for c in range(k):
            m = lab == c
            if m.any():
                C[c] = S[m].mean(0)
    out = np.empty(len(X), np.int64)
    for i in range(0, len(X), 1 << 16):
        B = X[i:i + (1 << 16)]
        out[i:i + len(B)] = np.argmin(-2 * B @ C.T + (C * C).sum(1)[None, :], axis=1)
    return out


def clustered(labels: np.ndarray, rounds: int = 5, seed: int = 11):
    g = _rng(seed)
    k = int(labels.max()) + 1
    members = [g.permutation(np.flatnonzero(labels == c)) for c in range(k)]
    slices = [np.array_split(m, rounds) for m in members]
    live = [np.empty(0, np.int64) for _ in range(k)]
    steps = []
    for r in range(rounds):
        for c in range(k):  # insertion phase, cluster by cluster
            live[c] = np.concatenate([live[c], slices[c][r]])
            steps.append({"insert": slices[c][r], "delete": np.empty(0, np.int64), "search": False})
        steps[-1]["search"] = True
        for c in range(k):  # deletion phase, cluster by cluster
            drop = g.choice(live[c], size=len(live[c]) // 2, replace=False) if len(live[c]) else live[c]
            live[c] = np.setdiff1d(live[c], drop)
            steps.append({"insert": np.empty(0, np.int64), "delete": drop, "search": False})
        steps[-1]["search"] = True
    return steps


def insert_heavy(n: int, n0: int, steps: int = 100, seed: int = 13):
    rest = np.arange(n0, n)
    chunks = np.array_split(rest, steps)
    out = [{"insert": np.arange(n0), "delete": np.empty(0, np.int64), "search": True}]
    for i, ch in enumerate(chunks):
        out.append({"insert": ch, "delete": np.empty(0, np.int64), "search": (i % 10) == 9})
    return out
