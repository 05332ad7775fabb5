"""The streaming trace generators (workloads/traces.py, paper P:L698-711) produce well-formed operation streams."""
import numpy as np

from workloads import GLM, traces


def _replay(steps, n):
    inserted = np.zeros(n, bool)
    deleted = np.zeros(n, bool)
    for s in steps:
        ins, dele = np.asarray(s["insert"]), np.asarray(s["delete"])
        assert not inserted[ins].any()                     # each row inserted once
        inserted[ins] = True
        assert inserted[dele].all() and not deleted[dele].any()   # delete only live rows, once
        deleted[dele] = True
    return inserted, deleted


def test_sliding_window():
    n, T = 10_000, 200
    steps = traces.sliding_window(n, T)
    ins, dele = _replay(steps, n)
    assert ins.all() and dele.sum() == sum(len(s) for s in np.array_split(np.arange(n), T)[: T // 2])
    assert sum(s["search"] for s in steps) == T // 2


def test_expiration_time_ratio_and_order():
    n, T = 26_000, 200
    steps = traces.expiration_time(n, T)
    ins, dele = _replay(steps, n)
    assert ins.all()
    # lifetimes 10:2:1 -> about 10/13 of early rows expire within 10 steps
    early = np.arange(n // T * 50)
    died_by = {}
    for t, s in enumerate(steps):
        for r in s["delete"]:
            died_by[int(r)] = t
    short = np.mean([died_by.get(int(r), 10**9) - r // (n // T) == 10 for r in early])
    assert abs(short - 10 / 13) < 0.03


def test_clustered():
    X = GLM(dim=16, ell=6).rows(1, 1, 0, 20_000)
    lab = traces.kmeans_labels(X, k=16, iters=3, sample=5000)
    assert lab.min() >= 0 and lab.max() < 16 and len(np.unique(lab)) > 8
    steps = traces.clustered(lab, rounds=5)
    ins, dele = _replay(steps, len(X))
    assert ins.all() and 0 < dele.sum() < len(X)


def test_insert_heavy():
    steps = traces.insert_heavy(10_000, 1_000, 90)
    ins, dele = _replay(steps, 10_000)
    assert ins.all() and not dele.any()
    assert abs(np.mean([s["search"] for s in steps[1:]]) - 0.1) < 0.02
