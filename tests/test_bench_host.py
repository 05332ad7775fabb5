"""Host-side logic of bench.py (no GPU): the iteration-cap candidates and the per-config build/insert sizes."""
import importlib.util
import os

from workloads import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_mi_caps_descending_and_cover_fixed_sweep():
    b = _bench()
    for L in (10, 14, 32, 40, 192, 512):
        caps = b.mi_caps(L)
        assert caps == sorted(set(caps), reverse=True)          # strictly descending: the sweep stops at a miss
        assert set(b.MI_SWEEP) <= set(caps) and min(caps) >= 1
        assert max(caps) >= max(64, 3 * L - 1)                  # the first cap tried is loose for any pool size


def test_build_and_insert_sizes_valid():
    b = _bench()
    assert set(b.BUILD_ITOPK) <= set(CONFIGS)
    for name, L in b.BUILD_ITOPK.items():
        assert L == 0 or CONFIGS[name]["degree"] < L <= 512     # L_build 0 = insert_itopk; else > R, <= 512
    for name, L in b.INSERT_ITOPK.items():
        assert CONFIGS[name]["degree"] < L <= 512               # L_insert <= R would disable the detour pruning


def test_bench_recall_equals_the_oracles_pinned_definitions():
    """bench.py measures recall with its own copy (only its cpu_baseline leg may call the oracle); it must equal
    O7's pinned id-based and tie-aware recall on random inputs with ties, padding and negative (IP) distances."""
    import numpy as np

    import oracle

    b = _bench()
    rng = np.random.default_rng(0)
    for _ in range(20):
        nq, k = 7, 10
        gt = rng.integers(0, 30, size=(nq, k)).astype(np.uint32)
        res = rng.integers(0, 30, size=(nq, k)).astype(np.uint32)
        gd = np.sort(rng.integers(-5, 5, size=(nq, k)).astype(np.float32), axis=1)
        rd = np.sort(rng.integers(-5, 6, size=(nq, k)).astype(np.float32), axis=1)
        rd[0, -2:] = np.inf
        # the oracle's id recall counts set intersections: use distinct ids per row so both definitions apply
        gt = np.argsort(rng.random((nq, 30)), axis=1)[:, :k].astype(np.uint32)
        res = np.argsort(rng.random((nq, 30)), axis=1)[:, :k].astype(np.uint32)
        assert abs(b.recall_at_k(res, gt, k) - oracle.recall_ids(res, gt, k)) < 1e-12
        assert abs(b.recall_tie_aware(rd, gd, k) - oracle.recall_tie_aware(rd, gd, k)) < 1e-12


def test_bench_defaults_and_selection_seed():
    b = _bench()
    a = b.parse([])
    assert a.config == "C2" and a.gpus == 1 and a.steps >= 10 and a.warmup >= 3
    assert b.SELECT_SEED != 2                     # itopk / cap are chosen on a batch other than the timed one
    assert set(b.EXTRA_CONFIGS) <= set(CONFIGS) and "C2" not in b.EXTRA_CONFIGS
