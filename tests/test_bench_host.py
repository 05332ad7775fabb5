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
