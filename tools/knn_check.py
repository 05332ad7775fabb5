"""Quick GPU check + timing of the exact-kNN engines (tcgen05 TF32 + re-rank vs FFMA tiles) against the oracle.
Usage: python tools/knn_check.py [--n N] [--nq Q] [--k K] [--float]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2601_08528_b200 as svf  # noqa: E402
from workloads import GLM, random_graph  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=5000)
    ap.add_argument("--nq", type=int, default=300)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--float", action="store_true")
    ap.add_argument("--check", type=int, default=200, help="queries checked against the oracle")
    a = ap.parse_args()
    gen = GLM(dim=a.dim, ell=32, s=1.0, m=0.0, sigma=0.05, normalize=True) if a.float else \
        GLM(dim=a.dim, ell=32, integer=True)
    X = gen.rows(1, 1, 0, a.n)
    Q = gen.rows(1, 2, 0, a.nq)
    idx = svf.Index.from_state(X, random_graph(min(a.n, 2000), 4, seed=1) if False else np.full((a.n, 4), 0xFFFFFFFF, np.uint32))
    Qd = torch.from_numpy(Q).cuda()
    res = {}
    for mode in (0, 1):
        idx.set_knn_mode(mode)
        ids, d = idx.knn_exact(Qd, a.k)
        torch.cuda.synchronize()
        t = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ids, d = idx.knn_exact(Qd, a.k)
            e1.record()
            torch.cuda.synchronize()
            t.append(e0.elapsed_time(e1))
        ms = min(t)
        tf = 2.0 * a.nq * a.n * a.dim / (ms * 1e-3) / 1e12
        res[mode] = (ids.cpu().numpy().view(np.uint32), d.cpu().numpy())
        print(f"mode {mode} ({'tcgen05' if mode == 0 else 'ffma'}): {ms:.3f} ms  {tf:.1f} TFLOP/s  stats {idx.knn_stats()}",
              flush=True)
    m = min(a.check, a.nq)
    ri, rd = oracle.bf_knn(X, Q[:m], a.k)
    for mode in (0, 1):
        ids, d = res[mode]
        same = np.mean(ids[:m] == ri)
        derr = np.max(np.abs(d[:m] - rd) / np.maximum(np.abs(rd), 1e-30))
        print(f"mode {mode}: id agreement {same:.5f}  max rel dist err {derr:.2e}  bit-exact {np.array_equal(ids[:m], ri) and np.array_equal(d[:m], rd)}")


if __name__ == "__main__":
    main()
