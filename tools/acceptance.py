"""Generator acceptance checks of SURVEY §8(d) ("run before any performance claim, on C1 and on a 1M slice") and the
G-LM calibration pass they call for, plus the G-CL second curve on C2:
  * BFS from node 0 over out-edges reaches every live node;
  * query MLE-LID (Levina-Bickel, k = 20, Euclidean distances) lies in 12-20;
  * on G-LM, recall@10 at itopk 16 is BELOW 0.95 (the itopk sweep is informative) and >= 0.95 is reachable at
    itopk <= 128.
For each latent dimension ell of --ells (C2's generator otherwise unchanged) the tool builds the C2-shaped index the
way bench.py does (L_build 256), computes exact ground truth (svf_knn_exact), and reports the uncapped itopk sweep.

  python tools/acceptance.py --ells 32,40,48 [--gcl] [--out profiles/r02_acceptance.json]
"""
import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from workloads import CONFIGS, GCL  # noqa: E402

SENT = 0xFFFFFFFF
SWEEP = [10, 12, 14, 16, 20, 24, 32, 48, 64, 96, 128]


def bfs_reach(graph: np.ndarray) -> float:
    n = len(graph)
    seen = np.zeros(n, bool)
    seen[0] = True
    front = np.array([0], np.int64)
    while len(front):
        nb = graph[front].ravel()
        nb = nb[nb != SENT].astype(np.int64)
        nb = np.unique(nb[~seen[nb]])
        seen[nb] = True
        front = nb
    return float(seen.mean())


def mle_lid(d_sq: np.ndarray) -> float:
    """Levina-Bickel MLE with k = d_sq.shape[1] neighbours, from SQUARED distances (ln r_i/r_k = ln(d_i/d_k)/2)."""
    d = np.maximum(d_sq.astype(np.float64), 1e-30)
    lr = 0.5 * np.log(d[:, :-1] / d[:, -1:])
    est = -1.0 / lr.mean(axis=1)
    return float(np.mean(est[np.isfinite(est)]))


def recall(ids, gt, k=10):
    ids, gt = np.asarray(ids)[:, :k], np.asarray(gt)[:, :k]
    return float((ids[:, :, None] == gt[:, None, :]).any(axis=2).mean())


def evaluate(gen, n: int, nq: int, build_L: int, label: str) -> dict:
    dev = torch.device("cuda:0")
    t0 = time.time()
    X = gen.rows(1, 1, 0, n)
    Q = gen.rows(1, 2, 0, nq)
    idx = svf.Index.build(torch.from_numpy(X).to(dev), degree=64, build_itopk=build_L)
    Qd = torch.from_numpy(Q).to(dev)
    gi, gd = idx.knn_exact(Qd, 20)
    gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    sweep = []
    for L in SWEEP:
        ids, _ = idx.search(Qd, 10, L)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        idx.search(Qd, 10, L)
        e1.record()
        torch.cuda.synchronize()
        sweep.append({"itopk": L, "recall": round(recall(ids.cpu().numpy(), gi), 4),
                      "ms": round(e0.elapsed_time(e1), 3)})
    reach = bfs_reach(idx.export()["graph"])
    lid = mle_lid(gd)
    r16 = next(s["recall"] for s in sweep if s["itopk"] == 16)
    first = next((s["itopk"] for s in sweep if s["recall"] >= 0.95), None)
    row = {"data": label, "n": n, "L_build": build_L, "bfs_reach_from_0": reach, "query_mle_lid_k20": round(lid, 2),
           "recall_at_itopk16": r16, "lowest_itopk_at_0.95": first,
           "checks": {"reachable": reach == 1.0, "lid_in_12_20": 12.0 <= lid <= 20.0,
                      "sweep_informative": r16 < 0.95, "0.95_reachable_by_128": first is not None and first <= 128},
           "sweep": sweep, "s": round(time.time() - t0, 1)}
    idx.close()
    print(json.dumps(row), flush=True)
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ells", default="32,40,48")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--build-itopk", type=int, default=256)
    ap.add_argument("--gcl", action="store_true", help="also the G-CL stress curve (1024 clusters, SURVEY §8(d) C2)")
    ap.add_argument("--c1", action="store_true", help="also C1 (10K rows) at its own build")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    base = CONFIGS["C2"]["gen"]
    rows = []
    for ell in [int(x) for x in a.ells.split(",") if x]:
        rows.append(evaluate(dataclasses.replace(base, ell=ell), a.n, a.nq, a.build_itopk, f"G-LM ell={ell}"))
    if a.c1:
        rows.append(evaluate(CONFIGS["C1"]["gen"], 10_000, 100, 0, "C1 G-LM ell=32 (10K)"))
    if a.gcl:
        rows.append(evaluate(GCL(dim=128, n_clusters=1024), a.n, a.nq, a.build_itopk, "G-CL 1024 clusters"))
    if a.out:
        json.dump({"note": "SURVEY §8(d) generator acceptance checks + calibration; C2 shape (R=64, 10K queries)",
                   "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
