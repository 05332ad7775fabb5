"""Streaming rounds on the GPU index (SURVEY §8(d) C3 / C4 shapes; paper workloads P:L698-711).

Each round: search the 10K-query batch (recall@10 vs exact ground truth over the live set, from svf_knn_exact),
insert `--ins` fresh vectors, delete `--del` ids (uniform live ids, or the oldest window for --sliding), and, with
--repair, run the localized repair.  Prints one JSON line per round and a summary.

  python tools/streaming.py --config C3 --n 10000000 --rounds 20 --repair
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from workloads import base_rows, config_spec, query_rows  # noqa: E402


def recall(ids, gt, k=10):
    ids, gt = ids[:, :k], gt[:, :k]
    return float((ids[:, :, None] == gt[:, None, :]).any(axis=2).sum()) / (k * ids.shape[0])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--ins", type=float, default=0.01, help="fraction of n inserted per round")
    ap.add_argument("--dele", type=float, default=0.01, help="fraction of n deleted per round")
    ap.add_argument("--sliding", action="store_true", help="delete the oldest live ids (sliding window)")
    ap.add_argument("--repair", action="store_true")
    ap.add_argument("--repair-threshold", type=float, default=0.5)
    ap.add_argument("--itopk", type=int, default=32)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    c = config_spec(a.config)
    n = a.n or c["n"]
    B_ins, B_del = int(n * a.ins), int(n * a.dele)
    dev = torch.device("cuda:0")
    t0 = time.time()
    X = torch.from_numpy(base_rows(a.config, 0, n)).to(dev)
    Q = torch.from_numpy(query_rows(a.config, a.nq)).to(dev)
    t_gen = time.time() - t0
    cap = n + B_ins * a.rounds
    torch.cuda.synchronize()
    t0 = time.time()
    idx = svf.Index.build(X, degree=c["degree"], metric=c["metric"], capacity=cap)
    torch.cuda.synchronize()
    t_build = time.time() - t0
    del X
    rng = np.random.default_rng(1000)
    alive = np.ones(cap, bool)
    alive[n:] = False
    n_alloc, oldest = n, 0
    log = []
    ev = lambda: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))  # noqa: E731
    for r in range(a.rounds + 1):
        rec = {"round": r, "live": int(alive[:n_alloc].sum())}
        e0, e1 = ev()
        e0.record()
        ids, _ = idx.search(Q, 10, a.itopk)
        e1.record()
        gi, _ = idx.knn_exact(Q, 10)
        torch.cuda.synchronize()
        rec["search_ms"] = round(e0.elapsed_time(e1), 3)
        rec["qps"] = round(a.nq / (e0.elapsed_time(e1) / 1e3))
        rec["recall"] = round(recall(ids.cpu().numpy(), gi.cpu().numpy()), 4)
        if r == a.rounds:
            log.append(rec)
            print(json.dumps(rec), flush=True)
            break
        newX = torch.from_numpy(base_rows(a.config, 100_000_000 + r * B_ins, B_ins, row_seed=1000 + r)).to(dev)
        e0, e1 = ev()
        e0.record()
        idx.insert(newX)
        e1.record()
        torch.cuda.synchronize()
        rec["insert_ms"] = round(e0.elapsed_time(e1), 3)
        rec["inserts_per_s"] = round(B_ins / (e0.elapsed_time(e1) / 1e3))
        alive[n_alloc:n_alloc + B_ins] = True
        n_alloc += B_ins
        if a.sliding:
            live_ids = np.flatnonzero(alive[:n_alloc])
            dels = live_ids[:B_del]
        else:
            dels = rng.choice(np.flatnonzero(alive[:n_alloc]), B_del, replace=False)
        alive[dels] = False
        e0, e1 = ev()
        e0.record()
        idx.delete(torch.from_numpy(dels.astype(np.int32)).to(dev))
        e1.record()
        torch.cuda.synchronize()
        rec["delete_ms"] = round(e0.elapsed_time(e1), 3)
        if a.repair:
            t1 = time.perf_counter()
            out = idx.repair(threshold=a.repair_threshold)
            rec["repair_ms"] = round((time.perf_counter() - t1) * 1e3, 3)
            rec["repaired"] = out["repaired"]
            rec["deleted_neighbour_hist"] = out["hist"]
        log.append(rec)
        print(json.dumps(rec), flush=True)
    summ = {"config": a.config, "n": n, "nq": a.nq, "itopk": a.itopk, "rounds": a.rounds, "B_ins": B_ins,
            "B_del": B_del, "sliding": a.sliding, "repair": a.repair, "repair_threshold": a.repair_threshold, "gen_s": round(t_gen, 2),
            "build_s": round(t_build, 2), "build_inserts_per_s": round(n / t_build),
            "recall_first": log[0]["recall"], "recall_last": log[-1]["recall"],
            "mean_inserts_per_s": round(float(np.mean([x["inserts_per_s"] for x in log if "inserts_per_s" in x]))),
            "mean_qps": round(float(np.mean([x["qps"] for x in log])))}
    print(json.dumps({"summary": summ}), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"summary": summ, "rounds": log}, f, indent=1)


if __name__ == "__main__":
    main()
