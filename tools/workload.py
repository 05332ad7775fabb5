"""Replay a paper-style streaming trace (workloads/traces.py) on the GPU index and report recall@10 against exact
ground truth over the live set, search QPS, insert and delete rates per evaluated step.

  python tools/workload.py --trace expiration --config C2 --n 1000000 --itopk 32 [--repair 0.15] [--consolidate 0.2]
      --out f.json
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
from workloads import traces  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trace", choices=["sliding", "expiration", "clustered", "insert_heavy"], default="expiration")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--t-max", type=int, default=200)
    ap.add_argument("--itopk", type=int, default=32)
    ap.add_argument("--repair", type=float, default=0.0, help="repair threshold after each delete (0 = off)")
    ap.add_argument("--consolidate", type=float, default=0.0,
                    help="automatic global consolidation ratio (svf_set_consolidation; 0 = off, paper: 0.2)")
    ap.add_argument("--max-evals", type=int, default=12)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    c = config_spec(a.config)
    dev = torch.device("cuda:0")
    X = base_rows(a.config, 0, a.n)
    Q = torch.from_numpy(query_rows(a.config, a.nq)).to(dev)
    if a.trace == "sliding":
        steps = traces.sliding_window(a.n, a.t_max)
    elif a.trace == "expiration":
        steps = traces.expiration_time(a.n, a.t_max)
    elif a.trace == "clustered":
        steps = traces.clustered(traces.kmeans_labels(X, 64, 5))
    else:
        steps = traces.insert_heavy(a.n, a.n // 10, 90)
    Xd = torch.from_numpy(X).to(dev)
    idx = None
    row_of_id = np.full(2 * a.n + 1, -1, np.int64)  # index id -> dataset row
    id_of_row = np.full(a.n, -1, np.int64)
    evals, t_ins, t_del = [], [], []
    ev = lambda: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))  # noqa: E731
    searchable = [i for i, s in enumerate(steps) if s["search"]]
    eval_at = set(searchable[:: max(1, len(searchable) // a.max_evals)])
    t_start = time.time()
    for si, s in enumerate(steps):
        ins = np.asarray(s["insert"], np.int64)
        if len(ins):
            if idx is None:
                idx = svf.Index.build(Xd[ins], degree=c["degree"], metric=c["metric"], capacity=a.n + 1)
                if a.consolidate > 0:
                    idx.set_consolidation(a.consolidate)
                new = np.arange(len(ins))
            else:
                e0, e1 = ev()
                e0.record()
                new = idx.insert(Xd[ins]).astype(np.int64)
                e1.record()
                torch.cuda.synchronize()
                t_ins.append((len(ins), e0.elapsed_time(e1)))
            row_of_id[new] = ins
            id_of_row[ins] = new
        dele = np.asarray(s["delete"], np.int64)
        if len(dele) and idx is not None:
            ids = id_of_row[dele]
            ids = ids[ids >= 0]
            e0, e1 = ev()
            e0.record()
            idx.delete(torch.from_numpy(ids.astype(np.int32)).to(dev))
            e1.record()
            torch.cuda.synchronize()
            t_del.append((len(ids), e0.elapsed_time(e1)))
            if a.repair > 0:
                idx.repair(threshold=a.repair)
        if si in eval_at and idx is not None:
            e0, e1 = ev()
            e0.record()
            ids, _ = idx.search(Q, 10, a.itopk)
            e1.record()
            gi, _ = idx.knn_exact(Q, 10)
            torch.cuda.synchronize()
            ids, gi = ids.cpu().numpy(), gi.cpu().numpy()
            rec = float((ids[:, :, None] == gi[:, None, :]).any(axis=2).sum()) / ids.size
            info = idx.info()
            r = {"step": si, "live": info["n_alloc"] - info["n_deleted"], "recall": round(rec, 4),
                 "qps": round(a.nq / (e0.elapsed_time(e1) / 1e3))}
            evals.append(r)
            print(json.dumps(r), flush=True)
    summ = {"trace": a.trace, "config": a.config, "n": a.n, "itopk": a.itopk, "repair": a.repair,
            "consolidate": a.consolidate, "consolidations": idx.consolidation_stats()["consolidations"],
            "steps": len(steps), "wall_s": round(time.time() - t_start, 1),
            "inserts_per_s": round(sum(n for n, _ in t_ins) / max(1e-9, sum(t for _, t in t_ins) / 1e3)),
            "deletes_per_s": round(sum(n for n, _ in t_del) / max(1e-9, sum(t for _, t in t_del) / 1e3)),
            "recall_min": min(e["recall"] for e in evals), "recall_mean": round(float(np.mean([e["recall"] for e in evals])), 4),
            "recall_last": evals[-1]["recall"]}
    print(json.dumps({"summary": summ}), flush=True)
    if a.out:
        json.dump({"summary": summ, "evals": evals}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
