"""Update-batch-size sweep (paper Fig. 17 / SURVEY E18: "larger batches substantially increase
throughput but degrade recall beyond 2^13"): build C2 with insert sub-batches of B and report build inserts/s,
the inserts/s of a further 1% insert batch, and recall@10 of the resulting graph at fixed itopk.

  python tools/batch_sweep.py [--batches 1024,2048,4096,8192,16384,32768] [--itopk 14] [--out f.json]
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
from workloads import base_rows, query_rows  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1024,2048,4096,8192,16384,32768")
    ap.add_argument("--itopk", type=int, default=14)
    ap.add_argument("--wpq", type=int, default=0)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    X = torch.from_numpy(base_rows("C2")).to(dev)
    Xn = torch.from_numpy(base_rows("C2", 1_000_000, 10_000)).to(dev)
    Q = torch.from_numpy(query_rows("C2")).to(dev)
    res = []
    gt = None
    for B in [int(b) for b in a.batches.split(",")]:
        torch.cuda.synchronize()
        t0 = time.time()
        idx = svf.Index.build(X, degree=64, capacity=1_010_000, insert_batch=B)
        torch.cuda.synchronize()
        tb = time.time() - t0
        if gt is None:
            gt = idx.knn_exact(Q, 10)[0].cpu().numpy()
        idx.set_warps_per_query(a.wpq)
        ids, _ = idx.search(Q, 10, a.itopk)
        ids = ids.cpu().numpy()
        rec = float((ids[:, :, None] == gt[:, None, :]).any(axis=2).mean())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        idx.insert(Xn)
        e1.record()
        torch.cuda.synchronize()
        r = {"insert_batch": B, "build_s": round(tb, 3), "build_inserts_per_s": round(1e6 / tb),
             "insert_1pct_ms": round(e0.elapsed_time(e1), 3),
             "inserts_per_s": round(len(Xn) / (e0.elapsed_time(e1) / 1e3)), "recall_at_10": round(rec, 4),
             "itopk": a.itopk, "wpq": a.wpq}
        print(json.dumps(r), flush=True)
        res.append(r)
        idx.close()
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
