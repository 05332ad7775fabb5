"""Small-batch search latency (paper Fig. 8 latency metrics) on the C2 index:
per-batch device latency p50/p95/p99 for batch sizes 1..1024, with 1 and 2 warps per query.

  python tools/latency.py [--itopk 14] [--reps 200] [--out file.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from workloads import base_rows, query_rows  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--itopk", type=int, default=14)
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--batches", default="1,8,64,256,1024,4096")
    ap.add_argument("--out", default="")
    ap.add_argument("--build-itopk", type=int, default=0)
    ap.add_argument("--max-iter", type=int, default=0)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    idx = svf.Index.build(torch.from_numpy(base_rows("C2")).to(dev), degree=64, build_itopk=a.build_itopk)
    idx.set_search_params(1, 0, a.max_iter, 0)
    Q = torch.from_numpy(query_rows("C2")).to(dev)
    res = []
    for b in [int(x) for x in a.batches.split(",")]:
        for wpq in (1, 2):
            idx.set_warps_per_query(wpq)
            oi = torch.empty((b, 10), dtype=torch.int32, device=dev)
            od = torch.empty((b, 10), dtype=torch.float32, device=dev)
            g = torch.cuda.CUDAGraph()
            qb = Q[:b].clone()
            idx.search_into(qb, 10, a.itopk, oi, od)
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                idx.search_into(qb, 10, a.itopk, oi, od)
            rng = np.random.default_rng(b)
            ts = []
            for i in range(a.reps):
                s = int(rng.integers(0, Q.shape[0] - b + 1))
                qb.copy_(Q[s:s + b])
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts = np.array(ts)
            r = {"batch": b, "wpq": wpq, "p50_ms": round(float(np.percentile(ts, 50)), 4),
                 "p95_ms": round(float(np.percentile(ts, 95)), 4), "p99_ms": round(float(np.percentile(ts, 99)), 4),
                 "qps_at_p50": round(b / (np.percentile(ts, 50) / 1e3))}
            print(json.dumps(r), flush=True)
            res.append(r)
    if a.out:
        json.dump({"itopk": a.itopk, "reps": a.reps, "results": res}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
