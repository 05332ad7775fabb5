"""Pair-mode handoff sweep on the C2 index: device time of one search batch (CUDA-graph replay, L2 flushed between
steps, median of --reps) for each `svf_set_search_handoff` value, and a check that the results are identical to the
handoff-off run (the handoff changes only which warps serve the stragglers, never the search).

  python tools/tail_sweep.py [--itopk 14] [--batches 10000,20000] [--tails 0,10,20,...] [--out file.json]
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
    ap.add_argument("--reps", type=int, default=60)
    ap.add_argument("--batches", default="10000")
    ap.add_argument("--tails", default="0,10,20,30,40,60", help="handoff thresholds (%% of warps)")
    ap.add_argument("--hash-bits", type=int, default=0, help="visited-table slots 2^b (0 = auto)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    idx = svf.Index.build(torch.from_numpy(base_rows("C2")).to(dev), degree=64)
    idx.set_search_params(1, 0, 0, a.hash_bits)
    nqmax = max(int(b) for b in a.batches.split(","))
    Qall = torch.from_numpy(query_rows("C2", nqmax)).to(dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    k, L = 10, a.itopk
    res = []
    for b in [int(x) for x in a.batches.split(",")]:
        Q = Qall[:b].contiguous()
        ref = None
        for t in [int(x) for x in a.tails.split(",")]:
            idx.set_search_handoff(t)
            oi = torch.empty((b, k), dtype=torch.int32, device=dev)
            od = torch.empty((b, k), dtype=torch.float32, device=dev)
            idx.search_into(Q, k, L, oi, od)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                idx.search_into(Q, k, L, oi, od)
            torch.cuda.synchronize()
            for _ in range(5):
                g.replay()
            ts = []
            for _ in range(a.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            out = (oi.cpu().numpy(), od.cpu().numpy())
            if ref is None:
                ref = out
            same = bool(np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1]))
            r = {"batch": b, "tail": t, "median_ms": round(float(np.median(ts)), 4),
                 "min_ms": round(float(np.min(ts)), 4), "qps": round(b / (np.median(ts) * 1e-3), 1),
                 "identical_to_first": same}
            print(json.dumps(r), flush=True)
            res.append(r)
            del g
    if a.out:
        json.dump({"config": "C2 1M x 128, R=64, itopk %d, k=10; CUDA-graph replay, L2 flushed" % L,
                   "rows": res}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
