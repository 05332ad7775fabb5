"""Quick GPU calibration: build a config's graph on the GPU, exact GT, recall / QPS sweep over itopk.
Usage: python tools/calib.py [C2] [--n N] [--nq Q]"""
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--widths", default="1")
    ap.add_argument("--Ls", default="10,16,24,32,48,64,96,128")
    ap.add_argument("--hbits", default="0")
    ap.add_argument("--wpq", default="0")
    a = ap.parse_args()
    c = config_spec(a.config)
    n = a.n or c["n"]
    nq = a.nq or c["nq"]
    t = time.time()
    X = base_rows(a.config, 0, n)
    Q = query_rows(a.config, nq)
    print(f"gen {time.time() - t:.1f}s", flush=True)
    dev = torch.device("cuda:0")
    Xd = torch.from_numpy(X).to(dev)
    Qd = torch.from_numpy(Q).to(dev)
    torch.cuda.synchronize()
    t = time.time()
    idx = svf.Index.build(Xd, degree=c["degree"], metric=c["metric"])
    torch.cuda.synchronize()
    tb = time.time() - t
    print(f"build {n} in {tb:.2f}s = {n / tb:.0f} inserts/s", flush=True)
    t = time.time()
    gt, gtd = idx.knn_exact(Qd, 10)
    torch.cuda.synchronize()
    print(f"knn_exact {nq} in {time.time() - t:.3f}s", flush=True)
    gt = gt.cpu().numpy()
    res = []
    for w, hb, wq in [(int(x), int(h), int(q)) for x in a.widths.split(",") for h in a.hbits.split(",")
                      for q in a.wpq.split(",")]:
        idx.set_search_params(w, 0, 0, hb)
        idx.set_warps_per_query(wq)
        for L in [int(x) for x in a.Ls.split(",")]:
            for _ in range(2):
                ids, d = idx.search(Qd, 10, L)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ids, d = idx.search(Qd, 10, L)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            ids = ids.cpu().numpy()
            rec = np.mean([len(set(ids[i]) & set(gt[i])) / 10 for i in range(nq)])
            cnt = idx.last_search_counters()
            r = dict(width=w, hbits=hb, wpq=wq, L=L, recall=round(float(rec), 4), ms=round(ms, 3), qps=round(nq / ms * 1e3),
                     n_dist=cnt["n_dist"] / nq, iters=cnt["iters"] / nq)
            gbs = nq * (r["n_dist"] * c["dim"] * 4 + r["iters"] * w * c["degree"] * 4) / (ms * 1e-3) / 1e9
            r["alg_GBps"] = round(gbs, 1)
            print(json.dumps(r), flush=True)
            res.append(r)


if __name__ == "__main__":
    main()
