"""Search-parameter sweep on one built index (any config): for each (itopk, search_width, hash_bits) the device time
of a 10K-query batch (CUDA-graph replay, L2 flushed, median of --reps) and recall@10 against exact ground truth.

  python tools/param_sweep.py --config C3 --itopk 64,96 --width 1,2 --hash-bits 0,11 [--out f.json]
"""
import argparse
import itertools
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from workloads import base_rows, config_spec, query_rows  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--itopk", default="64,96")
    ap.add_argument("--width", default="1,2")
    ap.add_argument("--hash-bits", default="0,11")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--build-itopk", type=int, default=0)
    ap.add_argument("--max-iter", default="0")
    ap.add_argument("--n-init", default="0", help="random entry points (0 = itopk)")
    ap.add_argument("--handoff", default="-1", help="pair-mode handoff thresholds %% (-1 = auto, 0 = off)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    c = config_spec(a.config)
    n = a.n or c["n"]
    dev = torch.device("cuda:0")
    idx = svf.Index.build(torch.from_numpy(base_rows(a.config, 0, n)).to(dev), degree=c["degree"], metric=c["metric"],
                          build_itopk=a.build_itopk)
    Q = torch.from_numpy(query_rows(a.config)).to(dev)
    gt = idx.knn_exact(Q, 10)[0].cpu().numpy()
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    oi = torch.empty((len(Q), 10), dtype=torch.int32, device=dev)
    od = torch.empty((len(Q), 10), dtype=torch.float32, device=dev)
    rows = []
    for L, p, hb, mi, ho, ni in itertools.product(*[[int(x) for x in v.split(",")] for v in
                                                   (a.itopk, a.width, a.hash_bits, a.max_iter, a.handoff, a.n_init)]):
        try:
            idx.set_search_params(p, ni, mi, hb)
            idx.set_search_handoff(ho)
            idx.search_into(Q, 10, L, oi, od)
        except Exception as e:  # noqa: BLE001 (invalid combinations are reported, not fatal)
            print(json.dumps({"itopk": L, "width": p, "hash_bits": hb, "error": str(e)[:80]}), flush=True)
            continue
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            idx.search_into(Q, 10, L, oi, od)
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ids = oi.cpu().numpy()
        rec = float((ids[:, :, None] == gt[:, None, :]).any(axis=2).sum()) / ids.size
        cnt = idx.last_search_counters()
        r = {"itopk": L, "width": p, "hash_bits": hb, "max_iter": mi, "handoff": ho, "n_init": ni, "median_ms": round(float(np.median(ts)), 4),
             "qps": round(len(Q) / (np.median(ts) * 1e-3)), "recall": round(rec, 4),
             "n_dist": round(cnt["n_dist"] / max(1, cnt["queries"]), 1),
             "iters": round(cnt["iters"] / max(1, cnt["queries"]), 2)}
        rows.append(r)
        print(json.dumps(r), flush=True)
        del g
    if a.out:
        json.dump({"config": a.config, "n": n, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
