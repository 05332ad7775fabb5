"""Graph-quality probe for the inner-product, out-of-distribution shape (C4): one index per build variant
(insert_itopk = L_insert, protect_prefix = P, seed_size = n0), each searched at several itopk / search widths;
recall@10 against exact IP ground truth (svf_knn_exact) and the device time of the 10K batch.

  python tools/ip_quality.py --n 2000000 --variants 128:32,256:32,128:16 --itopk 128,256 --width 1,2
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--n", type=int, default=2000000)
    ap.add_argument("--variants", default="128:32,256:32")  # insert_itopk:protect_prefix[:seed_size]
    ap.add_argument("--itopk", default="128,256")
    ap.add_argument("--width", default="1")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    c = config_spec(a.config)
    dev = torch.device("cuda:0")
    X = torch.from_numpy(base_rows(a.config, 0, a.n)).to(dev)
    Q = torch.from_numpy(query_rows(a.config)).to(dev)
    oi = torch.empty((len(Q), 10), dtype=torch.int32, device=dev)
    od = torch.empty((len(Q), 10), dtype=torch.float32, device=dev)
    gt, rows = None, []
    for v in a.variants.split(","):
        f = [int(t) for t in v.split(":")]
        kw = dict(insert_itopk=f[0], protect_prefix=f[1])
        if len(f) > 2:
            kw["seed_size"] = f[2]
        torch.cuda.synchronize()
        t0 = time.time()
        idx = svf.Index.build(X, degree=c["degree"], metric=c["metric"], **kw)
        torch.cuda.synchronize()
        tb = time.time() - t0
        if gt is None:
            gt = idx.knn_exact(Q, 10)[0].cpu().numpy()
        for w in [int(t) for t in a.width.split(",")]:
            for L in [int(t) for t in a.itopk.split(",")]:
                idx.set_search_params(w, 0, 0, 0)
                idx.search_into(Q, 10, L, oi, od)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                idx.search_into(Q, 10, L, oi, od)
                e1.record()
                torch.cuda.synchronize()
                ids = oi.cpu().numpy()
                rec = float((ids[:, :, None] == gt[:, None, :]).any(axis=2).sum()) / ids.size
                r = {"variant": v, "build_s": round(tb, 2), "width": w, "itopk": L, "recall": round(rec, 4),
                     "ms": round(e0.elapsed_time(e1), 3)}
                rows.append(r)
                print(json.dumps(r), flush=True)
        idx.close()
        del idx
    if a.out:
        json.dump({"config": a.config, "n": a.n, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
