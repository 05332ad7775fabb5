"""Graph quality under the inner product: build on the raw rows (IP) vs on norm-augmented rows
x' = [x, sqrt(M^2 - |x|^2), 0, 0, 0] (the MIPS -> NNS reduction; on the sphere |x'| = M the IP order of x' equals
its L2 order), searched with q' = [q, 0, 0, 0, 0] so that q'.x' = q.x. Recall@10 against exact IP ground truth.

  python tools/mips_probe.py --config C4 --n 2000000 --itopk 64,128,256
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


def recall(ids, gt):
    return float((ids[:, :, None] == gt[:, None, :]).any(axis=2).sum()) / ids.size


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--n", type=int, default=2000000)
    ap.add_argument("--itopk", default="64,128,256")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    c = config_spec(a.config)
    dev = torch.device("cuda:0")
    X = torch.from_numpy(base_rows(a.config, 0, a.n)).to(dev)
    Q = torch.from_numpy(query_rows(a.config)).to(dev)
    n2 = (X.double() ** 2).sum(1)
    M2 = n2.max()
    aug = torch.sqrt(torch.clamp(M2 - n2, min=0)).float()
    Xa = torch.zeros((a.n, X.shape[1] + 4), dtype=torch.float32, device=dev)
    Xa[:, :X.shape[1]] = X
    Xa[:, X.shape[1]] = aug
    Qa = torch.zeros((Q.shape[0], X.shape[1] + 4), dtype=torch.float32, device=dev)
    Qa[:, :X.shape[1]] = Q
    out = {"config": a.config, "n": a.n, "norm_min": float(n2.min().sqrt()), "norm_max": float(M2.sqrt()), "rows": []}
    gt = None
    for name, base, qq in (("ip_raw", X, Q), ("ip_augmented", Xa, Qa)):
        torch.cuda.synchronize()
        t0 = time.time()
        idx = svf.Index.build(base, degree=c["degree"], metric="ip")
        torch.cuda.synchronize()
        tb = time.time() - t0
        if gt is None:
            gt = idx.knn_exact(Q, 10)[0].cpu().numpy()
        for L in [int(x) for x in a.itopk.split(",")]:
            ids = idx.search(qq, 10, L)[0].cpu().numpy()
            r = {"build": name, "build_s": round(tb, 2), "itopk": L, "recall": round(recall(ids, gt), 4)}
            out["rows"].append(r)
            print(json.dumps(r), flush=True)
        idx.close()
        del idx
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
