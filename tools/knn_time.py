"""Device time of svf_knn_exact on C2 (1M x 128 integer G-LM base, 10K queries, k=10): median of --reps calls.
  python tools/knn_time.py [--reps 5]     (SVF_LIB selects a tuning variant of libsvf.so)"""
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
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--config", default="C2")
    a = ap.parse_args()
    X = base_rows(a.config)
    Q = torch.from_numpy(query_rows(a.config)).cuda()
    # a built graph: svf_knn_exact prunes with a short graph search over it (SVF_KNN_BOUND=0: the sample pass)
    idx = svf.Index.build(torch.from_numpy(X).cuda(), degree=64, build_itopk=256)
    idx.knn_exact(Q, 10)
    torch.cuda.synchronize()
    t = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        idx.knn_exact(Q, 10)
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    ms = float(np.median(t))
    print(json.dumps({"lib": os.environ.get("SVF_LIB", "default"), "bound": os.environ.get("SVF_KNN_BOUND", "1"),
                      "ms": round(ms, 3),
                      "tflops": round(2.0 * len(Q) * X.shape[0] * X.shape[1] / (ms * 1e-3) / 1e12, 1),
                      "stats": idx.knn_stats()}))


if __name__ == "__main__":
    main()
