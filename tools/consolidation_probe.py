"""Consolidation quality on C2 at L_build 256: 12 x 1% inserts + 10 x 1% random deletes, then recall@10 (itopk 10,
converged and cap 16) before and after svf_consolidate.  The candidate-list cut is taken from SVF_REPAIR_CAP.

  SVF_REPAIR_CAP=512 python tools/consolidation_probe.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from workloads import base_rows, query_rows  # noqa: E402

X = torch.from_numpy(base_rows("C2")).cuda()
Xn = torch.from_numpy(base_rows("C2", 1_000_000, 120_000)).cuda()
Q = torch.from_numpy(query_rows("C2")).cuda()
idx = svf.Index.build(X, degree=64, capacity=1_120_000, build_itopk=256)
for j in range(12):
    idx.insert(Xn[j * 10_000:(j + 1) * 10_000])
rng = np.random.default_rng(1000)
for j in range(10):
    idx.delete(torch.from_numpy(rng.choice(1_120_000, 10_000, replace=False).astype(np.int32)).cuda())
gt = idx.knn_exact(Q, 10)[0].cpu().numpy()


def rec():
    out = {}
    for cap in (0, 16):
        idx.set_search_params(1, 0, cap, 0)
        ids = idx.search(Q, 10, 10)[0].cpu().numpy()
        out[cap] = round(float((ids[:, :, None] == gt[:, None, :]).any(axis=2).sum()) / ids.size, 4)
    return out


before = rec()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
n = idx.consolidate()
e1.record()
torch.cuda.synchronize()
print(json.dumps({"repair_cap": os.environ.get("SVF_REPAIR_CAP"), "rewritten": n, "ms": round(e0.elapsed_time(e1), 1),
                  "recall_before": before, "recall_after": rec()}))
