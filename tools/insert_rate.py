"""Build + 1%-batch insert rate on C2 (the knob under test comes from the environment, e.g. SVF_HANDOFF, which
svf_build reads before any per-index setting exists).  Prints one JSON line.

  SVF_HANDOFF=45 python tools/insert_rate.py
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from workloads import base_rows, query_rows  # noqa: E402

X = torch.from_numpy(base_rows("C2")).cuda()
Xn = torch.from_numpy(base_rows("C2", 1_000_000, 120_000)).cuda()
torch.cuda.synchronize()
t0 = time.time()
w = int(os.environ.get("SVF_INS_WIDTH", "1"))        # search width of the insert search (svf_params.search_width)
lb = int(os.environ.get("SVF_BUILD_ITOPK", "0"))     # L_build
li = int(os.environ.get("SVF_INS_ITOPK", "128"))     # L_insert
idx = svf.Index.build(X, degree=64, capacity=1_120_000, search_width=w, build_itopk=lb, insert_itopk=li)
torch.cuda.synchronize()
t_build = time.time() - t0
hb = int(os.environ.get("SVF_HB", "0"))  # visited-table bits for the timed inserts (0 = automatic)
idx.set_search_params(1, 0, 0, hb)
idx.insert(Xn[:20_000])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(10):
    idx.insert(Xn[20_000 + i * 10_000: 30_000 + i * 10_000])
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
Q = torch.from_numpy(query_rows("C2")).cuda()
gt = idx.knn_exact(Q, 10)[0].cpu().numpy()
idx.set_search_params(1, 0, 0, 0)
rec = {}
for L in (10, 14):
    ids = idx.search(Q, 10, L)[0].cpu().numpy()
    rec[L] = round(float((ids[:, :, None] == gt[:, None, :]).any(axis=2).sum()) / ids.size, 4)
print(json.dumps({"ins_width": w, "build_itopk": lb, "insert_itopk": li, "recall_after_120k_inserts": rec,
                  "handoff_env": os.environ.get("SVF_HANDOFF"), "hash_bits": hb, "build_s": round(t_build, 3),
                  "build_inserts_per_s": round(1e6 / t_build), "insert_ms_per_10k": round(ms, 3),
                  "inserts_per_s": round(1e4 / (ms / 1e3))}))
