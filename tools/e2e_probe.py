"""Where the end-to-end (pinned host in / host out) search time goes on C2: host wall time per call for device
I/O vs pinned host I/O, and the device time of the same calls (CUDA events), percentiles over --reps calls."""
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

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=100)
ap.add_argument("--itopk", type=int, default=14)
a = ap.parse_args()
dev = torch.device("cuda:0")
idx = svf.Index.build(torch.from_numpy(base_rows("C2")).to(dev), degree=64)
Q = query_rows("C2")
Qd = torch.from_numpy(Q).to(dev)
Qh = torch.from_numpy(Q).pin_memory()
k, L = 10, a.itopk
od_i = torch.empty((len(Q), k), dtype=torch.int32, device=dev)
od_d = torch.empty((len(Q), k), dtype=torch.float32, device=dev)
oh_i = torch.empty((len(Q), k), dtype=torch.int32, pin_memory=True)
oh_d = torch.empty((len(Q), k), dtype=torch.float32, pin_memory=True)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
res = {}
for name, (qq, oi, od) in {"device_io": (Qd, od_i, od_d), "pinned_host_io": (Qh, oh_i, oh_d)}.items():
    for _ in range(10):
        idx.search_into(qq, k, L, oi, od)
    torch.cuda.synchronize()
    host, devt = [], []
    for _ in range(a.reps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        idx.search_into(qq, k, L, oi, od)
        e1.record()
        torch.cuda.synchronize()
        host.append((time.perf_counter() - t0) * 1e3)
        devt.append(e0.elapsed_time(e1))
    res[name] = {"host_ms": {p: round(float(np.percentile(host, p)), 4) for p in (10, 50, 90)},
                 "device_ms": {p: round(float(np.percentile(devt, p)), 4) for p in (10, 50, 90)}}
    print(json.dumps({name: res[name]}), flush=True)
