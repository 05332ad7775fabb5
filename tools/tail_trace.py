"""Timeline of one C2 search batch (svf_set_trace): when the query queue drains, how long the batch then runs,
how many queries are in flight over time, and how iteration counts relate to per-query latency.  Used for the
batch-tail analysis in DESIGN.md §6.

  python tools/tail_trace.py [--itopk 14] [--nq 10000] [--tails 0,30] (handoff thresholds, %% of warps) [--out file.json]
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


def analyse(t0, t1, sm, it, ph, bins=40):
    s = t0 - t0.min()
    e = t1 - t0.min()
    span = float(e.max())
    drain = float(s.max())                      # the last query was taken from the queue
    dur = (e - s).astype(np.float64)
    edges = np.linspace(0, span, bins + 1)
    mids = 0.5 * (edges[1:] + edges[:-1])
    inflight = [int(((s <= m) & (e > m)).sum()) for m in mids]
    last = np.argsort(e)[-20:]
    return {
        "span_us": round(span / 1e3, 2), "drain_us": round(drain / 1e3, 2),
        "after_drain_us": round((span - drain) / 1e3, 2),
        "first_end_us": round(float(e.min()) / 1e3, 2),
        "dur_us": {p: round(float(np.percentile(dur, q)) / 1e3, 2) for p, q in
                   (("p50", 50), ("p90", 90), ("p99", 99), ("max", 100))},
        "iters": {p: int(np.percentile(it, q)) for p, q in (("p50", 50), ("p90", 90), ("p99", 99), ("max", 100))},
        "ns_per_iter_median": round(float(np.median(dur / np.maximum(it, 1))), 1),
        "last20_iters": [int(x) for x in it[last]], "last20_dur_us": [round(float(x) / 1e3, 1) for x in dur[last]],
        "last20_start_us": [round(float(x) / 1e3, 1) for x in s[last]],
        "inflight_timeline": {"bin_us": round(span / bins / 1e3, 2), "inflight": inflight},
        "sms_used": int(len(np.unique(sm))),
        "phase_cycles_per_iter": {n: round(float(ph[:, i].sum()) / max(int(it.sum()), 1), 1) for i, n in
                                  enumerate(("select", "row", "filter", "distance", "merge"))},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--itopk", type=int, default=14)
    ap.add_argument("--nq", type=int, default=10000)
    ap.add_argument("--tails", default="0")
    ap.add_argument("--batch1", action="store_true", help="also trace batch 1 (zero-load latency)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    idx = svf.Index.build(torch.from_numpy(base_rows("C2")).to(dev), degree=64)
    Q = torch.from_numpy(query_rows("C2", a.nq)).to(dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    res = {}
    for t in [int(x) for x in a.tails.split(",")]:
        idx.set_search_handoff(t)
        idx.set_trace(False)
        for _ in range(5):
            idx.search(Q, 10, a.itopk)
        idx.set_trace(True)
        runs = []
        for _ in range(3):
            flush.zero_()
            torch.cuda.synchronize()
            idx.search(Q, 10, a.itopk)
            torch.cuda.synchronize()
            runs.append(analyse(*idx.read_trace(a.nq)))
        idx.set_trace(False)
        res[str(t)] = runs
        r = runs[-1]
        print(json.dumps({"tail": t, **{k: r[k] for k in ("span_us", "drain_us", "after_drain_us", "dur_us", "iters",
                                                          "ns_per_iter_median", "sms_used",
                                                          "phase_cycles_per_iter")}}), flush=True)
        print(json.dumps({"last20_iters": r["last20_iters"], "last20_dur_us": r["last20_dur_us"],
                          "last20_start_us": r["last20_start_us"]}), flush=True)
        print(json.dumps(r["inflight_timeline"]), flush=True)
    if a.batch1:
        idx.set_search_handoff(0)
        idx.set_trace(True)
        rows = []
        for i in range(200):
            idx.search(Q[i:i + 1].contiguous(), 10, a.itopk)
            torch.cuda.synchronize()
            t0, t1, sm, it, ph = idx.read_trace(1)
            rows.append((int(t1[0] - t0[0]), int(it[0]), ph[0]))
        idx.set_trace(False)
        its = sum(r[1] for r in rows)
        b1 = {"batch1_ns_per_iter": round(sum(r[0] for r in rows) / its, 1),
              "batch1_phase_cycles_per_iter": {n: round(float(sum(r[2][i] for r in rows)) / its, 1) for i, n in
                                               enumerate(("select", "row", "filter", "distance", "merge"))}}
        print(json.dumps(b1), flush=True)
        res["batch1"] = b1
    if a.out:
        json.dump({"config": f"C2 1M x 128, R=64, itopk {a.itopk}, batch {a.nq}; L2 flushed; direct launch",
                   "runs": res}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
