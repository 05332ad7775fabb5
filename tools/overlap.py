"""Two-stream search/update overlap (paper P:L495-498 "multiple search streams plus one update
stream"): on the C2 index, a 10K-query search batch on stream S and a 1% insert batch (10K) on stream U
- each alone, then both issued back to back on the two streams.  Device time from a start event on S (U waits for
it) to both streams' end events; results of the concurrent searches are checked for validity.

  python tools/overlap.py [--itopk 14] [--reps 20] [--out file.json]
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
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--searches", type=int, default=1, help="search batches per insert batch")
    ap.add_argument("--out", default="")
    ap.add_argument("--build-itopk", type=int, default=0)
    ap.add_argument("--max-iter", type=int, default=0)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    n, nb = 1_000_000, 10_000
    X = torch.from_numpy(base_rows("C2")).to(dev)
    Xn = torch.from_numpy(base_rows("C2", n, nb * (3 * a.reps + 2))).to(dev)
    Q = torch.from_numpy(query_rows("C2")).to(dev)
    idx = svf.Index.build(X, degree=64, capacity=n + len(Xn), build_itopk=a.build_itopk)
    idx.set_search_params(1, 0, a.max_iter, 0)
    s_q, s_u = torch.cuda.Stream(), torch.cuda.Stream()
    k, L = 10, a.itopk
    used = [0]

    def next_rows():
        r = Xn[used[0]:used[0] + nb]
        used[0] += nb
        return r

    def run(do_search, do_insert):
        t0 = torch.cuda.Event(enable_timing=True)
        eq, eu = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(s_q)
        s_u.wait_event(t0)
        outs = []
        if do_insert:
            with torch.cuda.stream(s_u):
                idx.insert_async(next_rows())
        if do_search:
            with torch.cuda.stream(s_q):
                for _ in range(a.searches):
                    outs.append(idx.search(Q, k, L))
        eq.record(s_q)
        eu.record(s_u)
        torch.cuda.synchronize()
        return max(t0.elapsed_time(eq), t0.elapsed_time(eu)), t0.elapsed_time(eq), outs

    run(True, True)                                    # warm-up (allocations, graph of caches)
    res = {}
    for name, fs, fi in (("search_only", True, False), ("insert_only", False, True), ("both", True, True)):
        ts, tq, bad = [], [], 0
        for _ in range(a.reps):
            ms, msq, outs = run(fs, fi)
            ts.append(ms)
            tq.append(msq)
            for ids, d in outs:                       # validity of concurrent results
                ids = ids.cpu().numpy().view(np.uint32)
                d = d.cpu().numpy()
                na = idx.info()["n_alloc"]
                bad += int((ids >= na).sum()) + int((np.diff(d, axis=1) < 0).sum())
        res[name] = {"median_ms": round(float(np.median(ts)), 4), "min_ms": round(float(np.min(ts)), 4),
                     "search_done_ms": round(float(np.median(tq)), 4) if fs else None, "invalid_results": bad}
        print(json.dumps({name: res[name]}), flush=True)
    s, i, b = (res[x]["median_ms"] for x in ("search_only", "insert_only", "both"))
    res["overlap_gain"] = round((s + i) / b, 3)
    # a search issued behind the insert on the same stream would finish at insert + search; on its own stream
    # it finishes at search_done_ms of "both"
    res["search_latency_behind_insert_ms"] = {"same_stream": round(s + i, 4),
                                              "own_stream": res["both"]["search_done_ms"]}
    print(json.dumps({"serial_sum_ms": round(s + i, 4), "both_ms": b, "gain": res["overlap_gain"],
                      "search_latency": res["search_latency_behind_insert_ms"]}))
    if a.out:
        json.dump({"config": f"C2 1M x 128 R=64, search {a.searches}x 10K queries itopk {L} on stream S, "
                             f"insert 10K (1%) on stream U; device time, median of {a.reps}",
                   "results": res}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
