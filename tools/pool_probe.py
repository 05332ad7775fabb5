"""Where does a large-pool search spend its time?  Per-query timelines (svf_set_trace) of itopk >= 128 searches on
the C2 graph (the insert search's shape: L_insert = 128 over 4096-query sub-batches), with per-phase SM cycles when
the library is the -DSVF_PHASE_PROF variant (SVF_LIB=...).  Also times one 10K insert with its stage breakdown.

  SVF_LIB=paper_2601_08528_b200/libsvf_phase.so python tools/pool_probe.py --out gpurun_out/pool_probe.json
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from tools.tail_trace import analyse  # noqa: E402
from workloads import base_rows  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--build-itopk", type=int, default=256)
    ap.add_argument("--itopks", default="128,192,256")
    ap.add_argument("--batches", default="4096,10000")
    ap.add_argument("--width", type=int, default=1)
    ap.add_argument("--n", type=int, default=0, help="base rows (0 = the config's)")
    ap.add_argument("--degree", type=int, default=64)
    ap.add_argument("--no-insert", action="store_true")
    ap.add_argument("--hbits", default="0", help="visited-cache sizes 2^b to try (0 = the library's default)")
    ap.add_argument("--no-trace", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    from workloads import config_spec

    X = base_rows(a.config, 0, a.n or None)
    n = len(X)
    idx = svf.Index.build(torch.from_numpy(X).to(dev), degree=a.degree, capacity=n + 80_000, build_itopk=a.build_itopk,
                          metric=config_spec(a.config)["metric"])
    Qn = torch.from_numpy(base_rows(a.config, n, 20_000)).to(dev)
    if a.config == "C4":   # C4's queries come from another modality (OOD): probe with those
        from workloads import query_rows

        Qn = torch.from_numpy(query_rows("C4", 20_000)).to(dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    res = {"config": f"{a.config} graph at L_build {a.build_itopk}; queries = fresh insert vectors", "runs": []}
    idx.set_search_handoff(0)
    for L, nq, hb in [(L, nq, hb) for L in map(int, a.itopks.split(",")) for nq in map(int, a.batches.split(","))
                      for hb in map(int, a.hbits.split(","))]:
        if True:
            idx.set_search_params(a.width, 0, 0, hb)
            Q = Qn[:nq].contiguous()
            for _ in range(2):
                idx.search(Q, 10, L)
            ts = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                idx.search(Q, 10, L)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            c = idx.last_search_counters()
            if a.no_trace:
                row = {"itopk": L, "nq": nq, "width": a.width, "hbits": hb, "ms_median": round(float(np.median(ts)), 4),
                       "n_dist_per_q": round(c["n_dist"] / c["queries"], 1),
                       "iters_per_q": round(c["iters"] / c["queries"], 1)}
                print(json.dumps(row), flush=True)
                res["runs"].append(row)
                continue
            idx.set_trace(True)
            flush.zero_()
            idx.search(Q, 10, L)
            torch.cuda.synchronize()
            r = analyse(*idx.read_trace(nq))
            idx.set_trace(False)
            row = {"itopk": L, "nq": nq, "width": a.width, "hbits": hb, "ms_median": round(float(np.median(ts)), 4),
                   "n_dist_per_q": round(c["n_dist"] / c["queries"], 1), "iters_per_q": round(c["iters"] / c["queries"], 1),
                   **{k: r[k] for k in ("span_us", "drain_us", "after_drain_us", "dur_us", "ns_per_iter_median",
                                        "phase_cycles_per_iter")}}
            row["hbm_frac_alg"] = round(nq * (c["n_dist"] / c["queries"] * X.shape[1] * 4) / (row["ms_median"] * 1e-3)
                                        / 6545e9, 4)
            print(json.dumps(row), flush=True)
            res["runs"].append(row)
    if a.no_insert:
        if a.out:
            json.dump(res, open(a.out, "w"), indent=1)
        return
    idx.set_search_handoff(-1)
    idx.set_search_params(1, 0, 0, 0)
    tt = []
    for j in range(6):
        if j == 4:
            idx.profile(True)  # stage breakdown from two serialised (profiled) batches
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        idx.insert(Qn[(j % 2) * 10_000:(j % 2 + 1) * 10_000])
        e1.record()
        torch.cuda.synchronize()
        tt.append(e0.elapsed_time(e1))
    pr = idx.profile_read()
    res["insert_10k_ms"] = [round(t, 3) for t in tt[:4]]
    res["insert_10k_ms_profiled"] = [round(t, 3) for t in tt[4:]]
    res["insert_breakdown_ms_per_batch"] = {k: round(v[0] / 2, 3) for k, v in pr.items()}
    print(json.dumps({k: res[k] for k in ("insert_10k_ms", "insert_10k_ms_profiled", "insert_breakdown_ms_per_batch")}),
          flush=True)
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
