"""Summarise ncu artefacts into profiles/ (tracked): a --set full report of one kernel and/or a launch list.

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
      --nq 10000 --itopk 14 --out profiles/r01_search
writes <out>.json + <out>.md; with --latest also profiles/ncu_search_latest.json (read by bench.py for `traffic`).
"""
import argparse
import collections
import csv
import json
import os
import re
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor.sum", "launch__shared_mem_per_block_dynamic",
]


def to_float(v: str):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return v


def rep_summary(rep: str) -> list:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        m = {"kernel": d[h.index("Kernel Name")] if "Kernel Name" in h else "?"}
        for k in KEYS:
            if k in h:
                m[k] = to_float(d[h.index(k)])
                m[k + ".unit"] = units[h.index(k)]
        stalls = {}
        for i, name in enumerate(h):
            if name.startswith("smsp__pcsamp_warps_issue_stalled") and not name.endswith("not_issued"):
                v = to_float(d[i])
                if isinstance(v, float):
                    stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
        tot = sum(stalls.values()) or 1.0
        m["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
        res.append(m)
    return res


def launch_summary(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(to_float(r[vi]))
    tot = sum(sum(v) for v in agg.values()) or 1.0
    return {k: {"launches": len(v), "total_us": round(sum(v) / 1e3, 1), "avg_us": round(sum(v) / len(v) / 1e3, 2),
                "share": round(sum(v) / tot, 4)} for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--nq", type=int, default=10000)
    ap.add_argument("--itopk", type=int, default=0)
    ap.add_argument("--out", required=True)
    ap.add_argument("--latest", action="store_true")
    ap.add_argument("--config", default="C2", help="with --latest: which config's traffic file bench.py reads")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    js = {"note": a.note, "nq": a.nq, "itopk": a.itopk}
    if a.rep:
        js["kernels"] = rep_summary(a.rep)
        # one search step = every captured search_kernel grid (the one-warp grid + the chained handoff grid)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        step, seen = [], set()
        for k in js["kernels"]:  # one step = each distinct search grid once (a capture may hold two steps)
            if re.search(r"search(_lp)?_kernel", k["kernel"]) and k["kernel"] not in seen:
                seen.add(k["kernel"])
                step.append(k)
        step = step or js["kernels"][:1]
        if all(isinstance(k.get("dram__bytes_read.sum"), float) for k in step):
            tot = sum(k["dram__bytes_read.sum"] * scale.get(k["dram__bytes_read.sum.unit"], 1) +
                      k["dram__bytes_write.sum"] * scale.get(k["dram__bytes_write.sum.unit"], 1) for k in step)
            js["dram_bytes_per_launch"] = tot
            js["dram_bytes_per_query"] = tot / a.nq
            js["step_kernels"] = len(step)
    if a.launches:
        js["launch_list"] = launch_summary(a.launches)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(js, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as f:
        f.write(f"# ncu summary: {os.path.basename(a.out)}\n\n{a.note}\n\n")
        for k in js.get("kernels", []):
            f.write(f"## {k['kernel'][:120]}\n\n| metric | value | unit |\n|---|---|---|\n")
            for kk in KEYS:
                if kk in k:
                    f.write(f"| {kk} | {k[kk]} | {k.get(kk + '.unit', '')} |\n")
            f.write(f"\nstall reasons (share of samples): {k['stall_share']}\n\n")
        if "launch_list" in js:
            f.write("## launch list (gpu__time_duration.sum, --clock-control none; serialised, cold)\n\n"
                    "| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|\n")
            for kname, v in js["launch_list"].items():
                f.write(f"| {kname[:100]} | {v['launches']} | {v['total_us']} | {v['avg_us']} | {v['share']} |\n")
    if a.latest and "dram_bytes_per_query" in js:
        json.dump({"itopk": a.itopk, "dram_bytes_per_query": js["dram_bytes_per_query"],
                   "source": os.path.basename(a.out) + ".json"},
                  open(os.path.join(os.path.dirname(a.out), "ncu_search_latest.json" if a.config == "C2"
                                    else f"ncu_search_latest_{a.config}.json"), "w"), indent=1)
    print(json.dumps({k: v for k, v in js.items() if k != "kernels"}, indent=1)[:2000])


if __name__ == "__main__":
    main()
