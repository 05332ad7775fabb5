#!/usr/bin/env python
"""bench.py — throughput of the SVFusion hot path on B200 (DESIGN.md §8 "Measurement").

Default (N=1): BASELINE.json configs[1], SIFT1M-shaped C2: 1M x d128 fp32 (integer-valued G-LM), degree 64, 10K-query
batches, k=10, L2.  A *step* is one pass of the search hot path (S0-S8) over the 10K-query batch at the lowest itopk
(and then the smallest iteration cap) whose recall@10 is >= 0.95 on a HELD-OUT selection batch (another query seed);
recall is then reported on the timed batch.  Inserts/s and deletes/s (I0-I3, D1) are measured in the same run on 1%
batches.  The 10M configs C3 (Deep10M-shaped) and C4 (Text2Image-shaped, inner product, OOD queries) follow in the same
run under "more_configs", each with its roofline, CPU-oracle baseline and end-to-end number.

Multi-GPU (torchrun, one process per GPU):
  * C1-C4 (fit in one GPU): replicas -- every rank holds the whole index and answers its own 10K-query batch; value =
    all ranks' queries / max-over-ranks time (weak scaling, queries over the fixed dataset, no data-path collective);
  * C5 or --shards S: SURVEY §8(e) -- S logical shards (g -> g mod S), rank r holds shards s mod G = r, per-rank
    pre-merge, one NCCL all_gather_into_tensor of packed pairs, K-M merge; value = merged queries / time.

  python bench.py [--gpus N --steps K --warmup W] [--impl svf|reference] [--config C2] [--shards S]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import base_rows, config_spec, query_rows  # noqa: E402

METRIC = "QPS at recall@10>=0.95 (batch 10K) and inserts/sec"
# L_build per config (svf_params.build_itopk; reading I15): the graph is grown once at this candidate-list size, then
# streamed inserts run at insert_itopk = 128.  Measured (profiles/r01_build_itopk.md): C2 at L_build 256 reaches
# recall@10 0.974 at itopk 10; C4 at 10M: 0.70 -> 0.92 at itopk 128 with 512.
BUILD_ITOPK = {"C1": 0, "C2": 256, "C2G": 256, "C3": 512, "C4": 512, "C5": 512}
# L_insert per config (svf_params.insert_itopk; default 128).  Kept > R: at L_insert <= R the detour selection
# keeps every candidate (no pruning) and streamed rows drift toward a plain kNN graph.
INSERT_ITOPK: dict = {}
# iteration caps tried (descending) at the chosen itopk; the smallest that keeps recall >= target on the selection
# batch is used (I4: a cap ends a query's search early; 0 = run to convergence)
MI_SWEEP = [64, 48, 40, 32, 28, 24, 20, 18, 16, 14, 12]
SELECT_SEED = 3          # held-out query batch for choosing itopk and the cap (the timed batch is seed 2)
EXTRA_CONFIGS = ["C3", "C4", "C2G"]


def mi_caps(L: int) -> list:
    """Caps to try at itopk L, descending: MI_SWEEP plus multiples of L (large pools need ~L iterations)."""
    return sorted(set(MI_SWEEP) | {int(L * f) for f in (3, 2.5, 2, 1.75, 1.5, 1.25, 1.1)}, reverse=True)


L_SWEEP = [10, 11, 12, 13, 14, 16, 20, 24, 32, 40, 48, 64, 80, 96, 128, 160, 192, 256]
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}
BAD_REASONS = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "hw_power_brake_slowdown"}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="svf", choices=["svf", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--shards", type=int, default=0, help="logical shards (SURVEY §8(e)); 0 = per config (C5: 8)")
    ap.add_argument("--n", type=int, default=0, help="override the number of base rows")
    ap.add_argument("--nq", type=int, default=0, help="override query batch")
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--target-recall", type=float, default=0.95)
    ap.add_argument("--select-margin", type=float, default=0.003,
                    help="itopk / cap must reach target + margin on the selection batch (the timed batch is another draw)")
    ap.add_argument("--itopk", type=int, default=0, help="fix itopk (skip the sweep)")
    ap.add_argument("--search-width", type=int, default=1)
    ap.add_argument("--max-iter", type=int, default=-1, help="iteration cap (-1 = choose by recall, 0 = converge)")
    ap.add_argument("--build-itopk", type=int, default=-1, help="L_build (-1 = per-config default, 0 = insert_itopk)")
    ap.add_argument("--insert-itopk", type=int, default=-1, help="L_insert (-1 = per-config default)")
    ap.add_argument("--insert-batch", type=int, default=0, help="insert sub-batch B_ins (0 = library default)")
    ap.add_argument("--hash-bits", type=int, default=0, help="visited-table slots 2^b per query (0 = auto)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-insert", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C3/C4 blocks after the headline")
    ap.add_argument("--extra", default=",".join(EXTRA_CONFIGS), help="configs measured after the headline")
    ap.add_argument("--ncu", action="store_true", help="short run for ncu: no GT / sweep / baselines")
    ap.add_argument("--no-graph", action="store_true", help="launch the step directly instead of a CUDA graph")
    ap.add_argument("--wpq", type=int, default=0, help="warps per query (0 = auto)")
    ap.add_argument("--handoff", type=int, default=-1, help="pair-mode handoff threshold %% (-1 = auto, 0 = off)")
    return ap.parse_args(argv)


# ---- distributed plumbing -------------------------------------------------------------------------------------
class Dist:
    def __init__(self, n_gpus: int):
        import torch

        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != n_gpus and self.world > 1:
            raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={self.world}")
        # SVF_SAME_DEVICE=1 + SVF_BACKEND=gloo: every rank on cuda:0 (checks the N>1 plumbing on a 1-GPU box;
        # NCCL refuses two ranks on one device).  Production runs use one GPU per rank over NCCL.
        same = os.environ.get("SVF_SAME_DEVICE") == "1"
        self.dev = torch.device("cuda", 0 if same else self.local)
        torch.cuda.set_device(self.dev)
        self.pg = None
        self.backend = None
        if self.world > 1:
            import torch.distributed as dist

            self.backend = os.environ.get("SVF_BACKEND", "nccl")
            dist.init_process_group(self.backend, device_id=self.dev if self.backend == "nccl" else None)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, v: float) -> float:
        if not self.pg:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev if self.backend == "nccl" else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


class Clocks:
    """nvidia-smi sampler around the timed region (the recipe's clocks line)."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = subprocess.Popen(
            ["nvidia-smi", "-i", str(index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
             "clocks_event_reasons.active,utilization.gpu", "--format=csv,noheader,nounits", "-lms", "100"],
            stdout=self.f, stderr=subprocess.DEVNULL)

    def stop(self) -> dict:
        time.sleep(0.15)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.count(",") >= 4]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        for r in rows:
            try:
                s, m, _, act, util = float(r[0]), float(r[1]), r[2], int(r[3].strip(), 16), float(r[4])
            except ValueError:
                continue
            mx = max(mx, m)
            if util > 0:
                sm.append(s)
            for bit, name in REASONS.items():
                if act & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(rows), "samples_under_load": len(sm)}


def measured_peaks() -> dict:
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(config: str) -> dict | None:
    """Per-query DRAM bytes of the search kernel from the committed ncu --set full summary (if any)."""
    name = "ncu_search_latest.json" if config == "C2" else f"ncu_search_latest_{config}.json"
    try:
        return json.load(open(os.path.join(ROOT, "profiles", name)))
    except Exception:
        return None


def host_cpu() -> dict:
    """The host the CPU baseline ran on: model name (lscpu) and core count."""
    model = platform.processor() or None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"model": model, "nproc": os.cpu_count()}


# ---- recall (O7).  The oracle's pinned definitions are checked equal to these in tests/test_bench_host.py;
# bench.py measures with its own copy because only its cpu_baseline leg may call the oracle. ---------------------
def recall_at_k(ids: np.ndarray, gt: np.ndarray, k: int) -> float:
    ids, gt = np.asarray(ids)[:, :k], np.asarray(gt)[:, :k]
    hit = (ids[:, :, None] == gt[:, None, :]).any(axis=2).sum()
    return float(hit) / (k * ids.shape[0])


def recall_tie_aware(res_d: np.ndarray, gt_d: np.ndarray, k: int, rel: float = 1e-5) -> float:
    res_d, gt_d = np.asarray(res_d, np.float64)[:, :k], np.asarray(gt_d, np.float64)[:, :k]
    kth = gt_d[:, k - 1:k]
    return float(np.mean(res_d <= kth + np.abs(kth) * rel + 1e-30))


def rnd(x, n=4):
    return None if x is None else round(float(x), n)


# ---- one measured configuration ------------------------------------------------------------------------------
class Run:
    """Everything measured on one configuration: build, selection sweeps, timed steps, roofline, e2e, CPU oracle
    baseline, inserts/deletes and their roofline, recall after updates / repair / consolidation."""

    def __init__(self, a, D, config: str, headline: bool):
        import torch

        self.a, self.D, self.name, self.headline, self.torch = a, D, config, headline, torch
        self.c = config_spec(config)
        self.S = a.shards if a.shards > 0 else int(self.c.get("shards", 1))
        self.sharded = self.S > 1
        self.mode = "sharded" if self.sharded else ("replicas" if D.world > 1 else "single")
        self.n = (a.n or self.c["n"]) if headline else self.c["n"]
        self.nq = (a.nq or self.c["nq"]) if headline else self.c["nq"]
        self.k, self.R, self.dim = a.k, self.c["degree"], self.c["dim"]
        self.build_L = a.build_itopk if (a.build_itopk >= 0 and headline) else BUILD_ITOPK.get(config, 0)
        self.ins_L = a.insert_itopk if (a.insert_itopk > 0 and headline) else INSERT_ITOPK.get(config, 128)
        self.out = {}

    # -- index -------------------------------------------------------------------------------------------------
    def build(self):
        import paper_2601_08528_b200 as svf
        from paper_2601_08528_b200.sharded import ShardedIndex

        torch, D = self.torch, self.D
        a = self.a
        self.ins_batch = max(1, self.n // 100)                 # 1% insert / delete batches (C3-style rounds)
        self.ins_steps = 0 if a.no_insert else (10 if self.headline else 4)
        self.ins_warm = 0 if a.no_insert else 2
        t0 = time.time()
        X = base_rows(self.name, 0, self.n)
        # the timed batch: seed 2 (rank 0; replicas: rank r answers its own batch); the selection batch: seed 3
        qseed = 2 if (D.rank == 0 or self.sharded) else 1000 + D.rank
        self.Q = query_rows(self.name, self.nq, row_seed=qseed)
        self.Qsel = query_rows(self.name, self.nq, row_seed=SELECT_SEED)
        # + 2 batches for the two-stream measurement (search on one stream while an insert runs on another)
        n_new = self.ins_batch * (self.ins_steps + self.ins_warm + (2 if self.ins_steps else 0))
        self.Xnew = base_rows(self.name, self.n, n_new) if n_new else None
        self.t_gen = time.time() - t0
        kw = dict(degree=self.R, metric=self.c["metric"], search_width=a.search_width, build_itopk=self.build_L,
                  insert_itopk=self.ins_L)
        if a.insert_batch:
            kw["insert_batch"] = a.insert_batch
        t0 = time.time()
        if self.sharded:
            cap_extra = (n_new + self.S - 1) // self.S
            Xd = torch.from_numpy(X)
            shards = {}
            from paper_2601_08528_b200.sharded import owned_shards

            for s in owned_shards(self.S, D.rank if D.world > 1 else 0, D.world):
                rows = Xd[s::self.S].to(D.dev)
                shards[s] = svf.Index.build(rows, capacity=rows.shape[0] + cap_extra, device=D.dev.index, **kw)
                del rows
            self.sh = ShardedIndex(shards, self.S, D.rank, D.world)
            self.idx = None
        else:
            Xd = torch.from_numpy(X).to(D.dev)
            self.idx = svf.Index.build(Xd, capacity=self.n + n_new, device=D.dev.index, **kw)
            self.sh = None
            del Xd
        torch.cuda.synchronize()
        self.t_build = time.time() - t0
        del X
        self.Qd = torch.from_numpy(self.Q).to(D.dev)
        self.Qsd = torch.from_numpy(self.Qsel).to(D.dev)
        for ix in self.indexes():
            ix.set_search_params(a.search_width, 0, 0, a.hash_bits)
            ix.set_warps_per_query(a.wpq)
            ix.set_search_handoff(a.handoff)

    def indexes(self):
        return list(self.sh.shards.values()) if self.sharded else [self.idx]

    def set_cap(self, cap: int):
        for ix in self.indexes():
            ix.set_search_params(self.a.search_width, 0, cap, self.a.hash_bits)

    def search(self, Q, L: int, k: int | None = None):
        k = k or self.k
        return self.sh.search(Q, k, L) if self.sharded else self.idx.search(Q, k, L)

    def knn(self, Q, k: int | None = None):
        k = k or self.k
        return self.sh.knn_exact(Q, k) if self.sharded else self.idx.knn_exact(Q, k)

    # -- ground truth, selection sweeps ------------------------------------------------------------------------
    def select(self):
        torch, D, a, k = self.torch, self.D, self.a, self.k
        self.knn(self.Qd)                                        # warm-up (tensor maps, scratch)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):                                       # G1: exact kNN on tcgen05, median of 3
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            gi, gd = self.knn(self.Qd)
            g1.record()
            torch.cuda.synchronize()
            ts.append(g0.elapsed_time(g1))
        gt_ms = D.max(float(np.median(ts)))
        self.gt, self.gt_d = gi.cpu().numpy(), gd.cpu().numpy()
        si, sd = self.knn(self.Qsd)
        self.gt_sel = si.cpu().numpy()
        peaks = measured_peaks()
        tf32_peak = peaks.get("bf16_tflops", 1590.0) / 2.0
        tflops = 2.0 * self.nq * self.n * self.dim / (gt_ms * 1e-3) / 1e12
        stats = [ix.knn_stats() for ix in self.indexes()]
        self.out["exact_knn"] = {
            "kernel": "knn_tc_kernel + knn_rerank_kernel (svf_knn_exact)" + (" per shard + merge" if self.sharded else ""),
            "bound": "tensor", "ms": round(gt_ms, 3), "achieved": round(tflops, 1), "unit": "TFLOP/s",
            "peak": tf32_peak, "frac": round(tflops / tf32_peak, 4),
            "peak_source": "measured bf16 dense peak x 1/2 (nominal tf32:bf16 ratio)",
            "fallbacks": int(sum(s["fallbacks"] for s in stats)), "queries": int(sum(s["queries"] for s in stats))}
        # itopk: the lowest whose recall on the SELECTION batch reaches the target, converged (no cap)
        L, sweep = a.itopk if self.headline else 0, []
        for Ls in ([L] if L else L_SWEEP):
            ids, d = self.search(self.Qsd, Ls)
            rec = recall_at_k(ids.cpu().numpy(), self.gt_sel, k)
            sweep.append({"itopk": Ls, "recall_sel": round(rec, 4)})
            if not L and rec >= a.target_recall + a.select_margin:
                L = Ls
                break
        self.L = L or L_SWEEP[-1]
        self.out["itopk_sweep_uncapped"] = sweep
        # then the smallest iteration cap that keeps it there (on the selection batch)
        MI, mi_sweep = max(0, a.max_iter) if self.headline else 0, []
        goal = a.target_recall + a.select_margin
        if (a.max_iter < 0 or not self.headline) and sweep[-1]["recall_sel"] >= goal:
            for cap in mi_caps(self.L):
                self.set_cap(cap)
                ids, d = self.search(self.Qsd, self.L)
                rec = recall_at_k(ids.cpu().numpy(), self.gt_sel, k)
                mi_sweep.append({"max_iter": cap, "recall_sel": round(rec, 4)})
                if rec < goal:
                    break
                MI = cap
        self.MI = MI
        self.set_cap(MI)
        self.out["max_iter_sweep"] = mi_sweep
        # recall of the TIMED batch at the chosen point (id-based and tie-aware, O7)
        ids, d = self.search(self.Qd, self.L)
        self.recall = recall_at_k(ids.cpu().numpy(), self.gt, k)
        self.recall_tie = recall_tie_aware(d.cpu().numpy(), self.gt_d, k)

    # -- timed steps -------------------------------------------------------------------------------------------
    def timed(self):
        torch, D, a = self.torch, self.D, self.a
        k, L, nq = self.k, self.L, self.nq
        dev = D.dev
        out_i = torch.empty((nq, k), dtype=torch.int32, device=dev)
        out_d = torch.empty((nq, k), dtype=torch.float32, device=dev)
        graph = None
        if not self.sharded and not a.no_graph:
            # the step is launch-bound on the host side (ctypes); capture svf_search once and replay it
            self.idx.search_into(self.Qd, k, L, out_i, out_d)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                self.idx.search_into(self.Qd, k, L, out_i, out_d)
            torch.cuda.synchronize()

        def step():
            if graph is not None:
                graph.replay()             # svf_search: work-counter reset + search grid(s)
            else:
                self.search(self.Qd, L)    # sharded: per-shard searches + pre-merge + all-gather + merge

        flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]

        def region():
            clocks = Clocks(dev.index or 0) if not a.ncu else None
            for _ in range(a.warmup):
                step()
            D.barrier()
            torch.cuda.synchronize()
            torch.cuda.profiler.start()                       # ncu --profile-from-start off captures this range
            for i in range(a.steps):
                flush.zero_()                                 # L2 flush between timed iterations
                ev[i][0].record()
                step()
                ev[i][1].record()
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
            D.barrier()
            return sum(e0.elapsed_time(e1) for e0, e1 in ev), (clocks.stop() if clocks else None)

        ms_total, clk = region()
        if clk and (BAD_REASONS & set(clk["reasons"])):      # rejected by the timing rules: re-measure once
            ms_total, clk = region()
            clk["remeasured"] = True
        self.clocks = clk
        self.ms_step = D.max(ms_total) / a.steps
        # queries answered per second over the fixed dataset: replicas answer world x nq distinct queries
        self.value = nq * (D.world if self.mode == "replicas" else 1) / (self.ms_step / 1e3)
        # per-launch duration of the search kernel(s) alone: the library's CUDA events around each launch, on the
        # launching stream, over direct launches with the same L2 flush in between
        for ix in self.indexes():
            ix.profile(True)
        for _ in range(min(a.steps, 50)):
            flush.zero_()
            if self.sharded:
                self.search(self.Qd, L)
            else:
                self.idx.search_into(self.Qd, k, L, out_i, out_d)
        kern_ms, kern_n = 0.0, 0
        for ix in self.indexes():
            pr = ix.profile_read()
            ix.profile(False)
            kern_ms += pr["search"][0]
            kern_n += pr["search"][1]
        per_step = kern_n / max(1, min(a.steps, 50))
        self.kern_ms_per_step = kern_ms / max(1, min(a.steps, 50))     # all search grids of one step
        self.kern_launches = per_step
        cnt = [ix.last_search_counters() for ix in self.indexes()]
        self.gpu_counters = {kk: sum(c[kk] for c in cnt) for kk in ("n_dist", "iters", "n_exp", "queries")}
        self.launches_per_step = int(sum(c["launches"] for c in cnt)) + (2 if self.sharded else 0)
        self.flush = flush

    # -- end to end through the public API: pinned host queries in, host results out ------------------------------
    def e2e(self):
        torch, D, a = self.torch, self.D, self.a
        k, L, nq = self.k, self.L, self.nq
        Qh = torch.from_numpy(self.Q).pin_memory()
        if self.sharded:
            # the sharded path's public API takes device queries: the H2D copy and the D2H read are in the region
            def call():
                Qd = Qh.to(D.dev, non_blocking=True)
                i, d = self.sh.search(Qd, k, L)
                i.cpu()
                d.cpu()
        else:
            oi_h = torch.empty((nq, k), dtype=torch.int32, pin_memory=True)   # pinned result buffers, reused
            od_h = torch.empty((nq, k), dtype=torch.float32, pin_memory=True)

            def call():
                self.idx.search_into(Qh, k, L, oi_h, od_h)    # H2D + kernel + D2H + sync inside svf_search
        for _ in range(max(20, a.warmup)):
            call()
        D.barrier()
        tt = []
        for _ in range(max(60, a.steps // 2)):
            self.flush.zero_()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            call()
            tt.append(time.perf_counter() - t1)
        e2e_s = D.max(float(np.median(tt)))                  # host wall time per step: median (robust to jitter)
        mult = D.world if self.mode == "replicas" else 1
        self.out["e2e"] = {"value": round(nq * mult / e2e_s, 1), "unit": "queries/s",
                           "h2d_bytes_per_step": int(self.Q.nbytes), "d2h_bytes_per_step": int(nq * k * 8),
                           "host_ms_p10_p50_p90": [round(float(np.percentile(tt, p)) * 1e3, 4) for p in (10, 50, 90)],
                           "api": "ShardedIndex.search" if self.sharded else "svf_search (host buffers)"}

    # -- CPU baseline: the oracle as it stands, on the host cores, on the graph just timed (rank 0, N=1 only) ------
    def cpu(self):
        a = self.a
        self.alg = None
        if self.D.world != 1 or a.no_cpu or self.sharded:
            self.out["cpu_baseline"] = None
            return
        import oracle

        st = self.idx.export()
        secs = a.cpu_seconds if self.headline else a.cpu_seconds / 2
        cpu, cnt = cpu_baseline(oracle, st, self.Q, self.k, self.L, secs, self.MI, a.search_width,
                                metric=self.c["metric"])
        self.out["cpu_baseline"] = cpu
        self.alg = {"n_dist": float(cnt[:, 0].mean()), "n_exp": float(cnt[:, 1].mean()),
                    "source": f"oracle counters over {len(cnt)} timed-batch queries"}
        g = self.gpu_counters
        gq = max(1, g["queries"])
        full = len(cnt) == gq
        self.out["search_counters"] = {
            "gpu_n_dist_per_query": round(g["n_dist"] / gq, 2), "oracle_n_dist_per_query": round(float(cnt[:, 0].mean()), 2),
            "recompute_ratio": round(g["n_dist"] / gq / max(1e-9, float(cnt[:, 0].mean())), 4),
            "gpu_iters_per_query": round(g["iters"] / gq, 3), "oracle_iters_per_query": round(float(cnt[:, 2].mean()), 3),
            "iters_equal": bool(full and g["iters"] == int(cnt[:, 2].sum())), "oracle_sample_queries": int(len(cnt)),
            "max_iter": self.MI, "max_iter_cap_hits": int((cnt[:, 2] >= self.MI).sum()) if self.MI else 0}

    def roofline(self):
        if self.alg is None:
            g = self.gpu_counters
            self.alg = {"n_dist": g["n_dist"] / max(1, g["queries"]) * (self.S if self.sharded else 1),
                        "n_exp": g["n_exp"] / max(1, g["queries"]) * (self.S if self.sharded else 1),
                        "source": "GPU counters (include visited-cache recomputes)" +
                                  (f", summed over the {self.S} shards" if self.sharded else "")}
        k, R, dim = self.k, self.R, self.dim
        bq = self.alg["n_dist"] * dim * 4 + self.alg["n_exp"] * R * 4 + dim * 4 + k * 8   # SURVEY §8(d) B_q
        peaks = measured_peaks()
        peak = peaks.get("hbm_gbs", 6650.0)
        achieved = self.nq * bq / (self.kern_ms_per_step / 1e3) / 1e9
        tr = ncu_traffic(self.name)
        self.out["roofline"] = {
            "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": (round(tr["dram_bytes_per_query"] * self.nq) if tr and tr.get("itopk") == self.L else None),
            "kernel": "search_lp_kernel" if self.L > 64 else "search_kernel",
            "kernel_ms_per_step": round(self.kern_ms_per_step, 4), "kernel_launches_per_step": self.kern_launches,
            "alg_bytes_per_query": round(bq, 1), "alg_counts": self.alg,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst, measured)" if peaks else
                           "fallback 6650 GB/s (B200_PROFILING.md)"}

    # -- inserts / deletes (I0-I3, D1) on 1% batches -------------------------------------------------------------
    def updates(self):
        if not self.ins_steps:
            self.out["insert"] = None
            return
        torch, D, a = self.torch, self.D, self.a
        k, L, dim, R = self.k, self.L, self.dim, self.R
        B = self.ins_batch
        Xn = torch.from_numpy(self.Xnew).to(D.dev)
        t_ins, first = [], self.n
        sample_counts = None
        # per-stage breakdown from the warm-up batches (profiling events serialise the stages, which also turns off
        # the PDL chain of the detour selection behind the insert search); the timed batches run unprofiled
        for ix in self.indexes():
            ix.profile(True)
        for j in range(self.ins_warm + self.ins_steps):
            if j == self.ins_warm:
                iprof = {}
                for ix in self.indexes():
                    for kk, v in ix.profile_read().items():
                        iprof[kk] = iprof.get(kk, 0.0) + v[0]
                    ix.profile(False)
            if j == self.ins_warm and D.world == 1 and not self.sharded and not a.no_cpu:
                # B_i from the ORACLE's counters of the insert-mode searches of a sample of the vectors about to be
                # inserted, on the exact snapshot they are searched over
                sample_counts = insert_counts_oracle(self.idx, self.Xnew[j * B:j * B + 256], first, self.ins_L,
                                                     self.c["metric"], a.search_width)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if self.sharded:
                self.sh.insert(Xn[j * B:(j + 1) * B], first)
            else:
                self.idx.insert(Xn[j * B:(j + 1) * B])
            e1.record()
            torch.cuda.synchronize()
            first += B
            if j >= self.ins_warm:
                t_ins.append(e0.elapsed_time(e1))
        rng = np.random.default_rng(1000)
        t_del = []
        for j in range(self.ins_steps):
            ids_del = rng.choice(first, B, replace=False).astype(np.int64)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if self.sharded:
                self.sh.delete(ids_del)
            else:
                self.idx.delete(torch.from_numpy(ids_del.astype(np.int32)).to(D.dev))
            e1.record()
            torch.cuda.synchronize()
            t_del.append(e0.elapsed_time(e1))
        ins_ms, del_ms = D.max(float(np.mean(t_ins))), D.max(float(np.mean(t_del)))
        # every replica applies every update (no write scaling); sharded ranks each apply their shards' part
        ins = {"inserts_per_s": round(B / (ins_ms / 1e3), 1), "deletes_per_s": round(B / (del_ms / 1e3), 1),
               "batch": B, "ms_per_insert_batch": round(ins_ms, 3), "ms_per_delete_batch": round(del_ms, 3),
               "insert_breakdown_ms": {kk: round(v / max(1, self.ins_warm), 3) for kk, v in iprof.items()
                                       if kk != "search"},
               "insert_breakdown_note": "serialised stage times of the profiled warm-up batches",
               "build_inserts_per_s": round(self.n / self.t_build, 1),
               "updates": f"{self.ins_warm + self.ins_steps} insert batches + {self.ins_steps} delete batches of {B} "
                          f"(L_insert {self.ins_L}), random deletes over all ids"}
        # quality after the update rounds (fresh exact ground truth over the live set), at the timed point
        gt2, _ = self.knn(self.Qd)
        gt2 = gt2.cpu().numpy()
        ins["recall_after_updates"] = rnd(recall_at_k(self.search(self.Qd, L)[0].cpu().numpy(), gt2, k))
        gs2 = self.knn(self.Qsd)[0].cpu().numpy()
        self.set_cap(0)
        need = None
        for Ls in [x for x in L_SWEEP if x >= L]:       # itopk that holds the target after the updates (uncapped)
            if recall_at_k(self.search(self.Qsd, Ls)[0].cpu().numpy(), gs2, k) >= a.target_recall:
                need = Ls
                break
        self.set_cap(self.MI)
        ins["itopk_needed_after_updates_uncapped"] = need
        if not self.sharded:
            # localized repair of vertices with > 50% deleted neighbours (NEXT-1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rs = self.idx.repair()
            e1.record()
            torch.cuda.synchronize()
            rep = {"ms": round(D.max(e0.elapsed_time(e1)), 3), **{kk: v for kk, v in rs.items() if kk != "hist"},
                   "recall_after": rnd(recall_at_k(self.search(self.Qd, L)[0].cpu().numpy(), gt2, k))}
            # and the global consolidation (NEXT-4; reading C2: vacancies refilled, live entries kept)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ncons = self.idx.consolidate()
            e1.record()
            torch.cuda.synchronize()
            rep["consolidation"] = {"ms": round(D.max(e0.elapsed_time(e1)), 3), "rewritten": int(ncons),
                                    "recall_after": rnd(recall_at_k(self.search(self.Qd, L)[0].cpu().numpy(), gt2, k))}
            ins["repair"] = rep
            ins["concurrent_search"] = self.concurrent(Xn[(self.ins_warm + self.ins_steps) * B:])
        # insert roofline: B_i = B_q(L_insert; whole pool out) + |C| R 4 + 2 R (R 8) + (D 4 + R 8)
        if sample_counts is not None:
            nd_i, ne_i = float(sample_counts[:, 0].mean()), float(sample_counts[:, 1].mean())
            src = (f"oracle insert-mode counters (L_insert {self.ins_L}) of {len(sample_counts)} of the vectors of the "
                   "first timed insert batch, on the snapshot they were searched over")
        else:
            nd_i, ne_i, src = None, None, None
        if nd_i is not None:
            Li = self.ins_L
            b_i = (nd_i * dim * 4 + ne_i * R * 4 + dim * 4 + Li * 8) + Li * R * 4 + 2 * R * (R * 8) + (dim * 4 + R * 8)
            pk = measured_peaks().get("hbm_gbs", 6650.0)
            ach = B / (ins_ms / 1e3) * b_i / 1e9
            ins["roofline"] = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk, "unit": "GB/s",
                               "frac": round(ach / pk, 4), "alg_bytes_per_insert": round(b_i, 1),
                               "alg_counts": {"n_dist": round(nd_i, 2), "n_exp": round(ne_i, 2), "source": src}}
        self.out["insert"] = ins

    def concurrent(self, Xrest):
        """NEXT-2 / C4's "concurrent search" ("multiple search streams plus one update stream"): the timed
        search batch on stream S while a 1% insert runs on stream U, against each alone; device time
        from a start event on S to both streams' end events; the concurrent results are checked for validity."""
        torch, k, L, B = self.torch, self.k, self.L, self.ins_batch
        s_q, s_u = torch.cuda.Stream(), torch.cuda.Stream()

        def run(do_search, rows):
            t0 = torch.cuda.Event(enable_timing=True)
            eq, eu = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0.record(s_q)
            s_u.wait_event(t0)
            out = None
            if rows is not None:
                with torch.cuda.stream(s_u):
                    self.idx.insert_async(rows)
            if do_search:
                with torch.cuda.stream(s_q):
                    out = self.idx.search(self.Qd, k, L)
            eq.record(s_q)
            eu.record(s_u)
            torch.cuda.synchronize()
            return max(t0.elapsed_time(eq), t0.elapsed_time(eu)), t0.elapsed_time(eq), out

        run(True, None)                                   # warm-up: the first search on s_q allocates its outputs
        t_s, _, _ = run(True, None)
        t_i, _, _ = run(False, Xrest[:B])
        t_b, t_bq, out = run(True, Xrest[B:2 * B])
        ids, d = out[0].cpu().numpy().view(np.uint32), out[1].cpu().numpy()
        bad = int((ids >= self.idx.info()["n_alloc"]).sum()) + int((np.diff(d, axis=1) < 0).sum())
        return {"search_alone_ms": round(t_s, 3), "insert_alone_ms": round(t_i, 3), "both_ms": round(t_b, 3),
                "search_done_under_insert_ms": round(t_bq, 3), "search_behind_insert_same_stream_ms": round(t_s + t_i, 3),
                "invalid_results": bad}

    # -- the JSON block ------------------------------------------------------------------------------------------
    def block(self) -> dict:
        c = self.c
        cfg = {"workload": c["workload"], "n": self.n, "dim": self.dim, "degree": self.R, "batch": self.nq,
               "k": self.k, "metric": "ip" if c["metric"] else "l2", "itopk": self.L,
               "search_width": self.a.search_width, "max_iter": self.MI, "build_itopk": self.build_L,
               "insert_itopk": self.ins_L, "recall_at_10": rnd(self.recall), "recall_at_10_tie_aware": rnd(self.recall_tie),
               "recall_batch": f"timed batch (query seed 2); itopk and max_iter chosen on a held-out batch (seed 3) "
                               f"to reach {self.a.target_recall} + {self.a.select_margin}",
               "l2": "flushed between timed steps (256 MB write)",
               "launch": "CUDA graph replay of svf_search" if (not self.sharded and not self.a.no_graph) else "direct",
               "parallelism": {"single": "1 GPU",
                               "replicas": f"{self.D.world} replicas, each answering its own {self.nq}-query batch",
                               "sharded": f"{self.S} logical shards over {self.D.world} rank(s), per-rank pre-merge, "
                                          "all_gather_into_tensor + svf_merge_pairs"}[self.mode]}
        b = {"value": round(self.value, 1), "unit": "queries/s", "ms_per_step": round(self.ms_step, 4),
             "config": cfg, "roofline": self.out["roofline"], "exact_knn": self.out.get("exact_knn"),
             "cpu_baseline": self.out.get("cpu_baseline"), "e2e": self.out.get("e2e"), "insert": self.out.get("insert"),
             "search_counters": self.out.get("search_counters"),
             "itopk_sweep_uncapped": self.out.get("itopk_sweep_uncapped"),
             "max_iter_sweep": self.out.get("max_iter_sweep"),
             "setup_s": {"gen": round(self.t_gen, 2), "build": round(self.t_build, 2)}}
        return b

    def close(self):
        for ix in self.indexes():
            ix.close()
        self.idx, self.sh = None, None
        self.torch.cuda.empty_cache()


def measure(a, D, config: str, headline: bool) -> tuple:
    r = Run(a, D, config, headline)
    r.build()
    if a.ncu:
        r.L, r.MI = a.itopk or 16, max(0, a.max_iter)
        r.set_cap(r.MI)
        r.recall = r.recall_tie = None
        r.timed()
        return r, None
    r.select()
    r.timed()
    r.e2e()
    r.cpu()
    r.roofline()
    r.updates()
    return r, r.block()


def run_svf(a):
    D = Dist(a.gpus)
    t_start = time.time()
    r, head = measure(a, D, a.config, headline=True)
    clk = r.clocks
    launches = r.launches_per_step
    mode, S = r.mode, r.S
    r.close()
    more = {}
    if D.world == 1 and not a.ncu and not a.no_extra and not a.n and not a.nq:
        for name in [x for x in a.extra.split(",") if x and x != a.config]:
            try:
                rr, blk = measure(a, D, name, headline=False)
                blk["clocks"] = rr.clocks
                more[name] = blk
                rr.close()
            except Exception as e:  # a failed extra config must not lose the headline line
                more[name] = {"error": f"{type(e).__name__}: {e}"}
    if D.rank == 0:
        line = {"metric": METRIC, "value": head["value"] if head else round(r.value, 1), "unit": "queries/s",
                "n_gpus": D.world, "steps": a.steps, "warmup": a.warmup,
                "ms_per_step": head["ms_per_step"] if head else round(r.ms_step, 4), "higher_is_better": True,
                "scaling": "weak" if mode == "replicas" else ("strong" if mode == "sharded" else "weak"),
                "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded G-LM; DESIGN.md §4)",
                "config": head["config"] if head else {"workload": a.config},
                "roofline": head["roofline"] if head else None, "exact_knn": head and head["exact_knn"],
                "cpu_baseline": head and head["cpu_baseline"], "e2e": head and head["e2e"],
                "insert": head and head["insert"], "clocks": clk, "search_counters": head and head["search_counters"],
                "itopk_sweep_uncapped": head and head["itopk_sweep_uncapped"],
                "max_iter_sweep": head and head["max_iter_sweep"],
                # search grids per step [+ pre-merge and merge kernels when sharded], every step
                "gpu_launches": a.steps * launches,
                "setup_s": head and head["setup_s"], "more_configs": more or None,
                "host_cpu": host_cpu(), "wall_s": round(time.time() - t_start, 1)}
        if mode == "sharded":
            line["config"]["shards"] = S
        print(json.dumps(line), flush=True)
    D.close()


def cpu_baseline(oracle, st, Q, k, L, seconds, max_iter=0, p=1, metric=0):
    """Time oracle.graph_search (as it stands) on the exported graph with all host cores, bounded to ~seconds."""
    threads = os.cpu_count() or 1
    X, G = st["vec"], st["graph"]
    tomb = st["tomb"] if st["tomb"].any() else None
    probe = Q[:256]
    t0 = time.perf_counter()
    oracle.graph_search(X, G, probe, k, L, tomb=tomb, n_alloc=st["n_alloc"], threads=threads, max_iter=max_iter, p=p,
                        metric=metric)
    per_q = (time.perf_counter() - t0) / len(probe)
    nq_s = int(min(len(Q), max(256, seconds / max(per_q, 1e-9))))
    sample = Q[:nq_s]
    t0 = time.perf_counter()
    _, _, cnt = oracle.graph_search(X, G, sample, k, L, tomb=tomb, n_alloc=st["n_alloc"], threads=threads,
                                    max_iter=max_iter, p=p, metric=metric)
    dt = time.perf_counter() - t0
    reps = 1
    while dt * (reps + 1) / reps < seconds and reps < 50 and nq_s == len(Q):
        t1 = time.perf_counter()
        oracle.graph_search(X, G, sample, k, L, tomb=tomb, n_alloc=st["n_alloc"], threads=threads, max_iter=max_iter,
                            p=p, metric=metric)
        dt += time.perf_counter() - t1
        reps += 1
    hc = host_cpu()
    return ({"value": round(nq_s * reps / dt, 1), "unit": "queries/s", "cores": threads, "kind": "oracle",
             "cpu_model": hc["model"],
             "sample": f"{nq_s} queries x {reps} pass(es) at itopk={L}, width={p}, max_iter={max_iter} on the exported "
                       f"GPU-built graph (oracle graph_search_ref, std::thread x {threads})"}, cnt)


def insert_counts_oracle(idx, Xs, first: int, L_ins: int, metric: int, p: int):
    """The oracle's O2 counters (n_dist, n_exp, iters) of insert-mode searches of the rows Xs, which are about to
    be inserted as ids first.., over the current state (the first sub-batch's snapshot)."""
    import oracle

    st = idx.export()
    tomb = st["tomb"] if st["tomb"].any() else None
    _, _, cnt = oracle.graph_search(st["vec"], st["graph"], Xs, 1, L_ins, p=p, metric=metric, tomb=tomb,
                                    n_alloc=st["n_alloc"], qidx=np.arange(first, first + len(Xs)), insert_mode=True)
    return cnt


# ---- the reference arm: the oracle, timed on the host cores ---------------------------------------------------------
def run_reference(a):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import torch

    import oracle
    import paper_2601_08528_b200 as svf

    c = config_spec(a.config)
    n = a.n or c["n"]
    nq = a.nq or c["nq"]
    k, R = a.k, c["degree"]
    X = base_rows(a.config, 0, n)
    Q = query_rows(a.config, nq)
    Qsel = query_rows(a.config, nq, row_seed=SELECT_SEED)
    # Input preparation (untimed): the graph is built by svf_build, which is bit-identical to oracle.build on this
    # integer-valued workload (tests/test_gpu_parity.py::test_build_bit_exact_integer_data); exact ground truth by
    # svf_knn_exact.  Only the oracle's search is timed.  Same L_build as the svf arm, so the same graph.
    build_L = a.build_itopk if a.build_itopk >= 0 else BUILD_ITOPK.get(a.config, 0)
    idx = svf.Index.build(torch.from_numpy(X).cuda(), degree=R, metric=c["metric"], build_itopk=build_L)
    gt = idx.knn_exact(torch.from_numpy(Qsel[:1000]).cuda(), k)[0].cpu().numpy()
    st = idx.export()
    idx.close()
    threads = os.cpu_count() or 1
    L = a.itopk
    sweep = []
    probe = Qsel[:1000]
    for Ls in ([L] if L else L_SWEEP):
        ids, _, _ = oracle.graph_search(st["vec"], st["graph"], probe, k, Ls, threads=threads, metric=c["metric"])
        rec = recall_at_k(ids.astype(np.int64).astype(np.int32), gt, k)
        sweep.append({"itopk": Ls, "recall_sel": round(rec, 4)})
        if not L and rec >= a.target_recall + a.select_margin:
            L = Ls
            break
    L = L or L_SWEEP[-1]
    MI, mi_sweep = max(0, a.max_iter), []
    if a.max_iter < 0 and sweep[-1]["recall_sel"] >= a.target_recall + a.select_margin:     # same cap selection as the svf arm
        for cap in mi_caps(L):
            ids, _, _ = oracle.graph_search(st["vec"], st["graph"], probe, k, L, max_iter=cap, threads=threads,
                                            metric=c["metric"])
            rec = recall_at_k(ids.astype(np.int64).astype(np.int32), gt, k)
            mi_sweep.append({"max_iter": cap, "recall_sel": round(rec, 4)})
            if rec < a.target_recall + a.select_margin:
                break
            MI = cap
    t0 = time.perf_counter()
    oracle.graph_search(st["vec"], st["graph"], Q[:256], k, L, threads=threads, max_iter=MI, metric=c["metric"])
    per_q = (time.perf_counter() - t0) / 256
    budget = 150.0 / max(1, a.steps + a.warmup)
    m = int(min(nq, max(64, budget / max(per_q, 1e-9))))
    times = []
    for i in range(a.warmup + a.steps):
        s0 = (i * m) % nq
        sample = np.roll(Q, -s0, axis=0)[:m]
        t1 = time.perf_counter()
        oracle.graph_search(st["vec"], st["graph"], sample, k, L, threads=threads, max_iter=MI, metric=c["metric"])
        if i >= a.warmup:
            times.append(time.perf_counter() - t1)
    ms = 1e3 * float(np.mean(times))
    qps = m / (ms / 1e3)
    hc = host_cpu()
    line = {"impl": "reference", "metric": METRIC,
            "value": round(qps, 1), "unit": "queries/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64-accumulate (fp32 decisions)", "data": "synthetic (seeded G-LM; DESIGN.md §4)",
            "config": {"workload": c["workload"], "n": n, "batch": nq, "k": k, "itopk": L, "max_iter": MI,
                       "max_iter_sweep_1000q": mi_sweep, "build_itopk": build_L, "recall_sweep_1000q": sweep,
                       "step_sample_queries": m},
            "cpu_baseline": {"value": round(qps, 1), "unit": "queries/s", "cores": threads, "kind": "oracle",
                             "cpu_model": hc["model"], "sample": f"{m} queries per step at itopk={L}, max_iter={MI}"},
            "e2e": {"value": round(qps, 1), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_svf(args)
