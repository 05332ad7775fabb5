"""Multi-rank check of the sharded path: 8 logical shards over the ranks, per-rank pre-merge
(svf_shard_premerge), one all_gather_into_tensor of packed pairs, svf_merge_pairs -- against a single-index exact
reference and against the same 8 shards searched in one process.  Run under torchrun; SVF_SAME_DEVICE=1 puts every
rank on cuda:0 (then SVF_BACKEND=gloo: NCCL refuses two ranks on one device).

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 tools/nccl_check.py
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from paper_2601_08528_b200.sharded import ShardedIndex  # noqa: E402
from workloads import GLM  # noqa: E402

S = 8


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev_idx = 0 if os.environ.get("SVF_SAME_DEVICE") else int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", dev_idx)
    torch.cuda.set_device(dev)
    backend = os.environ.get("SVF_BACKEND", "nccl")
    dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    gen = GLM(dim=64, ell=16, integer=True)
    n = 40_000
    X = torch.from_numpy(gen.rows(5, 5, 0, n)).to(dev)       # the global dataset (every rank generates it)
    Q = torch.from_numpy(gen.rows(5, 6, 0, 500)).to(dev)
    sh = ShardedIndex.build(X, S=S, rank=rank, world=world, degree=32, device=dev_idx)
    gi, gd = sh.knn_exact(Q, 10)                              # exact over the union of the shards
    ids, d = sh.search(Q, 10, 64)
    torch.cuda.synchronize()
    ok = True
    if rank == 0:
        full = svf.Index.build(X, degree=32, device=dev_idx)
        fi, fd = full.knn_exact(Q, 10)
        same = np.array_equal(gi.cpu().numpy(), fi.cpu().numpy()) and np.array_equal(gd.cpu().numpy(), fd.cpu().numpy())
        # the same 8 shards in this one process (G = 1): graph search must give the identical merged answer
        one = ShardedIndex.build(X, S=S, rank=0, world=1, degree=32, device=dev_idx)
        oi, od = one.search(Q, 10, 64)
        regroup = np.array_equal(oi.cpu().numpy(), ids.cpu().numpy()) and np.array_equal(od.cpu().numpy(), d.cpu().numpy())
        rec = float((ids.cpu().numpy()[:, :, None] == fi.cpu().numpy()[:, None, :]).any(axis=2).mean())
        print(f"world={world} backend={backend}: sharded exact kNN == single-index exact kNN: {same}; "
              f"G={world} search == G=1 search: {regroup}; sharded graph-search recall@10 = {rec:.4f}", flush=True)
        ok = same and regroup and rec > 0.9
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
