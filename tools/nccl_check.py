"""Multi-rank check of the sharded path (NCCL all-gather + svf_merge_topk) against a single-index exact reference.
Run under torchrun; SVF_SAME_DEVICE=1 puts every rank on cuda:0 (for a 1-GPU box, if NCCL allows it).

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


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev_idx = 0 if os.environ.get("SVF_SAME_DEVICE") else int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", dev_idx)
    torch.cuda.set_device(dev)
    backend = os.environ.get("SVF_BACKEND", "nccl")
    dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    gen = GLM(dim=64, ell=16, integer=True)
    n = 40_000
    X = gen.rows(5, 5, 0, n)                    # the global dataset (every rank generates it)
    Q = gen.rows(5, 6, 0, 500)
    gid = np.arange(rank, n, world)             # shard r holds global ids g = l*G + r
    idx = svf.Index.build(torch.from_numpy(X[gid]).to(dev), degree=32, device=dev_idx)
    sh = ShardedIndex(idx, rank, world)
    gi, gd = sh.knn_exact(torch.from_numpy(Q).to(dev), 10)     # exact over the union of the shards
    ids, d = sh.search(torch.from_numpy(Q).to(dev), 10, 64)
    torch.cuda.synchronize()
    ok = True
    if rank == 0:
        full = svf.Index.build(torch.from_numpy(X).to(dev), degree=32, device=dev_idx)
        fi, fd = full.knn_exact(torch.from_numpy(Q).to(dev), 10)
        same = np.array_equal(gi.cpu().numpy(), fi.cpu().numpy()) and np.array_equal(gd.cpu().numpy(), fd.cpu().numpy())
        rec = float((ids.cpu().numpy()[:, :, None] == fi.cpu().numpy()[:, None, :]).any(axis=2).mean())
        print(f"world={world} backend={backend}: sharded exact kNN == single-index exact kNN: {same}; "
              f"sharded graph-search recall@10 = {rec:.4f}", flush=True)
        ok = same and rec > 0.9
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
