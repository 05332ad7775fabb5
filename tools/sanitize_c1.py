"""One pass over every kernel family on C1-sized data, for compute-sanitizer (memcheck / racecheck / synccheck):
search (one-warp grid + PDL-chained pair-mode handoff grid, pair mode, K-S-L large pools), insert (search, detour,
reverse), delete, repair, consolidation, exact kNN (tcgen05 + re-rank), the shard pre-merge and pair merge.

  compute-sanitizer --tool racecheck python tools/sanitize_c1.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from workloads import base_rows, query_rows  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    X = base_rows("C1")
    Q = torch.from_numpy(query_rows("C1", 1000)).to(dev)
    idx = svf.Index.build(torch.from_numpy(X[:8000]).to(dev), degree=64, capacity=10_000, seed_size=1000,
                          insert_batch=1000, build_itopk=160)
    idx.set_warps_per_query(1)
    idx.set_search_handoff(100)                       # every straggler handed to the pair-mode grid
    idx.search(Q, 10, 32)
    assert idx.last_search_counters()["launches"] == 2
    idx.set_search_handoff(-1)
    idx.set_warps_per_query(2)
    idx.search(Q[:100], 10, 32)                       # pair mode
    idx.set_warps_per_query(0)
    idx.search(Q, 10, 128)                            # K-S-L
    idx.search(Q, 10, 256)
    idx.insert(torch.from_numpy(X[8000:]).to(dev))   # insert search (K-S-L at L_insert 128), detour, reverse
    idx.delete(torch.arange(0, 10_000, 7, dtype=torch.int32, device=dev))
    idx.repair(8, 0.3)
    idx.consolidate()
    idx.search(Q, 10, 64)
    idx.knn_exact(Q, 10)
    from paper_2601_08528_b200.sharded import ShardedIndex

    sh = ShardedIndex.build(torch.from_numpy(X).to(dev), S=8, degree=16, seed_size=300, insert_batch=300)
    sh.search(Q, 10, 32)
    sh.knn_exact(Q, 10)
    torch.cuda.synchronize()
    print("sanitize pass done", flush=True)


if __name__ == "__main__":
    main()
