"""One large-pool search inside a cudaProfilerStart/Stop range, for ncu --profile-from-start off: C2 (graph grown at
L_build 256) searched at itopk 128 by 4096 fresh vectors (the insert sub-batch shape), or C4 at itopk 192 by its 10K
OOD queries.   python tools/lp_prof.py [--config C4]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from workloads import base_rows, config_spec, query_rows  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
a = ap.parse_args()
c4 = a.config == "C4"
X = base_rows(a.config)
idx = svf.Index.build(torch.from_numpy(X).cuda(), degree=64, build_itopk=512 if c4 else 256,
                      metric=config_spec(a.config)["metric"])
Q = torch.from_numpy(query_rows("C4") if c4 else base_rows("C2", len(X), 4096)).cuda()
L = 192 if c4 else 128
for _ in range(2):
    idx.search(Q, 10, L)
torch.cuda.synchronize()
torch.cuda.profiler.start()
idx.search(Q, 10, L)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
