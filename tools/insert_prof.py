"""Profile one 1% insert batch (10K) into the C2 index as bench.py builds it (L_build 256, L_insert 128).
Run under ncu --profile-from-start off: only the second insert batch is in the profiled range."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from workloads import base_rows  # noqa: E402

L_BUILD = int(os.environ.get("SVF_L_BUILD", "256"))
X = base_rows("C2")
Xn = torch.from_numpy(base_rows("C2", 1_000_000, 20_000)).cuda()
idx = svf.Index.build(torch.from_numpy(X).cuda(), degree=64, capacity=1_020_000, build_itopk=L_BUILD)
idx.insert(Xn[:10_000])
torch.cuda.synchronize()
torch.cuda.profiler.start()
idx.insert(Xn[10_000:])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
