"""Profile one 1% insert batch (10K) into the C2 index: run under ncu --profile-from-start off."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08528_b200 as svf  # noqa: E402
from workloads import base_rows  # noqa: E402

X = base_rows("C2")
Xn = torch.from_numpy(base_rows("C2", 1_000_000, 20_000)).cuda()
idx = svf.Index.build(torch.from_numpy(X).cuda(), degree=64, capacity=1_020_000)
idx.insert(Xn[:10_000])
torch.cuda.synchronize()
torch.cuda.profiler.start()
idx.insert(Xn[10_000:])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
