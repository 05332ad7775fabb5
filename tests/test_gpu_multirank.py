"""Multi-process sharded search on the GPU kernels (tools/nccl_check.py under torchrun).  One GPU box => every rank
shares cuda:0 and the all-gather runs over gloo (NCCL refuses duplicate devices); the kernels (per-shard search,
exact kNN, svf_merge_topk) and the host plumbing are the production ones."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.timeout(600)
def test_sharded_search_multi_process(world):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, SVF_SAME_DEVICE="1", SVF_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                          "--master-addr", "127.0.0.1", "--master-port", str(29530 + world),
                          os.path.join(ROOT, "tools", "nccl_check.py")], env=env, capture_output=True, text=True,
                         timeout=540)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "sharded exact kNN == single-index exact kNN: True" in out.stdout
    assert "G=1 search: True" in out.stdout
