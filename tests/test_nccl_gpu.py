"""Row-sharded parity with one process per GPU (torchrun): the NVLink peer-memory exchange
(CUDA IPC windows) and the NCCL grouped send/recv.  Needs >= 2 GPUs (skipped otherwise; the loopback tests cover W up to 8 on one GPU)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
@pytest.mark.parametrize("name", ["toy", "wdl", "toy_cache", "wdl_cache", "criteo", "uneven", "toy_graph",
                                  "criteo_graph", "criteok2", "criteok2_graph", "wdlk", "wdlk_graph"])
def test_nccl_sharded_parity(name, exchange):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    if name.endswith("_graph") and exchange == "nccl":
        pytest.skip("the NCCL exchange synchronises with the host inside a step: not capturable")
    import __graft_entry__

    __graft_entry__.build()
    W = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={W}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "nccl_worker.py"), name]
    env = {**os.environ, "PICASSO_EXCHANGE": exchange}
    if name.endswith("_cache") and exchange == "nccl":
        env["PICASSO_NVLS"] = "0"
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
