"""Row-sharded step across PROCESSES on one GPU: every rank a separate process (torchrun, gloo
for the one-time IPC-handle exchange) on cuda:0, the peer-memory exchange with no NCCL
communicator.  This runs on a one-GPU box the cross-process pieces the loopback group cannot
reach — CUDA IPC windows opened by another process, the system-scope device barriers (release /
acquire epoch flags), K-Interleaving's per-(phase, pack) split barriers on two streams, and CUDA
graph replay of a whole row-sharded step — checked against the oracle like tests/nccl_worker.py
(forward bit-exact, every rank's shard bit-exact under dyadic dY).  The processes time-slice the
GPU, so a barrier wait spans a context switch: slow, but each case is a few seconds."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("W", [2, 3])
@pytest.mark.parametrize("name", ["toy", "wdl", "criteo", "uneven", "toy_graph", "criteok2", "criteok2_graph", "wdlk",
                                  "wdlk_graph"])
def test_xproc_same_gpu_parity(name, W):
    if W == 3 and name not in ("toy", "criteok2", "wdlk"):
        pytest.skip("W = 3 (non-power-of-two owner arithmetic): two cases suffice")
    import __graft_entry__

    __graft_entry__.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={W}",
           "--master-addr=127.0.0.1", "--master-port=29541", os.path.join(ROOT, "tests", "nccl_worker.py"), name]
    env = {**os.environ, "PICASSO_EXCHANGE": "p2p", "PICASSO_XPROC_SAMEDEV": "1"}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
