"""Two NCCL ranks on two B200s (skipped with fewer GPUs): the N-sharded GEMM, the NCCL
all-gather of C and the fused GEMM + gather kernel across real NVLink peers, against
the CPU oracle (tests/dist_worker_gpu.py).  SURVEY 8(e); BASELINE.json north_star."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs (this pool's gpurun gives one)")
def test_two_rank_nshard_nccl_and_fused_gather(tmp_path):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "dist.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "dist_worker_gpu.py"), str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["nranks"] == 2
    for acc in ("f32", "f16"):
        assert res[acc]["bitwise_equal"], res
