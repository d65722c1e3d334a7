"""The NCCL transport at world size 2 (one process per GPU, torchrun over 127.0.0.1): the
library's own distributed loops over real ncclSend/ncclRecv, ncclAllGather and ncclBroadcast,
each rank checked against the oracle on the undivided array (tests/workers/nccl_ranks.py).
Skips on a box with fewer than 2 GPUs; the same loops run at p = 2..8 on one GPU through the
virtual-rank transport (tests/test_gpu_virtual_ranks.py)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_nccl_two_ranks_vs_oracle():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "workers", "nccl_ranks.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "NCCL-RANKS OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
