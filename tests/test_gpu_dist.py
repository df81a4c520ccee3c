"""-m gpu: the sharded tensorwise quantize over real NCCL (a9).  With >= 2 visible GPUs it runs
tools/dist_check.py under torchrun (bit-identity of the gathered codes with the single-GPU and
oracle quantization); with one GPU it runs the same script as a single rank."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_sharded_tensorwise_over_nccl():
    n = min(torch.cuda.device_count(), 4)
    script = os.path.join(ROOT, "tools", "dist_check.py")
    if n >= 2:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), script, "8192", "1024"]
    else:
        cmd = [sys.executable, script, "8192", "1024"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["bit_identical"] and line["world"] == n
