"""-m gpu: the quantized DP gradient reduction (NEXT-4, D39).  loka_dequant_reduce with P
simulated ranks on one GPU against oracle/gradcomm.py (bit-exact on representable gradients, FP32
tolerance otherwise); the multi-rank protocol (p2p over CUDA IPC and the NCCL all_to_all baseline)
under torchrun when >= 2 GPUs are visible (tools/dist_grad_check.py)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, f64

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("fmt", ["e4m3", "e5m2"])
def test_exact_on_representable_gradients(fmt):
    g = torch.Generator().manual_seed(5)
    P, rows, cols = 8, 96, 256
    grads = [(torch.randint(-3, 4, (rows, cols), generator=g) * 2.0 ** torch.randint(-2, 3, (rows, 1), generator=g))
             .float() for _ in range(P)]
    # power-of-two (UE8M0) row scales: every product and partial sum is exact in FP32
    qs = [lk.loka_quantize(x.to(DEV), fmt, "row", "ue8m0") for x in grads]
    y = lk.loka_dequant_reduce([q for q, _ in qs], [s for _, s in qs], fmt)
    torch.cuda.synchronize()
    ref = oracle.gradcomm.reduce_dequantized([q.cpu().numpy() for q, _ in qs], [s.cpu().numpy() for _, s in qs], fmt)
    assert np.array_equal(f64(y), ref)


@pytest.mark.parametrize("P,rows,cols", [(1, 7, 16), (2, 300, 4096), (3, 129, 1040), (8, 1000, 512)])
def test_vs_oracle(P, rows, cols):
    grads = [synth.grad(rows, cols, 40 + p) for p in range(P)]
    codes, scales = [], []
    for x in grads:
        q, s = lk.loka_quantize(x.to(DEV), "e5m2", "row")
        codes.append(q)
        scales.append(s)
    y = lk.loka_dequant_reduce(codes, scales, "e5m2")
    torch.cuda.synchronize()
    ref = oracle.gradcomm.reduce_dequantized([q.cpu().numpy() for q in codes], [s.cpu().numpy() for s in scales])
    mag = sum(np.abs(oracle.quantize.dequantize(q.cpu().numpy(), s.cpu().numpy(), "e5m2", "row"))
              for q, s in zip(codes, scales))
    assert (np.abs(f64(y) - ref) <= P * 2.0 ** -24 * mag + 1e-30).all()
    ro, _, _ = oracle.gradcomm.quantized_allreduce([x.double().numpy() for x in grads], "e5m2")
    assert np.array_equal(ro, ref)  # the device quantize feeding the reduction is the oracle's


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_multi_rank_protocol(transport):
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "dist_grad_check.py"), transport,
           "1024", "1024"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["ok"] and line["world"] == n
