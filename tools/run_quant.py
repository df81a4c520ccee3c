"""Minimal driver for profiling the quantize kernels at the cfg4 shape (32768 x 4096 bf16)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

R, Cc = 32768, 4096
x = synth.heavy(R, Cc, 3, device="cuda")
for _ in range(2):
    lk.loka_quantize(x, "e4m3", "row")
    lk.loka_quantize(x, "e4m3", "tensor", transpose=True)
torch.cuda.synchronize()
print("ok")
