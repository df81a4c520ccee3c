"""Minimal driver for profiling the probe kernels (one 32768 x 4096 bf16 pair)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

ref = synth.gaussian(32768, 4096, 10, device="cuda")
out = (ref.float() * 1.01).to(torch.bfloat16)
for _ in range(2):
    lk.loka_probe_error([(out, ref)])
torch.cuda.synchronize()
print("ok")
