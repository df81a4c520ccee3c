"""Minimal driver for profiling the quantize kernels at the cfg4 shape (32768 x 4096 bf16):
  python tools/run_quant.py [gran ...]   (default: blk_1x128 blk_128x128 blk_128x1 dual)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

R, Cc = 32768, 4096
x = synth.heavy(R, Cc, 3, device="cuda")
grans = sys.argv[1:] or ["blk_1x128", "blk_128x128", "blk_128x1", "dual"]
for _ in range(2):
    for g in grans:
        if g == "dual":
            lk.loka_quantize(x, "e4m3", "blk_1x128", "ue8m0", transpose=True, gran_t="blk_1x128")
        else:
            lk.loka_quantize(x, "e4m3", g)
torch.cuda.synchronize()
print("ok")
