"""One production cfg2 stack launch after warm-ups (for ncu captures of stack_kernel<false, 4, L2StAsync>)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

DIMS = synth.CFG2_DIMS
x = synth.gaussian(4096, DIMS[0], 0, device="cuda")
xq, xs = lk.loka_quantize(x, "e4m3", "row")
ws = [lk.loka_quantize(synth.weight(DIMS[l + 1], DIMS[l], 100 + l, device="cuda"), "e4m3", "row") for l in range(8)]
for _ in range(4):
    y, _ = lk.loka_fp8_mlp_stack(xq, xs, ws, norms="layer", out_dtype="bf16")
torch.cuda.synchronize()
print("ok")
