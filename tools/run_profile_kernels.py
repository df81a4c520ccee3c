"""Driver for ncu captures of the round's main kernels at their benchmark shapes (one launch each
after a warm-up): CTA-pair FP8 GEMM (cfg4 fwd, 32768x4096x4096 tensorwise, bf16 out), the UE8M0
block-scaled pair GEMM (same shape), streaming rowwise quantize (32768x4096 bf16), the cast-
transpose tile kernel (tensor+transpose), and the probe (32768x4096 bf16 pair)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

M = N = K = 4096
M = 32768
dev = torch.device("cuda")
x = synth.gaussian(M, K, 0, device=dev)
w = synth.weight(N, K, 1, device=dev)
for rep in range(2):
    xq, xs = lk.loka_quantize(x, "e4m3", "tensor")
    wq, ws = lk.loka_quantize(w, "e4m3", "tensor")
    lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="tensor", b_gran="tensor", out_dtype="bf16")
    xb, xbs = lk.loka_quantize(x, "e4m3", "blk_1x128", "ue8m0")
    wb, wbs = lk.loka_quantize(w, "e4m3", "blk_128x128", "ue8m0")
    lk.loka_fp8_linear_norm(xb, xbs, wb, wbs, a_gran="blk_1x128", b_gran="blk_128x128", a_scale_fmt="ue8m0",
                            b_scale_fmt="ue8m0", out_dtype="bf16")
    lk.loka_quantize(x, "e4m3", "row")
    lk.loka_quantize(x, "e4m3", "tensor", transpose=True)
    ref = x
    out = (x.float() * 1.01).to(torch.bfloat16)
    lk.loka_probe_error([(out, ref)])
torch.cuda.synchronize()
print("ok")
