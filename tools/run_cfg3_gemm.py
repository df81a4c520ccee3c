"""Minimal driver for profiling: the cfg3 64-GEMM grouped FP8 launch, repeated R times."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

dev = torch.device("cuda")
S, M = synth.CFG3_DIMS, 2048
R = int(os.environ.get("R", "3"))
keep, args = [], []
for i, k in enumerate(S):
    xq, xs = lk.loka_quantize(synth.gaussian(M, k, i, device=dev), "e4m3", "row")
    for j, n in enumerate(S):
        wq, ws = lk.loka_quantize(synth.weight(n, k, 1000 + 8 * i + j, device=dev), "e4m3", "row")
        a, y, _ = lk.make_linear_args(xq, xs, wq, ws, out_dtype="bf16", keep=keep)
        args.append(a)
for _ in range(R):
    lk.loka_grouped_fp8_linear(args)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(10):
    lk.loka_grouped_fp8_linear(args)
ev[1].record()
torch.cuda.synchronize()
print(f"grouped 64-GEMM call: {ev[0].elapsed_time(ev[1]) / 10 * 1e3:.1f} us (no L2 flush, host enqueue included)")
