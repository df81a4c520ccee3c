"""One configuration of the pair-norm / plain pair GEMM, launched `--reps` times (for ncu captures).
  LOKA_PAIRNORM=256|512 LOKA_PAIR_WIDE=0|1 python tools/run_pairnorm_once.py --M 32768 --norm layer|none
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=32768)
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--norm", default="layer")
ap.add_argument("--act", default="none")
ap.add_argument("--out", default="bf16")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
x = synth.heavy(a.M, a.K, 3, device="cuda")
w = synth.weight(a.N, a.K, 4, device="cuda")
xq, xs = lk.loka_quantize(x, "e4m3", "tensor")
wq, ws = lk.loka_quantize(w, "e4m3", "tensor")
for _ in range(a.reps):
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="tensor", b_gran="tensor", norm=a.norm, act=a.act,
                                   norm_block=256, out_dtype=a.out)
torch.cuda.synchronize()
print("ok", float(y.float().abs().mean()))
