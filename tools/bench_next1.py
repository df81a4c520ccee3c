"""NEXT-1 measurement: one LRM layer with BlockNorm-256 + Hard
Swish fused into the FP8 GEMM epilogue vs the BF16 path (cuBLAS F.linear, then the grouped RMSNorm
and hardswish as separate torch ops).  Shapes: the cfg2 layer sizes at M=4096 and a cfg5-size layer.

  python tools/bench_next1.py [--out profiles/r01_next1.json]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402
from bench import ClockSampler, capture, time_steps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    _clk = ClockSampler(torch.cuda.current_device())  # NVML clocks during the whole measurement
    _clk.__enter__()
    dev = torch.device("cuda")
    stream = torch.cuda.Stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    res = {"what": "linear + BlockNorm(256) + Hard Swish; FP8: bf16 X quantized rowwise in the step, "
                   "fused epilogue, e4m3 (+row scales) out; BF16: F.linear + rms over 256-blocks + hardswish",
           "cases": []}
    for M, K, N in [(4096, 1024, 1024), (4096, 512, 1024), (32768, 4096, 4096)]:
        x = synth.heavy(M, K, 1, device=dev)
        w = synth.weight(N, K, 2, device=dev)
        wq, wsc = lk.loka_quantize(w, "e4m3", "row")
        xq = torch.empty(M, K, dtype=torch.uint8, device=dev)
        xs = torch.empty(M, dtype=torch.float32, device=dev)
        keep = []
        od = "e4m3" if N <= 2048 else "bf16"  # FP8 out needs the whole row in one cluster (N <= 2048)
        args, y, ys = lk.make_linear_args(xq, xs, wq, wsc, norm="block_rms", norm_block=256, act="hardswish",
                                          out_dtype=od, keep=keep)
        sh = stream.cuda_stream

        def fp8_step():
            lk.loka_quantize(x, "e4m3", "row", out=xq, scales=xs, stream=stream)
            st = lk._lib.loka_fp8_linear_norm(ctypes.byref(args), None, 0, sh)
            assert st == 0, st

        wb = w

        def bf16_step():
            yb = F.linear(x, wb)
            yb = F.rms_norm(yb.view(M, N // 256, 256), (256,), eps=1e-6).view(M, N)
            return F.hardswish(yb)

        with torch.cuda.stream(stream):
            t8 = time_steps(capture(fp8_step, stream).replay, a.steps, 3, flush, stream)
            tb = time_steps(capture(bf16_step, stream).replay, a.steps, 3, flush, stream)
        ms8, msb = sum(t8) / len(t8), sum(tb) / len(tb)
        fl = 2.0 * M * N * K
        res["cases"].append({"M": M, "K": K, "N": N, "fp8_out": od, "fp8_fused_ms": round(ms8, 4), "bf16_ms": round(msb, 4),
                             "fp8_tflops": round(fl / ms8 / 1e9, 1), "bf16_tflops": round(fl / msb / 1e9, 1),
                             "speedup": round(msb / ms8, 3)})
    _clk.__exit__()
    res["clocks"] = _clk.summary()
    print(json.dumps(res))
    if a.out:
        open(a.out, "w").write(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
