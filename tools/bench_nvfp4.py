"""NEXT-4 NVFP4 forward (D35-D38) vs the FP8 tensorwise path and BF16 cuBLAS on the same shapes.

  python tools/bench_nvfp4.py [--out profiles/r01_nvfp4.json]

Per shape: the NVFP4 GEMM alone (operands already quantized; bf16 out), the NVFP4 forward incl. the
quantize of X and W (tensor amax pass + cast each), the FP8 tensorwise GEMM / forward, BF16 F.linear.
CUDA-graph replays, L2 flushed before each, CUDA events.  FP4 peak = 4 x the measured BF16 peak
(nominal dense 9 PF / 2.25 PF, blackwell guide)."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402
from bench import ClockSampler, capture, peaks, time_steps  # noqa: E402

SHAPES = [(32768, 4096, 4096), (8192, 4096, 4096), (4096, 1024, 1024), (2048, 2048, 2048)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    _clk = ClockSampler(torch.cuda.current_device())  # NVML clocks during the whole measurement
    _clk.__enter__()
    dev = torch.device("cuda")
    stream = torch.cuda.Stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    bf16_peak, _, _, src = peaks()
    res = {"fp4_peak_tflops": 4 * bf16_peak, "fp8_peak_tflops": 2 * bf16_peak, "peak_source": src, "shapes": []}

    def tmean(fn):
        g = capture(fn, stream)
        t = time_steps(g.replay, a.steps, a.warmup, flush, stream)
        return sum(t) / len(t)

    for M, N, K in SHAPES:
        x = synth.gaussian(M, K, 0, device=dev)
        w = synth.weight(N, K, 1, device=dev)
        fl = 2.0 * M * N * K
        with torch.cuda.stream(stream):
            qa, qb = lk.loka_quantize_nvfp4(x), lk.loka_quantize_nvfp4(w)
            args, y, _ = lk.make_nvfp4_linear_args(qa, qb, out_dtype="bf16")
            nws = int(lk._lib.loka_nvfp4_linear_workspace_size(lk.C.byref(args)))
            ws = torch.empty(nws, dtype=torch.uint8, device=dev)
            xq8, xs8 = lk.loka_quantize(x, "e4m3", "tensor")
            wq8, ws8 = lk.loka_quantize(w, "e4m3", "tensor")
        torch.cuda.synchronize()

        def nv_gemm():
            lk.loka_nvfp4_linear_norm(qa, qb, ws=ws, out_dtype="bf16", y=y, stream=stream)

        def nv_fwd():
            lk.loka_quantize_nvfp4(x, out=qa, stream=stream)
            lk.loka_quantize_nvfp4(w, out=qb, stream=stream)
            lk.loka_nvfp4_linear_norm(qa, qb, ws=ws, out_dtype="bf16", y=y, stream=stream)

        def f8_gemm():
            lk.loka_fp8_linear_norm(xq8, xs8, wq8, ws8, a_gran="tensor", b_gran="tensor", out_dtype="bf16",
                                    stream=stream)

        def f8_fwd():
            lk.loka_quantize(x, "e4m3", "tensor", out=xq8, scales=xs8, stream=stream)
            lk.loka_quantize(w, "e4m3", "tensor", out=wq8, scales=ws8, stream=stream)
            f8_gemm()

        def bf16():
            torch.nn.functional.linear(x, w)

        r = {"M": M, "N": N, "K": K}
        for name, fn in [("nvfp4_gemm", nv_gemm), ("nvfp4_fwd", nv_fwd), ("fp8_tensorwise_gemm", f8_gemm),
                         ("fp8_tensorwise_fwd", f8_fwd), ("bf16_cublas", bf16)]:
            ms = tmean(fn)
            r[name] = {"ms": round(ms, 5), "tflops": round(fl / (ms * 1e-3) / 1e12, 1)}
        r["nvfp4_gemm"]["frac_of_fp4_peak"] = round(r["nvfp4_gemm"]["tflops"] / (4 * bf16_peak), 3)
        r["nvfp4_fwd_speedup_vs_bf16"] = round(r["bf16_cublas"]["ms"] / r["nvfp4_fwd"]["ms"], 3)
        r["fp8_fwd_speedup_vs_bf16"] = round(r["bf16_cublas"]["ms"] / r["fp8_tensorwise_fwd"]["ms"], 3)
        res["shapes"].append(r)
        print(json.dumps(r), flush=True)
    _clk.__exit__()
    res["clocks"] = _clk.summary()
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
