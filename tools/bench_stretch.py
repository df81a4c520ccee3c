"""The paper's largest LRM GEMM (SURVEY.md §8(d) "stretch"): X[2048,123200] . W[1024,123200]^T,
rowwise e4m3, bf16 out.  Only 2048x1024 outputs (32 tiles of 256x256) over a 123200-long K: without
split-K at most 64 of 148 SMs work.  GEMM-only time (operands pre-quantized), CUDA graph, L2 flushed.

  python tools/bench_stretch.py [--out profiles/r01_stretch.json]
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

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402
from bench import ClockSampler, capture, peaks, time_steps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=2048)
    ap.add_argument("--K", type=int, default=123200)
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    _clk = ClockSampler(torch.cuda.current_device())  # NVML clocks during the whole measurement
    _clk.__enter__()
    M, K, N = a.M, a.K, a.N
    dev = torch.device("cuda")
    x = synth.heavy(M, K, 3, device=dev)
    w = synth.weight(N, K, 4, device=dev)
    xq, xs = lk.loka_quantize(x, "e4m3", "row")
    wq, ws = lk.loka_quantize(w, "e4m3", "row")
    del x, w
    stream = torch.cuda.Stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    keep = []
    args, y, _ = lk.make_linear_args(xq, xs, wq, ws, out_dtype="bf16", keep=keep)
    ws_t = torch.empty(max(1, lk.linear_workspace(args)), dtype=torch.uint8, device=dev)
    sh = stream.cuda_stream
    fn = lambda: lk._lib.loka_fp8_linear_norm(ctypes.byref(args), ctypes.c_void_p(ws_t.data_ptr()), ws_t.numel(), sh)
    with torch.cuda.stream(stream):
        g = capture(fn, stream)
        t = time_steps(g.replay, a.steps, 3, flush, stream)
    ms = sum(t) / len(t)
    fl = 2.0 * M * N * K
    bf16_peak, _, _, src = peaks()
    # BF16 reference time on the same shape
    xb = synth.heavy(M, K, 3, device=dev)
    wb = synth.weight(N, K, 4, device=dev)
    yb = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    with torch.cuda.stream(stream):
        gb = capture(lambda: torch.matmul(xb, wb.t(), out=yb), stream)
        tb = time_steps(gb.replay, a.steps, 3, flush, stream)
    msb = sum(tb) / len(tb)
    res = {"workload": f"stretch GEMM M={M} K={K} N={N} rowwise e4m3, bf16 out", "ms": round(ms, 4),
           "tflops": round(fl / ms / 1e9, 1), "frac_of_measured_fp8_peak": round(fl / ms / 1e9 / (2 * bf16_peak), 4),
           "frac_of_4500": round(fl / ms / 1e9 / 4500, 4), "bf16_ms": round(msb, 4),
           "bf16_tflops": round(fl / msb / 1e9, 1), "speedup_vs_bf16": round(msb / ms, 3), "peak_source": src}
    _clk.__exit__()
    res["clocks"] = _clk.summary()
    print(json.dumps(res))
    if a.out:
        open(a.out, "w").write(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
