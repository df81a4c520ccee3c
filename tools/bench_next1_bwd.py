"""NEXT-1 backward measurement: dL/dz of a LayerNorm layer fused into the dgrad GEMM epilogue
(dh = dY . W, then the norm backward with the forward's saved x-hat / rstd) vs the BF16 path
(cuBLAS dY @ W, then aten's native_layer_norm_backward).  FP8 step = rowwise e5m2 quantize of dY +
one fused launch (bf16 or e5m2 dz out).  CUDA graphs, L2 flushed, CUDA events.

  python tools/bench_next1_bwd.py [--out profiles/r01_next1_bwd.json]
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
    res = {"what": "dz = LayerNorm backward(dh = dY . W) with saved x-hat/rstd; FP8: e5m2 rowwise dY quantize + "
                   "fused dgrad GEMM + norm-backward epilogue; BF16: cuBLAS matmul + aten native_layer_norm_backward",
           "cases": []}
    for M, N, K2 in [(4096, 1024, 1024), (32768, 2048, 2048), (32768, 4096, 4096)]:
        dy = synth.grad(M, K2, 1, device=dev) * 1024
        w = synth.weight(K2, N, 2, device=dev)          # dh = dY @ w  -> [M, N]; B (K-major) = w^T [N, K2]
        wtq, wts = lk.loka_quantize(w.t().contiguous(), "e4m3", "row")
        z = synth.gaussian(M, N, 3, device=dev).float()
        mean = z.mean(1)
        rstd = torch.rsqrt(z.var(1, unbiased=False) + 1e-5)
        xh = ((z - mean[:, None]) * rstd[:, None]).to(torch.bfloat16)
        dq = torch.empty(M, K2, dtype=torch.uint8, device=dev)
        ds = torch.empty(M, dtype=torch.float32, device=dev)
        sh = stream.cuda_stream
        row = {"M": M, "N": N, "K": K2}
        for od in ("bf16", "e5m2", "e5m2_1x128"):
            keep = []
            yg = "blk_1x128" if od.endswith("1x128") else "row"
            args, y, _ = lk.make_linear_args(dq, ds, wtq, wts, a_fmt="e5m2", norm="layer", out_dtype=od[:4],
                                             bwd_xhat=xh, bwd_rstd=rstd, direction="dgrad", keep=keep, y_gran=yg)

            wsb = torch.empty(max(1, lk.linear_workspace(args)), dtype=torch.uint8, device=dev)
            tiles = -(-M // 256) * -(-N // 256)
            row[f"path_{od}"] = ("CTA-pair engine, norm backward fused in its epilogue (pairnorm.cu)"
                                 if od in ("bf16", "e5m2_1x128") and (tiles >= 74 or od != "bf16") else
                                 "CTA-pair GEMM (FP32) + row-wise backward pass (FP8 dz needs the row amax)"
                                 if tiles >= 74 else "single-CTA fused epilogue (linear.cu)")

            def fp8_step():
                lk.loka_quantize(dy, "e5m2", "row", out=dq, scales=ds, stream=stream)
                st = lk._lib.loka_fp8_linear_norm(ctypes.byref(args), ctypes.c_void_p(wsb.data_ptr()), wsb.numel(), sh)
                assert st == 0, st
            with torch.cuda.stream(stream):
                t8 = time_steps(capture(fp8_step, stream).replay, a.steps, 3, flush, stream)
            row[f"fp8_{od}_ms"] = round(sum(t8) / len(t8), 4)
        zb, wb, dyb = z.to(torch.bfloat16), w, dy
        mb, rb = mean, rstd

        def bf16_step():
            dh = torch.matmul(dyb, wb)
            return torch.ops.aten.native_layer_norm_backward(dh, zb, [N], mb, rb, None, None, [True, False, False])
        with torch.cuda.stream(stream):
            tb = time_steps(capture(bf16_step, stream).replay, a.steps, 3, flush, stream)
        row["bf16_ms"] = round(sum(tb) / len(tb), 4)
        fl = 2.0 * M * N * K2
        row["fp8_bf16out_tflops"] = round(fl / row["fp8_bf16_ms"] / 1e9, 1)
        row["speedup_bf16out"] = round(row["bf16_ms"] / row["fp8_bf16_ms"], 3)
        row["speedup_e5m2out"] = round(row["bf16_ms"] / row["fp8_e5m2_ms"], 3)
        row["speedup_e5m2out_1x128_fused"] = round(row["bf16_ms"] / row["fp8_e5m2_1x128_ms"], 3)
        res["cases"].append(row)
    _clk.__exit__()
    res["clocks"] = _clk.summary()
    print(json.dumps(res))
    if a.out:
        open(a.out, "w").write(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
