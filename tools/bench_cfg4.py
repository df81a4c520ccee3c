"""cfg4 (BASELINE.json configs[3]): training step fwd + dgrad + wgrad, M=32768, K=N=4096, e4m3
X/W and e5m2 dY, tensorwise vs blockwise (1x128 x 128x128, FP32 promotion) vs the BF16 path.

  python tools/bench_cfg4.py [--steps 20] [--warmup 3] [--out profiles/r01_cfg4.json]

Per recipe: each GEMM alone (compute-only: operands already quantized) and the whole step
(end-to-end: every quantize incl. the cast-transposed K-major copies + the three GEMMs), CUDA-
graph replays, L2 flushed before each, CUDA events.  Y, dX in bf16; dW in f32.
"""
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

RECIPES = {
    "tensorwise": dict(fx="tensor", fw="tensor", gdy="tensor", gw="tensor", wdy="tensor", wx="tensor"),
    "blockwise": dict(fx="blk_1x128", fw="blk_128x128", gdy="blk_1x128", gw="blk_128x128", wdy="blk_128x1",
                      wx="blk_128x1"),
    # same granules with UE8M0 scales: native block-scaled MMA (kind::mxf8f6f4.block_scale)
    "blockwise_ue8m0": dict(fx="blk_1x128", fw="blk_128x128", gdy="blk_1x128", gw="blk_128x128", wdy="blk_128x1",
                            wx="blk_128x1", sf="ue8m0"),
}
T = {"row": "col", "col": "row", "blk_1x128": "blk_128x1", "blk_128x1": "blk_1x128"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--M", type=int, default=32768)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    _clk = ClockSampler(torch.cuda.current_device())  # NVML clocks during the whole measurement
    _clk.__enter__()
    M, N, K = a.M, a.N, a.K
    dev = torch.device("cuda")
    x = synth.gaussian(M, K, 0, device=dev)
    w = synth.weight(N, K, 1, device=dev)
    dy = synth.grad(M, N, 2, device=dev)
    stream = torch.cuda.Stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    fl = 2.0 * M * N * K
    bf16_peak, _, _, src = peaks()
    res = {"workload": f"cfg4 training step M={M} K={K} N={N}: fwd Y=XW^T, dgrad dX=dY W, wgrad dW=dY^T X",
           "flop_per_gemm": fl, "fp8_peak_tflops": 2 * bf16_peak, "peak_source": src}

    def tmean(fn, steps=a.steps):
        g = capture(fn, stream)
        t = time_steps(g.replay, steps, a.warmup, flush, stream)
        return sum(t) / len(t)

    with torch.cuda.stream(stream):
        for name, g in RECIPES.items():
            # quantized operands (and their K-major transposed copies)
            sf = g.get("sf", "f32")
            xq, xs = lk.loka_quantize(x, "e4m3", g["fx"], sf)
            wq, ws = lk.loka_quantize(w, "e4m3", g["fw"], sf)
            gq, gs = lk.loka_quantize(dy, "e5m2", g["gdy"], sf)
            _, _, wtq, wts = lk.loka_quantize(w, "e4m3", g["gw"], sf, want_q=False, transpose=True)
            _, _, gtq, gts = lk.loka_quantize(dy, "e5m2", g["wdy"], sf, want_q=False, transpose=True)
            _, _, xtq, xts = lk.loka_quantize(x, "e4m3", g["wx"], sf, want_q=False, transpose=True)
            keep = []
            kw = dict(a_scale_fmt=sf, b_scale_fmt=sf, keep=keep)
            fa, yy, _ = lk.make_linear_args(xq, xs, wq, ws, a_gran=g["fx"], b_gran=g["fw"], out_dtype="bf16", **kw)
            da, dx, _ = lk.make_linear_args(gq, gs, wtq, wts, a_fmt="e5m2", a_gran=g["gdy"],
                                            b_gran=T.get(g["gw"], g["gw"]), out_dtype="bf16", **kw)
            wa, dw, _ = lk.make_linear_args(gtq, gts, xtq, xts, a_fmt="e5m2", a_gran=T.get(g["wdy"], g["wdy"]),
                                            b_gran=T.get(g["wx"], g["wx"]), out_dtype="f32", **kw)
            sh = stream.cuda_stream
            import ctypes
            wsb = {id(ar): torch.empty(max(1, lk.linear_workspace(ar)), dtype=torch.uint8, device=dev)
                   for ar in (fa, da, wa)}
            call = lambda ar: lk._lib.loka_fp8_linear_norm(ctypes.byref(ar), ctypes.c_void_p(wsb[id(ar)].data_ptr()),
                                                           wsb[id(ar)].numel(), sh)
            one = lambda ar: (lambda: call(ar))
            t_f, t_d, t_w = tmean(one(fa)), tmean(one(da)), tmean(one(wa))

            def quant(src, fmt, g_plain, g_t, q, s, qt, st):
                # one pass writes both layouts when the two directions share the granules, or for the
                # 1x128 / 128x1-transposed pair (the tile kernel's dual mode)
                if g_plain == g_t:
                    lk.loka_quantize(src, fmt, g_plain, sf, out=q, scales=s, transpose=True, out_t=qt, scales_t=st)
                elif g_plain == "blk_1x128" and g_t == "blk_128x1":
                    lk.loka_quantize(src, fmt, g_plain, sf, out=q, scales=s, transpose=True, out_t=qt, scales_t=st,
                                     gran_t="blk_1x128")
                else:
                    lk.loka_quantize(src, fmt, g_plain, sf, out=q, scales=s)
                    lk.loka_quantize(src, fmt, g_t, sf, want_q=False, transpose=True, out_t=qt, scales_t=st)

            def step():  # every quantize (incl. the K-major copies) and the three GEMMs
                quant(x, "e4m3", g["fx"], g["wx"], xq, xs, xtq, xts)
                quant(w, "e4m3", g["fw"], g["gw"], wq, ws, wtq, wts)
                quant(dy, "e5m2", g["gdy"], g["wdy"], gq, gs, gtq, gts)
                for ar in (fa, da, wa):
                    assert call(ar) == 0

            t_s = tmean(step, max(5, a.steps // 2))
            res[name] = {
                "fwd": {"ms": round(t_f, 4), "tflops": round(fl / t_f / 1e9, 1)},
                "dgrad": {"ms": round(t_d, 4), "tflops": round(fl / t_d / 1e9, 1)},
                "wgrad": {"ms": round(t_w, 4), "tflops": round(fl / t_w / 1e9, 1)},
                "gemm_only_tflops": round(3 * fl / (t_f + t_d + t_w) / 1e9, 1),
                "gemm_only_frac_of_fp8_peak": round(3 * fl / (t_f + t_d + t_w) / 1e9 / (2 * bf16_peak), 4),
                "step_ms_end_to_end": round(t_s, 4),
                "end_to_end_tflops": round(3 * fl / t_s / 1e9, 1),
            }
            del keep
        # MXFP8 forward (NEXT-4): 1x32 UE8M0 blocks on A and B (the MMA's native granule); forward only
        # (the transposed 32x1 copies the backward needs are not built)
        xm, xms = lk.loka_quantize(x, "e4m3", "blk_1x32", "ue8m0")
        wm, wms = lk.loka_quantize(w, "e4m3", "blk_1x32", "ue8m0")
        keep = []
        ma, ym, _ = lk.make_linear_args(xm, xms, wm, wms, a_gran="blk_1x32", b_gran="blk_1x32", a_scale_fmt="ue8m0",
                                        b_scale_fmt="ue8m0", out_dtype="bf16", keep=keep)
        wsm = torch.empty(max(1, lk.linear_workspace(ma)), dtype=torch.uint8, device=dev)
        import ctypes
        callm = lambda: lk._lib.loka_fp8_linear_norm(ctypes.byref(ma), ctypes.c_void_p(wsm.data_ptr()), wsm.numel(),
                                                     stream.cuda_stream)
        t_m = tmean(callm)

        def mstep():
            lk.loka_quantize(x, "e4m3", "blk_1x32", "ue8m0", out=xm, scales=xms)
            lk.loka_quantize(w, "e4m3", "blk_1x32", "ue8m0", out=wm, scales=wms)
            assert callm() == 0
        t_ms = tmean(mstep)
        res["mxfp8_fwd"] = {"gemm_ms": round(t_m, 4), "gemm_tflops": round(fl / t_m / 1e9, 1),
                            "fwd_with_quantize_ms": round(t_ms, 4)}
        del keep
        # BF16 path
        xb, wb, dyb = x, w, dy
        yb = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
        dxb = torch.empty(M, K, dtype=torch.bfloat16, device=dev)
        dwb = torch.empty(N, K, dtype=torch.float32, device=dev)
        b_f = tmean(lambda: torch.matmul(xb, wb.t(), out=yb))
        b_d = tmean(lambda: torch.matmul(dyb, wb, out=dxb))
        b_w = tmean(lambda: dwb.copy_(torch.matmul(dyb.t(), xb)))
        res["bf16"] = {"fwd_ms": round(b_f, 4), "dgrad_ms": round(b_d, 4), "wgrad_ms": round(b_w, 4),
                       "step_tflops": round(3 * fl / (b_f + b_d + b_w) / 1e9, 1), "impl": "torch.matmul (cuBLAS)"}
        for name in RECIPES:
            res[name]["speedup_vs_bf16_end_to_end"] = round((b_f + b_d + b_w) / res[name]["step_ms_end_to_end"], 3)
        res["mxfp8_fwd"]["speedup_vs_bf16_fwd"] = round(b_f / res["mxfp8_fwd"]["fwd_with_quantize_ms"], 3)
    _clk.__exit__()
    res["clocks"] = _clk.summary()
    print(json.dumps(res))
    if a.out:
        open(a.out, "w").write(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
