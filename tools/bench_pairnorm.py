"""Kernel-level timing of the norm fused into the CTA-pair engine (pairnorm.cu) vs the plain-epilogue
GEMM of the same shape and vs the round-1 route (pair GEMM FP32 -> workspace + row-wise pass).
Pre-quantized operands (compute-only), CUDA events over `reps` launches after
warm-up, NVML clocks sampled during the timed region.

  python tools/bench_pairnorm.py [--out f.json] [--quick]
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
from bench import ClockSampler  # noqa: E402


def timed(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run_case(name, M, N, K, norm, od, act="none", gran="tensor", reps=10, modes=("512", "256", "0")):
    dev = torch.device("cuda")
    x = synth.heavy(M, K, 3, device=dev)
    w = synth.weight(N, K, 4, device=dev)
    xq, xs = lk.loka_quantize(x, "e4m3", gran)
    wq, ws = lk.loka_quantize(w, "e4m3", gran)
    del x
    y = torch.empty(M, N, dtype=torch.bfloat16 if od == "bf16" else torch.float32, device=dev)
    res = {"case": name, "M": M, "N": N, "K": K, "norm": norm, "act": act, "out": od, "gran": gran}
    fl = 2.0 * M * N * K
    out = {}
    for mode in modes:
        os.environ["LOKA_PAIRNORM"] = mode
        wsb = None
        args, _, _ = lk.make_linear_args(xq, xs, wq, ws, a_gran=gran, b_gran=gran, norm=norm, act=act,
                                         norm_block=256, out_dtype=od, y=y)
        nws = lk.linear_workspace(args)
        if nws:
            wsb = torch.empty(nws, dtype=torch.uint8, device=dev)

        def f():
            lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran=gran, b_gran=gran, norm=norm, act=act, norm_block=256,
                                    out_dtype=od, y=y, ws=wsb)
        with ClockSampler(torch.cuda.current_device()) as cs:
            ms = timed(f, reps)
        out[{"512": "pair_tn512", "256": "pair_tn256", "0": "round1_route"}[mode]] = {
            "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1), "clocks": cs.summary()}
        del wsb
    os.environ.pop("LOKA_PAIRNORM", None)

    os.environ["LOKA_PAIR_WIDE"] = "0"

    def plain256():
        lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran=gran, b_gran=gran, norm="none", out_dtype=od, y=y)
    with ClockSampler(torch.cuda.current_device()) as cs:
        ms = timed(plain256, reps)
    out["plain_gemm_256_tiles"] = {"ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1), "clocks": cs.summary()}
    os.environ.pop("LOKA_PAIR_WIDE", None)

    def plain():
        lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran=gran, b_gran=gran, norm="none", out_dtype=od, y=y)
    with ClockSampler(torch.cuda.current_device()) as cs:
        ms = timed(plain, reps)
    out["plain_gemm_same_shape"] = {"ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1), "clocks": cs.summary()}
    # achievability reference: cuBLASLt FP8 (torch._scaled_mm, tensorwise scales, bf16 out) on the same
    # operands (library GEMM, no norm)
    try:
        a8 = xq.view(torch.float8_e4m3fn)
        b8 = wq.view(torch.float8_e4m3fn)
        sa = xs.reshape(()) if xs.numel() == 1 else xs.reshape(-1, 1)
        sb = ws.reshape(()) if ws.numel() == 1 else ws.reshape(1, -1)
        def smm():
            torch._scaled_mm(a8, b8.t(), scale_a=sa, scale_b=sb, out_dtype=torch.bfloat16)
        with ClockSampler(torch.cuda.current_device()) as cs:
            ms = timed(smm, reps)
        out["cublaslt_scaled_mm_same_shape"] = {"ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1),
                                                "clocks": cs.summary()}
    except Exception as e:  # noqa: BLE001
        out["cublaslt_scaled_mm_same_shape"] = {"error": str(e)[:200]}
    res.update(out)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    cases = [("cfg5_p1_layernorm", 262144, 4096, 4096, "layer", "bf16"),
             ("cfg5_p8_layernorm", 32768, 4096, 4096, "layer", "bf16"),
             ("blocknorm256_hswish_32768x4096", 32768, 4096, 4096, "block_rms", "bf16", "hardswish"),
             ("cfg4_rms_f32", 32768, 4096, 4096, "rms", "f32")]
    if a.quick:
        cases = cases[1:3]
    res = []
    for c in cases:
        r = run_case(*c, reps=5 if c[1] > 100000 else 20)
        print(json.dumps(r), flush=True)
        res.append(r)
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
