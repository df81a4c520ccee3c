"""cfg3 (BASELINE.json configs[2]): DHEN/Wukong-style ensemble of 64 heterogeneous GEMMs (M=2048,
K,N in {128,...,2048}, 8 shared inputs; odd-indexed inputs heavy-tailed) — grouped FP8 launch vs the
BF16 path, LoKA Probe MERE per layer against the BF16 outputs, and the LoKA Dispatch plan.

  python tools/bench_cfg3.py [--steps 50] [--warmup 5] [--out profiles/r01_cfg3.json]

FP8 step = one grouped rowwise quantize of the 8 inputs + the grouped FP8 GEMM (weights quantized
once, inference-style); BF16 step = 64 torch F.linear (cuBLAS) calls.  Both CUDA-graph replays,
L2 flushed before every timed step, CUDA events.  Per-layer dispatch timing: each GEMM alone (FP8
fused launch incl. its input quantize vs BF16), graph replays.  All statistics computed by
libloka (loka_probe_error, loka_dispatch_select).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
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
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda")
    S, M = synth.CFG3_DIMS, 2048
    xs = [(synth.heavy(M, k, i, device=dev) if i % 2 else synth.gaussian(M, k, i, device=dev)) for i, k in enumerate(S)]
    ws = [[synth.weight(n, k, 1000 + 8 * i + j, device=dev) for j, n in enumerate(S)] for i, k in enumerate(S)]
    stream = torch.cuda.Stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    flops = sum(2.0 * M * k * n for k in S for n in S)

    # ---- FP8: grouped quantize of the 8 inputs + grouped GEMM ----
    xq = [(torch.empty(M, k, dtype=torch.uint8, device=dev), torch.empty(M, dtype=torch.float32, device=dev)) for k in S]
    wq = [[lk.loka_quantize(w, "e4m3", "row") for w in row] for row in ws]
    keep, args, ys = [], [], []
    for i in range(8):
        for j in range(8):
            ar, y, _ = lk.make_linear_args(xq[i][0], xq[i][1], wq[i][j][0], wq[i][j][1], out_dtype="bf16", keep=keep)
            args.append(ar)
            ys.append(y)
    arr = (lk.loka_linear_args * 64)(*args)
    G = 8
    qx = (lk.loka_tensor * G)()
    qq = (lk.loka_tensor * G)()
    for i, k in enumerate(S):
        qx[i] = lk._tensor(xs[i], lk.BF16, M, k)
        qq[i] = lk._tensor(xq[i][0], lk.E4M3, M, k, xq[i][1], "row")
    sh = stream.cuda_stream

    def fp8_step():
        assert lk._lib.loka_quantize_grouped(G, qx, qq, None, sh) == 0
        assert lk._lib.loka_grouped_fp8_linear(64, arr, None, 0, sh) == 0

    def fp8_gemm_only():
        assert lk._lib.loka_grouped_fp8_linear(64, arr, None, 0, sh) == 0

    clk = ClockSampler(torch.cuda.current_device())
    clk.__enter__()
    g8 = capture(fp8_step, stream)
    t8 = time_steps(g8.replay, a.steps, a.warmup, flush, stream)
    gg = capture(fp8_gemm_only, stream)
    tg = time_steps(gg.replay, a.steps, a.warmup, flush, stream)

    # ---- BF16 path ----
    yb = [[torch.empty(M, n, dtype=torch.bfloat16, device=dev) for n in S] for _ in S]

    def bf16_step():
        for i in range(8):
            for j in range(8):
                torch.matmul(xs[i], ws[i][j].t(), out=yb[i][j])

    gb = capture(bf16_step, stream)
    tb = time_steps(gb.replay, a.steps, a.warmup, flush, stream)
    ms8, msg, msb = sum(t8) / len(t8), sum(tg) / len(tg), sum(tb) / len(tb)
    clk.__exit__()

    # ---- LoKA Probe: MERE of every FP8 layer against the BF16 path (one libloka call) ----
    g8.replay()
    gb.replay()
    torch.cuda.synchronize()
    pairs = [(ys[8 * i + j], yb[i][j]) for i in range(8) for j in range(8)]
    stats = lk.probe_stats_to_dicts(lk.loka_probe_error(pairs))
    mere = [s["mere"] for s in stats]
    geo = lambda v: math.exp(sum(math.log(max(x, 1e-6)) for x in v) / len(v))
    normal = [mere[8 * i + j] for i in range(0, 8, 2) for j in range(8)]
    heavy = [mere[8 * i + j] for i in range(1, 8, 2) for j in range(8)]

    # ---- LoKA Dispatch per layer: FP8 (fused, incl. its input quantize) vs BF16 ----
    plan = []
    for i, k in enumerate(S):
        for j, n in enumerate(S):
            a1 = (lk.loka_linear_args * 1)(args[8 * i + j])
            x1 = (lk.loka_tensor * 1)(qx[i])
            q1 = (lk.loka_tensor * 1)(qq[i])

            nws1 = int(lk._lib.loka_grouped_workspace_size(1, a1))
            ws1 = torch.empty(max(nws1, 16), dtype=torch.uint8, device=dev)

            def one_fp8():
                assert lk._lib.loka_quantize_grouped(1, x1, q1, None, sh) == 0
                assert lk._lib.loka_grouped_fp8_linear(1, a1, ctypes.c_void_p(ws1.data_ptr()), ws1.numel(), sh) == 0

            def one_bf16():
                torch.matmul(xs[i], ws[i][j].t(), out=yb[i][j])

            reps = max(10, a.steps // 5)
            f = sum(time_steps(capture(one_fp8, stream).replay, reps, 3, flush, stream)) / reps
            b = sum(time_steps(capture(one_bf16, stream).replay, reps, 3, flush, stream)) / reps
            ch = lk.loka_dispatch_select([("fp8_rowwise", "fwd", mere[8 * i + j], 1e3 * f)], 1e3 * b, 0.2, 1.05)
            # the same decision on the layer's share of the grouped steps (how the layer runs inside the
            # ensemble: one grouped FP8 launch vs 64 BF16 GEMMs), FLOP-proportional
            share = 2.0 * M * k * n / flops
            chg = lk.loka_dispatch_select([("fp8_rowwise", "fwd", mere[8 * i + j], 1e3 * ms8 * share)],
                                          1e3 * msb * share, 0.2, 1.05)
            plan.append({"K": k, "N": n, "mere": round(mere[8 * i + j], 5), "max_rel": round(stats[8 * i + j]["max_rel"], 3),
                         "n_floored": stats[8 * i + j]["n_floored"],
                         "fp8_us_alone": round(1e3 * f, 2), "bf16_us_alone": round(1e3 * b, 2),
                         "speedup_alone": round(b / f, 3), "choice_alone": "fp8_rowwise" if ch == 0 else "baseline",
                         "speedup_grouped_share": round(msb / ms8, 3),
                         "choice_grouped": "fp8_rowwise" if chg == 0 else "baseline",
                         "binding": ("mere" if mere[8 * i + j] >= 0.2 else "") +
                                    ("+speedup_alone" if b / f <= 1.05 else "")})
    out = {
        "workload": "cfg3: 64 GEMMs M=2048, K,N in " + str(S) + ", 8 shared inputs (odd ones heavy-tailed), bf16 out",
        "flop_per_step": flops,
        "fp8_end_to_end": {"ms_per_step": round(ms8, 5), "tflops": round(flops / ms8 / 1e9, 2),
                           "step": "grouped quantize of 8 inputs + grouped FP8 GEMM (2 persistent launches)"},
        "fp8_gemm_only": {"ms_per_step": round(msg, 5), "tflops": round(flops / msg / 1e9, 2)},
        "bf16": {"ms_per_step": round(msb, 5), "tflops": round(flops / msb / 1e9, 2), "impl": "64 x torch.matmul"},
        "speedup_vs_bf16_end_to_end": round(msb / ms8, 3),
        "speedup_vs_bf16_gemm_only": round(msb / msg, 3),
        "probe": {"geomean_mere_all": round(geo(mere), 5), "geomean_mere_gaussian_inputs": round(geo(normal), 5),
                  "geomean_mere_heavy_inputs": round(geo(heavy), 5), "ref": "BF16 path (DESIGN.md D9)"},
        "dispatch": {"budget": 0.2, "min_speedup": 1.05,
                     "fp8_layers_alone": sum(p["choice_alone"] != "baseline" for p in plan),
                     "fp8_layers_grouped": sum(p["choice_grouped"] != "baseline" for p in plan),
                     "layers_mere_below_budget": sum(p["mere"] < 0.2 for p in plan),
                     "why": "MERE (P:192) is a mean of per-element relative errors; these synthetic layers' outputs "
                            "are zero-centred, so elements near 0 dominate it (the floor f = 1e-6 mean|ref| "
                            "barely clips them) and FP8's ~3-4% per-element error turns into MERE 0.2-0.6 > the "
                            "paper's 0.2 budget (P:541) for most layers; alone, each small GEMM is launch/latency-"
                            "bound and FP8's extra quantize launch makes it slower than BF16 (speedup_alone < 1), "
                            "while inside the grouped launch FP8 is faster for every layer",
                     "plan": plan},
        "l2": "flushed before every timed step", "timing": "CUDA-graph replays, CUDA events",
        "clocks": clk.summary(),
    }
    s = json.dumps(out)
    print(s)
    if a.out:
        open(a.out, "w").write(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
