"""LoKA Probe (a7) against the HBM roofline: MERE statistics of one large (out, ref) pair and of
the cfg3 64-layer set.  Algorithmic bytes = out + ref read once (M*N*(b_out + b_ref)); the floor
pass's second read of ref is an implementation cost.  CUDA graphs, L2 flushed, CUDA events.

  python tools/bench_probe.py [--out profiles/r01_probe.json]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    _clk = ClockSampler(torch.cuda.current_device())  # NVML clocks during the whole measurement
    _clk.__enter__()
    dev = torch.device("cuda")
    stream = torch.cuda.Stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    _, _, hbm, src = peaks()
    res = {"hbm_peak_gbs": hbm, "peak_source": src, "cases": []}
    cases = [("32768x4096 bf16 pair", [(32768, 4096)]),
             ("cfg3: 64 layers 2048 x N (N in S), bf16", [(2048, n) for _ in range(8) for n in synth.CFG3_DIMS])]
    for name, shapes in cases:
        pairs = []
        for i, (M, N) in enumerate(shapes):
            ref = synth.gaussian(M, N, 10 + i, device=dev)
            out = (ref.float() * (1 + 0.01 * torch.randn(M, N, device=dev))).to(torch.bfloat16)
            pairs.append((out, ref))
        stats = torch.empty(len(pairs), 5, dtype=torch.float64, device=dev)
        nws = 1 << 20
        ws = torch.empty(nws, dtype=torch.uint8, device=dev)
        with torch.cuda.stream(stream):
            lk.loka_probe_error(pairs, stream=stream, stats=stats, ws=ws)
            g = capture(lambda: lk.loka_probe_error(pairs, stream=stream, stats=stats, ws=ws), stream)
            t = time_steps(g.replay, a.steps, 3, flush, stream)
        ms = sum(t) / len(t)
        algo = sum(M * N * 4 for M, N in shapes)
        res["cases"].append({"case": name, "ms": round(ms, 4), "algorithmic_bytes": algo,
                             "gbs": round(algo / ms / 1e6, 1), "frac_of_hbm": round(algo / ms / 1e6 / hbm, 3)})
    _clk.__exit__()
    res["clocks"] = _clk.summary()
    print(json.dumps(res))
    if a.out:
        open(a.out, "w").write(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
