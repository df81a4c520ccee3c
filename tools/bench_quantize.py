"""Quantize kernels (a1-a3) against the HBM roofline: achieved GB/s = algorithmic bytes / time.

  python tools/bench_quantize.py [--rows 32768 --cols 4096] [--out profiles/r01_quantize.json]

Algorithmic bytes per element: 2 (bf16 read) + 1 per FP8 layout written (+ 4 B per granule).
The tensorwise amax pass re-reads X (an implementation cost, reported separately).  CUDA-graph
replays, L2 flushed before each, CUDA events; peak = MEASURED_PEAKS.json hbm_gbs.
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
from bench import capture, peaks, time_steps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=32768)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    R, Cc = a.rows, a.cols
    dev = torch.device("cuda")
    x = synth.heavy(R, Cc, 3, device=dev)
    stream = torch.cuda.Stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    _, _, hbm, src = peaks()
    q = torch.empty(R, Cc, dtype=torch.uint8, device=dev)
    qt = torch.empty(Cc, R, dtype=torch.uint8, device=dev)
    out = {"shape": [R, Cc], "hbm_peak_gbs": hbm, "peak_source": src, "kernels": {}}
    cases = [("row", "row", False), ("blk_1x128", "blk_1x128", False), ("blk_128x128", "blk_128x128", False),
             ("tensor", "tensor", False), ("col", "col", False), ("blk_128x1", "blk_128x1", False),
             ("row+transpose", "row", True), ("tensor+transpose", "tensor", True),
             ("blk_128x1+transpose", "blk_128x1", True)]
    from bench import ClockSampler
    clk = ClockSampler(torch.cuda.current_device())
    clk.__enter__()
    with torch.cuda.stream(stream):
        for name, gran, tr in cases:
            s = torch.empty(lk.scale_shape(R, Cc, gran), dtype=torch.float32, device=dev)
            st = None
            if tr:
                tg = {"row": "col", "col": "row", "blk_1x128": "blk_128x1", "blk_128x1": "blk_1x128"}.get(gran, gran)
                st = torch.empty(lk.scale_shape(Cc, R, tg), dtype=torch.float32, device=dev)
            fn = (lambda g=gran, s=s, st=st, tr=tr:
                  lk.loka_quantize(x, "e4m3", g, out=q, scales=s, transpose=tr, out_t=qt if tr else None,
                                   scales_t=st))
            g = capture(fn, stream)
            t = time_steps(g.replay, a.steps, 3, flush, stream)
            ms = sum(t) / len(t)
            nbytes = R * Cc * (2 + (2 if tr else 1))
            gbs = nbytes / (ms * 1e-3) / 1e9
            # the granularities whose amax spans the whole tensor / row / column beyond one tile
            # read x twice (amax pre-pass, then the cast): the bytes HBM actually moves
            moved = nbytes + (R * Cc * 2 if gran in ("tensor", "col") or (gran == "row" and tr) else 0)
            out["kernels"][name] = {"ms": round(ms, 4), "algorithmic_bytes": nbytes, "gbs": round(gbs, 1),
                                    "frac_of_hbm": round(gbs / hbm, 3), "moved_bytes": moved,
                                    "gbs_moved": round(moved / (ms * 1e-3) / 1e9, 1)}
        # the tensorwise recipe's two phases separately (split-phase for the DP all-reduce)
        amax = torch.zeros(1, dtype=torch.float32, device=dev)
        s1 = torch.empty(1, dtype=torch.float32, device=dev)
        amax = torch.zeros(2, dtype=torch.float32, device=dev)
        lk.loka_quantize(x, "e4m3", "tensor", phase="amax", amax=amax, want_q=False, scales=s1)
        for name, ph, nbytes in (("tensor_amax_pass", "amax", R * Cc * 2), ("tensor_cast_pass", "cast", R * Cc * 3),
                                 ("tensor_cast_delayed_with_amax", "delayed", R * Cc * 3)):
            fn = (lambda ph=ph: lk.loka_quantize(x, "e4m3", "tensor", phase=ph, amax=amax, out=q, scales=s1,
                                                 want_q=ph != "amax"))
            g = capture(fn, stream)
            t = time_steps(g.replay, a.steps, 3, flush, stream)
            ms = sum(t) / len(t)
            gbs = nbytes / (ms * 1e-3) / 1e9
            out["kernels"][name] = {"ms": round(ms, 4), "algorithmic_bytes": nbytes, "gbs": round(gbs, 1),
                                    "frac_of_hbm": round(gbs / hbm, 3)}
    clk.__exit__()
    out["clocks"] = clk.summary()
    print(json.dumps(out))
    if a.out:
        open(a.out, "w").write(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
