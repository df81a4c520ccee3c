"""Per-launch interleaved timing of the cfg5 step variants: fused cast (pacing 1 / 3 / 8 / none) vs the
unfused quantize + GEMM (drift-free A/B).  python tools/seq_castx.py --n 12"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402
from bench import CFG5_K, CFG5_N, Cfg5, ClockSampler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=262144)
ap.add_argument("--n", type=int, default=12)
a = ap.parse_args()
x = synth.heavy(a.M, CFG5_K, 3, device="cuda", total_rows=a.M)
w = synth.weight(CFG5_N, CFG5_K, 4, device="cuda")
step = Cfg5(lk, x, w)
sh = torch.cuda.current_stream().cuda_stream
os.environ["LOKA_FUSED_CAST"] = "1"
variants = {"fused_ahead1": ("1", step.step_castx), "fused_ahead3": ("3", step.step_castx),
            "fused_ahead8": ("8", step.step_castx), "fused_free": ("100000", step.step_castx),
            "unfused": (None, step.step)}
res = {k: [] for k in variants}
for _ in range(2):
    for k, (ah, fn) in variants.items():
        if ah:
            os.environ["LOKA_CAST_AHEAD"] = ah
        fn(sh)
torch.cuda.synchronize()
ev = []
with ClockSampler(torch.cuda.current_device()) as cs:
    for _ in range(a.n):
        for k, (ah, fn) in variants.items():
            if ah:
                os.environ["LOKA_CAST_AHEAD"] = ah
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(sh)
            e1.record()
            ev.append((k, e0, e1))
    torch.cuda.synchronize()
for k, e0, e1 in ev:
    res[k].append(e0.elapsed_time(e1))
print(json.dumps({"clocks": cs.summary(), "median_ms": {k: round(statistics.median(v), 4) for k, v in res.items()},
                  "ms": {k: [round(t, 3) for t in v] for k, v in res.items()}}))
