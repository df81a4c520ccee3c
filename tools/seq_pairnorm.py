"""Per-launch event timing of a long back-to-back sequence (drift check), variants interleaved
launch by launch.  python tools/seq_pairnorm.py --n 60"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402
from bench import ClockSampler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=32768)
ap.add_argument("--n", type=int, default=60)
ap.add_argument("--gap_ms", type=float, default=0.0)
a = ap.parse_args()
K = N = 4096
x = synth.heavy(a.M, K, 3, device="cuda")
w = synth.weight(N, K, 4, device="cuda")
xq, xs = lk.loka_quantize(x, "e4m3", "tensor")
wq, ws = lk.loka_quantize(w, "e4m3", "tensor")
y = torch.empty(a.M, N, dtype=torch.bfloat16, device="cuda")
wsb = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
variants = {"pn256_o0": ("layer", {"LOKA_PAIRNORM": "256", "LOKA_PN_ORDER": "0"}),
            "pn256_o1": ("layer", {"LOKA_PAIRNORM": "256", "LOKA_PN_ORDER": "1"}),
            "pn256_rms": ("rms", {"LOKA_PAIRNORM": "256"}),
            "pn512_o1": ("layer", {"LOKA_PAIRNORM": "512", "LOKA_PN_ORDER": "1"}),
            "pn256_nowait": ("layer", {"LOKA_PAIRNORM": "256", "LOKA_PN_ORDER": "0", "LOKA_PN_DEBUG": "1"}),
            "plain": ("none", {"LOKA_PAIR_WIDE": "0"})}
res = {k: [] for k in variants}
ev = []
with ClockSampler(torch.cuda.current_device()) as cs:
    for i in range(a.n):
        for k, (norm, env) in variants.items():
            for kk in ("LOKA_PAIRNORM", "LOKA_PN_ORDER", "LOKA_PAIR_WIDE", "LOKA_PN_DEBUG"):
                os.environ.pop(kk, None)
            os.environ.update(env)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="tensor", b_gran="tensor", norm=norm, out_dtype="bf16",
                                    y=y, ws=wsb)
            e1.record()
            ev.append((k, e0, e1))
        if a.gap_ms:
            torch.cuda._sleep(int(a.gap_ms * 1.9e6))
    torch.cuda.synchronize()
for k, e0, e1 in ev:
    res[k].append(round(e0.elapsed_time(e1), 4))
print(json.dumps({"clocks": cs.summary(), "ms": res}))
