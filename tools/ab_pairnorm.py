"""A/B timing of pair-norm variants (env settings) at one shape, interleaved rounds, median ms.
  python tools/ab_pairnorm.py --M 32768 --variants "PN=256" "PN=256,DBG=1" ...
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402
from bench import ClockSampler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=32768)
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--norm", default="layer")
ap.add_argument("--act", default="none")
ap.add_argument("--out", default="bf16")
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--variants", nargs="+", default=["PN=256", "PN=256,DBG=1", "PN=256,DBG=2", "PN=256,DBG=3",
                                                   "NORM=none,WIDE=0", "NORM=none,WIDE=1"])
a = ap.parse_args()
x = synth.heavy(a.M, a.K, 3, device="cuda")
w = synth.weight(a.N, a.K, 4, device="cuda")
xq, xs = lk.loka_quantize(x, "e4m3", "tensor")
wq, ws = lk.loka_quantize(w, "e4m3", "tensor")
del x
y = torch.empty(a.M, a.N, dtype=torch.bfloat16 if a.out == "bf16" else torch.float32, device="cuda")
wsb = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
KEYS = {"PN": "LOKA_PAIRNORM", "DBG": "LOKA_PN_DEBUG", "WIDE": "LOKA_PAIR_WIDE", "ORDER": "LOKA_PN_ORDER", "MC": "LOKA_PN_MC"}


def setenv(v):
    norm = a.norm
    for k in KEYS.values():
        os.environ.pop(k, None)
    for kv in v.split(","):
        k, val = kv.split("=")
        if k == "NORM":
            norm = val
        else:
            os.environ[KEYS[k]] = val
    return norm


def run(v):
    norm = setenv(v)
    fn = lambda: lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="tensor", b_gran="tensor", norm=norm, act=a.act,
                                         norm_block=256, out_dtype=a.out, y=y, ws=wsb)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


res = {v: [] for v in a.variants}
with ClockSampler(torch.cuda.current_device()) as cs:
    for _ in range(a.rounds):
        for v in a.variants:
            res[v].append(run(v))
fl = 2.0 * a.M * a.N * a.K
out = {"shape": [a.M, a.N, a.K], "norm": a.norm, "act": a.act, "clocks": cs.summary(),
       "variants": {v: {"ms_median": round(statistics.median(t), 4), "tflops": round(fl / statistics.median(t) / 1e9, 1),
                        "ms_all": [round(u, 4) for u in t]} for v, t in res.items()}}
print(json.dumps(out))
