"""Phase trace of the pair-norm kernel (loka_debug_pairnorm_trace): where a tile's time goes.
  LOKA_PAIRNORM=256 python tools/trace_pairnorm.py --M 32768
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=32768)
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--norm", default="layer")
ap.add_argument("--out", default=None)
a = ap.parse_args()
x = synth.heavy(a.M, a.K, 3, device="cuda")
w = synth.weight(a.N, a.K, 4, device="cuda")
xq, xs = lk.loka_quantize(x, "e4m3", "tensor")
wq, ws = lk.loka_quantize(w, "e4m3", "tensor")
buf = torch.zeros(148 * 64 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="tensor", b_gran="tensor", norm=a.norm, out_dtype="bf16")
torch.cuda.synchronize()
lk._lib.loka_debug_pairnorm_trace(buf.data_ptr())
lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="tensor", b_gran="tensor", norm=a.norm, out_dtype="bf16")
torch.cuda.synchronize()
lk._lib.loka_debug_pairnorm_trace(None)
t = buf.cpu().numpy().reshape(148, 64, 8).astype(np.float64)
valid = t[:, :, 0] > 0
t0 = t[valid][:, 0].min()
us = lambda v: (v / 1e3)
ep = t[valid]
res = {"tiles_traced": int(valid.sum()),
       "span_us": us(ep[:, 3].max() - t0)}
for name, (i, j) in {"pass_S": (0, 1), "exchange_wait": (1, 2), "pass_N": (2, 3), "until_flags_seen": (1, 7),
                     "gather_merge": (7, 2)}.items():
    d = us(ep[:, j] - ep[:, i])
    res[name] = {"mean": float(d.mean()), "p50": float(np.median(d)), "p90": float(np.percentile(d, 90)),
                 "max": float(d.max())}
lead = t[0::2]
lv = lead[:, :, 4] > 0
mm = lead[lv]
for name, (i, j) in {"mma_wait_for_acc_buffer": (4, 5), "mma_tile": (5, 6)}.items():
    d = us(mm[:, j] - mm[:, i])
    res[name] = {"mean": float(d.mean()), "p50": float(np.median(d)), "p90": float(np.percentile(d, 90)),
                 "max": float(d.max()), "sum_per_cta_mean": float(d.sum() / 74)}
# per-wave view: mean MMA stall by wave index
waves = {}
for c in range(74):
    for k in range(64):
        if lead[c, k, 4] > 0:
            waves.setdefault(k, []).append(us(lead[c, k, 5] - lead[c, k, 4]))
res["mma_stall_by_wave_mean"] = {k: round(float(np.mean(v)), 2) for k, v in sorted(waves.items())}
res["stalled_pairs_gt2us_by_wave"] = {k: int(np.sum(np.array(v) > 2.0)) for k, v in sorted(waves.items())}
# MMA-completion skew inside a row block: spread of the accumulator-ready stamps of its tiles
G = -(-a.N // int(os.environ.get("LOKA_PAIRNORM", "256")))
print(json.dumps(res, indent=1))
if a.out:
    np.save(a.out, t)
