"""Per-CTA phase timeline of the cfg2 linear+LayerNorm launches (loka_debug_trace)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

DIMS = synth.CFG2_DIMS
dev = torch.device("cuda")
M = 4096
x = synth.gaussian(M, DIMS[0], 0, device=dev)
hq, hs = lk.loka_quantize(x, "e4m3", "row")
names = ["entry", "pdl", "tma0", "stage0", "mma", "acc", "pre2", "stored", "p1", "halves", "clus", "fin"]
for l in range(8):
    K, N = DIMS[l], DIMS[l + 1]
    wq, ws = lk.loka_quantize(synth.weight(N, K, 100 + l, device=dev), "e4m3", "row")
    for rep in range(3):
        torch.cuda.synchronize()
        if rep == 2:
            lk.debug_trace(1)
        y, ys = lk.loka_fp8_linear_norm(hq, hs, wq, ws, norm="layer", out_dtype="bf16" if l == 7 else "e4m3")
        torch.cuda.synchronize()
    t = np.array(lk.debug_trace(0, 4096 * 16), dtype=np.int64).reshape(-1, 16)[:, :12]
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()
    rel = (t - base) / 1000.0  # us
    med = np.median(rel, axis=0)
    mx = rel.max(axis=0)
    print(f"layer {l} K={K} N={N} ctas={len(t)}: " + " ".join(f"{n}={m:.1f}/{x_:.1f}" for n, m, x_ in zip(names, med, mx)))
    hq, hs = y, ys
