"""Per-CTA phase timeline of the fused stack launch (loka_debug_trace, stack slots).
Usage: python tools/trace_stack.py [dims (comma list, default cfg2)] [M]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

DIMS = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else synth.CFG2_DIMS
L = len(DIMS) - 1
dev = torch.device("cuda")
M = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
x = synth.gaussian(M, DIMS[0], 0, device=dev)
xq, xs = lk.loka_quantize(x, "e4m3", "row")
ws = [lk.loka_quantize(synth.weight(DIMS[l + 1], DIMS[l], 100 + l, device=dev), "e4m3", "row") for l in range(L)]
for rep in range(4):
    torch.cuda.synchronize()
    if rep == 3:
        lk.debug_trace(1)
    y, _ = lk.loka_fp8_mlp_stack(xq, xs, ws, norms="layer", out_dtype="bf16")
    torch.cuda.synchronize()
t = np.array(lk.debug_trace(0, 65536 + 512 * 64), dtype=np.int64)[65536:].reshape(-1, 64)[:, :64]
t = t[t[:, 0] > 0]
base = t[:, 0].min()
rel = np.where(t > 0, (t - base) / 1000.0, np.nan)
print("raw stamps of CTA 0 (ns from its entry):", [int(v) for v in (t[0][t[0] > 0] - t[0, 0])][:24])
med = np.nanmedian(rel, axis=0)
mx = np.nanmax(rel, axis=0)
print(f"ctas={len(t)} entry {med[0]:.2f}/{mx[0]:.2f} setup {med[1]:.2f}/{mx[1]:.2f} end(max last stamp) {np.nanmax(rel):.2f} us")
d = rel[:, 58:62]
if np.isfinite(d).any():
    print("L1 epilogue detail (median): normalized %.2f scales %.2f codes_stored %.2f fenced+barrier %.2f" %
          tuple(np.nanmedian(d, axis=0)))
names = ["w_landed", "mma_done", "acc_ready", "q_merged", "cl_merged", "pushed", "A_ready"]
for l in range(min(L, 8)):
    b = 2 + 7 * l
    print(f"L{l} K={DIMS[l]} N={DIMS[l + 1]}: " + " ".join(f"{n}={med[b + i]:.2f}/{mx[b + i]:.2f}" for i, n in enumerate(names)))
