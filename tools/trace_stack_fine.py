"""Fine (clock64) timeline of layer 1's epilogue in the fused stack launch, thread 0 and warp 15.
Usage: python tools/trace_stack_fine.py [dims] [M]"""
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
n0 = 65536 + 512 * 64
t = np.array(lk.debug_trace(0, n0 + 512 * 64), dtype=np.int64)[n0:].reshape(-1, 64)
t = t[t[:, 0] > 0].astype(np.float64)
names = {16: "loop_top", 17: "col_staged", 0: "epi_entry", 1: "acc_ready", 2: "tmem_loaded", 3: "dequant", 4: "seg_stats",
         5: "qbar", 6: "qmerge", 7: "dsmem_push", 8: "cluster_sync", 9: "cmerge", 10: "normalized", 11: "scales",
         12: "codes_stored", 15: "hs_saved", 13: "fence_bar", 14: "tma_store_wait"}
order = [16, 17, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 15, 13, 14]
for who, off in (("thread0", 0), ("warp15", 32)):
    base = t[:, off + 16]
    row = []
    prev = None
    for i in order:
        v = t[:, off + i]
        ok = (v > 0) & (base > 0)
        if not ok.any():
            continue
        d = np.median(v[ok] - base[ok])
        row.append(f"{names[i]}={d:.0f}" + (f"(+{d - prev:.0f})" if prev is not None else ""))
        prev = d
    print(who, "cycles from loop top:", " ".join(row))
