"""One small launch of every hot kernel family, for compute-sanitizer (racecheck / synccheck /
memcheck): quantize (bulk-copy row + tensor, 1x128, tiled cast-transpose), linear_norm (cluster
LayerNorm, FP8 out), the CTA-pair engine (plain + WIDE), pair-norm (Case-2 exchange, both tile
widths), the fused stack, the probe.  Prints "sanitize-run ok".
  compute-sanitizer --tool racecheck python tools/sanitize_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

dev = torch.device("cuda")
which = set(sys.argv[1:]) or {"quant", "linear", "pair", "pairnorm", "stack", "probe"}
x = synth.heavy(512, 1024, 1, device=dev)
if "quant" in which:
    for g in ("row", "tensor", "blk_1x128", "blk_128x128"):
        lk.loka_quantize(x, "e4m3", g)
    lk.loka_quantize(x, "e5m2", "row", transpose=True)
    torch.cuda.synchronize()
xq, xs = lk.loka_quantize(x, "e4m3", "row")
w = synth.weight(1024, 1024, 2, device=dev)
wq, ws = lk.loka_quantize(w, "e4m3", "row")
if "linear" in which:
    lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="layer", out_dtype="e4m3")
    torch.cuda.synchronize()
if "pair" in which:
    for wide in ("0", "1"):
        os.environ["LOKA_PAIR_WIDE"] = wide
        xb = synth.heavy(4864, 2048, 3, device=dev)
        wb = synth.weight(2048, 2048, 4, device=dev)
        aq, asc = lk.loka_quantize(xb, "e4m3", "tensor")
        bq, bsc = lk.loka_quantize(wb, "e4m3", "tensor")
        lk.loka_fp8_linear_norm(aq, asc, bq, bsc, a_gran="tensor", b_gran="tensor", out_dtype="bf16")
        torch.cuda.synchronize()
    os.environ.pop("LOKA_PAIR_WIDE", None)
if "pairnorm" in which:
    for tn in ("256", "512"):
        os.environ["LOKA_PAIRNORM"] = tn
        w4 = synth.weight(2048, 1024, 5, device=dev)
        q4, s4 = lk.loka_quantize(w4, "e4m3", "row")
        lk.loka_fp8_linear_norm(xq, xs, q4, s4, norm="layer", out_dtype="bf16")
        lk.loka_fp8_linear_norm(xq, xs, q4, s4, norm="rms", out_dtype="e4m3")
        torch.cuda.synchronize()
    os.environ.pop("LOKA_PAIRNORM", None)
if "stack" in which:
    dims = synth.CFG2_DIMS
    hq = lk.loka_quantize(synth.gaussian(256, dims[0], 0, device=dev), "e4m3", "row")
    wts = [lk.loka_quantize(synth.weight(dims[l + 1], dims[l], 100 + l, device=dev), "e4m3", "row")
           for l in range(len(dims) - 1)]
    lk.loka_fp8_mlp_stack(hq[0], hq[1], wts, norms="layer", out_dtype="bf16")
    torch.cuda.synchronize()
if "probe" in which:
    y = torch.randn(512, 1024, device=dev)
    lk.loka_probe_error([(y.to(torch.bfloat16), y)])
    torch.cuda.synchronize()
print("sanitize-run ok")
