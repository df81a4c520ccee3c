"""The README example, run as a check (tools/gpu_run.sh)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_10886_b200 as lk
x = torch.randn(32768, 4096, device="cuda", dtype=torch.bfloat16)          # activation X [M, K]
w = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16) / 64      # weight W [N, K]
xq, xs = lk.loka_quantize(x, "e4m3", "tensor")                              # a1 (split phases: phase="amax"/"cast")
wq, ws = lk.loka_quantize(w, "e4m3", "tensor")                              # a2
y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="tensor", b_gran="tensor",
                               norm="layer", out_dtype="bf16")              # a4 + a5 fused
ref = torch.nn.functional.layer_norm(x @ w.t(), (4096,))                    # the BF16 path
st = lk.probe_stats_to_dicts(lk.loka_probe_error([(y, ref)]))[0]            # a7: MERE, max_rel, ...
plan = lk.loka_dispatch_select([("fp8_tw", "fwd", st["mere"], 500.0)], 900.0, 0.2, 1.05)  # a8
print(st, plan)
