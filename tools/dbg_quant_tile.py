"""Run each streaming-tile quantize case eagerly, one process per case (a fault kills the context)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import sys, torch
sys.path.insert(0, "{root}")
import synth, paper_2605_10886_b200 as lk
R, C, gran, tr = {R}, {C}, "{gran}", {tr}
x = synth.heavy(R, C, 3, device="cuda")
q = torch.empty(R, C, dtype=torch.uint8, device="cuda"); qt = torch.empty(C, R, dtype=torch.uint8, device="cuda")
s = torch.empty(lk.scale_shape(R, C, gran), dtype=torch.float32, device="cuda")
st = None
if tr:
    tg = {{"row": "col", "col": "row", "blk_1x128": "blk_128x1", "blk_128x1": "blk_1x128"}}.get(gran, gran)
    st = torch.empty(lk.scale_shape(C, R, tg), dtype=torch.float32, device="cuda")
for it in range(3):
    lk.loka_quantize(x, "e4m3", gran, out=q, scales=s, transpose=tr, out_t=qt if tr else None, scales_t=st)
torch.cuda.synchronize()
print("OK")
'''
for R in (8192, 16384, 32768):
    for gran, tr in (("blk_1x128", False), ("blk_128x128", False), ("blk_128x1", False), ("col", False),
                     ("row", True), ("tensor", True), ("blk_128x1", True)):
        code = CASE.format(root=ROOT, R=R, C=4096, gran=gran, tr=tr)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
        last = (r.stdout.strip().splitlines() or [""])[-1]
        err = [l for l in r.stderr.splitlines() if "Error" in l or "error" in l][-1:] 
        print(R, gran, tr, last or "FAIL", err, flush=True)
