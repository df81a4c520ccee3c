import sys, os, json
sys.path.insert(0, "/root/repo")
import torch, synth, paper_2605_10886_b200 as lk
from bench import capture, time_steps
dev = torch.device("cuda")
R, C = 262144, 4096
stream = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
q = torch.empty(R, C, dtype=torch.uint8, device=dev)
res = {}
for dist in ("gaussian", "heavy"):
    x = synth.heavy(R, C, 3, device=dev) if dist == "heavy" else synth.gaussian(R, C, 3, device=dev)
    amax = torch.zeros(1, dtype=torch.float32, device=dev)
    s1 = torch.empty(1, dtype=torch.float32, device=dev)
    sr = torch.empty(R, dtype=torch.float32, device=dev)
    lk.loka_quantize(x, "e4m3", "tensor", phase="amax", amax=amax, want_q=False, scales=s1)
    for name, fn in (("row", lambda: lk.loka_quantize(x, "e4m3", "row", out=q, scales=sr)),
                     ("tensor_cast", lambda: lk.loka_quantize(x, "e4m3", "tensor", phase="cast", amax=amax, out=q, scales=s1)),
                     ("tensor_cast_amax_x16", lambda: lk.loka_quantize(x, "e4m3", "tensor", phase="cast", amax=amax16, out=q, scales=s1))):
        amax16 = amax * 16
        with torch.cuda.stream(stream):
            g = capture(fn, stream)
            t = time_steps(g.replay, 10, 3, flush, stream)
        res[f"{dist}_{name}"] = round(sum(t) / len(t), 4)
    del x
print(json.dumps(res))
