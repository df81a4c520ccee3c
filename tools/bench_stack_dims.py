"""Time the fused stack launch for arbitrary layer dims (CUDA graph of the launch, L2 flushed before
each replay, CUDA events); used to compare stack variants (e.g. LOKA_STACK_PAIR=0/1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

dims = [int(v) for v in sys.argv[1].split(",")]
M = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dev = torch.device("cuda")
x = synth.gaussian(M, dims[0], 0, device=dev)
xq, xs = lk.loka_quantize(x, "e4m3", "row")
ws = [lk.loka_quantize(synth.weight(dims[l + 1], dims[l], 100 + l, device=dev), "e4m3", "row") for l in range(len(dims) - 1)]
a, y, ys = lk.make_stack_args(xq, xs, ws, norms="layer", out_dtype="bf16")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        lk._check(lk._lib.loka_fp8_mlp_stack(lk.C.byref(a), s.cuda_stream), "stack")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        lk._check(lk._lib.loka_fp8_mlp_stack(lk.C.byref(a), s.cuda_stream), "stack")
ts = []
for _ in range(30):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
fl = sum(2 * M * dims[i] * dims[i + 1] for i in range(len(dims) - 1))
print(f"dims={dims} M={M} pair={os.environ.get('LOKA_STACK_PAIR', 'default')} median {ts[15]:.1f} us "
      f"{fl / ts[15] / 1e6:.1f} TF/s")
