"""Time the parts of the cfg2 bench step separately (graph of each, L2 flushed before every replay,
CUDA events): grouped quantize alone, stack alone, the whole step."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

dev = torch.device("cuda")
x = synth.gaussian(bench.M_PER_GPU, bench.DIMS[0], 0, device=dev)
w = [synth.weight(bench.DIMS[l + 1], bench.DIMS[l], 100 + l, device=dev) for l in range(8)]
st = bench.Fp8Stack(lk, x, w)
s = torch.cuda.Stream()
sh = s.cuda_stream
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for name, fn in [("quantize", lambda: st.quantize_all(sh)), ("stack", lambda: st.stack_only(sh)),
                 ("step", lambda: st.step(sh)), ("quantize", lambda: st.quantize_all(sh))]:
    g = bench.capture(fn, s)
    ts = sorted(bench.time_steps(g.replay, 40, 5, flush, s))
    print(f"{name:10s} median {1e3 * ts[20]:.2f} us  min {1e3 * ts[0]:.2f} us")
