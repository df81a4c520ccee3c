"""Scratch: the event-to-event floor of one graph replay (write-flushed L2 before each), for a
trivial torch kernel, an empty graph, and the library's tiny grouped quantize (TMA and register
variants via LOKA_QUANT_TMA)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

dev = torch.device("cuda")
s = torch.cuda.Stream()
big = torch.empty(64 << 20, dtype=torch.float32, device=dev)
small = torch.zeros(1024, device=dev)
tiny = [torch.randn(16, 1024, device=dev).bfloat16() for _ in range(9)]
outs = [(torch.empty(t.shape, dtype=torch.uint8, device=dev), torch.empty(t.shape[0], device=dev)) for t in tiny]
one = [tiny[0]]
for name, fn in [("torch add_ (1 kernel)", lambda: small.add_(1)),
                 ("torch add_ x2", lambda: (small.add_(1), small.mul_(1))),
                 ("grouped quantize 9x16 rows", lambda: lk.loka_quantize_grouped(tiny, outs=[o for o, _ in outs], scales=[c for _, c in outs])),
                 ("quantize 16 rows", lambda: lk.loka_quantize_grouped(one, outs=[outs[0][0]], scales=[outs[0][1]]))]:
    g = bench.capture(fn, s)
    t = sorted(bench.time_steps(g.replay, 60, 5, big, s))
    print(f"{name:28s} median {1e3 * t[30]:.2f} us  min {1e3 * t[0]:.2f} us", flush=True)
