"""Scratch: is the ~8-10 us 'fixed cost' of a small graph replay GPU time or host submission lag?
Times the cfg2 grouped quantize and the tiny case with a write flush, and with a GPU spin
(torch.cuda._sleep) before each timed replay that lets the host run ahead."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

dev = torch.device("cuda")
s = torch.cuda.Stream()
big = torch.empty(64 << 20, dtype=torch.float32, device=dev)


class Spin:
    def __init__(self, flush):
        self.flush = flush

    def zero_(self):
        if self.flush is not None:
            self.flush.zero_()
        torch.cuda._sleep(200000)  # ~100 us of GPU spin: the host gets ahead of the GPU


x = synth.gaussian(bench.M_PER_GPU, bench.DIMS[0], 0, device=dev)
w = [synth.weight(bench.DIMS[l + 1], bench.DIMS[l], 100 + l, device=dev) for l in range(8)]
tiny = [torch.randn(16, 1024, device=dev).bfloat16() for _ in range(9)]
st = bench.Fp8Stack(lk, x, w)
cases = {"tiny 9x16 rows": tiny, "X + 8 W": [x] + w}
for name, ts_in in cases.items():
    outs = [(torch.empty(t.shape, dtype=torch.uint8, device=dev), torch.empty(t.shape[0], device=dev)) for t in ts_in]
    fn = lambda: lk.loka_quantize_grouped(ts_in, outs=[o for o, _ in outs], scales=[c for _, c in outs])  # noqa: E731
    g = bench.capture(fn, s)
    for fname, fl in [("flush", big), ("flush+spin", Spin(big)), ("spin only", Spin(None))]:
        t = sorted(bench.time_steps(g.replay, 40, 5, fl, s))
        print(f"{name:16s} {fname:10s} median {1e3 * t[20]:.2f} us  min {1e3 * t[0]:.2f} us", flush=True)
for name, fn in [("stack", lambda: st.stack_only(s.cuda_stream)), ("step", lambda: st.step(s.cuda_stream))]:
    g = bench.capture(fn, s)
    for fname, fl in [("flush", big), ("flush+spin", Spin(big))]:
        t = sorted(bench.time_steps(g.replay, 40, 5, fl, s))
        print(f"{name:16s} {fname:10s} median {1e3 * t[20]:.2f} us  min {1e3 * t[0]:.2f} us", flush=True)
