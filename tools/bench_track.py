"""NEXT-2 measurement: one batched Welford update of LoKA Probe's input tracker
on a B x K bf16 activation batch, vs the same update in torch (column mean, centring, cuBLAS BF16
GEMM xc^T xc, FP32 merge).  CUDA graphs, L2 flushed, CUDA events.

  python tools/bench_track.py [--out profiles/r01_track.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402
from bench import ClockSampler, capture, time_steps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    _clk = ClockSampler(torch.cuda.current_device())  # NVML clocks during the whole measurement
    _clk.__enter__()
    dev = torch.device("cuda")
    stream = torch.cuda.Stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    res = {"what": "one tracker update: column mean, centred transpose, S_b = Xc^T Xc (tensor cores, BF16 in, "
                   "FP32 acc), Sigma += S_b + c delta delta^T", "cases": []}
    for B, K in [(32768, 1024), (32768, 4096), (4096, 4096)]:
        x = synth.heavy(B, K, 5, device=dev)
        tr = lk.InputTracker(K, dev)
        with torch.cuda.stream(stream):
            tr.update(x, stream=stream)
            t = time_steps(capture(lambda: tr.update(x, stream=stream), stream).replay, a.steps, 3, flush, stream)
        ms = sum(t) / len(t)
        mean = torch.zeros(K, dtype=torch.float32, device=dev)
        scat = torch.zeros(K, K, dtype=torch.float32, device=dev)
        n = [B]

        def torch_update():
            mb = x.float().mean(0)
            xc = (x.float() - mb).to(torch.bfloat16)
            sb = torch.matmul(xc.t(), xc, out_dtype=torch.float32) if hasattr(torch.matmul, "out_dtype") else \
                torch.mm(xc.t(), xc).float()
            d = mb - mean
            nn = n[0] + B
            mean.add_(d * (B / nn))
            scat.add_(sb + (n[0] * B / nn) * torch.outer(d, d))
        with torch.cuda.stream(stream):
            torch_update()
            tt = time_steps(capture(torch_update, stream).replay, a.steps, 3, flush, stream)
        mst = sum(tt) / len(tt)
        fl = 2.0 * K * K * B
        res["cases"].append({"B": B, "K": K, "ms": round(ms, 4), "gemm_equiv_tflops": round(fl / ms / 1e9, 1),
                             "torch_ms": round(mst, 4), "speedup_vs_torch": round(mst / ms, 3)})
    _clk.__exit__()
    res["clocks"] = _clk.summary()
    print(json.dumps(res))
    if a.out:
        open(a.out, "w").write(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
