"""cfg5 (BASELINE.json configs[4]): batch-sharded M (global 262144) x K = N = 4096, heavy-tailed X,
tensorwise e4m3 with the NCCL MAX all-reduce of amax (a9), linear + LayerNorm (16-CTA clusters per
4096-wide row), bf16 out, across P GPUs (one process per GPU, torchrun).  Per step and rank:
loka_quantize(AMAX_ONLY) -> all_reduce(MAX) -> loka_quantize(CAST_WITH_AMAX) -> loka_fp8_linear_norm.
Timed with CUDA events between barriers, max over ranks; BF16 path = F.linear + F.layer_norm.

  torchrun --nproc-per-node P --master-addr 127.0.0.1 tools/bench_cfg5.py [--M 262144] [--out f.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402
from paper_2605_10886_b200 import dist as ldist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=262144)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    M, K, N = a.M, a.K, a.N
    r0, r1 = ldist.shard_rows(M, world, rank)
    Ml = r1 - r0
    x = synth.heavy(Ml, K, 3, device=dev, row0=r0, total_rows=M)
    w = synth.weight(N, K, 4, device=dev)
    wq, wsc = lk.loka_quantize(w, "e4m3", "tensor")
    xq = torch.empty(Ml, K, dtype=torch.uint8, device=dev)
    xs = torch.empty(1, dtype=torch.float32, device=dev)
    amax = torch.zeros(1, dtype=torch.float32, device=dev)
    keep = []
    args, y, _ = lk.make_linear_args(xq, xs, wq, wsc, a_gran="tensor", b_gran="tensor", norm="layer",
                                     out_dtype="bf16", keep=keep)
    import ctypes
    wsb = torch.empty(max(1, lk.linear_workspace(args)), dtype=torch.uint8, device=dev)

    def fp8_step():
        lk.loka_quantize(x, "e4m3", "tensor", phase="amax", amax=amax, want_q=False, scales=xs)
        if world > 1:
            dist.all_reduce(amax, op=dist.ReduceOp.MAX)
        lk.loka_quantize(x, "e4m3", "tensor", phase="cast", amax=amax, out=xq, scales=xs)
        st = lk._lib.loka_fp8_linear_norm(ctypes.byref(args), ctypes.c_void_p(wsb.data_ptr()), wsb.numel(),
                                          torch.cuda.current_stream().cuda_stream)
        assert st == 0, st

    amax_local = torch.zeros(1, dtype=torch.float32, device=dev)
    lk.loka_quantize(x, "e4m3", "tensor", phase="amax", amax=amax_local, want_q=False, scales=xs)

    def fp8_step_producer_amax():
        # NEXT-4: X's local amax came from the previous layer's epilogue (amax_out); only the
        # all-reduce + cast + GEMM remain in the step (the amax pass over X disappears)
        amax.copy_(amax_local)
        if world > 1:
            dist.all_reduce(amax, op=dist.ReduceOp.MAX)
        lk.loka_quantize(x, "e4m3", "tensor", phase="cast", amax=amax, out=xq, scales=xs)
        st = lk._lib.loka_fp8_linear_norm(ctypes.byref(args), ctypes.c_void_p(wsb.data_ptr()), wsb.numel(),
                                          torch.cuda.current_stream().cuda_stream)
        assert st == 0, st

    def bf16_step():
        return F.layer_norm(F.linear(x, w), (N,))

    def timed(fn):
        for _ in range(a.warmup):
            fn()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / a.steps], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms8 = timed(fp8_step)
    ms8p = timed(fp8_step_producer_amax)
    msb = timed(bf16_step)
    fl = 2.0 * M * N * K
    if rank == 0:
        res = {"workload": f"cfg5: M={M} (sharded over {world}), K={K}, N={N}, heavy-tailed X, tensorwise e4m3 + NCCL "
                           f"MAX all-reduce of amax, linear + LayerNorm, bf16 out",
               "n_gpus": world, "fp8_ms": round(ms8, 4), "fp8_tflops_total": round(fl / ms8 / 1e9, 1),
               "bf16_ms": round(msb, 4), "bf16_tflops_total": round(fl / msb / 1e9, 1),
               "speedup_vs_bf16": round(msb / ms8, 3),
               "fp8_producer_amax_ms": round(ms8p, 4), "speedup_vs_bf16_producer_amax": round(msb / ms8p, 3),
               "producer_amax_note": "NEXT-4: X's amax supplied by the previous layer's epilogue (amax_out), so the "
                                     "step is all-reduce + cast + GEMM + norm",
               "path": "N > 2048: CTA-pair GEMM (FP32, workspace) + row-wise LayerNorm pass" if lk.linear_workspace(args)
                       else "fused linear_norm", 
               "timing": "CUDA events over the steps (eager; the all-reduce is not graph-captured), max over ranks"}
        print(json.dumps(res))
        if a.out:
            open(a.out, "w").write(json.dumps(res, indent=1))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
