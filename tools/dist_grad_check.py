"""Multi-GPU check + timing of the quantized DP gradient reduce-scatter (NEXT-4, D39):

  torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port P tools/dist_grad_check.py \
      [p2p|nccl] [rows cols] [--bench]

Rank p's gradient is synth.grad(rows, cols, 100 + p) (bf16, regenerated on every rank for the
check); each rank reduces its row shard with QuantizedGradReducer and compares it with
oracle/gradcomm.py (FP32 tolerance).  --bench times the call (CUDA events, max over ranks) next to
NCCL reduce_scatter of the FP32 and BF16 gradients.  Prints one JSON line on rank 0."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402,F401
from paper_2605_10886_b200 import dist as ldist  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    transport = args[0] if args else "p2p"
    rows = int(args[1]) if len(args) > 1 else 4096
    cols = int(args[2]) if len(args) > 2 else 4096
    bench = "--bench" in sys.argv
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    red = ldist.QuantizedGradReducer(rows, cols, "e5m2", transport=transport, device=dev)
    g = synth.grad(rows, cols, 100 + rank, device=dev)
    out = red.reduce_scatter(g)
    torch.cuda.synchronize()
    import oracle  # the check (test infrastructure)
    grads = [synth.grad(rows, cols, 100 + p, device=dev).double().cpu().numpy() for p in range(world)]
    ref, _, _ = oracle.gradcomm.quantized_allreduce(grads, "e5m2")
    r0, r1 = red.r0, red.r1
    mag = sum(np.abs(x) for x in grads)[r0:r1] * 1.25 + 1e-30
    err = np.abs(out.double().cpu().numpy() - ref[r0:r1])
    ok = bool((err <= world * 2.0 ** -23 * mag).all())
    line = {"world": world, "transport": red.transport, "rows": rows, "cols": cols, "ok": ok,
            "max_abs_err": float(err.max()) if err.size else 0.0}
    if bench:
        def timed(fn, n=20):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                fn()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / n], device=dev, dtype=torch.float64)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        g32 = g.float()
        n = r1 - r0
        o32 = torch.empty(n, cols, dtype=torch.float32, device=dev)
        o16 = torch.empty(n, cols, dtype=torch.bfloat16, device=dev)
        line["ms_quantized"] = timed(lambda: red.reduce_scatter(g, out))
        if world > 1 and rows % world == 0:
            line["ms_nccl_fp32_reduce_scatter"] = timed(lambda: dist.reduce_scatter_tensor(o32, g32))
            line["ms_nccl_bf16_reduce_scatter"] = timed(lambda: dist.reduce_scatter_tensor(o16, g))
        line["payload_bytes_per_rank"] = {"fp8": rows * cols + 4 * rows, "fp32": 4 * rows * cols,
                                          "bf16": 2 * rows * cols}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
