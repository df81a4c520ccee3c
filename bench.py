#!/usr/bin/env python
"""bench.py — FP8 linear+norm hot path of LoKA on B200 (BASELINE.json metric), one JSON line.

Workload (BASELINE.json configs[1], "cfg2"): LRM MLP stack, batch M = 4096 per GPU, 8 layers with
dims [1024,1024,1024,512,512,256,256,512,1024]; every layer is rowwise-e4m3 FP8 linear + LayerNorm;
layers 0-6 hand their output to the next layer as e4m3 + row scales (fused in the epilogue),
layer 7 emits bf16.  One step = quantize X + quantize the 8 weights + 8 fused linear+LayerNorm
launches, captured once in a CUDA graph and replayed.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun, one process per GPU): every rank runs its own batch of 4096 rows (data
parallel, weak scaling, no data-path collective: the rowwise recipe needs none); the time is the
max over ranks.  Timing: CUDA events on the launching stream around each step, L2 flushed
(256 MiB write) before every timed step, W warm-up steps, exactly K timed steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP8 linear+norm TFLOP/s (% of 4.5 PF) and speedup vs BF16, 1/2/4/8 B200"
DIMS = [1024, 1024, 1024, 512, 512, 256, 256, 512, 1024]
M_PER_GPU = 4096
WORKLOAD = ("cfg2 LRM MLP stack: M=4096 per GPU, 8 layers dims " + str(DIMS) +
            ", rowwise e4m3 X/W fwd, FP32 accumulate, fused LayerNorm, e4m3+row-scale hand-off, bf16 out")


def flops_per_step(M=M_PER_GPU, dims=DIMS):
    return 2.0 * M * sum(dims[l] * dims[l + 1] for l in range(len(dims) - 1))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="loka", choices=["loka", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=0, help="run N eager steps only (for ncu), no JSON")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------
# clocks (NVML polled from a thread during the timed region)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x10: "sync_boost",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            print(f"[bench] NVML unavailable: {e}", file=sys.stderr)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b], "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------
# the LoKA FP8 step and the BF16 baseline step
# ------------------------------------------------------------------------------------------
class Fp8Stack:
    """Preallocated cfg2 forward through the C ABI (libloka.so)."""

    def __init__(self, lk, x_bf16, w_bf16):
        import ctypes as C
        import torch
        self.lk, self.C = lk, C
        dev = x_bf16.device
        M = x_bf16.shape[0]
        self.x, self.w = x_bf16, w_bf16
        self.keep = []
        self.xq = torch.empty(M, DIMS[0], dtype=torch.uint8, device=dev)
        self.xs = torch.empty(M, dtype=torch.float32, device=dev)
        self.wq = [torch.empty_like(w, dtype=torch.uint8) for w in w_bf16]
        self.wsc = [torch.empty(w.shape[0], dtype=torch.float32, device=dev) for w in w_bf16]
        self.hq = [torch.empty(M, DIMS[l + 1], dtype=torch.uint8, device=dev) for l in range(7)]
        self.hs = [torch.empty(M, dtype=torch.float32, device=dev) for l in range(7)]
        self.y = torch.empty(M, DIMS[8], dtype=torch.bfloat16, device=dev)
        self.ws = torch.empty(256, dtype=torch.uint8, device=dev)
        # one grouped quantize launch: X and every layer's weight (rowwise e4m3)
        srcs = [(self.x, self.xq, self.xs)] + list(zip(self.w, self.wq, self.wsc))
        self.G = len(srcs)
        self.qx = (lk.loka_tensor * self.G)()
        self.qq = (lk.loka_tensor * self.G)()
        for g, (src, dst, sc) in enumerate(srcs):
            r, c = src.shape
            self.qx[g] = lk._tensor(src, lk.BF16, r, c)
            self.qq[g] = lk._tensor(dst, lk.E4M3, r, c, sc, "row")
        # linear argument structs
        self.largs = []
        for l in range(8):
            a, asc = (self.xq, self.xs) if l == 0 else (self.hq[l - 1], self.hs[l - 1])
            last = l == 7
            args, _, _ = lk.make_linear_args(a, asc, self.wq[l], self.wsc[l], norm="layer",
                                             out_dtype="bf16" if last else "e4m3",
                                             y=self.y if last else self.hq[l], y_scales=None if last else self.hs[l],
                                             keep=self.keep)
            self.largs.append(args)
        # the fused stack: all 8 layers in one launch, same output bits as the per-layer chain
        self.sargs, _, _ = lk.make_stack_args(self.xq, self.xs, list(zip(self.wq, self.wsc)), norms="layer",
                                              out_dtype="bf16", y=self.y)

    def quantize_all(self, stream_handle):
        st = self.lk._lib.loka_quantize_grouped(self.G, self.qx, self.qq, None, stream_handle)
        if st:
            raise self.lk.LokaError(st, "loka_quantize_grouped")

    def stack_only(self, stream_handle):
        st = self.lk._lib.loka_fp8_mlp_stack(self.C.byref(self.sargs), stream_handle)
        if st:
            raise self.lk.LokaError(st, "loka_fp8_mlp_stack")

    def step(self, stream_handle):
        """The bench step: 1 grouped quantize launch + 1 fused stack launch."""
        self.quantize_all(stream_handle)
        self.stack_only(stream_handle)

    def step_per_layer(self, stream_handle):
        """Reference path: the same step with one fused linear+norm launch per layer."""
        lib, C = self.lk._lib, self.C
        self.quantize_all(stream_handle)
        for a in self.largs:
            st = lib.loka_fp8_linear_norm(C.byref(a), None, 0, stream_handle)
            if st:
                raise self.lk.LokaError(st, "loka_fp8_linear_norm")

    def linear_only(self, l, stream_handle):
        st = self.lk._lib.loka_fp8_linear_norm(self.C.byref(self.largs[l]), None, 0, stream_handle)
        if st:
            raise self.lk.LokaError(st, "loka_fp8_linear_norm")


def bf16_step(x, w, out):
    import torch.nn.functional as F
    h = x
    for l in range(8):
        h = F.layer_norm(F.linear(h, w[l]), (DIMS[l + 1],))
    out.copy_(h)


def capture(fn, stream):
    import torch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        fn()  # warm (allocations, attributes)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=stream):
            fn()
    torch.cuda.synchronize()
    return g


def time_steps(run, steps, warmup, flush, stream, barrier=None):
    """W untimed warm-ups, then exactly K timed steps; events around each step, L2 flushed before."""
    import torch
    for _ in range(warmup):
        run()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for e0, e1 in ev:
            flush.zero_()
            e0.record(stream)
            run()
            e1.record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    return [e0.elapsed_time(e1) for e0, e1 in ev]  # ms


def time_pipelined(sets, xh, steps, warmup, flush, stream, barrier=None):
    """End-to-end loop through the public API with double buffering: step i's H2D copy (pinned host
    X -> sets[i%2].x) on an H2D stream, its graph (L2 flush first) on `stream`, its D2H copy
    (y -> pinned host) on a D2H stream; events order reuse of each buffer set.  Returns the total ms
    of exactly `steps` steps, one event pair around the whole loop (all streams joined)."""
    import torch
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    yh = [torch.empty_like(s.y, device="cpu").pin_memory() for s, _ in sets]
    nb = len(sets)

    def run(n):
        ev_in = [None] * nb
        ev_c = [None] * nb
        ev_out = [None] * nb
        for i in range(n):
            b = i % nb
            s, g = sets[b]
            with torch.cuda.stream(h2d):
                if ev_c[b] is not None:
                    h2d.wait_event(ev_c[b])  # the previous user of x[b] finished
                s.x.copy_(xh, non_blocking=True)
                ev_in[b] = torch.cuda.Event()
                ev_in[b].record(h2d)
            stream.wait_event(ev_in[b])
            if ev_out[b] is not None:
                stream.wait_event(ev_out[b])  # y[b] of step i-nb copied out
            with torch.cuda.stream(stream):
                flush.zero_()
                g.replay()
            ev_c[b] = torch.cuda.Event()
            ev_c[b].record(stream)
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_c[b])
                yh[b].copy_(s.y, non_blocking=True)
                ev_out[b] = torch.cuda.Event()
                ev_out[b].record(d2h)
        for e in ev_out:
            if e is not None:
                stream.wait_event(e)

    run(warmup)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h2d.wait_event(e0)
    d2h.wait_event(e0)
    run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["bf16_tflops"]), float(d["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 1590.0, 6650.0, "fallback"


# ------------------------------------------------------------------------------------------
# oracle (CPU) legs: cpu_baseline (rank 0, N=1) and --impl reference
# ------------------------------------------------------------------------------------------
def oracle_forward(x_np, w_np):
    import numpy as np
    import oracle
    hq, hs = oracle.quantize.quantize(x_np, "e4m3", "row")
    y = None
    for l in range(8):
        wq, wsc = oracle.quantize.quantize(w_np[l], "e4m3", "row")
        y = oracle.linear.linear_norm(hq, hs, "e4m3", "row", wq, wsc, "e4m3", "row", norm="layer")
        if l < 7:
            hq, hs = oracle.quantize.quantize(y.astype(np.float32).astype(np.float64), "e4m3", "row")
    return y


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        return max(int(i.get("num_threads", 1)) for i in threadpool_info()) or 1
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def oracle_inputs(rows, seed):
    import synth
    x = synth.gaussian(rows, DIMS[0], seed).double().numpy()
    w = [synth.weight(DIMS[l + 1], DIMS[l], 100 + l).double().numpy() for l in range(8)]
    return x, w


def cpu_baseline(rows=M_PER_GPU, seed=0):
    x, w = oracle_inputs(rows, seed)
    t0 = time.perf_counter()
    oracle_forward(x, w)
    dt = time.perf_counter() - t0
    return {"value": flops_per_step(rows) / dt / 1e12, "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "oracle",
            "sample": f"full cfg2 step on {rows} rows (8 layers, weight quantize included), numpy FP64 oracle, "
                      f"{dt:.2f} s", "seconds": dt}


def run_reference(args, rank, world):
    if rank != 0:
        return
    rows = 512
    x, w = oracle_inputs(rows, 0)
    for _ in range(args.warmup):
        oracle_forward(x, w)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle_forward(x, w)
        ts.append(time.perf_counter() - t0)
    tot = sum(ts)
    val = flops_per_step(rows) * args.steps / tot / 1e12
    cb = {"value": val, "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "oracle",
          "sample": f"each step = cfg2 forward on {rows} of the 4096 rows (8 layers incl. weight quantize), "
                    "numpy FP64 oracle on the host"}
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "rows_per_step": rows, "parallelism": "host"},
            "cpu_baseline": cb, "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import synth
    import paper_2605_10886_b200 as lk

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    barrier = (lambda: dist.barrier(device_ids=[local])) if world > 1 else None

    # inputs: rank r owns its own 4096-row batch (seed r); weights identical on every rank
    x = synth.gaussian(M_PER_GPU, DIMS[0], rank, device=dev)
    w = [synth.weight(DIMS[l + 1], DIMS[l], 100 + l, device=dev) for l in range(8)]
    stack = Fp8Stack(lk, x, w)
    stream = torch.cuda.Stream(device=dev)
    sh = stream.cuda_stream

    if args.profile_steps:
        with torch.cuda.stream(stream):
            for _ in range(args.profile_steps):
                stack.step(sh)
        torch.cuda.synchronize()
        return

    n0 = lk.launch_count()
    with torch.cuda.stream(stream):
        stack.step(sh)
    torch.cuda.synchronize()
    launches_per_step = lk.launch_count() - n0

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    g8 = capture(lambda: stack.step(sh), stream)
    with ClockSampler(local) as clk:
        t_fp8 = time_steps(g8.replay, args.steps, args.warmup, flush, stream, barrier)
    clocks = clk.summary()

    # The dominant kernel (the fused stack launch): a graph of that one launch, replayed with the L2
    # flushed before each replay, timed with events on the launching stream.
    gst = capture(lambda: stack.stack_only(sh), stream)
    t_st = time_steps(gst.replay, args.steps, args.warmup, flush, stream, None)
    stack_ms = sum(t_st) / len(t_st)
    # the per-layer path (one linear_norm launch per layer) for comparison
    gpl = capture(lambda: stack.step_per_layer(sh), stream)
    t_pl = time_steps(gpl.replay, args.steps, args.warmup, flush, stream, None)
    per_layer_ms = sum(t_pl) / len(t_pl)

    # BF16 baseline (torch F.linear + F.layer_norm, graph-captured) on the same inputs
    out_bf = torch.empty(M_PER_GPU, DIMS[8], dtype=torch.bfloat16, device=dev)
    gb = capture(lambda: bf16_step(x, w, out_bf), stream)
    t_bf = time_steps(gb.replay, args.steps, args.warmup, flush, stream, barrier)

    # e2e through the public API: pinned host X -> device, graph step, device Y -> pinned host
    xh = x.cpu().pin_memory()
    yh = torch.empty(M_PER_GPU, DIMS[8], dtype=torch.bfloat16).pin_memory()

    def e2e_step():
        stack.x.copy_(xh, non_blocking=True)
        g8.replay()
        yh.copy_(stack.y, non_blocking=True)

    t_e2e = time_steps(e2e_step, args.steps, args.warmup, flush, stream, barrier)
    # the same, pipelined as a serving loop would run it: two buffer sets, the H2D copy of step i+1
    # and the D2H copy of step i-1 on their own streams (PCIe is full duplex) under step i's kernels
    stack2 = Fp8Stack(lk, torch.empty_like(x), w)
    g8b = capture(lambda: stack2.step(sh), stream)
    t_pipe = time_pipelined([(stack, g8), (stack2, g8b)], xh, args.steps, args.warmup, flush, stream, barrier)

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_fp8 = max_over_ranks(sum(t_fp8)) / args.steps
    ms_bf = max_over_ranks(sum(t_bf)) / args.steps
    ms_e2e_serial = max_over_ranks(sum(t_e2e)) / args.steps
    ms_e2e = max_over_ranks(t_pipe) / args.steps
    fl = flops_per_step() * world
    value = fl / (ms_fp8 * 1e-3) / 1e12
    bf_value = fl / (ms_bf * 1e-3) / 1e12
    e2e_value = fl / (ms_e2e * 1e-3) / 1e12
    e2e_serial_value = fl / (ms_e2e_serial * 1e-3) / 1e12

    bf16_peak, hbm_peak, src = peaks()
    fp8_peak = 2.0 * bf16_peak  # nominal dense fp8/bf16 ratio 4500/2250
    stack_fl = flops_per_step()  # one stack launch = the 8 layers' 2 M K N
    achieved = stack_fl / (stack_ms * 1e-3) / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("stack_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_fp8, 5), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "e4m3", "data": "synthetic",
            "config": {"workload": WORKLOAD, "model": "cfg2", "global_batch": M_PER_GPU * world,
                       "seq_len": None, "parallelism": f"dp{world}",
                       "l2": "flushed before every timed step (256 MiB write)",
                       "step": "1 grouped quantize launch (X + 8 W, rowwise e4m3) + 1 fused 8-layer FP8 "
                               "linear+LayerNorm stack launch, CUDA-graph replay"},
            "pct_of_4500_tflops": round(100.0 * value / world / 4500.0, 2),
            "bf16_baseline": {"value": round(bf_value, 3), "unit": "TFLOP/s", "ms_per_step": round(ms_bf, 5),
                              "impl": "torch F.linear + F.layer_norm (bf16, cuBLAS), CUDA-graph replay"},
            "speedup_vs_bf16": round(ms_bf / ms_fp8, 3),
            "roofline": {"kernel": "stack_kernel (8 fused FP8 GEMM + LayerNorm layers), 1 launch/step",
                         "bound": "tensor", "achieved": round(achieved, 2), "peak": round(fp8_peak, 1),
                         "unit": "TFLOP/s", "frac": round(achieved / fp8_peak, 4), "traffic": traffic,
                         "peak_source": f"{src}: 2 x bf16 {bf16_peak} TF/s (nominal fp8/bf16 ratio)",
                         "flop_per_launch": stack_fl, "launch_us": round(1e3 * stack_ms, 3),
                         "timing": "graph of the launch, L2 flushed before each replay, CUDA events"},
            "per_layer_path": {"ms_per_step": round(per_layer_ms, 5),
                               "value": round(flops_per_step() / (per_layer_ms * 1e-3) / 1e12, 3),
                               "impl": "grouped quantize + 8 linear_norm launches (same layers, per-layer kernels)"},
            "e2e": {"value": round(e2e_value, 3), "unit": "TFLOP/s", "ms_per_step": round(ms_e2e, 5),
                    "h2d_bytes_per_step": int(x.numel() * 2), "d2h_bytes_per_step": int(stack.y.numel() * 2),
                    "how": "pinned host X -> device, graph step (quantize + stack, L2 flushed first), "
                           "device Y -> pinned host, every step; double-buffered: H2D / compute / D2H on three "
                           "streams, one event pair around all K steps",
                    "serial": {"value": round(e2e_serial_value, 3), "ms_per_step": round(ms_e2e_serial, 5),
                               "how": "same copies, one stream, no overlap"}},
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clocks,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
