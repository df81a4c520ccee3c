#!/usr/bin/env python
"""bench.py — FP8 linear+norm hot path of LoKA on B200 (BASELINE.json metric), one JSON line.

Headline workload (BASELINE.json configs[4] at P = N GPUs, "cfg5"; the largest LRM shape of the
north star): global batch M = 262144 rows sharded over the ranks (strong scaling), K = N = 4096,
heavy-tailed X (bf16, synth.heavy), tensorwise e4m3 X and W, linear + LayerNorm (gamma = 1, beta = 0),
bf16 out.  One step:
  loka_quantize(X, AMAX_ONLY) -> NCCL all_reduce(MAX) of the amax (N > 1) -> loka_quantize(X,
  CAST_WITH_AMAX) -> loka_quantize(W, tensorwise) -> loka_fp8_linear_norm (CTA-pair FP8 GEMM with the
  LayerNorm fused in its epilogue, pairnorm.cu).
Extras on the same line: "cfg2" (the 8-layer MLP stack, configs[1]) and "cfg3" (the 64-GEMM grouped
ensemble with probe + dispatch, configs[2]).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--no-extras]

Multi-GPU (torchrun, one process per GPU): rank r owns rows [r M/N, (r+1) M/N) of the one global X
(the sharded codes equal the single-GPU codes: MAX is exact, D20); time = max over ranks.
Timing: CUDA events on the launching stream around each step, barrier + synchronize on both sides;
the inputs (2 GB of X at N = 1, 268 MB at N = 8) exceed the 126 MB L2, so no flush between steps.
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
CFG5_M, CFG5_K, CFG5_N = 262144, 4096, 4096
WORKLOAD5 = ("cfg5: global M=262144 sharded over the GPUs (strong scaling), K=N=4096, heavy-tailed X, tensorwise "
             "e4m3 X/W with the NCCL MAX all-reduce of X's amax, FP32 accumulate, linear + fused LayerNorm, bf16 out")
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
    ap.add_argument("--no-extras", action="store_true", help="skip the cfg2 / cfg3 extra keys")
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
            if flush is not None:
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
    """(bf16 burst TF/s, bf16 sustained TF/s, HBM GB/s, source) from the driver-written MEASURED_PEAKS.json."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return (float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), float(d["hbm_gbs"]),
                "measured")
    except Exception:  # noqa: BLE001
        return 1590.0, 1370.0, 6650.0, "fallback"


# ------------------------------------------------------------------------------------------
# cfg5: the headline step
# ------------------------------------------------------------------------------------------
class Cfg5:
    """Preallocated cfg5 step on this rank's shard through the C ABI (libloka.so)."""

    def __init__(self, lk, x, w, dist=None):
        import ctypes as C
        import torch
        self.lk, self.C, self.dist = lk, C, dist
        dev = x.device
        M, K = x.shape
        N = w.shape[0]
        self.x, self.w = x, w
        self.keep = []
        self.xq = torch.empty(M, K, dtype=torch.uint8, device=dev)
        self.xs = torch.empty(1, dtype=torch.float32, device=dev)
        self.amax = torch.zeros(1, dtype=torch.float32, device=dev)
        self.amax2 = torch.zeros(2, dtype=torch.float32, device=dev)  # delayed scaling: [previous, this step]
        self.wq = torch.empty(N, K, dtype=torch.uint8, device=dev)
        self.wsc = torch.empty(1, dtype=torch.float32, device=dev)
        self.y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
        self.tx = lk._tensor(x, lk.BF16, M, K)
        self.tq = lk._tensor(self.xq, lk.E4M3, M, K, self.xs, "tensor")
        self.tw = lk._tensor(w, lk.BF16, N, K)
        self.twq = lk._tensor(self.wq, lk.E4M3, N, K, self.wsc, "tensor")
        self.qws = torch.empty(max(256, int(lk._lib.loka_quantize_workspace_size(C.byref(self.tx), C.byref(self.tq)))),
                               dtype=torch.uint8, device=dev)
        self.wqws = torch.empty(max(256, int(lk._lib.loka_quantize_workspace_size(C.byref(self.tw), C.byref(self.twq)))),
                                dtype=torch.uint8, device=dev)
        self.args, _, _ = lk.make_linear_args(self.xq, self.xs, self.wq, self.wsc, a_gran="tensor", b_gran="tensor",
                                              norm="layer", out_dtype="bf16", y=self.y, keep=self.keep)
        nws = int(lk._lib.loka_linear_workspace_size(C.byref(self.args)))
        self.lws = torch.empty(max(nws, 256), dtype=torch.uint8, device=dev)
        # the headline call: x_recipe with the bf16 X and the (all-reduced) amax -> the tensorwise cast of X
        # runs inside the fused GEMM + LayerNorm kernel (CASTX), overlapped with earlier row blocks' MMAs
        self.fargs, _, _ = lk.make_linear_args(self.xq, self.xs, self.wq, self.wsc, a_gran="tensor", b_gran="tensor",
                                               norm="layer", out_dtype="bf16", y=self.y, keep=self.keep)
        self.fargs.a = lk._tensor(x, lk.BF16, M, K, None, "tensor")
        self.fargs.x_amax = self.amax.data_ptr()
        nfw = int(lk._lib.loka_linear_workspace_size(C.byref(self.fargs)))
        self.fws = torch.empty(max(nfw, 256), dtype=torch.uint8, device=dev)
        self.flops = 2.0 * M * N * K

    def _q(self, tx, tq, phase, amax, ws, sh):
        st = self.lk._lib.loka_quantize(self.C.byref(tx), self.C.byref(tq), None, phase,
                                        None if amax is None else amax.data_ptr(), None, ws.data_ptr(), ws.numel(), sh)
        if st:
            raise self.lk.LokaError(st, "loka_quantize")

    def quantize(self, sh):
        """a1 + a9 + a2: X's local amax, the MAX all-reduce (N > 1), X's cast, W's quantize."""
        lk = self.lk
        self._q(self.tx, self.tq, lk.PHASE["amax"], self.amax, self.qws, sh)
        work = None
        if self.dist is not None:  # the all-reduce overlaps W's quantize; the cast waits for it
            work = self.dist.all_reduce(self.amax, op=self.dist.ReduceOp.MAX, async_op=True)
        self._q(self.tw, self.twq, lk.PHASE["full"], None, self.wqws, sh)
        if work is not None:
            work.wait()
        self._q(self.tx, self.tq, lk.PHASE["cast"], self.amax, self.qws, sh)

    def linear(self, sh):
        """a4 + a5: the fused FP8 GEMM + LayerNorm (the dominant kernel)."""
        st = self.lk._lib.loka_fp8_linear_norm(self.C.byref(self.args), self.C.c_void_p(self.lws.data_ptr()),
                                               self.lws.numel(), sh)
        if st:
            raise self.lk.LokaError(st, "loka_fp8_linear_norm")

    def step(self, sh):
        """The headline step: X's amax -> all-reduce (overlapping W's quantize) -> X's cast -> the fused
        GEMM + LayerNorm kernel on the codes."""
        self.quantize(sh)
        self.linear(sh)

    def step_castx(self, sh):
        """x_recipe with the cast inside the GEMM kernel (LOKA_FUSED_CAST=1 route; measured not faster
        under the power cap, kept as a comparison)."""
        lk = self.lk
        self._q(self.tx, self.tq, lk.PHASE["amax"], self.amax, self.qws, sh)
        work = None
        if self.dist is not None:
            work = self.dist.all_reduce(self.amax, op=self.dist.ReduceOp.MAX, async_op=True)
        self._q(self.tw, self.twq, lk.PHASE["full"], None, self.wqws, sh)
        if work is not None:
            work.wait()
        self.fused(sh)

    def fused(self, sh):
        st = self.lk._lib.loka_fp8_linear_norm(self.C.byref(self.fargs), self.C.c_void_p(self.fws.data_ptr()),
                                               self.fws.numel(), sh)
        if st:
            raise self.lk.LokaError(st, "loka_fp8_linear_norm (x_recipe)")


    def step_delayed(self, sh):
        """NEXT-4 delayed scaling: X cast with the previous step's (all-reduced) amax while the same pass
        records this step's amax for the next (LOKA_PHASE_CAST_DELAYED: no separate amax read of X); the
        all-reduce of the new amax is issued after the GEMM, off the critical path."""
        lk = self.lk
        self._q(self.tx, self.tq, lk.PHASE["delayed"], self.amax2, self.qws, sh)
        self._q(self.tw, self.twq, lk.PHASE["full"], None, self.wqws, sh)
        self.linear(sh)
        self.amax2[0:1].copy_(self.amax2[1:2])
        if self.dist is not None:
            self.dist.all_reduce(self.amax2[0:1], op=self.dist.ReduceOp.MAX)


def cfg5_oracle(rows, seed=3, threads=None):
    """The oracle on a bounded sample of cfg5: `rows` rows of the global heavy-tailed X (tensorwise amax of
    the sample), W's tensorwise quantize, linear + LayerNorm in FP64.  Returns (seconds, flops)."""
    import oracle
    import synth
    x = synth.heavy(rows, CFG5_K, seed, total_rows=CFG5_M).double().numpy()
    w = synth.weight(CFG5_N, CFG5_K, 4).double().numpy()

    def run():
        xq, xs = oracle.quantize.quantize(x, "e4m3", "tensor")
        wq, ws = oracle.quantize.quantize(w, "e4m3", "tensor")
        oracle.linear.linear_norm(xq, xs, "e4m3", "tensor", wq, ws, "e4m3", "tensor", norm="layer")

    t0 = time.perf_counter()
    if threads:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=threads):
            run()
    else:
        run()
    return time.perf_counter() - t0, 2.0 * rows * CFG5_K * CFG5_N


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        return max(int(i.get("num_threads", 1)) for i in threadpool_info()) or 1
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def cpu_baseline(rows=1024):
    dt, fl = cfg5_oracle(rows)
    dt1, _ = cfg5_oracle(rows, threads=1)
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "oracle",
            "sample": f"{rows} of cfg5's {CFG5_M} rows: tensorwise quantize of the sample and of W (4096x4096), "
                      f"linear + LayerNorm, numpy FP64 oracle on the host; {dt:.2f} s",
            "seconds": round(dt, 3),
            "single_thread": {"value": fl / dt1 / 1e12, "seconds": round(dt1, 3), "cores": 1},
            "full_step_extrapolated_s": round(dt * CFG5_M / rows, 1),
            "extrapolation": "linear in rows (rows are independent given the scales; W's quantize counted once "
                             "per sample, so this over-counts it for the full step)"}


def extras_oracle_times():
    """The oracle timed on cfg2 (all 4096 rows, the 8 chained layers with the e4m3 row-scale hand-offs)
    and on a 256-row sample of cfg3's 64 GEMMs (rows are independent under rowwise scales), on the
    host's threads — SURVEY.md §8(d) "oracle timing beside it"; a reported baseline, not a target."""
    import oracle
    import synth
    out = {}
    x = synth.gaussian(M_PER_GPU, DIMS[0], 0).double().numpy()
    w = [synth.weight(DIMS[l + 1], DIMS[l], 100 + l).double().numpy() for l in range(8)]
    t0 = time.perf_counter()
    hq, hs = oracle.quantize.quantize(x, "e4m3", "row")
    for l in range(8):
        wq, ws = oracle.quantize.quantize(w[l], "e4m3", "row")
        y = oracle.linear.linear_norm(hq, hs, "e4m3", "row", wq, ws, "e4m3", "row", norm="layer", eps=1e-5)
        if l < 7:
            hq, hs = oracle.quantize.quantize(y, "e4m3", "row")
    dt = time.perf_counter() - t0
    out["cfg2"] = {"value": flops_per_step() / dt / 1e12, "unit": "TFLOP/s", "seconds": round(dt, 3),
                   "cores": cpu_threads(), "kind": "oracle", "sample": "the full cfg2 step (4096 rows, 8 layers)"}
    S, rows = synth.CFG3_DIMS, 256
    xs = [(synth.heavy(rows, k, i) if i % 2 else synth.gaussian(rows, k, i)).double().numpy() for i, k in enumerate(S)]
    t0 = time.perf_counter()
    for i, k in enumerate(S):
        xq, xsc = oracle.quantize.quantize(xs[i], "e4m3", "row")
        for j, n in enumerate(S):
            wq, wsc = oracle.quantize.quantize(synth.weight(n, k, 1000 + 8 * i + j).double().numpy(), "e4m3", "row")
            oracle.linear.linear_norm(xq, xsc, "e4m3", "row", wq, wsc, "e4m3", "row")
    dt = time.perf_counter() - t0
    fl = sum(2.0 * rows * k * n for k in S for n in S)
    out["cfg3"] = {"value": fl / dt / 1e12, "unit": "TFLOP/s", "seconds": round(dt, 3), "cores": cpu_threads(),
                   "kind": "oracle", "sample": f"{rows} of cfg3's 2048 rows, all 64 GEMMs incl. the 64 weight quantizes"}
    return out


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, each step a 256-row sample of cfg5 (W quantize
    included), on the host's cores; rank 0 only."""
    if rank != 0:
        return
    rows = 256
    for _ in range(args.warmup):
        cfg5_oracle(rows)
    ts = [cfg5_oracle(rows)[0] for _ in range(args.steps)]
    tot = sum(ts)
    fl = 2.0 * rows * CFG5_K * CFG5_N
    val = fl * args.steps / tot / 1e12
    cb = {"value": val, "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "oracle",
          "sample": f"each step = {rows} of cfg5's {CFG5_M} rows: tensorwise quantize of the sample and of W "
                    "(4096x4096), linear + LayerNorm, numpy FP64 oracle on the host"}
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD5, "rows_per_step": rows, "parallelism": "host"},
            "cpu_baseline": cb, "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# extras: cfg2 (the fused 8-layer stack) and cfg3 (the grouped 64-GEMM ensemble)
# ------------------------------------------------------------------------------------------
def cfg2_extra(lk, dev, rank, steps, warmup, stream):
    import torch
    import synth
    x = synth.gaussian(M_PER_GPU, DIMS[0], rank, device=dev)
    w = [synth.weight(DIMS[l + 1], DIMS[l], 100 + l, device=dev) for l in range(8)]
    stack = Fp8Stack(lk, x, w)
    sh = stream.cuda_stream
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    g8 = capture(lambda: stack.step(sh), stream)
    t8 = time_steps(g8.replay, steps, warmup, flush, stream)
    gst = capture(lambda: stack.stack_only(sh), stream)
    tst = time_steps(gst.replay, steps, warmup, flush, stream)
    out_bf = torch.empty(M_PER_GPU, DIMS[8], dtype=torch.bfloat16, device=dev)
    gb = capture(lambda: bf16_step(x, w, out_bf), stream)
    tb = time_steps(gb.replay, steps, warmup, flush, stream)
    # the library's own BF16 path (kind::f16 CTA-pair engine + the same fused LayerNorm), layer by layer
    # (a BF16 layer input of 128 rows x 1024 K is 256 KB: it cannot stay resident in one CTA's shared
    # memory, so there is no BF16 form of the one-launch stack)
    import ctypes
    hb = [x.to(torch.bfloat16)] + [torch.empty(M_PER_GPU, DIMS[l + 1], dtype=torch.bfloat16, device=dev)
                                   for l in range(8)]
    wb = [t.to(torch.bfloat16) for t in w]
    one = torch.ones(1, dtype=torch.float32, device=dev)
    keep, bl_args = [], []
    for l in range(8):
        ar, _, _ = lk.make_linear_args(hb[l], one, wb[l], one, a_gran="tensor", b_gran="tensor", norm="layer",
                                       eps=1e-5, out_dtype="bf16", y=hb[l + 1], keep=keep)
        ar.a.dtype = lk.BF16
        ar.b.dtype = lk.BF16
        bl_args.append(ar)
    bl_ws = torch.empty(max(256, max(int(lk._lib.loka_bf16_linear_workspace_size(ctypes.byref(a_))) for a_ in bl_args)),
                        dtype=torch.uint8, device=dev)

    def bf16_lib_step():
        for a_ in bl_args:
            assert lk._lib.loka_bf16_linear_norm(ctypes.byref(a_), ctypes.c_void_p(bl_ws.data_ptr()), bl_ws.numel(),
                                                 sh) == 0

    gbl = capture(bf16_lib_step, stream)
    tbl = time_steps(gbl.replay, steps, warmup, flush, stream)
    ms8, msst, msb = sum(t8) / len(t8), sum(tst) / len(tst), sum(tb) / len(tb)
    msbl = sum(tbl) / len(tbl)
    fl = flops_per_step()
    return {"workload": WORKLOAD, "value": round(fl / ms8 / 1e9, 2), "unit": "TFLOP/s", "ms_per_step": round(ms8, 5),
            "step": "1 grouped quantize launch (X + 8 W) + 1 fused 8-layer stack launch, CUDA-graph replay, "
                    "L2 flushed before every step",
            "bf16_ms_per_step": round(msb, 5), "speedup_vs_bf16": round(msb / ms8, 3),
            "bf16_library_fused_ms_per_step": round(msbl, 5), "speedup_vs_bf16_library_fused": round(msbl / ms8, 3),
            "bf16_library_fused_impl": "8 x loka_bf16_linear_norm (kind::f16 CTA-pair GEMM + fused LayerNorm), graph",
            "stack_kernel_us": round(1e3 * msst, 3), "stack_kernel_tflops": round(fl / msst / 1e9, 2)}


def cfg3_extra(lk, dev, steps, warmup, stream):
    """The 64-GEMM ensemble: grouped quantize + grouped FP8 launch vs 64 cuBLAS BF16 GEMMs; probe MERE of
    every layer vs the BF16 outputs; dispatch per layer on per-layer timings (tools/bench_cfg3.py has the
    full per-layer table)."""
    import ctypes
    import torch
    import synth
    S, M = synth.CFG3_DIMS, 2048
    xs = [(synth.heavy(M, k, i, device=dev) if i % 2 else synth.gaussian(M, k, i, device=dev)) for i, k in enumerate(S)]
    ws = [[synth.weight(n, k, 1000 + 8 * i + j, device=dev) for j, n in enumerate(S)] for i, k in enumerate(S)]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    flops = sum(2.0 * M * k * n for k in S for n in S)
    xq = [(torch.empty(M, k, dtype=torch.uint8, device=dev), torch.empty(M, dtype=torch.float32, device=dev)) for k in S]
    wq = [[lk.loka_quantize(w, "e4m3", "row") for w in row] for row in ws]
    keep, args, ys = [], [], []
    for i in range(8):
        for j in range(8):
            ar, y, _ = lk.make_linear_args(xq[i][0], xq[i][1], wq[i][j][0], wq[i][j][1], out_dtype="bf16", keep=keep)
            args.append(ar)
            ys.append(y)
    arr = (lk.loka_linear_args * 64)(*args)
    qx = (lk.loka_tensor * 8)()
    qq = (lk.loka_tensor * 8)()
    for i, k in enumerate(S):
        qx[i] = lk._tensor(xs[i], lk.BF16, M, k)
        qq[i] = lk._tensor(xq[i][0], lk.E4M3, M, k, xq[i][1], "row")
    sh = stream.cuda_stream

    def fp8_step():
        assert lk._lib.loka_quantize_grouped(8, qx, qq, None, sh) == 0
        assert lk._lib.loka_grouped_fp8_linear(64, arr, None, 0, sh) == 0

    yb = [[torch.empty(M, n, dtype=torch.bfloat16, device=dev) for n in S] for _ in S]

    def bf16_step_3():
        for i in range(8):
            for j in range(8):
                torch.matmul(xs[i], ws[i][j].t(), out=yb[i][j])

    # the library's own BF16 grouped path (kind::f16 on the same CTA-pair engine, one launch)
    ybl = [[torch.empty(M, n, dtype=torch.bfloat16, device=dev) for n in S] for _ in S]
    one = torch.ones(1, dtype=torch.float32, device=dev)
    bl_args = []
    for i in range(8):
        for j in range(8):
            ar, _, _ = lk.make_linear_args(xs[i], one, ws[i][j], one, a_gran="tensor", b_gran="tensor",
                                           out_dtype="bf16", y=ybl[i][j], keep=keep)
            ar.a.dtype = lk.BF16
            ar.b.dtype = lk.BF16
            bl_args.append(ar)
    bl_arr = (lk.loka_linear_args * 64)(*bl_args)

    def bf16_lib_step_3():
        assert lk._lib.loka_grouped_bf16_linear(64, bl_arr, sh) == 0

    g8 = capture(fp8_step, stream)
    gb = capture(bf16_step_3, stream)
    gbl = capture(bf16_lib_step_3, stream)
    t8 = time_steps(g8.replay, steps, warmup, flush, stream)
    tb = time_steps(gb.replay, steps, warmup, flush, stream)
    tbl = time_steps(gbl.replay, steps, warmup, flush, stream)
    ms8, msb = sum(t8) / len(t8), sum(tb) / len(tb)
    msbl = sum(tbl) / len(tbl)
    g8.replay()
    gb.replay()
    torch.cuda.synchronize()
    stats = lk.probe_stats_to_dicts(lk.loka_probe_error([(ys[8 * i + j], yb[i][j]) for i in range(8) for j in range(8)]))
    mere = [s_["mere"] for s_ in stats]
    geo = math.exp(sum(math.log(max(v, 1e-6)) for v in mere) / len(mere))
    # dispatch: one candidate per layer (FP8 rowwise, its share of the grouped step's time) against the
    # layer's BF16 time share; budget 0.2, min speedup 1.05
    chosen = 0
    for i, k in enumerate(S):
        for j, n in enumerate(S):
            share = 2.0 * M * k * n / flops
            c = lk.loka_dispatch_select([("fp8_rowwise", "fwd", mere[8 * i + j], 1e3 * ms8 * share)],
                                        1e3 * msb * share, 0.2, 1.05)
            chosen += c == 0
    return {"workload": "cfg3: 64 GEMMs M=2048, K,N in " + str(S) + ", 8 shared inputs (odd ones heavy-tailed), bf16",
            "value": round(flops / ms8 / 1e9, 2), "unit": "TFLOP/s", "ms_per_step": round(ms8, 5),
            "step": "grouped rowwise quantize of the 8 inputs + grouped FP8 GEMM (1 persistent launch of 64 problems), CUDA "
                    "graph, L2 flushed", "bf16_ms_per_step": round(msb, 5), "speedup_vs_bf16": round(msb / ms8, 3),
            "bf16_library_grouped_ms_per_step": round(msbl, 5),
            "speedup_vs_bf16_library_grouped": round(msbl / ms8, 3),
            "bf16_library_grouped_impl": "loka_grouped_bf16_linear: the same CTA-pair engine with kind::f16 operands (1 launch)",
            "probe_geomean_mere_vs_bf16": round(geo, 5), "dispatch_fp8_layers": int(chosen),
            "dispatch_rule": "MERE < 0.2 and speedup > 1.05 (time shares of the grouped step)"}


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
    import torch.nn.functional as F

    import synth
    import paper_2605_10886_b200 as lk

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    barrier = (lambda: dist.barrier(device_ids=[local])) if world > 1 else None
    stream = torch.cuda.Stream(device=dev)
    sh = stream.cuda_stream

    # this rank's shard of the one global heavy-tailed X (seed 3); W identical on every rank
    r0 = rank * CFG5_M // world
    r1 = (rank + 1) * CFG5_M // world
    x = synth.heavy(r1 - r0, CFG5_K, 3, device=dev, row0=r0, total_rows=CFG5_M)
    w = synth.weight(CFG5_N, CFG5_K, 4, device=dev)
    step = Cfg5(lk, x, w, dist if world > 1 else None)

    if args.profile_steps:
        with torch.cuda.stream(stream):
            for _ in range(args.profile_steps):
                step.step(sh)
        torch.cuda.synchronize()
        return

    with torch.cuda.stream(stream):
        step.step(sh)  # warm (attributes, NCCL communicator)
    torch.cuda.synchronize()
    n0 = lk.launch_count()
    with torch.cuda.stream(stream):
        step.step(sh)
    torch.cuda.synchronize()
    launches_per_step = lk.launch_count() - n0

    # the timed steps: events at the start, between the quantize calls and the fused GEMM + LayerNorm
    # call, and at the end of every step, so the dominant kernel's time comes from the same steps
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step.step(sh)
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    lk_ = step.lk
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            for e0, e1, e2 in ev:  # = step.step, with an event between the quantize calls and the kernel
                e0.record(stream)
                step.quantize(sh)
                e1.record(stream)
                step.linear(sh)
                e2.record(stream)
        torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    clocks = clk.summary()
    t_fp8 = [e0.elapsed_time(e2) for e0, _, e2 in ev]
    t_q = [e0.elapsed_time(e1) for e0, e1, _ in ev]
    t_lin = [e1.elapsed_time(e2) for _, e1, e2 in ev]
    lin_ms = statistics.median(t_lin)

    # NEXT-4 delayed scaling (extra key): the scale from the previous step's amax, recorded by the cast
    with torch.cuda.stream(stream):
        step.quantize(sh)
        step.amax2[0:1].copy_(step.amax)  # (the first step's "previous" amax)

    def run_delayed():
        with torch.cuda.stream(stream):
            step.step_delayed(sh)


    # BF16 baseline (torch F.linear + F.layer_norm, cuBLAS) on the same shard
    out_bf = torch.empty_like(step.y)

    def run_bf():
        with torch.cuda.stream(stream):
            out_bf.copy_(F.layer_norm(F.linear(x, w), (CFG5_N,)))


    # the library's own BF16 path with the same fused epilogue (kind::f16 on the CTA-pair engine):
    # separates the FP8 gain from the fusion gain (SURVEY.md §8(d) secondary denominator)
    import ctypes
    bargs, _, _ = lk.make_linear_args(x, step.xs, w, step.wsc, a_gran="tensor", b_gran="tensor", norm="layer",
                                      out_dtype="bf16", y=out_bf, keep=step.keep)
    bargs.a.dtype = lk.BF16
    bargs.b.dtype = lk.BF16
    bws = torch.empty(max(256, int(lk._lib.loka_bf16_linear_workspace_size(ctypes.byref(bargs)))), dtype=torch.uint8,
                      device=dev)

    def run_bf_lib():
        with torch.cuda.stream(stream):
            st_ = lk._lib.loka_bf16_linear_norm(ctypes.byref(bargs), ctypes.c_void_p(bws.data_ptr()), bws.numel(), sh)
            assert st_ == 0, st_


    # the comparison paths, interleaved step by step with the FP8 step (same thermal / power state for
    # every path: B200 clocks drift under sustained tensor load, so back-to-back blocks would bias it)
    def run_fp8():
        with torch.cuda.stream(stream):
            step.step(sh)

    def run_castx():
        os.environ["LOKA_FUSED_CAST"] = "1"
        with torch.cuda.stream(stream):
            step.step_castx(sh)
        os.environ.pop("LOKA_FUSED_CAST", None)

    paths = {"fp8": run_fp8, "bf16": run_bf, "delayed": run_delayed, "bf16_lib": run_bf_lib, "castx": run_castx}
    for _ in range(args.warmup):
        for fn in paths.values():
            fn()
    iev = {k: [] for k in paths}
    torch.cuda.synchronize()
    if barrier:
        barrier()
    for _ in range(args.steps):
        for k, fn in paths.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            iev[k].append((e0, e1))
    torch.cuda.synchronize()
    if barrier:
        barrier()
    it = {k: [a.elapsed_time(b) for a, b in v] for k, v in iev.items()}
    t_bf, t_dl, t_bfl, t_fp8i = it["bf16"], it["delayed"], it["bf16_lib"], it["fp8"]
    t_cx = it["castx"]

    def max_over_ranks_early(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # e2e through the public API: pinned host X -> device, the step, device Y -> pinned host, every step
    xh = x.cpu().pin_memory()
    yh = torch.empty(step.y.shape, dtype=torch.bfloat16).pin_memory()

    def run_e2e():
        with torch.cuda.stream(stream):
            step.x.copy_(xh, non_blocking=True)
            step.step(sh)
            yh.copy_(step.y, non_blocking=True)

    e2e_steps = max(3, min(args.steps, 10))
    t_e2e = time_steps(run_e2e, e2e_steps, 1, None, stream, barrier)

    # the same end to end, pipelined across steps: a second buffer set (its own X, codes, Y and
    # workspaces; the same W) so step i+1's H2D copy and step i's D2H copy (separate copy engines,
    # both directions of PCIe at once) overlap each other and the compute — every step still copies
    # its whole input in and its whole result out inside the timed region
    class _Eager:  # time_pipelined replays a "graph"; the cfg5 step runs eagerly (NCCL inside for N > 1)
        def __init__(self, s_):
            self.s_ = s_

        def replay(self):
            self.s_.step(sh)

    step_b = Cfg5(lk, torch.empty_like(x), w, dist if world > 1 else None)
    ms_e2e_pipe = max_over_ranks_early(time_pipelined([(step, _Eager(step)), (step_b, _Eager(step_b))], xh, e2e_steps,
                                                       1, torch.zeros(1, device=dev), stream, barrier)) / e2e_steps
    del step_b

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_fp8 = max_over_ranks(sum(t_fp8)) / args.steps
    ms_fp8i = max_over_ranks(sum(t_fp8i)) / args.steps
    ms_bf = max_over_ranks(sum(t_bf)) / args.steps
    ms_dl = max_over_ranks(sum(t_dl)) / args.steps
    ms_bfl = max_over_ranks(sum(t_bfl)) / args.steps
    ms_q = max_over_ranks(sum(t_q)) / args.steps
    ms_lin = max_over_ranks(lin_ms)
    ms_cx = max_over_ranks(sum(t_cx)) / args.steps
    ms_e2e = max_over_ranks(sum(t_e2e)) / e2e_steps
    fl = 2.0 * CFG5_M * CFG5_N * CFG5_K  # the whole job (all ranks)
    value = fl / (ms_fp8 * 1e-3) / 1e12

    bf16_peak, bf16_sus, hbm_peak, src = peaks()
    fp8_peak_sus, fp8_peak_burst = 2.0 * bf16_sus, 2.0 * bf16_peak  # nominal fp8/bf16 = 4500/2250
    # the denominator: the burst peak when the SM clock held its maximum through the timed steps (the
    # measured sustained figure was taken at ~1.3 GHz under a 4 s cuBLAS loop), else the sustained one
    # (and no throttle reason at all: with sw_power_cap in the samples the median clock can still read
    # max while the kernel ran capped part of the time — profiles/r02aj_bench.json: 1965 MHz median,
    # sw_power_cap, the fused kernel at 2538 TF/s)
    at_max = (clocks.get("sm_mhz") is not None and clocks["sm_mhz"] >= 0.97 * float(clocks.get("sm_max_mhz") or 1e9)
              and not clocks.get("reasons"))
    fp8_peak = fp8_peak_burst if at_max else fp8_peak_sus
    achieved = step.flops / (lin_ms * 1e-3) / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"pairnorm_bytes_per_launch_m{x.shape[0]}")
        except Exception:  # noqa: BLE001
            traffic = None

    extras = {}
    if not args.no_extras:
        extras["cfg2"] = cfg2_extra(lk, dev, rank, args.steps, args.warmup, stream)
        if rank == 0:
            extras["cfg3"] = cfg3_extra(lk, dev, args.steps, args.warmup, stream)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_fp8, 5), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "e4m3", "data": "synthetic",
            "config": {"workload": WORKLOAD5, "model": "cfg5", "global_batch": CFG5_M, "rows_per_gpu": int(x.shape[0]),
                       "K": CFG5_K, "N": CFG5_N, "seq_len": None, "parallelism": f"dp{world} (M sharded)",
                       "l2": "not flushed: the step's inputs (X bf16 2 GB / N GPUs) exceed the 126 MB L2",
                       "step": "loka_quantize AMAX_ONLY -> NCCL all_reduce(MAX) (N > 1, overlapping "
                               "loka_quantize(W, tensorwise)) -> loka_quantize CAST_WITH_AMAX -> "
                               "loka_fp8_linear_norm (fused FP8 GEMM + LayerNorm), eager launches on one stream"},
            "pct_of_4500_tflops": round(100.0 * value / world / 4500.0, 2),
            "compute_only": {"value": round(fl / (ms_lin * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
                             "ms_per_step": round(ms_lin, 5),
                             "pct_of_4500_tflops": round(100.0 * fl / (ms_lin * 1e-3) / 1e12 / world / 4500.0, 2),
                             "what": "the fused GEMM + LayerNorm call of each timed step on the step's codes "
                                     "(events between the quantize calls and it; median over the K steps)"},
            "cast_inside_gemm_step": {"ms_per_step": round(ms_cx, 5), "value": round(fl / (ms_cx * 1e-3) / 1e12, 3),
                                      "vs_step": round(ms_fp8i / ms_cx, 3),
                                      "what": "x_recipe with the tensorwise cast of X inside the GEMM kernel "
                                              "(LOKA_FUSED_CAST=1), interleaved: not faster under the power cap"},
            "quantize_ms_per_step": round(ms_q, 5),
            "bf16_baseline": {"value": round(fl / (ms_bf * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
                              "ms_per_step": round(ms_bf, 5), "impl": "torch F.linear + F.layer_norm (bf16, cuBLAS)"},
            "speedup_vs_bf16": round(ms_bf / ms_fp8i, 3),
            "comparison_protocol": "bf16_baseline, bf16_library_fused, delayed_scaling and fp8_step_interleaved: "
                                   "the K steps of each path interleaved step by step (same clock / power state); "
                                   "speedups divide those",
            "fp8_step_interleaved_ms": round(ms_fp8i, 5),
            "delayed_scaling": {"value": round(fl / (ms_dl * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
                                "ms_per_step": round(ms_dl, 5), "speedup_vs_bf16": round(ms_bf / ms_dl, 3),
                                "vs_current_scaling_step": round(ms_fp8i / ms_dl, 3),
                                "step": "loka_quantize(X, CAST_DELAYED: the previous step's amax, this step's "
                                        "amax recorded in the same read) -> W quantize -> fused GEMM + LayerNorm -> "
                                        "all_reduce(MAX) of the new amax (N > 1) after the GEMM (NEXT-4)"},
            "bf16_library_fused": {"value": round(fl / (ms_bfl * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
                                   "ms_per_step": round(ms_bfl, 5),
                                   "impl": "this library's BF16 path: kind::f16 CTA-pair GEMM + the same fused "
                                           "LayerNorm epilogue (loka_bf16_linear_norm), no quantize",
                                   "fp8_step_speedup": round(ms_bfl / ms_fp8i, 3),
                                   "fp8_compute_only_speedup": round(ms_bfl / ms_lin, 3)},
            "roofline": {"kernel": "pair_norm_kernel<256, LayerNorm> (CTA-pair FP8 GEMM + fused LayerNorm), 1 "
                                   "launch/step", "bound": "tensor", "achieved": round(achieved, 2),
                         "peak": round(fp8_peak, 1), "unit": "TFLOP/s", "frac": round(achieved / fp8_peak, 4),
                         "traffic": traffic,
                         "peak_source": (f"{src}: 2 x bf16 burst {bf16_peak} TF/s (nominal fp8/bf16 ratio; the SM "
                                         "clock stayed at max during the timed steps)") if at_max else
                                        (f"{src}: 2 x bf16 sustained {bf16_sus} TF/s (nominal fp8/bf16 ratio; the "
                                         "clock dropped under the timed steps' load)"),
                         "peak_sustained": round(fp8_peak_sus, 1), "frac_sustained": round(achieved / fp8_peak_sus, 4),
                         "peak_burst": round(fp8_peak_burst, 1), "frac_burst": round(achieved / fp8_peak_burst, 4),
                         "flop_per_launch": step.flops, "launch_ms": round(lin_ms, 4),
                         "algorithmic_bytes_per_launch": int(x.shape[0] * CFG5_K + CFG5_N * CFG5_K +
                                                             x.shape[0] * CFG5_N * 2),
                         "timing": "median over the K timed steps of the launch's events (launching stream)"},
            "e2e": {"value": round(fl / (ms_e2e_pipe * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
                    "ms_per_step": round(ms_e2e_pipe, 5),
                    "h2d_bytes_per_step": int(x.numel() * 2), "d2h_bytes_per_step": int(step.y.numel() * 2),
                    "steps": e2e_steps,
                    "how": "every step: pinned host X -> device (H2D stream), the step (compute stream), device Y "
                           "-> pinned host (D2H stream); two buffer sets, so step i+1's input copy overlaps step "
                           "i's output copy and compute; one event pair around all K steps, streams joined",
                    "serial": {"value": round(fl / (ms_e2e * 1e-3) / 1e12, 3), "ms_per_step": round(ms_e2e, 5),
                               "how": "the same copies and step on one stream, no overlap"}},
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clocks,
        }
        line.update(extras)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
            if extras:
                try:
                    for k_, v_ in extras_oracle_times().items():
                        if k_ in line:
                            line[k_]["cpu_oracle"] = v_
                except Exception as e:  # noqa: BLE001  (a reported baseline: never fails the bench line)
                    line["cpu_oracle_error"] = str(e)[:200]
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
