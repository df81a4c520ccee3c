"""Data-parallel plumbing for the LoKA hot path (a9) — host glue only.

The batch dimension M is sharded over ranks (one process per GPU, torch.distributed over NCCL).
Rowwise / 1x128 / 128x128 granules never cross a shard, so they need no
communication.  Tensorwise scaling is the one real exchange step (BASELINE.json north_star
"NCCL over NVLink is used only for ... the tensorwise amax all-reduce"):

    loka_quantize(PHASE_AMAX_ONLY)  -> local amax (device float, libloka kernel)
    all_reduce(amax, op=MAX)        -> global amax (4 bytes over NVLink / NVSwitch)
    loka_quantize(PHASE_CAST)       -> codes with the global scale (libloka kernel)

MAX is exact and order-independent, so every rank's codes equal the single-GPU codes of the
concatenated tensor (D20).  The amax / cast steps are injectable only so the protocol
can be exercised by CPU gloo tests; the default is libloka on the current CUDA stream.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(total_rows: int, world: int, rank: int):
    """Rows [r0, r1) of rank `rank` when `total_rows` are split over `world` ranks as evenly as
    possible (the first total % world ranks get one extra row)."""
    base, extra = divmod(total_rows, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def _lk():
    import paper_2605_10886_b200 as lk  # the CUDA library; raises if it is missing
    return lk


def _default_amax(x, fmt):
    lk = _lk()
    amax = torch.empty(1, dtype=torch.float32, device=x.device)
    lk.loka_quantize(x, fmt, "tensor", phase="amax", amax=amax, want_q=False)
    return amax


def _default_cast(x, fmt, amax, scale_fmt):
    lk = _lk()
    return lk.loka_quantize(x, fmt, "tensor", scale_fmt, phase="cast", amax=amax)


def quantize_tensorwise_sharded(x_local: torch.Tensor, fmt: str = "e4m3", scale_fmt: str = "f32", group=None,
                                amax_fn=None, cast_fn=None):
    """Tensorwise quantization of a row-sharded tensor with a global scale.

    Returns (codes_local, scale[1], global_amax[1]).  With world_size 1 (or no initialised
    process group) this is exactly loka_quantize(..., "tensor")."""
    amax = (amax_fn or _default_amax)(x_local, fmt)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(amax, op=dist.ReduceOp.MAX, group=group)
    q, s = (cast_fn or _default_cast)(x_local, fmt, amax, scale_fmt)
    return q, s, amax


def reduce_probe_stats(stats_list, group=None):
    """Combine per-rank probe statistics of one layer: counts and sums add,
    maxima max; MERE = sum of per-element relative errors / total count."""
    keys = ("mere", "max_rel", "sum_abs_ref", "count", "n_floored")
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return stats_list
    out = []
    for st in stats_list:
        t = torch.tensor([st["mere"] * st["count"], st["sum_abs_ref"], float(st["count"]), float(st["n_floored"])],
                         dtype=torch.float64)
        m = torch.tensor([st["max_rel"]], dtype=torch.float64)
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else t.device
        t, m = t.to(dev), m.to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
        t, m = t.cpu(), m.cpu()
        cnt = int(t[2])
        out.append(dict(zip(keys, (float(t[0]) / cnt if cnt else 0.0, float(m[0]), float(t[1]), cnt, int(t[3])))))
    return out
