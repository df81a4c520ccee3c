"""Quantized data-parallel gradient reduction (SURVEY.md §8(f) NEXT-4 "quantized (FP8) DP gradient
communication"; PAPER.md:562 FSDP gradient sync, PAPER.md:778 future work) — TEST INFRASTRUCTURE ONLY.

Reading D39: every rank p quantizes its local gradient G_p [N, K] rowwise (O3-O5,
one FP32 scale per row; e5m2 for gradients by D5, e4m3 selectable), the codes and scales are
exchanged instead of FP32 values (1 byte + 4/K bytes per element instead of 4), and the owner of a
row shard reduces the dequantized shards:  R = sum_{p=0}^{P-1} decode(q_p) * s_p  (O6, then a sum).
The GPU accumulates in FP32 in rank order p = 0..P-1; this oracle sums the exact dequantized values
in float64 (the difference is the FP32 rounding of P partial sums)."""
from __future__ import annotations

import numpy as np

from . import quantize


def reduce_dequantized(codes_list, scales_list, fmt="e5m2") -> np.ndarray:
    """R = sum_p dequantize(q_p, s_p) (rowwise scales), float64."""
    out = None
    for q, s in zip(codes_list, scales_list):
        d = quantize.dequantize(q, s, fmt, "row")
        out = d if out is None else out + d
    return out


def quantized_allreduce(grads, fmt="e5m2"):
    """Each rank's gradient quantized rowwise (O5), then reduced (D39).  Returns (R, codes, scales)."""
    codes, scales = [], []
    for g in grads:
        q, s = quantize.quantize(g, fmt, "row")
        codes.append(q)
        scales.append(s)
    return reduce_dequantized(codes, scales, fmt), codes, scales
