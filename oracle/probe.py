"""O11/O12 — LoKA Probe error statistic (TEST INFRASTRUCTURE ONLY).

PAPER.md:192 (§II-C) defines MERE(out, ref) = sum_m sum_n |(out - ref) / ref|.
Readings:
  D8  "Mean": divide by M*N (the name and Table II magnitudes ~0.5 imply a mean;
      SPEC.md:326, 360).
  D9  ``ref`` is the BF16 path's output of the same op (BJ north_star: "relative
      error against the BF16 result"); the TF32 reference of P:192 is the
      paper's hardware choice.
  D10 near-zero references: denominator max(|ref|, f), f = 1e-6 * mean(|ref|)
      (SPEC.md:361); n_floored counts the elements that used the floor.
Also reported: max relative error, sum |ref|, element count.
All sums are exactly-rounded float64 sums (math.fsum), so the oracle's value
does not depend on summation order.
"""
from __future__ import annotations

import math

import numpy as np


def mere_stats(out, ref, floor_rel: float = 1e-6, floor: float | None = None) -> dict:
    """``floor`` (optional) is the absolute floor f of a row shard of a larger tensor: D10 applied
    to the whole tensor (f = floor_rel * mean |ref| over every shard), as the data-parallel probe
    uses it; by default f is this array's own floor_rel * mean |ref|."""
    out = np.asarray(out, np.float64)
    ref = np.asarray(ref, np.float64)
    if out.shape != ref.shape:
        raise ValueError("ShapeMismatch")
    n = out.size
    if n == 0:
        return dict(mere=0.0, max_rel=0.0, sum_abs_ref=0.0, count=0, n_floored=0)
    aref = np.abs(ref).reshape(-1)
    sum_abs_ref = math.fsum(aref)
    f = floor_rel * (sum_abs_ref / n) if floor is None else float(floor)
    denom = np.maximum(aref, f)
    n_floored = int(np.count_nonzero(aref < f))
    rel = np.abs(out.reshape(-1) - ref.reshape(-1))
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(denom > 0, rel / np.where(denom > 0, denom, 1.0), np.where(rel > 0, np.inf, 0.0))
    return dict(mere=math.fsum(rel) / n, max_rel=float(rel.max()), sum_abs_ref=sum_abs_ref,
                count=int(n), n_floored=n_floored)


def mere(out, ref, floor_rel: float = 1e-6) -> float:
    return mere_stats(out, ref, floor_rel)["mere"]


def geomean(values, floor: float = 1e-6) -> float:
    """Table II aggregate (PAPER.md:176 caption "Geometric mean of MERE"):
    exp(mean(log(max(v, 1e-6))))."""
    v = [max(float(x), floor) for x in values]
    if not v:
        raise ValueError("EmptyList")
    return math.exp(math.fsum(math.log(x) for x in v) / len(v))
