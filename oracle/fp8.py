"""O1/O2 — FP8 formats by exhaustive table (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Follows SURVEY.md §8(c) O1-O2 and DESIGN.md readings D3/D4:
  * OCP E4M3FN: bias 7, no infinities, NaN = S.1111.111, max finite 448.
  * OCP E5M2:   bias 15, IEEE-like, Inf = S.11111.00, NaN = S.11111.{01,10,11}, max 57344.
  (PAPER.md:38 says only "FP8"; SPEC.md:22-26/85 fixes these two formats.)

Encoding is "saturating round-to-nearest-even" (PAPER.md:425
"clamped and quantized"): the value is compared against the sorted table of
all non-negative finite codes; the nearest wins, an exact midpoint goes to the
code with mantissa LSB 0 ("even"), magnitudes above the max finite value
(including +-Inf) saturate to +-max, and the sign bit is always OR'd in so
underflow keeps -0.  NaN is not encodable here (the caller raises
NonFiniteInput first, D3).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Fp8Format:
    name: str
    ebits: int
    mbits: int
    bias: int
    has_inf: bool


E4M3 = Fp8Format("e4m3", 4, 3, 7, False)
E5M2 = Fp8Format("e5m2", 5, 2, 15, True)
FORMATS = {"e4m3": E4M3, "e5m2": E5M2}


def fmt_of(f) -> Fp8Format:
    return FORMATS[f] if isinstance(f, str) else f


def decode_code(c: int, fmt) -> float:
    """Closed-form value of one 8-bit code."""
    fmt = fmt_of(fmt)
    s = (c >> 7) & 1
    e = (c >> fmt.mbits) & ((1 << fmt.ebits) - 1)
    m = c & ((1 << fmt.mbits) - 1)
    emax_field = (1 << fmt.ebits) - 1
    sign = -1.0 if s else 1.0
    if fmt.has_inf:  # E5M2: top exponent is Inf / NaN (IEEE)
        if e == emax_field:
            return sign * float("inf") if m == 0 else float("nan")
    else:  # E4M3FN: only S.1111.111 is NaN
        if e == emax_field and m == (1 << fmt.mbits) - 1:
            return float("nan")
    if e == 0:  # subnormal: m * 2^(1-bias-mbits)
        return sign * m * 2.0 ** (1 - fmt.bias - fmt.mbits)
    return sign * (1.0 + m / float(1 << fmt.mbits)) * 2.0 ** (e - fmt.bias)


def decode_table(fmt) -> np.ndarray:
    """float64[256]: value of every code (NaN codes -> nan)."""
    return np.array([decode_code(c, fmt) for c in range(256)], dtype=np.float64)


def max_code(fmt) -> int:
    """Largest positive finite code (0x7E for e4m3, 0x7B for e5m2), by enumeration."""
    t = decode_table(fmt)
    best = 0
    for c in range(128):
        if np.isfinite(t[c]) and t[c] > t[best]:
            best = c
    return best


def max_finite(fmt) -> float:
    return float(decode_table(fmt)[max_code(fmt)])


def _positive_table(fmt):
    t = decode_table(fmt)
    cmax = max_code(fmt)
    pos = t[: cmax + 1]
    assert np.all(np.diff(pos) > 0), "positive finite codes must be increasing"
    return pos, cmax


def encode(v, fmt) -> np.ndarray:
    """Saturating RNE encode of values ``v`` (float64 holding FP32 values) -> uint8 codes.

    Pure table lookup: find the bracketing pair (P[c], P[c+1]) of non-negative
    finite table values and compare against their exact midpoint (the midpoint
    of two FP8 values has <= 6 significant bits, so it is exact in float64 and
    no arithmetic rounding enters the decision).
    """
    fmt = fmt_of(fmt)
    v = np.asarray(v, dtype=np.float64)
    if np.isnan(v).any():
        raise ValueError("NaN is not encodable (NonFiniteInput is raised upstream)")
    pos, cmax = _positive_table(fmt)
    a = np.abs(v)
    sign = np.signbit(v).astype(np.uint8) << 7
    out = np.empty(a.shape, dtype=np.uint8)
    sat = a >= pos[cmax]
    out[sat] = cmax
    rest = ~sat
    ar = a[rest]
    lo = np.searchsorted(pos, ar, side="right") - 1  # pos[lo] <= a < pos[lo+1]
    hi = lo + 1
    mid = (pos[lo] + pos[hi]) * 0.5
    code = np.where(ar < mid, lo, np.where(ar > mid, hi, np.where(lo % 2 == 0, lo, hi)))
    out[rest] = code.astype(np.uint8)
    return out | sign


def decode(codes, fmt) -> np.ndarray:
    t = decode_table(fmt)
    return t[np.asarray(codes, dtype=np.uint8).astype(np.int64)]
