"""O3-O6 — granule amax, scale, quantize, dequantize (TEST INFRASTRUCTURE ONLY).

Follows SURVEY.md §8(c) O3-O6, which restates:
  * PAPER.md:535 (§III-C) "quantization strategies (tensorwise, rowwise, blockwise)"
    and PAPER.md:171/692 (DeepGEMM 1x128 / 128x128 blockwise);
  * SPEC.md:57-75 [OP] compute_scales / quantize / dequantize:
    "scale = amax(granule) / format.max_finite; if amax = 0, scale = 1";
  * DESIGN.md readings D1 (multiply by the reciprocal r = fl32(max/amax) rather
    than divide per element; the SPEC's per-element divide is kept as
    ``mode="div"``; D1b: when max/amax overflows FP32, i.e. amax < max/FLT_MAX, the
    reciprocal is the largest finite FP32 value instead of +Inf), D2 (zero
    granule -> s = r = 1), D3 (non-finite input ->
    NonFiniteInput), D6 (blockwise geometry), D7 (F32 or UE8M0 scales).

Scale layouts (row-major arrays, shared with include/loka.h's contract):
  TENSOR [1] | ROW [R] | COL [C] | BLK_1x128 [R, ceil(C/128)]
  | BLK_128x1 [ceil(R/128), C] | BLK_128x128 [ceil(R/128), ceil(C/128)]
Scales are FP32 values (UE8M0 scales are powers of two stored as FP32).
"""
from __future__ import annotations

import math

import numpy as np

from . import fp8

# blk_1x32: the MX block (OCP MXFP8 block size 32; NEXT-4), one scale per row per 32 columns
GRANS = ("tensor", "row", "col", "blk_1x128", "blk_128x1", "blk_128x128", "blk_1x32")
FLT32_MAX = float(np.finfo(np.float32).max)
_BLK = {"blk_1x128": (1, 128), "blk_128x1": (128, 1), "blk_128x128": (128, 128), "blk_1x32": (1, 32)}


class NonFiniteInput(ValueError):
    """SPEC.md:61 errors: NonFiniteInput if any element is NaN/Inf."""


def _cdiv(a, b):
    return -(-a // b)


def scale_shape(rows: int, cols: int, gran: str):
    return {
        "tensor": (1,),
        "row": (rows,),
        "col": (cols,),
        "blk_1x128": (rows, _cdiv(cols, 128)),
        "blk_128x1": (_cdiv(rows, 128), cols),
        "blk_128x128": (_cdiv(rows, 128), _cdiv(cols, 128)),
        "blk_1x32": (rows, _cdiv(cols, 32)),
    }[gran]


def granule_index(i: int, j: int, gran: str):
    """Index into the scale array of element (i, j) (SURVEY.md §8(c) O3 granules)."""
    return {
        "tensor": (0,),
        "row": (i,),
        "col": (j,),
        "blk_1x128": (i, j // 128),
        "blk_128x1": (i // 128, j),
        "blk_128x128": (i // 128, j // 128),
        "blk_1x32": (i, j // 32),
    }[gran]


def granule_slices(rows: int, cols: int, gran: str):
    """Yield (scale_index, row_slice, col_slice) for every granule; edge granules are partial."""
    if gran == "tensor":
        yield (0,), slice(0, rows), slice(0, cols)
    elif gran == "row":
        for i in range(rows):
            yield (i,), slice(i, i + 1), slice(0, cols)
    elif gran == "col":
        for j in range(cols):
            yield (j,), slice(0, rows), slice(j, j + 1)
    else:
        br, bc = _BLK[gran]
        for bi in range(_cdiv(rows, br)):
            for bj in range(_cdiv(cols, bc)):
                yield (bi, bj), slice(bi * br, min(rows, (bi + 1) * br)), slice(bj * bc, min(cols, (bj + 1) * bc))


def _as_f64(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if not np.isfinite(x).all():
        raise NonFiniteInput("NaN/Inf in quantize input")
    return x


def granule_amax(x, gran: str) -> np.ndarray:
    """O3: exact max |x| over each granule's in-bounds elements."""
    x = _as_f64(x)
    rows, cols = x.shape
    amax = np.zeros(scale_shape(rows, cols, gran), dtype=np.float64)
    if gran == "row":  # same definition as the loop below, vectorised for speed
        return np.abs(x).max(axis=1) if cols else amax
    if gran == "col":
        return np.abs(x).max(axis=0) if rows else amax
    for idx, rs, cs in granule_slices(rows, cols, gran):
        blk = x[rs, cs]
        amax[idx] = np.abs(blk).max() if blk.size else 0.0
    return amax


def fl32(v) -> np.ndarray:
    """Round float64 values to the nearest FP32 (RNE, subnormals kept)."""
    return np.asarray(v, dtype=np.float64).astype(np.float32).astype(np.float64)


def ue8m0_scale(a: float, fmax: float) -> float:
    """Smallest power of two 2^e, e >= -127, with a <= fmax * 2^e (D7 / SURVEY O4).

    frexp only supplies a starting guess; the two loops then decide with exact
    float64 comparisons (a and fmax * 2^e are both exactly representable).
    """
    _, e = math.frexp(a / fmax)  # guess: a/fmax < 2^e
    while e - 1 >= -127 and a <= fmax * 2.0 ** (e - 1):
        e -= 1
    while a > fmax * 2.0 ** e:
        e += 1
    return 2.0 ** max(e, -127)


def scales_from_amax(amax, fmt, scale_fmt: str = "f32"):
    """O4: (s, r) per granule.  a = 0 -> s = r = 1."""
    fmax = fp8.max_finite(fmt)
    amax = np.asarray(amax, dtype=np.float64)
    s = np.ones_like(amax)
    r = np.ones_like(amax)
    nz = amax > 0
    if scale_fmt == "f32":
        s[nz] = fl32(amax[nz] / fmax)  # IEEE division correctly rounded to FP32
        # D1b: fl32(max/amax) is +Inf for amax < max/FLT_MAX (~1.3e-36 for e4m3); the reciprocal
        # is then the largest finite FP32, so x*r stays finite and below max (no NaN from 0*Inf)
        with np.errstate(over="ignore"):
            r[nz] = np.minimum(fl32(fmax / amax[nz]), FLT32_MAX)
    elif scale_fmt == "ue8m0":
        flat_s = s.reshape(-1)
        flat_r = r.reshape(-1)
        for k, a in enumerate(amax.reshape(-1)):
            if a > 0:
                flat_s[k] = ue8m0_scale(float(a), fmax)
                flat_r[k] = 1.0 / flat_s[k]  # exact: power of two
    else:
        raise ValueError(scale_fmt)
    return s, r


def expand(scale_arr, rows: int, cols: int, gran: str) -> np.ndarray:
    """Broadcast a per-granule array to a full [rows, cols] array (element -> its granule)."""
    a = np.asarray(scale_arr, dtype=np.float64)
    if gran == "tensor":
        return np.full((rows, cols), a.reshape(-1)[0])
    if gran == "row":
        return np.repeat(a.reshape(rows, 1), cols, axis=1)
    if gran == "col":
        return np.repeat(a.reshape(1, cols), rows, axis=0)
    br, bc = _BLK[gran]
    full = np.repeat(np.repeat(a, br, axis=0), bc, axis=1)
    return full[:rows, :cols]


def quantize(x, fmt="e4m3", gran="row", scale_fmt="f32", amax=None, mode="mul"):
    """O5: codes = encode_satRNE(fl32(x * r)) per granule; returns (codes uint8, scales float32).

    ``amax`` overrides the granule amax (tensorwise split phase: the caller
    passes the all-reduced global amax).  ``mode="div"`` is the
    SPEC.md:68 reading encode(fl32(x / s)) (D1).
    """
    x = _as_f64(x)
    rows, cols = x.shape
    if amax is None:
        amax = granule_amax(x, gran)
    else:
        amax = np.asarray(amax, dtype=np.float64).reshape(scale_shape(rows, cols, gran))
    s, r = scales_from_amax(amax, fmt, scale_fmt)
    if mode == "mul":
        v = fl32(x * expand(r, rows, cols, gran))  # FP32*FP32 product exact in float64, rounded once
    elif mode == "div":
        v = fl32(x / expand(s, rows, cols, gran))  # float64 quotient then FP32: innocuous double rounding
    else:
        raise ValueError(mode)
    codes = fp8.encode(v, fmt)
    return codes, s.astype(np.float32)


def dequantize(codes, scales, fmt="e4m3", gran="row") -> np.ndarray:
    """O6: x_hat = decode(q) * s, exact in float64."""
    codes = np.asarray(codes, dtype=np.uint8)
    rows, cols = codes.shape
    return fp8.decode(codes, fmt) * expand(np.asarray(scales, dtype=np.float64), rows, cols, gran)
