"""NVFP4 quantization and linear — TEST INFRASTRUCTURE ONLY.

The paper names FP4 as future work ("... FP4 ...", SURVEY.md §8(f) NEXT-4:
"NVFP4 / MXFP8 block-scaled recipes"); it fixes no algorithm, so this module follows the
readings D35-D38 of DESIGN.md §8.5, written in the same style as the FP8 recipe (D1: one IEEE
division per granule, one multiply per element):

  * E2M1 (D35): 4-bit code s.ee.m, exponent bias 1; e = 0 -> m * 0.5 (subnormal), else
    (1 + m/2) * 2^(e-1): magnitudes {0, 0.5, 1, 1.5, 2, 3, 4, 6}.  Encoding is saturating
    round-to-nearest-even exactly as O2 (nearest table value, ties to the code with m = 0,
    |v| > 6 -> 6, sign always kept so underflow gives -0).  Two codes per byte, element 2j in
    the low nibble of byte j.
  * Two-level scaling (D36): a tensor amax A (the all-reduced global amax under data parallel,
    as O3/D20), tensor scale s_t = fl32(A / 2688) and r_t = fl32(2688 / A) (2688 = 448 * 6, the
    largest value an E4M3 block scale times an E2M1 code can express; A = 0 -> s_t = r_t = 1);
    per 1x16 block (row i, columns 16b..16b+15) with amax a_b:
        sf_b = E4M3_satRNE( fl32( fl32(a_b * r_t) / 6 ) )      (a non-negative E4M3 code: UE4M3)
        d_b  = decode(sf_b);   codes = E2M1_satRNE( fl32(x * fl32(r_t / d_b)) )   (d_b > 0)
    and codes = +-0 when d_b = 0 (the block underflows the block-scale format).
  * Dequantization (D37): x_hat = e2m1(code) * d_b * s_t, exact in float64.
  * Linear (D38): the GEMM of the dequantized operands in float64 (O7) followed by the same
    bias / norm steps (O8, O9) as the FP8 path.
"""
from __future__ import annotations

import numpy as np

from . import fp8
from .quantize import fl32, NonFiniteInput, FLT32_MAX

BLOCK = 16
FP4_MAX = 6.0
SCALED_MAX = 448.0 * 6.0  # E4M3 max x E2M1 max


def e2m1_decode_code(c: int) -> float:
    """Closed-form value of a 4-bit E2M1 code (D35)."""
    s = (c >> 3) & 1
    e = (c >> 1) & 3
    m = c & 1
    v = m * 0.5 if e == 0 else (1.0 + m / 2.0) * 2.0 ** (e - 1)
    return -v if s else v


E2M1_TABLE = np.array([e2m1_decode_code(c) for c in range(16)], dtype=np.float64)


def e2m1_encode(v) -> np.ndarray:
    """Saturating RNE to E2M1 codes (uint8 values 0..15), following O2's table rule (D35)."""
    v = np.asarray(v, dtype=np.float64)
    if np.isnan(v).any():
        raise NonFiniteInput("NaN in e2m1 encode")
    mag = np.minimum(np.abs(v), FP4_MAX)
    pos = E2M1_TABLE[:8]  # codes 0..7, increasing
    d = np.abs(mag[..., None] - pos)  # distance to every positive code
    best = np.argmin(d, axis=-1)  # first minimum = the lower code of a tie ...
    dmin = np.take_along_axis(d, best[..., None], axis=-1)[..., 0]
    nxt = np.minimum(best + 1, 7)
    tie = (nxt != best) & (np.abs(mag - pos[nxt]) == dmin)
    best = np.where(tie & (best % 2 == 1), nxt, best)  # ... unless it is odd: ties go to m = 0
    sign = np.signbit(v).astype(np.uint8) << 3
    return (best.astype(np.uint8) | sign).astype(np.uint8)


def e2m1_decode(codes) -> np.ndarray:
    return E2M1_TABLE[np.asarray(codes, dtype=np.uint8) & 0xF]


def pack(codes) -> np.ndarray:
    """[rows, cols] codes -> [rows, cols/2] bytes, element 2j in the low nibble (D35)."""
    c = np.asarray(codes, dtype=np.uint8)
    return (c[:, 0::2] | (c[:, 1::2] << 4)).astype(np.uint8)


def unpack(packed) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty((p.shape[0], p.shape[1] * 2), dtype=np.uint8)
    out[:, 0::2] = p & 0xF
    out[:, 1::2] = p >> 4
    return out


def tensor_scales(A: float):
    """(s_t, r_t) from the tensor amax (D36)."""
    if A == 0.0:
        return 1.0, 1.0
    # D1b (as for FP8): a reciprocal that overflows FP32 (A < 2688/FLT_MAX) is the largest finite FP32
    with np.errstate(over="ignore"):
        r_t = float(min(fl32(SCALED_MAX / A), FLT32_MAX))
    return float(fl32(A / SCALED_MAX)), r_t


def quantize(x, amax=None):
    """NVFP4 quantize (D36).  x [rows, cols] finite, cols % 16 == 0.
    Returns (packed uint8 [rows, cols/2], sf uint8 [rows, cols/16] E4M3 codes, s_t float32 [1])."""
    x = np.asarray(x, dtype=np.float64)
    if not np.isfinite(x).all():
        raise NonFiniteInput("NaN/Inf in quantize input")
    rows, cols = x.shape
    if cols % BLOCK:
        raise ValueError("NVFP4 needs cols % 16 == 0")
    A = float(np.abs(x).max()) if amax is None else float(np.asarray(amax).reshape(-1)[0])
    if x.size == 0:
        A = 0.0 if amax is None else A
    s_t, r_t = tensor_scales(A)
    xb = x.reshape(rows, cols // BLOCK, BLOCK)
    a_b = np.abs(xb).max(axis=2) if x.size else np.zeros((rows, cols // BLOCK))
    u = fl32(a_b * r_t)  # FP32 * FP32: exact in float64, rounded once
    sf = fp8.encode(fl32(u / 6.0), "e4m3")  # IEEE division, then E4M3 satRNE (non-negative)
    d = fp8.decode(sf, "e4m3")
    safe = np.where(d > 0, d, 1.0)
    with np.errstate(over="ignore"):
        rb = np.where(d > 0, np.minimum(fl32(r_t / safe), FLT32_MAX), 0.0)  # D1b clamp
    v = fl32(xb * rb[:, :, None])
    v = np.where(d[:, :, None] > 0, v, np.copysign(0.0, xb))  # underflowed block: signed zeros
    codes = e2m1_encode(v).reshape(rows, cols)
    return pack(codes), sf.astype(np.uint8), np.array([s_t], dtype=np.float32)


def dequantize(packed, sf, s_t) -> np.ndarray:
    """x_hat = e2m1(code) * decode_e4m3(sf) * s_t (D37), exact in float64."""
    codes = unpack(packed)
    rows, cols = codes.shape
    d = fp8.decode(np.asarray(sf, dtype=np.uint8), "e4m3")
    full = np.repeat(d, BLOCK, axis=1)[:, :cols]
    return e2m1_decode(codes) * full * float(np.asarray(s_t, dtype=np.float64).reshape(-1)[0])


def linear_norm(a_packed, a_sf, a_st, b_packed, b_sf, b_st, norm="none", eps=None, bias=None, gamma=None, beta=None,
                block=256):
    """D38: y = norm(A_hat B_hat^T (+ bias)) in float64 (O7-O9 on NVFP4-dequantized operands)."""
    from . import linear
    y = linear.matmul_nt(dequantize(a_packed, a_sf, a_st), dequantize(b_packed, b_sf, b_st))
    if bias is not None:
        y = linear.add_bias(y, bias)
    return linear.apply_norm(y, norm, eps, gamma, beta, block)
