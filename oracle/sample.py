"""NEXT-3 — LoKA Probe's learned-distribution sampling (TEST INFRASTRUCTURE ONLY).

PAPER.md:368-393 (§III LoKA Probe, "Sampling learned distributions"):
  (a) inputs   T' = 1_B mu^T + Z L_Sigma^T,  Z ~ N(0, I_K) rows,  L_Sigma L_Sigma^T = Sigma + eps I
  (b) weights  W' = M + L_U Z L_V^T,         Z ~ N(0, I_{MxN}),  L_U L_U^T = U + eps I,
                                                                 L_V L_V^T = V + eps I
with the jitter of footnote PAPER.md:381: eps = 1e-6 * trace(Sigma) / K ("to maintain numerical
stability"), escalated x10 up to 4 times on a failed factorisation (reading D30).

The standard normals Z come from a counter-based generator that the CUDA side implements
independently (D31): Philox4x64-10 (Salmon et al., SC'11; the bit generator numpy ships
as ``np.random.Philox``) keyed by (seed, 0) on the counter (block, 0, 0, 0); element e of a draw
with offset o uses block (o + e) // 4, word pair ((o + e) % 4) // 2, and Box-Muller on the top 24
bits of the two 64-bit words:
    u1 = ((x_a >> 40) + 1) 2^-24  in (0, 1],   u2 = (x_b >> 40) 2^-24  in [0, 1)
    r = sqrt(-2 ln u1),  z_even = r cos(2 pi u2),  z_odd = r sin(2 pi u2)
(float64 here; the GPU evaluates the same uniforms in FP32, so Z agrees to FP32 rounding).
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2E7470EE14C6C93)
_M1 = np.uint64(0xCA5A826395121157)
_W0 = np.uint64(0x9E3779B97F4A7C15)
_W1 = np.uint64(0xBB67AE8584CAA73B)
_LO = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def _mulhilo64(a: np.ndarray, b: np.uint64):
    """128-bit product of uint64 arrays by a uint64 constant: (hi, lo), via 32-bit limbs."""
    al, ah = a & _LO, a >> _S32
    bl, bh = b & _LO, b >> _S32
    ll, lh, hl, hh = al * bl, al * bh, ah * bl, ah * bh
    mid = (ll >> _S32) + (lh & _LO) + (hl & _LO)
    lo = (ll & _LO) | ((mid & _LO) << _S32)
    hi = hh + (lh >> _S32) + (hl >> _S32) + (mid >> _S32)
    return hi, lo


def philox4x64_10(counter, key):
    """Philox4x64 with 10 rounds (Salmon et al. 2011, Random123): counter [n, 4] uint64, key (k0, k1).
    Round: (hi0, lo0) = M0 * c0, (hi1, lo1) = M1 * c2,
           c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); key += (W0, W1) between rounds."""
    c = np.array(counter, dtype=np.uint64).reshape(-1, 4)
    c0, c1, c2, c3 = (c[:, i].copy() for i in range(4))
    k0, k1 = np.uint64(key[0]), np.uint64(key[1])
    with np.errstate(over="ignore"):
        for rnd in range(10):
            hi0, lo0 = _mulhilo64(c0, _M0)
            hi1, lo1 = _mulhilo64(c2, _M1)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            if rnd < 9:
                k0 = k0 + _W0
                k1 = k1 + _W1
    return np.stack([c0, c1, c2, c3], axis=1)


def normals(seed: int, offset: int, n: int) -> np.ndarray:
    """n standard normals of the stream (seed, offset) as defined in the module docstring (float64)."""
    if n <= 0:
        return np.zeros(0)
    e = np.arange(offset, offset + n, dtype=np.int64)
    b0, b1 = int(e[0] // 4), int(e[-1] // 4)
    blocks = np.arange(b0, b1 + 1, dtype=np.uint64)
    ctr = np.zeros((len(blocks), 4), dtype=np.uint64)
    ctr[:, 0] = blocks
    x = philox4x64_10(ctr, (np.uint64(seed & 0xFFFFFFFFFFFFFFFF), np.uint64(0)))
    u_top = (x >> np.uint64(40)).astype(np.float64)  # 24-bit integers, exact in float64
    z = np.empty((len(blocks), 4))
    for p in range(2):
        u1 = (u_top[:, 2 * p] + 1.0) * 2.0 ** -24
        u2 = u_top[:, 2 * p + 1] * 2.0 ** -24
        r = np.sqrt(-2.0 * np.log(u1))
        z[:, 2 * p] = r * np.cos(2.0 * np.pi * u2)
        z[:, 2 * p + 1] = r * np.sin(2.0 * np.pi * u2)
    return z.reshape(-1)[e - 4 * b0]


class NotPositiveDefinite(ValueError):
    pass


def jitter(a: np.ndarray, eps_rel: float) -> float:
    """eps = eps_rel * trace(a) / n (PAPER.md:381 footnote); a zero / negative trace uses scale 1
    (reading D30: the footnote's relative jitter would vanish for a constant stream)."""
    n = a.shape[0]
    t = float(np.trace(a)) / n if n else 0.0
    return eps_rel * (t if t > 0.0 else 1.0)


def cholesky_jittered(a, eps_rel: float = 1e-6, escalations: int = 4):
    """L with L L^T = sym(a) + eps I, eps escalated x10 up to `escalations`
    times on failure.  Returns (L, eps_used); raises NotPositiveDefinite."""
    a = np.asarray(a, np.float64)
    a = 0.5 * (a + a.T)
    n = a.shape[0]
    eps = jitter(a, eps_rel)
    for _ in range(escalations + 1):
        try:
            return np.linalg.cholesky(a + eps * np.eye(n)), eps
        except np.linalg.LinAlgError:
            eps *= 10.0
    raise NotPositiveDefinite(f"not positive definite after {escalations} escalations")


def sample_input(mean, l_sigma, b: int, seed: int, offset: int = 0) -> np.ndarray:
    """(a) T' = 1_B mu^T + Z L_Sigma^T, Z [B, K] row-major from the stream."""
    mean = np.asarray(mean, np.float64)
    k = mean.shape[0]
    z = normals(seed, offset, b * k).reshape(b, k)
    return mean[None, :] + z @ np.asarray(l_sigma, np.float64).T


def sample_weight(mean, l_u, l_v, seed: int, offset: int = 0) -> np.ndarray:
    """(b) W' = M + L_U Z L_V^T, Z [M, N] row-major from the stream."""
    mean = np.asarray(mean, np.float64)
    m, n = mean.shape
    z = normals(seed, offset, m * n).reshape(m, n)
    return mean + np.asarray(l_u, np.float64) @ z @ np.asarray(l_v, np.float64).T
