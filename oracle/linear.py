"""O7-O10 — FP8 linear (3 directions), bias, norms, output casts (TEST INFRASTRUCTURE ONLY).

The method's linear layer is *defined* by its quantized operands: the FP8 GEMM
with FP32 accumulation approximates the exact product of the dequantized
operands (SURVEY.md §8(c) preamble; SPEC.md:123-133 gemm_ref / gemm_lowprec,
"product taken over dequantized values").  The oracle therefore computes
    Y_hat = X_hat @ W_hat^T          (fwd,   X[M,K], W[N,K] -> Y[M,N])
    dX_hat = dY_hat @ W_hat          (dgrad, dY[M,N], W[N,K] -> dX[M,K])
    dW_hat = dY_hat^T @ X_hat        (wgrad, dY[M,N], X[M,K] -> dW[N,K])
in float64 (numpy BLAS matmul serves as the library primitive, SPEC.md:123
"64-bit accumulation"), then bias ("(Wx + b)", before the norm,
DESIGN.md D15) and the norm that follows:
  * LayerNorm (Ba et al.; D13): mu = mean, var = biased
    mean of squared deviations, z = (y - mu) / sqrt(var + eps), eps = 1e-5,
    optional gamma/beta.
  * RMSNorm (Zhang & Sennrich; D14):
    z = y / sqrt(mean(y^2) + eps), eps = 1e-6, optional gamma.
  * BlockNorm ("RMSNorm((Wx + b).view(-1, BlockN)).view(B, N)";
    PAPER.md:473 block 256; "unparameterized Grouped RMSNorm"):
    RMSNorm over each contiguous block of B columns, no gamma; N % B != 0 is an
    error (SPEC.md:399 IndivisibleFeatureDim).
  * Hard Swish, applied to the norm's output
    ("integrates seamlessly with BlockNorm, allowing both operations to be fused"):
    h-swish(x) = x * ReLU6(x + 3) / 6, ReLU6(t) = min(max(t, 0), 6).
"""
from __future__ import annotations

import numpy as np

from . import quantize as Q


class IndivisibleFeatureDim(ValueError):
    """SPEC.md:399 errors: IndivisibleFeatureDim."""


def matmul_nt(a_hat: np.ndarray, b_hat: np.ndarray) -> np.ndarray:
    """C = A B^T in float64 (SPEC.md:123 gemm_ref with 64-bit accumulation)."""
    return np.asarray(a_hat, np.float64) @ np.asarray(b_hat, np.float64).T


def fwd(x_hat, w_hat):
    """Y = X W^T: X[M,K], W[N,K] (SPEC.md:130 Forward: x(B,K)·w(N,K)^T)."""
    return matmul_nt(x_hat, w_hat)


def dgrad(dy_hat, w_hat):
    """dX = dY W: dY[M,N], W[N,K] (SPEC.md:130 BackwardInputGrad: dy(B,N)·w(N,K))."""
    return np.asarray(dy_hat, np.float64) @ np.asarray(w_hat, np.float64)


def wgrad(dy_hat, x_hat):
    """dW = dY^T X: dY[M,N], X[M,K] (SPEC.md:130 BackwardWeightGrad: dy(B,N)^T·x(B,K))."""
    return np.asarray(dy_hat, np.float64).T @ np.asarray(x_hat, np.float64)


def add_bias(y, bias):
    if bias is None:
        return y
    return y + np.asarray(bias, np.float64)[None, :]


def layer_norm(y, eps=1e-5, gamma=None, beta=None):
    y = np.asarray(y, np.float64)
    mu = y.mean(axis=1, keepdims=True)
    var = ((y - mu) ** 2).mean(axis=1, keepdims=True)
    z = (y - mu) / np.sqrt(var + eps)
    if gamma is not None:
        z = z * np.asarray(gamma, np.float64)[None, :]
    if beta is not None:
        z = z + np.asarray(beta, np.float64)[None, :]
    return z


def rms_norm(y, eps=1e-6, gamma=None):
    y = np.asarray(y, np.float64)
    z = y / np.sqrt((y ** 2).mean(axis=1, keepdims=True) + eps)
    if gamma is not None:
        z = z * np.asarray(gamma, np.float64)[None, :]
    return z


def block_rms_norm(y, block=256, eps=1e-6):
    y = np.asarray(y, np.float64)
    m, n = y.shape
    if block < 1 or n % block != 0:
        raise IndivisibleFeatureDim(f"N={n} not divisible by block={block}")
    out = np.empty_like(y)
    for b in range(n // block):  # each block is an independent unparameterized RMSNorm
        sl = slice(b * block, (b + 1) * block)
        out[:, sl] = rms_norm(y[:, sl], eps)
    return out


def apply_norm(y, norm="none", eps=None, gamma=None, beta=None, block=256):
    if norm == "none":
        return np.asarray(y, np.float64)
    if norm == "layer":
        return layer_norm(y, 1e-5 if eps is None else eps, gamma, beta)
    if norm == "rms":
        return rms_norm(y, 1e-6 if eps is None else eps, gamma)
    if norm == "block_rms":
        return block_rms_norm(y, block, 1e-6 if eps is None else eps)
    raise ValueError(norm)


def hard_swish(x):
    """h-swish(x) = x * ReLU6(x + 3) / 6."""
    x = np.asarray(x, np.float64)
    return x * np.minimum(np.maximum(x + 3.0, 0.0), 6.0) / 6.0


def apply_act(y, act="none"):
    if act == "none":
        return y
    if act == "hardswish":
        return hard_swish(y)
    raise ValueError(act)


def linear_norm(a_codes, a_scales, a_fmt, a_gran, b_codes, b_scales, b_fmt, b_gran,
                bias=None, norm="none", eps=None, gamma=None, beta=None, block=256, act="none"):
    """O6-O9 chain for C = A B^T with K-major operands A[M,K], B[N,K] (every direction
    is this product once its operands are laid out K-major),
    then the optional activation after the norm (NEXT-1)."""
    a_hat = Q.dequantize(a_codes, a_scales, a_fmt, a_gran)
    b_hat = Q.dequantize(b_codes, b_scales, b_fmt, b_gran)
    y = add_bias(matmul_nt(a_hat, b_hat), bias)
    return apply_act(apply_norm(y, norm, eps, gamma, beta, block), act)


def norm_stats(y, norm="layer", eps=None, block=256):
    """The forward quantities the backward needs: xhat (normalised, before gamma/beta/act) and rstd
    (per row; BlockNorm: per row and block, [M, N/block])."""
    y = np.asarray(y, np.float64)
    if norm == "layer":
        eps = 1e-5 if eps is None else eps
        mu = y.mean(axis=1, keepdims=True)
        rstd = 1.0 / np.sqrt(((y - mu) ** 2).mean(axis=1, keepdims=True) + eps)
        return (y - mu) * rstd, rstd[:, 0]
    if norm == "rms":
        eps = 1e-6 if eps is None else eps
        rstd = 1.0 / np.sqrt((y ** 2).mean(axis=1, keepdims=True) + eps)
        return y * rstd, rstd[:, 0]
    if norm == "block_rms":
        eps = 1e-6 if eps is None else eps
        m, n = y.shape
        yb = y.reshape(m, n // block, block)
        rstd = 1.0 / np.sqrt((yb ** 2).mean(axis=2) + eps)
        return (yb * rstd[:, :, None]).reshape(m, n), rstd
    raise ValueError(norm)


def hard_swish_grad(x):
    """d h-swish / dx = 0 (x < -3), (2x + 3)/6 (-3 <= x <= 3), 1 (x > 3) (PyTorch's convention at
    the kinks)."""
    x = np.asarray(x, np.float64)
    return np.where(x < -3.0, 0.0, np.where(x <= 3.0, (2.0 * x + 3.0) / 6.0, 1.0))


def norm_backward(dh, xhat, rstd, norm="layer", gamma=None, beta=None, act="none", block=256):
    """NEXT-1: gradient wrt the norm's input z of h = act(xhat*gamma + beta),
    given dh = dL/dh and the saved xhat, rstd (norm_stats).  With g = dh * act'(y_pre) * gamma:
      LayerNorm (xhat = (z - mu) rstd):  dz = rstd (g - mean(g) - xhat mean(g xhat))
      RMSNorm   (xhat = z rstd):         dz = rstd (g - xhat mean(g xhat))
      BlockNorm: RMSNorm's formula per block (rstd [M, N/block])."""
    dh = np.asarray(dh, np.float64)
    xhat = np.asarray(xhat, np.float64)
    g = dh
    gam = np.ones(xhat.shape[1]) if gamma is None else np.asarray(gamma, np.float64)
    if act == "hardswish":
        ypre = xhat * gam[None, :] + (0.0 if beta is None else np.asarray(beta, np.float64)[None, :])
        g = g * hard_swish_grad(ypre)
    elif act != "none":
        raise ValueError(act)
    g = g * gam[None, :]
    if norm == "layer":
        r = np.asarray(rstd, np.float64)[:, None]
        return r * (g - g.mean(axis=1, keepdims=True) - xhat * (g * xhat).mean(axis=1, keepdims=True))
    if norm == "rms":
        r = np.asarray(rstd, np.float64)[:, None]
        return r * (g - xhat * (g * xhat).mean(axis=1, keepdims=True))
    if norm == "block_rms":
        m, n = xhat.shape
        gb, xb = g.reshape(m, n // block, block), xhat.reshape(m, n // block, block)
        r = np.asarray(rstd, np.float64).reshape(m, n // block, 1)
        return (r * (gb - xb * (gb * xb).mean(axis=2, keepdims=True))).reshape(m, n)
    raise ValueError(norm)


def round_bf16(v) -> np.ndarray:
    """O10: round float64 values to the nearest bf16 value, ties to even (8 significant
    bits; bf16 subnormal spacing 2^-133).  |v| = f 2^p with f in [0.5, 1) -> the bf16
    spacing there is 2^(p-8); |v| / spacing is exact and np.rint rounds half to even."""
    v = np.asarray(v, np.float64)
    _, p = np.frexp(v)
    spacing = np.exp2(np.maximum(p - 8, -133).astype(np.float64))
    return np.rint(v / spacing) * spacing
