"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no quantization, no GEMM, no
norm, no error statistic).  It only draws random tensors with the shapes and
value distributions of the paper's LRM workloads (DESIGN.md
"Input recipe") and rounds them to bf16, so that both sides consume the same
input bytes.

Distributions
-------------
* ``gaussian``   X ~ N(0, 1)                               ("standard normal")
* ``weight``     W ~ N(0, 1/K)                              (fan-in init of an nn.Linear)
* ``grad``       dY ~ 2^-10 * N(0, 1)                      (small gradients -> e5m2, BJ north_star)
* ``heavy``      X = t3/sqrt(3) * exp(N(0,1))_row * c_col   ("systematic outlier
                 activations"; Student-t nu=3 body, log-normal per-row scale, c_col = 32 on a
                 seeded 1% of columns, else 1)

Every generator takes an explicit integer ``seed`` and a ``device``; values are
drawn with ``torch.Generator(device).manual_seed(seed)`` and rounded RNE to
bf16.  The same seed on the same device type gives the same bytes.  CPU and
CUDA generators differ, so parity tests either generate on the CPU and copy to
the GPU, or copy GPU-generated rows back to the host for the oracle.
"""
from __future__ import annotations

import torch

__all__ = ["gaussian", "weight", "grad", "heavy", "make", "CFG3_DIMS", "CFG2_DIMS"]

# cfg2: LRM MLP stack dims: layer l maps DIMS[l] -> DIMS[l+1]
CFG2_DIMS = [1024, 1024, 1024, 512, 512, 256, 256, 512, 1024]
# cfg3: DHEN/Wukong-style ensemble feature sizes
CFG3_DIMS = [128, 256, 384, 512, 768, 1024, 1536, 2048]


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=torch.device(device))
    g.manual_seed(int(seed))
    return g


def gaussian(rows: int, cols: int, seed: int, device="cpu", std: float = 1.0) -> torch.Tensor:
    """N(0, std^2) rounded to bf16, shape [rows, cols] row-major."""
    g = _gen(seed, device)
    x = torch.randn(rows, cols, generator=g, device=device, dtype=torch.float32)
    if std != 1.0:
        x = x * std
    return x.to(torch.bfloat16)


def weight(n: int, k: int, seed: int, device="cpu") -> torch.Tensor:
    """W[N, K] ~ N(0, 1/K) in bf16."""
    return gaussian(n, k, seed, device, std=float(k) ** -0.5)


def grad(rows: int, cols: int, seed: int, device="cpu") -> torch.Tensor:
    """dY ~ 2^-10 N(0,1) in bf16."""
    return gaussian(rows, cols, seed, device, std=2.0 ** -10)


def heavy(rows: int, cols: int, seed: int, device="cpu", row0: int = 0, total_rows: int | None = None,
          outlier_frac: float = 0.01, outlier_scale: float = 32.0) -> torch.Tensor:
    """Heavy-tailed LRM-like activations (see module docstring), bf16 [rows, cols].

    ``row0``/``total_rows`` select rows [row0, row0+rows) of one global tensor of
    ``total_rows`` rows, so a rank's shard is bit-identical to the same rows of
    the unsharded tensor (SURVEY.md §8(d) seeds).  Rows are generated
    in fixed 4096-row chunks, each chunk seeded from (seed, chunk index); the
    outlier column set depends on ``seed`` only.
    """
    total_rows = rows if total_rows is None else total_rows
    assert 0 <= row0 and row0 + rows <= total_rows
    gc = _gen(seed * 1_000_003 + 17, "cpu")
    ncol_out = max(1, int(round(outlier_frac * cols)))
    out_cols = torch.randperm(cols, generator=gc)[:ncol_out]
    c_col = torch.ones(cols, dtype=torch.float32)
    c_col[out_cols] = outlier_scale
    c_col = c_col.to(device)
    chunk = 4096
    parts = []
    r = row0
    end = row0 + rows
    while r < end:
        ci = r // chunk
        c0 = ci * chunk
        c1 = min(c0 + chunk, total_rows)
        g = _gen(seed * 7919 + ci, device)
        n = c1 - c0
        z = torch.randn(n, cols, generator=g, device=device, dtype=torch.float32)
        chi = torch.randn(3, n, cols, generator=g, device=device, dtype=torch.float32).square_().sum(0)
        t3 = z / torch.sqrt(chi / 3.0)
        rs = torch.exp(torch.randn(n, 1, generator=g, device=device, dtype=torch.float32))
        blk = (t3 / (3.0 ** 0.5)) * rs * c_col
        lo = max(r, c0) - c0
        hi = min(end, c1) - c0
        parts.append(blk[lo:hi])
        r = c0 + hi
    return torch.cat(parts, 0).to(torch.bfloat16)


def make(dist: str, rows: int, cols: int, seed: int, device="cpu") -> torch.Tensor:
    if dist == "gaussian":
        return gaussian(rows, cols, seed, device)
    if dist == "heavy":
        return heavy(rows, cols, seed, device)
    if dist == "weight":
        return weight(rows, cols, seed, device)
    if dist == "grad":
        return grad(rows, cols, seed, device)
    raise ValueError(dist)
