"""NEXT-2 — LoKA Probe's online input-distribution tracker (TEST INFRASTRUCTURE ONLY).

PAPER.md:282-305 (§III LoKA Probe, "Optimized Input Distribution Modeling"): the batch dimension is
treated as independent, so a layer input X [B, K] (rows = samples, columns = features) is modelled
by its feature mean and K x K covariance, tracked online with a batched Welford (Chan et al.)
update.  For a batch with mean mu_b and scatter S_b = (X - 1 mu_b^T)^T (X - 1 mu_b^T):
    n_new     = n_old + B
    delta     = mu_b - mu_old
    mu_new    = mu_old + (B / n_new) delta
    Sigma_new = Sigma_old + S_b + (n_old B / n_new) delta delta^T     (unnormalised scatter)
and the unbiased covariance is Sigma_new / (n_new - 1) for n_new > 1.
Plain float64 (the paper keeps Sigma "in higher precision (e.g., FP32)"; the oracle's FP64 is
the definition the GPU's FP32 accumulation is checked against).
"""
from __future__ import annotations

import numpy as np


def init(k: int) -> dict:
    return {"n": 0, "mean": np.zeros(k), "scatter": np.zeros((k, k))}


def batch_stats(x):
    """mu_b and S_b of one batch."""
    x = np.asarray(x, np.float64)
    mu = x.mean(axis=0)
    xc = x - mu[None, :]
    return mu, xc.T @ xc


def update(state: dict, x) -> dict:
    """One batched Welford merge, in the paper's order and notation."""
    x = np.asarray(x, np.float64)
    b = x.shape[0]
    if b == 0:
        return dict(state)
    mu_b, s_b = batch_stats(x)
    n_old = state["n"]
    n_new = n_old + b
    delta = mu_b - state["mean"]
    mu_new = state["mean"] + (b / n_new) * delta
    sigma_new = state["scatter"] + s_b + (n_old * b / n_new) * np.outer(delta, delta)
    return {"n": n_new, "mean": mu_new, "scatter": sigma_new}


def covariance(state: dict) -> np.ndarray:
    """Unbiased (sample) covariance Sigma / (n - 1), n > 1."""
    if state["n"] < 2:
        raise ValueError("covariance needs n > 1")
    return state["scatter"] / (state["n"] - 1)
