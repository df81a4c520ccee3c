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


# ---- NEXT-3: matrix-normal weight tracker -------------------------------------
# W [M, N] ~ MN(Mean, U, V): vec(W) ~ N(vec(Mean), V (x) U), U [M, M] row covariance, V [N, N]
# column covariance.  Readings (D32-D34): the state starts at Mean = the first observed
# weight, U = I_M, V = I_N; W_c is centred by the CURRENT mean, which is then updated
# by an EMA with the same momentum m; both per-update estimates use the current (U, V)
# (the flip-flop of one update reads the factors as they were before it); eps_U = eps_rel tr(U)/M
# and eps_V = eps_rel tr(V)/N of the current factors are used both in the solves and in the
# "+ eps I" of the regularisation.

def weight_init(w, momentum: float = 0.95, eps_rel: float = 1e-6) -> dict:
    w = np.asarray(w, np.float64)
    m, n = w.shape
    return {"mean": w.copy(), "U": np.eye(m), "V": np.eye(n), "m": float(momentum), "eps_rel": float(eps_rel),
            "count": 0}


def _solve_lower(l, b):
    """x = L^{-1} b for lower-triangular L by forward substitution (column by column of b)."""
    n = l.shape[0]
    x = np.array(b, np.float64, copy=True)
    for i in range(n):
        x[i] = (x[i] - l[i, :i] @ x[:i]) / l[i, i]
    return x


def weight_update(state: dict, w) -> dict:
    """One Kronecker-factor (flip-flop) update with EMA, symmetrisation + eps I and the trace
    renormalisation, in the paper's order."""
    w = np.asarray(w, np.float64)
    mm, nn = w.shape
    u, v, m = state["U"], state["V"], state["m"]
    wc = w - state["mean"]
    eps_u = state["eps_rel"] * np.trace(u) / mm
    eps_v = state["eps_rel"] * np.trace(v) / nn
    # Solve L_V L_V^T = V + eps I, W~ = W_c L_V^{-T}, U' = (1/N) W~ W~^T
    l_v = np.linalg.cholesky(v + eps_v * np.eye(nn))
    w_t = _solve_lower(l_v, wc.T).T  # W_c L_V^{-T} = (L_V^{-1} W_c^T)^T
    u1 = (w_t @ w_t.T) / nn
    # Solve L_U L_U^T = U + eps I, W^ = L_U^{-1} W_c, V' = (1/M) W^^T W^
    l_u = np.linalg.cholesky(u + eps_u * np.eye(mm))
    w_h = _solve_lower(l_u, wc)
    v1 = (w_h.T @ w_h) / mm
    # EMA, symmetrise + eps I
    u2 = m * u + (1.0 - m) * u1
    v2 = m * v + (1.0 - m) * v1
    u_new = 0.5 * (u2 + u2.T) + eps_u * np.eye(mm)
    v_new = 0.5 * (v2 + v2.T) + eps_v * np.eye(nn)
    # scale identifiability: s = tr(U)/M, U <- U/s, V <- s V
    s = np.trace(u_new) / mm
    return {"mean": m * state["mean"] + (1.0 - m) * w, "U": u_new / s, "V": s * v_new, "m": m,
            "eps_rel": state["eps_rel"], "count": state["count"] + 1}
