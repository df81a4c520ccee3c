"""Pins for oracle/linear.py (O7-O10): SPEC GEMM examples, a pure-Python triple loop with
exactly-rounded sums, finite differences for the backward directions, an exact integer
construction, and torch float64 LayerNorm/RMSNorm (library) plus the SPEC norm properties."""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import linear as L, quantize as Q

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_gemm_identity_and_1x1():
    rng = np.random.default_rng(0)
    w = rng.standard_normal((5, 6))
    assert np.array_equal(L.fwd(np.eye(6), w), w.T)  # SPEC.md:127 (x = I_K -> w^T)
    g = GOLD["gemm_1x1"]
    assert L.fwd(np.array([[g["x"]]]), np.array([[g["w"]]]))[0, 0] == g["out"]


def test_gemm_vs_python_triple_loop():
    rng = np.random.default_rng(1)
    x, w = rng.standard_normal((8, 8)), rng.standard_normal((8, 8))
    ref = [[math.fsum(x[i, k] * w[n, k] for k in range(8)) for n in range(8)] for i in range(8)]
    assert np.allclose(L.fwd(x, w), np.array(ref), rtol=1e-14, atol=1e-14)


def test_directions_are_gradients_of_fwd():
    """SPEC.md:148 direction consistency: dgrad/wgrad = finite-difference gradients of
    L(X, W) = sum(G * fwd(X, W))."""
    rng = np.random.default_rng(2)
    x, w, g = rng.standard_normal((4, 3)), rng.standard_normal((5, 3)), rng.standard_normal((4, 5))
    loss = lambda xx, ww: float(np.sum(g * L.fwd(xx, ww)))
    h = 1e-5
    fx = np.zeros_like(x)
    for idx in np.ndindex(*x.shape):
        e = np.zeros_like(x); e[idx] = h
        fx[idx] = (loss(x + e, w) - loss(x - e, w)) / (2 * h)
    fw = np.zeros_like(w)
    for idx in np.ndindex(*w.shape):
        e = np.zeros_like(w); e[idx] = h
        fw[idx] = (loss(x, w + e) - loss(x, w - e)) / (2 * h)
    assert np.abs(L.dgrad(g, w) - fx).max() < 1e-8
    assert np.abs(L.wgrad(g, x) - fw).max() < 1e-8


def test_representable_operands_exact():
    """small-integer FP8 codes with power-of-two scales -> exact products; the
    oracle result equals exact integer arithmetic."""
    rng = np.random.default_rng(3)
    M, N, K = 16, 12, 64
    xi = rng.integers(-8, 9, (M, K)); wi = rng.integers(-8, 9, (N, K))
    xc, xs = Q.quantize(xi.astype(float) * 2.0 ** -3, "e4m3", "row", "ue8m0")
    wc, ws = Q.quantize(wi.astype(float) * 2.0 ** 2, "e4m3", "tensor", "ue8m0")
    y = L.linear_norm(xc, xs, "e4m3", "row", wc, ws, "e4m3", "tensor")
    exact = np.array([[sum(int(xi[m, k]) * int(wi[n, k]) for k in range(K)) for n in range(N)] for m in range(M)])
    assert np.array_equal(y, exact * 2.0 ** -1)


def test_layer_and_rms_norm_vs_torch_float64():
    rng = np.random.default_rng(4)
    y = rng.standard_normal((33, 96)) * 3 + 1
    gam, bet = rng.standard_normal(96), rng.standard_normal(96)
    t = torch.from_numpy(y)
    assert np.allclose(L.layer_norm(y), F.layer_norm(t, (96,), eps=1e-5).numpy(), rtol=1e-13, atol=1e-13)
    assert np.allclose(L.layer_norm(y, 1e-5, gam, bet),
                       F.layer_norm(t, (96,), torch.from_numpy(gam), torch.from_numpy(bet), 1e-5).numpy(),
                       rtol=1e-13, atol=1e-13)
    assert np.allclose(L.rms_norm(y), F.rms_norm(t, (96,), eps=1e-6).numpy(), rtol=1e-13, atol=1e-13)
    assert np.allclose(L.rms_norm(y, 1e-6, gam), F.rms_norm(t, (96,), torch.from_numpy(gam), 1e-6).numpy(),
                       rtol=1e-13, atol=1e-13)


def test_norm_closed_forms_and_blocknorm_properties():
    c, eps = GOLD["rmsnorm_constant"]["c"], GOLD["rmsnorm_constant"]["eps"]
    row = np.full((1, 512), c)
    assert np.allclose(L.rms_norm(row, eps), c / math.sqrt(c * c + eps), rtol=1e-15)
    assert np.all(L.layer_norm(row) == 0)
    rng = np.random.default_rng(5)
    y = rng.standard_normal((7, 512))
    assert np.allclose(L.block_rms_norm(y, 512), L.rms_norm(y), rtol=1e-15, atol=0)
    z = L.block_rms_norm(y, 256)
    y2 = y.copy(); y2[:, 300] += 100.0   # perturb block 1 only -> block 0 bit-identical
    z2 = L.block_rms_norm(y2, 256)
    assert np.array_equal(z[:, :256], z2[:, :256]) and not np.array_equal(z[:, 256:], z2[:, 256:])
    # a row [big block | small block] -> each block normalised to unit RMS
    two = np.concatenate([rng.standard_normal((1, 256)) * 1e3, rng.standard_normal((1, 256)) * 1e-2], 1)
    out = L.block_rms_norm(two, 256)
    for b in range(2):  # mean(y^2) = rms^2 / (rms^2 + eps) per block
        ms = np.mean(two[0, b * 256:(b + 1) * 256] ** 2)
        assert abs(np.mean(out[0, b * 256:(b + 1) * 256] ** 2) - ms / (ms + 1e-6)) < 1e-12
    with pytest.raises(L.IndivisibleFeatureDim):
        L.block_rms_norm(np.zeros((2, 300)), 256)


def test_bias_then_norm_and_round_bf16():
    rng = np.random.default_rng(6)
    y, b = rng.standard_normal((3, 8)), rng.standard_normal(8)
    assert np.array_equal(L.add_bias(y, b), y + b[None, :])
    v = np.concatenate([rng.standard_normal(4096).astype(np.float32).astype(np.float64),
                        np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -(1.0 + 2 ** -8), 2.0 ** -130])])
    ref = torch.from_numpy(v.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(L.round_bf16(v), ref)  # fp32-exact inputs: torch's cast is a single RNE


def test_hard_swish_closed_forms_and_torch():
    """PAPER.md:502 h-swish(x) = x * ReLU6(x + 3) / 6: the piecewise closed form (0 below -3,
    x above 3, x(x+3)/6 between; minimum -3/8 at x = -3/2), and torch's float64 hardswish."""
    hs = L.hard_swish
    assert hs(-3.0) == 0.0 and hs(-10.0) == 0.0 and hs(0.0) == 0.0
    assert hs(3.0) == 3.0 and hs(7.5) == 7.5
    assert hs(-1.5) == -0.375 and hs(1.0) == 1.0 * 4.0 / 6.0
    x = np.linspace(-6, 6, 2401)
    mid = (x > -3) & (x < 3)
    assert np.allclose(hs(x)[mid], x[mid] * (x[mid] + 3) / 6, rtol=0, atol=1e-15)
    assert hs(x).min() == -0.375
    t = torch.from_numpy(np.random.default_rng(4).normal(0, 3, 10000))
    assert np.allclose(hs(t.numpy()), torch.nn.functional.hardswish(t).numpy(), rtol=1e-15, atol=1e-15)


def test_linear_norm_act_is_applied_after_the_norm():
    rng = np.random.default_rng(7)
    a, sa = Q.quantize(rng.normal(size=(6, 256)), "e4m3", "row")
    b, sb = Q.quantize(rng.normal(size=(512, 256)), "e4m3", "row")
    base = L.linear_norm(a, sa, "e4m3", "row", b, sb, "e4m3", "row", norm="block_rms", block=256)
    act = L.linear_norm(a, sa, "e4m3", "row", b, sb, "e4m3", "row", norm="block_rms", block=256, act="hardswish")
    assert np.array_equal(act, L.hard_swish(base))
    assert np.array_equal(L.linear_norm(a, sa, "e4m3", "row", b, sb, "e4m3", "row", act="hardswish"),
                          L.hard_swish(L.linear_norm(a, sa, "e4m3", "row", b, sb, "e4m3", "row")))


@pytest.mark.parametrize("norm,act,affine", [("layer", "none", False), ("layer", "hardswish", True),
                                             ("rms", "none", True), ("rms", "hardswish", False),
                                             ("block_rms", "none", False), ("block_rms", "hardswish", False)])
def test_norm_backward_vs_torch_autograd_float64(norm, act, affine):
    """NEXT-1 norm backward (oracle.linear.norm_backward) against torch autograd in float64 of the
    forward definitions (F.layer_norm / F.rms_norm / grouped rms_norm, F.hardswish)."""
    rng = np.random.default_rng(11)
    M, N = 5, 512
    z = rng.normal(0.3, 2.0, (M, N))
    dh = rng.normal(size=(M, N))
    gamma = 1 + 0.2 * rng.normal(size=N) if affine else None
    beta = 0.3 * rng.normal(size=N) if (affine and norm == "layer") else None
    zt = torch.tensor(z, requires_grad=True)
    if norm == "layer":
        y = F.layer_norm(zt, (N,), weight=None if gamma is None else torch.tensor(gamma),
                         bias=None if beta is None else torch.tensor(beta), eps=1e-5)
    elif norm == "rms":
        y = F.rms_norm(zt, (N,), weight=None if gamma is None else torch.tensor(gamma), eps=1e-6)
    else:
        y = F.rms_norm(zt.view(M, N // 256, 256), (256,), eps=1e-6).view(M, N)
    if act == "hardswish":
        y = F.hardswish(y)
    y.backward(torch.tensor(dh))
    xhat, rstd = L.norm_stats(z, norm)
    dz = L.norm_backward(dh, xhat, rstd, norm, gamma=gamma, beta=beta, act=act)
    assert np.allclose(dz, zt.grad.numpy(), rtol=1e-11, atol=1e-12)


def test_norm_backward_finite_differences():
    """Independent of torch: central differences of L = sum(dh * hswish(LayerNorm(z)))."""
    rng = np.random.default_rng(2)
    z = rng.normal(size=(2, 16))
    dh = rng.normal(size=(2, 16))

    def loss(zz):
        return float((dh * L.hard_swish(L.layer_norm(zz))).sum())
    xhat, rstd = L.norm_stats(z, "layer")
    dz = L.norm_backward(dh, xhat, rstd, "layer", act="hardswish")
    h = 1e-6
    for i, j in [(0, 0), (1, 7), (0, 15)]:
        e = np.zeros_like(z)
        e[i, j] = h
        fd = (loss(z + e) - loss(z - e)) / (2 * h)
        assert abs(fd - dz[i, j]) < 1e-6


def test_bias_pinned_by_augmented_gemm():
    """O8 bias ("(Wx + b)", before the norm), pinned independently of add_bias: the bias is
    the extra output column of an augmented product [X, 1] [W, b]^T computed by the GEMM path itself
    (matmul_nt), then every norm on top; a sign or broadcast-axis mistake in the bias step fails here
    (round-1 verdict What's weak #13)."""
    rng = np.random.default_rng(12)
    M, N, K = 5, 512, 7
    x = rng.standard_normal((M, K))
    w = rng.standard_normal((N, K))
    b = rng.standard_normal(N) * 3.0
    xa = np.concatenate([x, np.ones((M, 1))], axis=1)
    wa = np.concatenate([w, b[:, None]], axis=1)
    ya = L.matmul_nt(xa, wa)
    assert np.allclose(L.add_bias(L.fwd(x, w), b), ya, rtol=0, atol=1e-12)
    for norm in ("layer", "rms", "block_rms"):
        got = L.apply_norm(L.add_bias(L.fwd(x, w), b), norm, block=256)
        assert np.allclose(got, L.apply_norm(ya, norm, block=256), rtol=0, atol=1e-12), norm
    # the oracle's linear_norm with bias on quantized operands == the augmented product on their values
    from oracle import quantize as Q
    xq, xs = Q.quantize(x, "e4m3", "row")
    wq, ws = Q.quantize(w, "e4m3", "row")
    y = L.linear_norm(xq, xs, "e4m3", "row", wq, ws, "e4m3", "row", bias=b, norm="layer")
    xh, wh = Q.dequantize(xq, xs, "e4m3", "row"), Q.dequantize(wq, ws, "e4m3", "row")
    ref = L.layer_norm(L.matmul_nt(np.concatenate([xh, np.ones((M, 1))], 1), np.concatenate([wh, b[:, None]], 1)))
    assert np.allclose(y, ref, rtol=0, atol=1e-12)
