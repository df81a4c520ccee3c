"""-m gpu: NEXT-1 — the norm backward fused into a GEMM epilogue, and the
forward's saves it consumes.  Forward: linear_norm(..., save_xhat, save_rstd) writes the normalised
values (bf16) and rstd of z; backward: A . B^T (e.g. the next layer's dgrad, dL/dh) -> epilogue
g = dh * act'(xhat*gamma+beta) * gamma -> dz = rstd (g - mean(g) - xhat mean(g xhat)) (LayerNorm;
RMSNorm / BlockNorm without the mean(g) term) -> f32 / bf16 / e5m2.  Compared with
oracle.linear.norm_stats / norm_backward on the same inputs."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, assert_bytes_equal, assert_scales_equal, f64, to_dev_padded

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None
TOL = 2e-3


def _q(x, fmt="e4m3"):
    return lk.loka_quantize(to_dev_padded(x), fmt, "row")


@pytest.mark.parametrize("norm,N", [("layer", 1024), ("rms", 256), ("block_rms", 512)])
def test_forward_saves_xhat_and_rstd(norm, N):
    M, K = 300, 384
    xq, xs = _q(synth.heavy(M, K, 1))
    wq, ws = _q(synth.weight(N, K, 2))
    nb = N // 256 if norm == "block_rms" else 1
    sx = torch.empty(M, N, dtype=torch.bfloat16, device=DEV)
    sr = torch.empty(M, nb, dtype=torch.float32, device=DEV) if nb > 1 else torch.empty(M, dtype=torch.float32,
                                                                                       device=DEV)
    lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, out_dtype="f32", save_xhat=sx, save_rstd=sr)
    torch.cuda.synchronize()
    z = oracle.linear.linear_norm(xq.cpu().numpy(), xs.cpu().numpy(), "e4m3", "row", wq.cpu().numpy(),
                                  ws.cpu().numpy(), "e4m3", "row")
    xh, rs = oracle.linear.norm_stats(z, norm)
    assert np.max(np.abs(f64(sx) - xh)) <= 2.0 ** -8 * np.max(np.abs(xh)) + 2e-3
    assert np.allclose(f64(sr).reshape(rs.shape), rs, rtol=2e-3, atol=0)


@pytest.mark.parametrize("norm,N,act,affine", [("layer", 1024, "none", False), ("layer", 256, "hardswish", True),
                                               ("rms", 512, "none", True), ("block_rms", 512, "hardswish", False),
                                               ("block_rms", 768, "none", False)])
def test_norm_backward_epilogue_f32(norm, N, act, affine):
    M, K2 = 300, 384
    aq, as_ = _q(synth.grad(M, K2, 3) * 1024, "e5m2")
    bq, bs = _q(synth.weight(N, K2, 4))
    rng = np.random.default_rng(N)
    xh = torch.tensor(rng.normal(size=(M, N)), dtype=torch.bfloat16)
    nb = N // 256
    rstd = torch.tensor(rng.uniform(0.5, 2.0, size=(M, nb) if norm == "block_rms" else (M,)), dtype=torch.float32)
    gamma = torch.tensor(1 + 0.2 * rng.normal(size=N), dtype=torch.float32) if affine else None
    beta = torch.tensor(0.3 * rng.normal(size=N), dtype=torch.float32) if (affine and norm == "layer") else None
    y, _ = lk.loka_fp8_linear_norm(aq, as_, bq, bs, a_fmt="e5m2", norm=norm, act=act, out_dtype="f32",
                                   bwd_xhat=xh.to(DEV), bwd_rstd=rstd.to(DEV), direction="dgrad",
                                   gamma=None if gamma is None else gamma.to(DEV),
                                   beta=None if beta is None else beta.to(DEV))
    torch.cuda.synchronize()
    dh = oracle.linear.linear_norm(aq.cpu().numpy(), as_.cpu().numpy(), "e5m2", "row", bq.cpu().numpy(),
                                   bs.cpu().numpy(), "e4m3", "row")
    dz = oracle.linear.norm_backward(dh, xh.double().numpy(), rstd.double().numpy(), norm,
                                     gamma=None if gamma is None else gamma.double().numpy(),
                                     beta=None if beta is None else beta.double().numpy(), act=act)
    rms = np.sqrt(np.mean(dz ** 2, axis=1, keepdims=True))
    assert np.max(np.abs(f64(y) - dz) / np.maximum(np.abs(dz), rms)) <= TOL


def test_norm_backward_e5m2_output_bit_exact():
    """dz as the next dgrad's e5m2 rowwise operand: codes + scales equal the oracle's quantize of
    the GPU's own pre-cast dz (cluster of 8 CTAs for N = 1024)."""
    M, N, K2 = 256, 1024, 512
    aq, as_ = _q(synth.grad(M, K2, 5) * 1024, "e5m2")
    bq, bs = _q(synth.weight(N, K2, 6))
    rng = np.random.default_rng(1)
    xh = torch.tensor(rng.normal(size=(M, N)), dtype=torch.bfloat16).to(DEV)
    rstd = torch.tensor(rng.uniform(0.5, 2.0, size=M), dtype=torch.float32).to(DEV)
    pre = torch.empty(M, N, dtype=torch.float32, device=DEV)
    y, ys = lk.loka_fp8_linear_norm(aq, as_, bq, bs, a_fmt="e5m2", norm="layer", out_dtype="e5m2", precast=pre,
                                    bwd_xhat=xh, bwd_rstd=rstd, direction="dgrad")
    torch.cuda.synchronize()
    oq, os_ = oracle.quantize.quantize(f64(pre), "e5m2", "row")
    assert_scales_equal(ys, os_)
    assert_bytes_equal(y, oq)
    dh = oracle.linear.linear_norm(aq.cpu().numpy(), as_.cpu().numpy(), "e5m2", "row", bq.cpu().numpy(),
                                   bs.cpu().numpy(), "e4m3", "row")
    dz = oracle.linear.norm_backward(dh, f64(xh), f64(rstd), "layer")
    rms = np.sqrt(np.mean(dz ** 2, axis=1, keepdims=True))
    assert np.max(np.abs(f64(pre) - dz) / np.maximum(np.abs(dz), rms)) <= TOL


@pytest.mark.parametrize("act", ["none", "hardswish"])
def test_forward_then_backward_chain_matches_autograd(act):
    """End to end on one layer: forward (saves) -> backward epilogue on dL/dh.  Exact parity with the
    oracle on the saved values, and closeness to torch float64 autograd of LayerNorm (+ hardswish)
    on the oracle's z (the bf16 x-hat rounding enters; h-swish' jumps at +-3, so elements whose
    pre-activation sits within that rounding of a kink may differ)."""
    M, K, N = 256, 256, 512
    xq, xs = _q(synth.heavy(M, K, 7))
    wq, ws = _q(synth.weight(N, K, 8))
    sx = torch.empty(M, N, dtype=torch.bfloat16, device=DEV)
    sr = torch.empty(M, dtype=torch.float32, device=DEV)
    lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="layer", act=act, out_dtype="bf16", save_xhat=sx,
                            save_rstd=sr)
    gq, gs = _q(synth.grad(M, 128, 9) * 1024, "e5m2")  # dL/dh = G . V^T, V [N, 128]
    vq, vs = _q(synth.weight(N, 128, 10))
    dz, _ = lk.loka_fp8_linear_norm(gq, gs, vq, vs, a_fmt="e5m2", norm="layer", act=act, out_dtype="f32",
                                    bwd_xhat=sx, bwd_rstd=sr)
    torch.cuda.synchronize()
    z = oracle.linear.linear_norm(xq.cpu().numpy(), xs.cpu().numpy(), "e4m3", "row", wq.cpu().numpy(),
                                  ws.cpu().numpy(), "e4m3", "row")
    dh = oracle.linear.linear_norm(gq.cpu().numpy(), gs.cpu().numpy(), "e5m2", "row", vq.cpu().numpy(),
                                   vs.cpu().numpy(), "e4m3", "row")
    own = oracle.linear.norm_backward(dh, f64(sx), f64(sr), "layer", act=act)
    rms = np.sqrt(np.mean(own ** 2, axis=1, keepdims=True))
    assert np.max(np.abs(f64(dz) - own) / np.maximum(np.abs(own), rms)) <= TOL
    zt = torch.tensor(z, requires_grad=True)
    h = torch.nn.functional.layer_norm(zt, (N,), eps=1e-5)
    (torch.nn.functional.hardswish(h) if act == "hardswish" else h).backward(torch.tensor(dh))
    ref = zt.grad.numpy()
    rms = np.sqrt(np.mean(ref ** 2, axis=1, keepdims=True))
    close = np.abs(f64(dz) - ref) <= 1e-2 * np.maximum(np.abs(ref), rms)
    assert np.mean(close) > (0.999 if act == "none" else 0.99)


@pytest.mark.parametrize("norm,N,act,od", [("layer", 1024, "hardswish", "f32"), ("rms", 2048, "none", "bf16"),
                                           ("block_rms", 512, "none", "e5m2")])
def test_norm_backward_unfused_at_scale(norm, N, act, od):
    """Enough rows for the CTA-pair engine: dh (FP32, workspace) + the row-wise backward pass."""
    M, K2 = 20480, 256
    aq, as_ = _q(synth.grad(M, K2, 12) * 1024, "e5m2")
    bq, bs = _q(synth.weight(N, K2, 13))
    rng = np.random.default_rng(3)
    xh = torch.tensor(rng.normal(size=(M, N)), dtype=torch.bfloat16)
    rstd = torch.tensor(rng.uniform(0.5, 2.0, size=(M, N // 256) if norm == "block_rms" else (M,)),
                        dtype=torch.float32)
    pre = torch.empty(M, N, dtype=torch.float32, device=DEV)
    y, ys = lk.loka_fp8_linear_norm(aq, as_, bq, bs, a_fmt="e5m2", norm=norm, act=act, out_dtype=od, precast=pre,
                                    bwd_xhat=xh.to(DEV), bwd_rstd=rstd.to(DEV), direction="dgrad")
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(4).choice(M, 40, replace=False))
    dh = oracle.linear.linear_norm(aq.cpu().numpy()[rows], as_.cpu().numpy()[rows], "e5m2", "row", bq.cpu().numpy(),
                                   bs.cpu().numpy(), "e4m3", "row")
    dz = oracle.linear.norm_backward(dh, xh.double().numpy()[rows], rstd.double().numpy()[rows], norm, act=act)
    rms = np.sqrt(np.mean(dz ** 2, axis=1, keepdims=True))
    assert np.max(np.abs(f64(pre)[rows] - dz) / np.maximum(np.abs(dz), rms)) <= TOL
    if od == "e5m2":
        oq, os_ = oracle.quantize.quantize(f64(pre)[rows], "e5m2", "row")
        assert_scales_equal(ys[rows], os_)
        assert_bytes_equal(y[rows], oq)
