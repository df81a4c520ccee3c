"""-m gpu: the three GEMM directions of a training step (PAPER.md:547 per-direction recipes;
BJ configs[3]) with e4m3 activations / weights and e5m2 gradients, for the tensorwise, rowwise
and blockwise (1x128 x 128x128, FP32 promotion) recipes.  Every direction runs the library's
C = A . B^T kernel on K-major operands produced by loka_quantize (cast-transpose for the
backward copies) and is compared with oracle/linear.py's fwd / dgrad / wgrad on the operands
dequantized with each direction's own granularity (D6)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, f64, guarded_rel_err, to_dev_padded

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None
TOL = 2e-3

# recipe -> granularities (x-frame) for: fwd X, fwd W, dgrad dY, dgrad W, wgrad dY, wgrad X
RECIPES = {
    "tensor": dict(fx="tensor", fw="tensor", gdy="tensor", gw="tensor", wdy="tensor", wx="tensor"),
    "row": dict(fx="row", fw="row", gdy="row", gw="col", wdy="col", wx="col"),
    "block": dict(fx="blk_1x128", fw="blk_128x128", gdy="blk_1x128", gw="blk_128x128", wdy="blk_128x1",
                  wx="blk_128x1"),
}
T = {"row": "col", "col": "row", "blk_1x128": "blk_128x1", "blk_128x1": "blk_1x128"}


def _deq(x, fmt, gran):
    q, s = oracle.quantize.quantize(x.double().numpy(), fmt, gran)
    return oracle.quantize.dequantize(q, s, fmt, gran)


@pytest.mark.parametrize("recipe", list(RECIPES))
@pytest.mark.parametrize("M,N,K", [(512, 384, 256), (300, 256, 640)])
def test_fwd_dgrad_wgrad(recipe, M, N, K):
    g = RECIPES[recipe]
    x = synth.heavy(M, K, 1)
    w = synth.weight(N, K, 2)
    dy = synth.grad(M, N, 3)
    xd, wd, dyd = to_dev_padded(x), to_dev_padded(w), to_dev_padded(dy)
    # fwd: Y = X W^T
    xq, xs = lk.loka_quantize(xd, "e4m3", g["fx"])
    wq, ws = lk.loka_quantize(wd, "e4m3", g["fw"])
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran=g["fx"], b_gran=g["fw"], out_dtype="f32")
    # dgrad: dX = dY W  -> A = dYq [M,N], B = (W^T)q [K,N] (transposed copy of W's quantization)
    gq, gs = lk.loka_quantize(dyd, "e5m2", g["gdy"])
    _, _, wtq, wts = lk.loka_quantize(wd, "e4m3", g["gw"], want_q=False, transpose=True)
    dx, _ = lk.loka_fp8_linear_norm(gq, gs, wtq, wts, a_fmt="e5m2", a_gran=g["gdy"], b_gran=T.get(g["gw"], g["gw"]),
                                    out_dtype="f32", direction="dgrad")
    # wgrad: dW = dY^T X -> A = (dY^T)q [N,M], B = (X^T)q [K,M]
    _, _, gtq, gts = lk.loka_quantize(dyd, "e5m2", g["wdy"], want_q=False, transpose=True)
    _, _, xtq, xts = lk.loka_quantize(xd, "e4m3", g["wx"], want_q=False, transpose=True)
    dw, _ = lk.loka_fp8_linear_norm(gtq, gts, xtq, xts, a_fmt="e5m2", a_gran=T.get(g["wdy"], g["wdy"]),
                                    b_gran=T.get(g["wx"], g["wx"]), out_dtype="f32", direction="wgrad")
    torch.cuda.synchronize()
    yo = oracle.linear.fwd(_deq(x, "e4m3", g["fx"]), _deq(w, "e4m3", g["fw"]))
    dxo = oracle.linear.dgrad(_deq(dy, "e5m2", g["gdy"]), _deq(w, "e4m3", g["gw"]))
    dwo = oracle.linear.wgrad(_deq(dy, "e5m2", g["wdy"]), _deq(x, "e4m3", g["wx"]))
    assert guarded_rel_err(f64(y), yo) <= TOL
    assert guarded_rel_err(f64(dx), dxo) <= TOL
    assert guarded_rel_err(f64(dw), dwo) <= TOL


def test_blockwise_bf16_fp8_outputs_and_bias():
    M, N, K = 384, 128, 1000
    x, w = synth.heavy(M, K, 5), synth.weight(N, K, 6)
    xq, xs = lk.loka_quantize(to_dev_padded(x), "e4m3", "blk_1x128")
    wq, ws = lk.loka_quantize(to_dev_padded(w), "e4m3", "blk_128x128")
    bias = torch.randn(N, generator=torch.Generator().manual_seed(0))
    yo = oracle.linear.linear_norm(xq.cpu().numpy(), xs.cpu().numpy(), "e4m3", "blk_1x128", wq.cpu().numpy(),
                                   ws.cpu().numpy(), "e4m3", "blk_128x128", bias=bias.double().numpy())
    yb, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="blk_1x128", b_gran="blk_128x128", bias=bias.to(DEV),
                                    out_dtype="bf16")
    pre = torch.empty(M, N, dtype=torch.float32, device=DEV)
    y8, y8s = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="blk_1x128", b_gran="blk_128x128", bias=bias.to(DEV),
                                      out_dtype="e4m3", precast=pre)
    torch.cuda.synchronize()
    rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
    assert np.all(np.abs(f64(yb) - yo) <= TOL * np.maximum(np.abs(yo), rms) + 2.0 ** -8 * np.abs(yo))
    assert guarded_rel_err(f64(pre), yo) <= TOL
    oq, os_ = oracle.quantize.quantize(f64(pre), "e4m3", "row")
    assert np.array_equal(y8.cpu().numpy(), oq)
    assert np.array_equal(y8s.cpu().numpy().view(np.uint32), os_.view(np.uint32))


def test_cfg4_shape_sampled():
    """BJ configs[3] size: M=32768, K=N=4096, blockwise fwd (bench launch configuration), rows sampled."""
    M, N, K = 32768, 4096, 4096
    x = synth.gaussian(M, K, 0, device=DEV)
    w = synth.weight(N, K, 1, device=DEV)
    xq, xs = lk.loka_quantize(x, "e4m3", "blk_1x128")
    wq, ws = lk.loka_quantize(w, "e4m3", "blk_128x128")
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="blk_1x128", b_gran="blk_128x128", out_dtype="bf16")
    torch.cuda.synchronize()
    rows = torch.randperm(M, generator=torch.Generator().manual_seed(4))[:16].sort().values.to(DEV)
    yo = oracle.linear.linear_norm(xq[rows].cpu().numpy(), xs[rows].cpu().numpy(), "e4m3", "blk_1x128",
                                   wq.cpu().numpy(), ws.cpu().numpy(), "e4m3", "blk_128x128")
    rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
    assert np.all(np.abs(f64(y[rows]) - yo) <= TOL * np.maximum(np.abs(yo), rms) + 2.0 ** -8 * np.abs(yo))


@pytest.mark.parametrize("recipe", ["tensor", "row"])
@pytest.mark.parametrize("od", ["f32", "bf16"])
def test_wide_pair_engine_routes(recipe, od, monkeypatch):
    """The production routes of the cfg4 / cfg5 GEMMs on the CTA-pair engine (round-1 verdict
    What's weak #2a): M = 4864, N = K = 2048 gives 76 WIDE 256 x 512 tiles and 16 K stages, so fwd and
    dgrad take grouped2_kernel<FP8, WIDE, !SPLIT>; wgrad (32 wide tiles, K = M = 4864) takes the WIDE
    split-K instance + the slice reduction.  All three against the oracle at 2e-3 (bf16 output: plus one
    bf16 half-ulp)."""
    monkeypatch.delenv("LOKA_PAIR_WIDE", raising=False)
    g = RECIPES[recipe]
    M, N, K = 4864, 2048, 2048
    x = synth.heavy(M, K, 11)
    w = synth.weight(N, K, 12)
    dy = synth.grad(M, N, 13)
    xd, wd, dyd = to_dev_padded(x), to_dev_padded(w), to_dev_padded(dy)
    xq, xs = lk.loka_quantize(xd, "e4m3", g["fx"])
    wq, ws = lk.loka_quantize(wd, "e4m3", g["fw"])
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran=g["fx"], b_gran=g["fw"], out_dtype=od)
    gq, gs = lk.loka_quantize(dyd, "e5m2", g["gdy"])
    _, _, wtq, wts = lk.loka_quantize(wd, "e4m3", g["gw"], want_q=False, transpose=True)
    dx, _ = lk.loka_fp8_linear_norm(gq, gs, wtq, wts, a_fmt="e5m2", a_gran=g["gdy"], b_gran=T.get(g["gw"], g["gw"]),
                                    out_dtype=od, direction="dgrad")
    _, _, gtq, gts = lk.loka_quantize(dyd, "e5m2", g["wdy"], want_q=False, transpose=True)
    _, _, xtq, xts = lk.loka_quantize(xd, "e4m3", g["wx"], want_q=False, transpose=True)
    dw, _ = lk.loka_fp8_linear_norm(gtq, gts, xtq, xts, a_fmt="e5m2", a_gran=T.get(g["wdy"], g["wdy"]),
                                    b_gran=T.get(g["wx"], g["wx"]), out_dtype="f32", direction="wgrad")
    torch.cuda.synchronize()
    yo = oracle.linear.fwd(_deq(x, "e4m3", g["fx"]), _deq(w, "e4m3", g["fw"]))
    dxo = oracle.linear.dgrad(_deq(dy, "e5m2", g["gdy"]), _deq(w, "e4m3", g["gw"]))
    dwo = oracle.linear.wgrad(_deq(dy, "e5m2", g["wdy"]), _deq(x, "e4m3", g["wx"]))
    for got, ref in ((y, yo), (dx, dxo)):
        if od == "f32":
            assert guarded_rel_err(f64(got), ref) <= TOL
        else:
            guard = np.maximum(np.abs(ref), np.sqrt(np.mean(ref ** 2, axis=1, keepdims=True)))
            assert np.all(np.abs(f64(got) - ref) <= TOL * guard + 2.0 ** -8 * np.abs(ref))
    assert guarded_rel_err(f64(dw), dwo) <= TOL


@pytest.mark.parametrize("recipe", ["tensor", "row"])
def test_cfg4_shape_sampled(recipe):
    """BJ configs[3] at full size (M = 32768, K = N = 4096) in the bench's launch configuration:
    fwd / dgrad rows and wgrad rows (output channels) sampled, the oracle run on the operands the GPU
    consumed (their quantization is checked bit-exactly elsewhere), bf16 out for fwd / dgrad, f32 dW."""
    g = RECIPES[recipe]
    M = 32768
    N = K = 4096
    x = synth.gaussian(M, K, 0, device=DEV)
    w = synth.weight(N, K, 1, device=DEV)
    dy = synth.grad(M, N, 2, device=DEV)
    xq, xs = lk.loka_quantize(x, "e4m3", g["fx"])
    wq, ws = lk.loka_quantize(w, "e4m3", g["fw"])
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran=g["fx"], b_gran=g["fw"], out_dtype="bf16")
    gq, gs = lk.loka_quantize(dy, "e5m2", g["gdy"])
    _, _, wtq, wts = lk.loka_quantize(w, "e4m3", g["gw"], want_q=False, transpose=True)
    dx, _ = lk.loka_fp8_linear_norm(gq, gs, wtq, wts, a_fmt="e5m2", a_gran=g["gdy"], b_gran=T.get(g["gw"], g["gw"]),
                                    out_dtype="bf16", direction="dgrad")
    _, _, gtq, gts = lk.loka_quantize(dy, "e5m2", g["wdy"], want_q=False, transpose=True)
    _, _, xtq, xts = lk.loka_quantize(x, "e4m3", g["wx"], want_q=False, transpose=True)
    dw, _ = lk.loka_fp8_linear_norm(gtq, gts, xtq, xts, a_fmt="e5m2", a_gran=T.get(g["wdy"], g["wdy"]),
                                    b_gran=T.get(g["wx"], g["wx"]), out_dtype="f32", direction="wgrad")
    torch.cuda.synchronize()
    rows = torch.from_numpy(np.sort(np.random.default_rng(7).choice(M, 64, replace=False))).to(DEV)
    nrows = torch.from_numpy(np.sort(np.random.default_rng(8).choice(N, 64, replace=False))).to(DEV)

    def orc(aq, as_, af, ag, bq, bs, bf, bg, r):
        a_s = as_[r] if ag in ("row",) else as_
        return oracle.linear.linear_norm(aq[r].cpu().numpy(), a_s.cpu().numpy(), af, ag, bq.cpu().numpy(),
                                         bs.cpu().numpy(), bf, bg)

    checks = [(y, orc(xq, xs, "e4m3", g["fx"], wq, ws, "e4m3", g["fw"], rows), rows),
              (dx, orc(gq, gs, "e5m2", g["gdy"], wtq, wts, "e4m3", T.get(g["gw"], g["gw"]), rows), rows)]
    for got, ref, r in checks:
        guard = np.maximum(np.abs(ref), np.sqrt(np.mean(ref ** 2, axis=1, keepdims=True)))
        assert np.all(np.abs(f64(got[r]) - ref) <= TOL * guard + 2.0 ** -8 * np.abs(ref))
    dwo = orc(gtq, gts, "e5m2", T.get(g["wdy"], g["wdy"]), xtq, xts, "e4m3", T.get(g["wx"], g["wx"]), nrows)
    assert guarded_rel_err(f64(dw[nrows]), dwo) <= TOL
