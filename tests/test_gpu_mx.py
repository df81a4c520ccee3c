"""-m gpu: the native block-scaled GEMM (SURVEY.md §8(a) a4 "UE8M0: kind::mxf8f6f4.block_scale
with scales in TMEM"; D7/D23).  Blockwise operands with UE8M0 scales (A 1x128, B 128x128
or 1x128) are multiplied by the tensor core with the scales applied per 32-wide K block, so the
accumulator is the dequantized product and the whole a5 epilogue applies.  Compared with
oracle/linear.py on the same codes and scales (FP64 on the dequantized operands)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, assert_bytes_equal, assert_scales_equal, f64, guarded_rel_err, to_dev_padded

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None
TOL = 2e-3


def _operands(M, N, K, seed, xdist="heavy", a_fmt="e4m3", b_gran="blk_128x128"):
    x = synth.heavy(M, K, seed) if xdist == "heavy" else synth.gaussian(M, K, seed)
    w = synth.weight(N, K, seed + 1)
    xq, xs = lk.loka_quantize(to_dev_padded(x), a_fmt, "blk_1x128", "ue8m0")
    wq, ws = lk.loka_quantize(to_dev_padded(w), "e4m3", b_gran, "ue8m0")
    return xq, xs, wq, ws


def _mx(xq, xs, wq, ws, a_fmt="e4m3", b_gran="blk_128x128", **kw):
    return lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_fmt=a_fmt, a_gran="blk_1x128", b_gran=b_gran,
                                   a_scale_fmt="ue8m0", b_scale_fmt="ue8m0", **kw)


def _oracle(xq, xs, wq, ws, a_fmt="e4m3", b_gran="blk_128x128", **kw):
    return oracle.linear.linear_norm(xq.cpu().numpy(), xs.cpu().numpy(), a_fmt, "blk_1x128", wq.cpu().numpy(),
                                     ws.cpu().numpy(), "e4m3", b_gran, **kw)


def test_block_scales_applied_exactly():
    """Integer-valued blocks times per-block powers of two: every product and partial sum is exact
    in FP32, so the result must equal the oracle bit for bit.  A scale applied to the wrong row,
    column or K block (a wrong scale-atom layout or sf_id) changes the value."""
    g = torch.Generator().manual_seed(3)
    M, N, K = 256, 256, 512
    xi = torch.randint(-8, 9, (M, K), generator=g).float()
    wi = torch.randint(-8, 9, (N, K), generator=g).float()
    ea = torch.randint(-1, 2, (M, K // 128), generator=g).float()
    eb = torch.randint(-1, 2, (N // 128, K // 128), generator=g).float()
    xv = xi * torch.repeat_interleave(2.0 ** ea, 128, dim=1)
    wv = wi * torch.repeat_interleave(torch.repeat_interleave(2.0 ** eb, 128, dim=0), 128, dim=1)
    xq, xs = lk.loka_quantize(xv.to(DEV), "e4m3", "blk_1x128", "ue8m0")
    wq, ws = lk.loka_quantize(wv.to(DEV), "e4m3", "blk_128x128", "ue8m0")
    y, _ = _mx(xq, xs, wq, ws, out_dtype="f32")
    torch.cuda.synchronize()
    yo = _oracle(xq, xs, wq, ws)
    assert np.array_equal(f64(y), yo), float(np.abs(f64(y) - yo).max())
    assert np.array_equal(yo, xv.double().numpy() @ wv.double().numpy().T)


@pytest.mark.parametrize("M,N,K", [(128, 128, 128), (300, 256, 640), (200, 384, 1000), (512, 1024, 512),
                                   (4096, 256, 2048), (130, 2048, 256)])
@pytest.mark.parametrize("norm", ["none", "layer", "rms"])
def test_mx_linear_norm_f32(M, N, K, norm):
    xq, xs, wq, ws = _operands(M, N, K, M + N + K)
    y, _ = _mx(xq, xs, wq, ws, norm=norm, out_dtype="f32")
    torch.cuda.synchronize()
    assert guarded_rel_err(f64(y), _oracle(xq, xs, wq, ws, norm=norm)) <= TOL


@pytest.mark.parametrize("b_gran", ["blk_128x128", "blk_1x128"])
@pytest.mark.parametrize("a_fmt", ["e4m3", "e5m2"])
def test_mx_granularities_and_formats(b_gran, a_fmt):
    M, N, K = 384, 512, 768
    xq, xs, wq, ws = _operands(M, N, K, 9, a_fmt=a_fmt, b_gran=b_gran)
    y, _ = _mx(xq, xs, wq, ws, a_fmt=a_fmt, b_gran=b_gran, out_dtype="f32")
    torch.cuda.synchronize()
    assert guarded_rel_err(f64(y), _oracle(xq, xs, wq, ws, a_fmt=a_fmt, b_gran=b_gran)) <= TOL


def test_mx_blocknorm_bias_bf16():
    M, N, K = 256, 1024, 384
    xq, xs, wq, ws = _operands(M, N, K, 21)
    bias = torch.randn(N, generator=torch.Generator().manual_seed(2))
    y, _ = _mx(xq, xs, wq, ws, norm="block_rms", norm_block=256, bias=bias.to(DEV), out_dtype="bf16")
    torch.cuda.synchronize()
    yo = _oracle(xq, xs, wq, ws, norm="block_rms", block=256, bias=bias.double().numpy())
    rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
    assert np.all(np.abs(f64(y) - yo) <= TOL * np.maximum(np.abs(yo), rms) + 2.0 ** -8 * np.abs(yo))


@pytest.mark.parametrize("norm", ["layer", "none"])
def test_mx_fp8_output_bit_exact(norm):
    M, N, K = 256, 1024, 512
    xq, xs, wq, ws = _operands(M, N, K, 13)
    pre = torch.empty(M, N, dtype=torch.float32, device=DEV)
    y, ys = _mx(xq, xs, wq, ws, norm=norm, out_dtype="e4m3", precast=pre)
    torch.cuda.synchronize()
    oq, os_ = oracle.quantize.quantize(f64(pre), "e4m3", "row")
    assert_scales_equal(ys, os_)
    assert_bytes_equal(y, oq)
    assert guarded_rel_err(f64(pre), _oracle(xq, xs, wq, ws, norm=norm)) <= TOL


def test_mx_training_directions():
    """fwd / dgrad / wgrad of the blockwise UE8M0 recipe (BJ configs[3] recipe, small shape)."""
    M, N, K = 384, 256, 640
    x, w, dy = synth.heavy(M, K, 1), synth.weight(N, K, 2), synth.grad(M, N, 3)
    xd, wd, dyd = to_dev_padded(x), to_dev_padded(w), to_dev_padded(dy)
    xq, xs = lk.loka_quantize(xd, "e4m3", "blk_1x128", "ue8m0")
    wq, ws = lk.loka_quantize(wd, "e4m3", "blk_128x128", "ue8m0")
    y, _ = _mx(xq, xs, wq, ws, out_dtype="f32")
    gq, gs = lk.loka_quantize(dyd, "e5m2", "blk_1x128", "ue8m0")
    _, _, wtq, wts = lk.loka_quantize(wd, "e4m3", "blk_128x128", "ue8m0", want_q=False, transpose=True)
    dx, _ = _mx(gq, gs, wtq, wts, a_fmt="e5m2", out_dtype="f32", direction="dgrad")
    _, _, gtq, gts = lk.loka_quantize(dyd, "e5m2", "blk_128x1", "ue8m0", want_q=False, transpose=True)
    _, _, xtq, xts = lk.loka_quantize(xd, "e4m3", "blk_128x1", "ue8m0", want_q=False, transpose=True)
    dw, _ = _mx(gtq, gts, xtq, xts, a_fmt="e5m2", b_gran="blk_1x128", out_dtype="f32", direction="wgrad")
    torch.cuda.synchronize()

    def deq(t, fmt, gran):
        q, s = oracle.quantize.quantize(t.double().numpy(), fmt, gran, "ue8m0")
        return oracle.quantize.dequantize(q, s, fmt, gran)
    assert guarded_rel_err(f64(y), oracle.linear.fwd(deq(x, "e4m3", "blk_1x128"), deq(w, "e4m3", "blk_128x128"))) <= TOL
    assert guarded_rel_err(f64(dx), oracle.linear.dgrad(deq(dy, "e5m2", "blk_1x128"),
                                                        deq(w, "e4m3", "blk_128x128"))) <= TOL
    assert guarded_rel_err(f64(dw), oracle.linear.wgrad(deq(dy, "e5m2", "blk_128x1"),
                                                        deq(x, "e4m3", "blk_128x1"))) <= TOL


def test_mx_workspace_required_and_grouped():
    M, N, K = 256, 256, 256
    xq, xs, wq, ws = _operands(M, N, K, 5)
    args, y, _ = lk.make_linear_args(xq, xs, wq, ws, a_gran="blk_1x128", b_gran="blk_128x128", a_scale_fmt="ue8m0",
                                     b_scale_fmt="ue8m0", out_dtype="f32")
    need = lk.linear_workspace(args)
    assert need == 2 * 2 * 512 + 2 * 2 * 512  # A: 2 row blocks x 2 k blocks; B: 1 pair of 128-row atoms x 2
    import ctypes as C
    assert lk._lib.loka_fp8_linear_norm(C.byref(args), None, 0, None) == lk.ERR_WORKSPACE
    # grouped: two MX problems + one rowwise, one call
    xr, xrs = lk.loka_quantize(to_dev_padded(synth.gaussian(M, K, 8)), "e4m3", "row")
    wr, wrs = lk.loka_quantize(to_dev_padded(synth.weight(N, K, 9)), "e4m3", "row")
    a1, y1, _ = lk.make_linear_args(xq, xs, wq, ws, a_gran="blk_1x128", b_gran="blk_128x128", a_scale_fmt="ue8m0",
                                    b_scale_fmt="ue8m0", out_dtype="bf16")
    a2, y2, _ = lk.make_linear_args(xq, xs, wq, ws, a_gran="blk_1x128", b_gran="blk_128x128", a_scale_fmt="ue8m0",
                                    b_scale_fmt="ue8m0", norm="layer", out_dtype="f32")
    a3, y3, _ = lk.make_linear_args(xr, xrs, wr, wrs, out_dtype="bf16")
    lk.loka_grouped_fp8_linear([a1, a2, a3])
    torch.cuda.synchronize()
    yo = _oracle(xq, xs, wq, ws)
    rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
    assert np.all(np.abs(f64(y1) - yo) <= TOL * np.maximum(np.abs(yo), rms) + 2.0 ** -8 * np.abs(yo))
    assert guarded_rel_err(f64(y2), _oracle(xq, xs, wq, ws, norm="layer")) <= TOL
    yr = oracle.linear.linear_norm(xr.cpu().numpy(), xrs.cpu().numpy(), "e4m3", "row", wr.cpu().numpy(),
                                   wrs.cpu().numpy(), "e4m3", "row")
    rms = np.sqrt(np.mean(yr ** 2, axis=1, keepdims=True))
    assert np.all(np.abs(f64(y3) - yr) <= TOL * np.maximum(np.abs(yr), rms) + 2.0 ** -8 * np.abs(yr))


def test_mx_pair_engine_exact_block_scales():
    """>= 74 tiles of 256 x 256: the CTA-pair block-scaled kernel (cta_group::2, scale atoms copied
    to both CTAs' TMEM).  Integer blocks x per-block powers of two -> exact in FP32; a ragged last
    row tile (rows past M) and several tiles per pair."""
    g = torch.Generator().manual_seed(11)
    M, N, K = 2176, 2560, 384
    xi = torch.randint(-8, 9, (M, K), generator=g).float()
    wi = torch.randint(-8, 9, (N, K), generator=g).float()
    ea = torch.randint(-1, 2, (M, K // 128), generator=g).float()
    eb = torch.randint(-1, 2, (N // 128, K // 128), generator=g).float()
    xv = xi * torch.repeat_interleave(2.0 ** ea, 128, dim=1)
    wv = wi * torch.repeat_interleave(torch.repeat_interleave(2.0 ** eb, 128, dim=0), 128, dim=1)
    xq, xs = lk.loka_quantize(xv.to(DEV), "e4m3", "blk_1x128", "ue8m0")
    wq, ws = lk.loka_quantize(wv.to(DEV), "e4m3", "blk_128x128", "ue8m0")
    y, _ = _mx(xq, xs, wq, ws, out_dtype="f32")
    torch.cuda.synchronize()
    assert np.array_equal(f64(y), xv.double().numpy() @ wv.double().numpy().T)


@pytest.mark.parametrize("b_gran,a_fmt,od", [("blk_128x128", "e4m3", "bf16"), ("blk_1x128", "e5m2", "f32")])
def test_mx_pair_engine_vs_oracle(b_gran, a_fmt, od):
    M, N, K = 2048, 2816, 1000
    xq, xs, wq, ws = _operands(M, N, K, 17, a_fmt=a_fmt, b_gran=b_gran)
    bias = torch.randn(N, generator=torch.Generator().manual_seed(4))
    y, _ = _mx(xq, xs, wq, ws, a_fmt=a_fmt, b_gran=b_gran, bias=bias.to(DEV), out_dtype=od)
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(2).choice(M, 64, replace=False))
    yo = oracle.linear.linear_norm(xq.cpu().numpy()[rows], xs.cpu().numpy()[rows], a_fmt, "blk_1x128",
                                   wq.cpu().numpy(), ws.cpu().numpy(), "e4m3", b_gran, bias=bias.double().numpy())
    yg = f64(y)[rows]
    rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
    extra = 2.0 ** -8 * np.abs(yo) if od == "bf16" else 0.0
    assert np.all(np.abs(yg - yo) <= TOL * np.maximum(np.abs(yo), rms) + extra)


# ---- MXFP8 (NEXT-4): 1x32 blocks, the block-scaled MMA's native granule ----------------------
def _exact_1x32(M, N, K, seed, b_gran):
    """Integer codes times per-32-block powers of two (A 1x32, B per b_gran): every product and
    partial sum exact in FP32, so any scale applied to the wrong row / column / 32-wide K block (a
    wrong byte in the scale atoms or a wrong sf_id) changes the result."""
    g = torch.Generator().manual_seed(seed)
    xi = torch.randint(-8, 9, (M, K), generator=g).float()
    wi = torch.randint(-8, 9, (N, K), generator=g).float()
    ea = torch.randint(-2, 3, (M, K // 32), generator=g).float()
    xv = xi * torch.repeat_interleave(2.0 ** ea, 32, dim=1)
    if b_gran == "blk_1x32":
        eb = torch.randint(-2, 3, (N, K // 32), generator=g).float()
        wv = wi * torch.repeat_interleave(2.0 ** eb, 32, dim=1)
    else:
        eb = torch.randint(-1, 2, (N // 128, K // 128), generator=g).float()
        wv = wi * torch.repeat_interleave(torch.repeat_interleave(2.0 ** eb, 128, dim=0), 128, dim=1)
    xq, xs = lk.loka_quantize(xv.to(DEV), "e4m3", "blk_1x32", "ue8m0")
    wq, ws = lk.loka_quantize(wv.to(DEV), "e4m3", b_gran, "ue8m0")
    return xv, wv, xq, xs, wq, ws


@pytest.mark.parametrize("M,N,K,b_gran", [(256, 256, 512, "blk_1x32"), (300, 384, 640, "blk_128x128"),
                                          (2176, 2560, 384, "blk_1x32")])
def test_mxfp8_1x32_exact(M, N, K, b_gran):
    xv, wv, xq, xs, wq, ws = _exact_1x32(M, N, K, M + K, b_gran)
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="blk_1x32", b_gran=b_gran, a_scale_fmt="ue8m0",
                                   b_scale_fmt="ue8m0", out_dtype="f32")
    torch.cuda.synchronize()
    assert np.array_equal(f64(y), xv.double().numpy() @ wv.double().numpy().T)


@pytest.mark.parametrize("M,N,K,norm", [(200, 384, 1000, "layer"), (512, 1024, 512, "none"),
                                        (2048, 2816, 1000, "none")])
def test_mxfp8_1x32_vs_oracle(M, N, K, norm):
    x, w = synth.heavy(M, K, 31), synth.weight(N, K, 32)
    xq, xs = lk.loka_quantize(to_dev_padded(x), "e4m3", "blk_1x32", "ue8m0")
    wq, ws = lk.loka_quantize(to_dev_padded(w), "e4m3", "blk_1x32", "ue8m0")
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="blk_1x32", b_gran="blk_1x32", a_scale_fmt="ue8m0",
                                   b_scale_fmt="ue8m0", norm=norm, out_dtype="f32")
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(3).choice(M, min(M, 64), replace=False))
    yo = oracle.linear.linear_norm(xq.cpu().numpy()[rows], xs.cpu().numpy()[rows], "e4m3", "blk_1x32",
                                   wq.cpu().numpy(), ws.cpu().numpy(), "e4m3", "blk_1x32", norm=norm)
    assert guarded_rel_err(f64(y)[rows], yo) <= TOL
