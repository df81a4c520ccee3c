"""-m gpu: loka_fp8_linear_norm (a4+a5) against oracle/linear.py (FP64 on the dequantized
operands the GPU consumed).  FP32 output: guarded max relative error <= 2e-3 (D17/D18);
FP8 output: codes + row scales bit-exact vs the oracle's quantize of the GPU's own pre-cast
values, and those values within 2e-3; BF16 output: 2e-3 plus one bf16 half-ulp."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, assert_bytes_equal, assert_scales_equal, f64, guarded_rel_err, to_dev_padded

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None
TOL = 2e-3


def _operands(M, N, K, seed, xdist="gaussian", a_fmt="e4m3", b_fmt="e4m3", a_gran="row", b_gran="row"):
    x = synth.heavy(M, K, seed) if xdist == "heavy" else synth.gaussian(M, K, seed)
    w = synth.weight(N, K, seed + 1)
    xq, xs = lk.loka_quantize(to_dev_padded(x), a_fmt, a_gran)
    wq, ws = lk.loka_quantize(to_dev_padded(w), b_fmt, b_gran)
    return xq, xs, wq, ws


def _oracle(xq, xs, wq, ws, a_fmt="e4m3", b_fmt="e4m3", a_gran="row", b_gran="row", **kw):
    return oracle.linear.linear_norm(xq.cpu().numpy(), xs.cpu().numpy(), a_fmt, a_gran, wq.cpu().numpy(),
                                     ws.cpu().numpy(), b_fmt, b_gran, **kw)


def test_cfg1_rowwise_layernorm():
    """BJ configs[0]: X[256,256] x W[256,256], rowwise e4m3, LayerNorm, seed 0."""
    M = N = K = 256
    xq, xs, wq, ws = _operands(M, N, K, 0)
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="layer", out_dtype="f32")
    torch.cuda.synchronize()
    yo = _oracle(xq, xs, wq, ws, norm="layer")
    assert guarded_rel_err(f64(y), yo) <= TOL


def test_accumulation_is_fp32_exact_on_representable_operands():
    """D21: small-integer codes with power-of-two scales make every partial sum exact in FP32
    (|sum| < 2^24), so any accumulation narrower than FP32 would show as a bit difference."""
    g = torch.Generator().manual_seed(5)
    for K in (128, 1024, 4096, 16384):
        M, N = 128, 128
        xi = torch.randint(-8, 9, (M, K), generator=g).float()
        wi = torch.randint(-8, 9, (N, K), generator=g).float()
        xq, xs = lk.loka_quantize(xi.to(DEV), "e4m3", "tensor", "ue8m0")
        wq, ws = lk.loka_quantize(wi.to(DEV), "e4m3", "tensor", "ue8m0")
        y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="tensor", b_gran="tensor", out_dtype="f32")
        torch.cuda.synchronize()
        yo = _oracle(xq, xs, wq, ws, a_gran="tensor", b_gran="tensor")
        assert np.array_equal(f64(y), yo), (K, float(np.abs(f64(y) - yo).max()))


@pytest.mark.parametrize("M,N,K", [(128, 64, 128), (300, 128, 208), (256, 256, 1024), (200, 384, 512),
                                   (4096 + 64, 1024, 1024), (256, 2048, 256), (130, 200, 96)])
@pytest.mark.parametrize("norm", ["none", "layer", "rms"])
def test_linear_norm_f32(M, N, K, norm):
    xq, xs, wq, ws = _operands(M, N, K, M + N + K, xdist="heavy" if N % 3 else "gaussian")
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, out_dtype="f32")
    torch.cuda.synchronize()
    yo = _oracle(xq, xs, wq, ws, norm=norm)
    assert guarded_rel_err(f64(y), yo) <= TOL


@pytest.mark.parametrize("N,block", [(256, 256), (512, 256), (1024, 128), (768, 256), (128, 64)])
def test_blocknorm(N, block):
    M, K = 384, 512
    xq, xs, wq, ws = _operands(M, N, K, 7)
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="block_rms", norm_block=block, out_dtype="f32")
    torch.cuda.synchronize()
    yo = _oracle(xq, xs, wq, ws, norm="block_rms", block=block)
    assert guarded_rel_err(f64(y), yo) <= TOL


def test_blocknorm_indivisible_is_shape_error():
    xq, xs, wq, ws = _operands(128, 300, 128, 1)
    with pytest.raises(lk.LokaError) as e:
        lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="block_rms", norm_block=256)
    assert e.value.status == lk.ERR_SHAPE


@pytest.mark.parametrize("norm", ["layer", "rms"])
def test_bias_gamma_beta_bf16_out(norm):
    M, N, K = 256, 512, 256
    xq, xs, wq, ws = _operands(M, N, K, 3)
    g = torch.Generator().manual_seed(1)
    bias = torch.randn(N, generator=g).to(torch.bfloat16)
    gamma = (1 + 0.1 * torch.randn(N, generator=g)).float()
    beta = (0.1 * torch.randn(N, generator=g)).float() if norm == "layer" else None
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, bias=bias.to(DEV), gamma=gamma.to(DEV),
                                   beta=None if beta is None else beta.to(DEV), out_dtype="bf16")
    torch.cuda.synchronize()
    yo = _oracle(xq, xs, wq, ws, norm=norm, bias=bias.double().numpy(), gamma=gamma.double().numpy(),
                 beta=None if beta is None else beta.double().numpy())
    yg = f64(y)
    rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
    assert np.all(np.abs(yg - yo) <= TOL * np.maximum(np.abs(yo), rms) + 2.0 ** -8 * np.abs(yo))


@pytest.mark.parametrize("norm,affine", [("layer", False), ("rms", False), ("none", False), ("block_rms", False),
                                         ("layer", True)])
@pytest.mark.parametrize("N", [256, 1024])
def test_fp8_output_bit_exact(norm, affine, N):
    """The epilogue's FP8 output (next layer's rowwise input): codes + row scales equal the
    oracle's rowwise quantize of the GPU's own pre-cast FP32 values."""
    M, K = 256, 512
    xq, xs, wq, ws = _operands(M, N, K, 11, xdist="heavy")
    pre = torch.empty(M, N, dtype=torch.float32, device=DEV)
    gamma = torch.linspace(0.5, 1.5, N, device=DEV) if affine else None
    y, ys = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, out_dtype="e4m3", precast=pre, gamma=gamma)
    torch.cuda.synchronize()
    oq, os_ = oracle.quantize.quantize(f64(pre), "e4m3", "row")
    assert_scales_equal(ys, os_)
    assert_bytes_equal(y, oq)
    yo = _oracle(xq, xs, wq, ws, norm=norm, gamma=None if gamma is None else f64(gamma))
    assert guarded_rel_err(f64(pre), yo) <= TOL


def test_tensorwise_e5m2_operands():
    M, N, K = 256, 256, 384
    xq, xs, wq, ws = _operands(M, N, K, 4, a_fmt="e5m2", b_fmt="e4m3", a_gran="tensor", b_gran="tensor")
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_fmt="e5m2", a_gran="tensor", b_gran="tensor", norm="rms")
    torch.cuda.synchronize()
    yo = _oracle(xq, xs, wq, ws, a_fmt="e5m2", a_gran="tensor", b_gran="tensor", norm="rms")
    assert guarded_rel_err(f64(y), yo) <= TOL


def test_cfg2_stack_full_size():
    """BJ configs[1] in the bench's launch configuration: M=4096, 8 layers, rowwise e4m3, LayerNorm,
    FP8 hand-off between layers; every layer checked on 64 sampled rows against the oracle run on
    the GPU's own layer inputs."""
    dims = synth.CFG2_DIMS
    M = 4096
    x = synth.gaussian(M, dims[0], 0, device=DEV)
    hq, hs = lk.loka_quantize(x, "e4m3", "row")
    rows = torch.randperm(M, generator=torch.Generator().manual_seed(1))[:64].sort().values.to(DEV)
    for l in range(8):
        K, N = dims[l], dims[l + 1]
        w = synth.weight(N, K, 100 + l, device=DEV)
        wq, ws = lk.loka_quantize(w, "e4m3", "row")
        last = l == 7
        pre = torch.empty(M, N, dtype=torch.float32, device=DEV)
        y, ys = lk.loka_fp8_linear_norm(hq, hs, wq, ws, norm="layer", out_dtype="bf16" if last else "e4m3",
                                        precast=pre)
        torch.cuda.synchronize()
        yo = oracle.linear.linear_norm(hq[rows].cpu().numpy(), hs[rows].cpu().numpy(), "e4m3", "row",
                                       wq.cpu().numpy(), ws.cpu().numpy(), "e4m3", "row", norm="layer")
        assert guarded_rel_err(f64(pre[rows]), yo) <= TOL, l
        if not last:
            oq, os_ = oracle.quantize.quantize(f64(pre[rows]), "e4m3", "row")
            assert_bytes_equal(y[rows], oq)
            assert_scales_equal(ys[rows], os_)
            hq, hs = y, ys


@pytest.mark.parametrize("norm,N", [("block_rms", 1024), ("block_rms", 256), ("layer", 512), ("rms", 2048),
                                    ("none", 384)])
def test_hardswish_after_norm_f32(norm, N):
    """NEXT-1: Hard Swish fused after the norm in the same epilogue."""
    M, K = 300, 512
    xq, xs, wq, ws = _operands(M, N, K, 31, xdist="heavy")
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, act="hardswish", out_dtype="f32")
    torch.cuda.synchronize()
    yo = _oracle(xq, xs, wq, ws, norm=norm, act="hardswish")
    # guard from the pre-activation scale: h-swish shrinks values near zero but its slope is <= 1.5
    pre = _oracle(xq, xs, wq, ws, norm=norm)
    rms = np.sqrt(np.mean(pre ** 2, axis=1, keepdims=True))
    assert np.max(np.abs(f64(y) - yo) / np.maximum(np.abs(pre), rms)) <= 1.5 * TOL


@pytest.mark.parametrize("norm,N", [("block_rms", 1024), ("layer", 256)])
def test_hardswish_fp8_output_bit_exact(norm, N):
    """The row amax of an activated row is reduced over the activated values (h-swish is not
    monotone): codes + scales equal the oracle's rowwise quantize of the GPU's pre-cast values."""
    M, K = 256, 384
    xq, xs, wq, ws = _operands(M, N, K, 33, xdist="heavy")
    pre = torch.empty(M, N, dtype=torch.float32, device=DEV)
    y, ys = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, act="hardswish", out_dtype="e4m3", precast=pre)
    torch.cuda.synchronize()
    oq, os_ = oracle.quantize.quantize(f64(pre), "e4m3", "row")
    assert_scales_equal(ys, os_)
    assert_bytes_equal(y, oq)
    yo = _oracle(xq, xs, wq, ws, norm=norm, act="hardswish")
    rms = np.sqrt(np.mean(_oracle(xq, xs, wq, ws, norm=norm) ** 2, axis=1, keepdims=True))
    assert np.max(np.abs(f64(pre) - yo) / np.maximum(np.abs(yo), rms)) <= 1.5 * TOL


def test_hardswish_with_gamma_beta_bf16():
    M, N, K = 256, 512, 256
    xq, xs, wq, ws = _operands(M, N, K, 35)
    g = torch.Generator().manual_seed(2)
    gamma = (1 + 0.2 * torch.randn(N, generator=g)).float()
    beta = (0.5 * torch.randn(N, generator=g)).float()
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="layer", gamma=gamma.to(DEV), beta=beta.to(DEV),
                                   act="hardswish", out_dtype="bf16")
    torch.cuda.synchronize()
    yo = _oracle(xq, xs, wq, ws, norm="layer", gamma=gamma.double().numpy(), beta=beta.double().numpy(),
                 act="hardswish")
    pre = _oracle(xq, xs, wq, ws, norm="layer", gamma=gamma.double().numpy(), beta=beta.double().numpy())
    rms = np.sqrt(np.mean(pre ** 2, axis=1, keepdims=True))
    assert np.all(np.abs(f64(y) - yo) <= 1.5 * TOL * np.maximum(np.abs(pre), rms) + 2.0 ** -8 * np.abs(yo))


@pytest.mark.parametrize("N,norm,od", [(4096, "layer", "f32"), (3000, "rms", "f32"), (4096, "layer", "e4m3"),
                                       (2560, "none", "e4m3")])
def test_full_row_norm_wide_rows_16_cta_cluster(N, norm, od):
    """BJ configs[4] (cfg5) layer: LayerNorm over N = 4096 needs a 16-CTA (non-portable) cluster."""
    M, K = 300, 384
    xq, xs, wq, ws = _operands(M, N, K, 41, xdist="heavy")
    if od == "f32":
        y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, out_dtype="f32")
        torch.cuda.synchronize()
        assert guarded_rel_err(f64(y), _oracle(xq, xs, wq, ws, norm=norm)) <= TOL
    else:
        pre = torch.empty(M, N, dtype=torch.float32, device=DEV)
        y, ys = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, out_dtype="e4m3", precast=pre)
        torch.cuda.synchronize()
        oq, os_ = oracle.quantize.quantize(f64(pre), "e4m3", "row")
        assert_scales_equal(ys, os_)
        assert_bytes_equal(y, oq)
        assert guarded_rel_err(f64(pre), _oracle(xq, xs, wq, ws, norm=norm)) <= TOL


@pytest.mark.parametrize("norm,od,act,affine", [("layer", "f32", "none", False), ("rms", "bf16", "hardswish", True),
                                                ("layer", "e4m3", "hardswish", False)])
def test_wide_rows_unfused_pair_plus_rownorm(norm, od, act, affine):
    """N > 2048 with enough rows: CTA-pair GEMM (FP32, workspace) + the row-wise norm pass
    (rownorm.cu).  Sampled rows vs the oracle; FP8 codes bit-exact vs the GPU's pre-cast values."""
    M, N, K = 1300, 4096, 512
    xq, xs, wq, ws = _operands(M, N, K, 43, xdist="heavy")
    g = torch.Generator().manual_seed(3)
    gamma = (1 + 0.2 * torch.randn(N, generator=g)).float() if affine else None
    pre = torch.empty(M, N, dtype=torch.float32, device=DEV)
    y, ys = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, act=act, out_dtype=od, precast=pre,
                                   gamma=None if gamma is None else gamma.to(DEV))
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(5).choice(M, 48, replace=False))
    kw = dict(norm=norm, act=act, gamma=None if gamma is None else gamma.double().numpy())
    yo = oracle.linear.linear_norm(xq.cpu().numpy()[rows], xs.cpu().numpy()[rows], "e4m3", "row", wq.cpu().numpy(),
                                   ws.cpu().numpy(), "e4m3", "row", **kw)
    kw0 = dict(kw, act="none")
    base = oracle.linear.linear_norm(xq.cpu().numpy()[rows], xs.cpu().numpy()[rows], "e4m3", "row",
                                     wq.cpu().numpy(), ws.cpu().numpy(), "e4m3", "row", **kw0)
    rms = np.sqrt(np.mean(base ** 2, axis=1, keepdims=True))
    guard = np.maximum(np.abs(base), rms)
    # the guard is taken on the pre-activation values; h-swish's slope (<= 1.5 on [-3, 3]) may scale
    # an error by up to 1.5 against it, so only the activated cases get the 1.5x
    tol = TOL if act == "none" else 1.5 * TOL
    assert np.max(np.abs(f64(pre)[rows] - yo) / guard) <= tol
    if od == "e4m3":
        oq, os_ = oracle.quantize.quantize(f64(pre), "e4m3", "row")
        assert_scales_equal(ys, os_)
        assert_bytes_equal(y, oq)
    elif od == "bf16":
        assert np.all(np.abs(f64(y)[rows] - yo) <= tol * guard + 2.0 ** -8 * np.abs(yo))
    else:
        assert np.max(np.abs(f64(y)[rows] - yo) / guard) <= tol


@pytest.mark.parametrize("gran,M,N,K", [("row", 300, 512, 384), ("tensor", 4864, 4096, 512), ("blk_1x128", 256, 256, 640)])
def test_x_recipe_quantizes_inside_the_call(gran, M, N, K):
    """loka_fp8_linear_norm with an unquantized bf16 X quantizes it internally with
    x's granularity (e4m3) into the workspace and runs the FP8 problem: bit-identical to loka_quantize
    followed by the call on the codes (both the single-CTA and the CTA-pair routes)."""
    import ctypes as C
    x = to_dev_padded(synth.heavy(M, K, 17))
    b_gran = "blk_128x128" if gran == "blk_1x128" else "row"
    sf = "ue8m0" if gran == "blk_1x128" else "f32"
    wq, ws = lk.loka_quantize(to_dev_padded(synth.weight(N, K, 18)), "e4m3", b_gran, sf)
    xq, xs = lk.loka_quantize(x, "e4m3", gran, sf)
    y_ref, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran=gran, b_gran=b_gran, a_scale_fmt=sf, b_scale_fmt=sf,
                                       norm="layer" if gran != "blk_1x128" else "none", out_dtype="f32")
    keep = []
    args, y, _ = lk.make_linear_args(xq, xs, wq, ws, a_gran=gran, b_gran=b_gran, a_scale_fmt=sf, b_scale_fmt=sf,
                                     norm="layer" if gran != "blk_1x128" else "none", out_dtype="f32", keep=keep)
    args.a = lk._tensor(x, lk.BF16, M, K, None, gran, sf)
    nws = int(lk._lib.loka_linear_workspace_size(C.byref(args)))
    wsb = torch.empty(nws, dtype=torch.uint8, device=DEV)
    assert lk._lib.loka_fp8_linear_norm(C.byref(args), C.c_void_p(wsb.data_ptr()), nws, None) == 0
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)
