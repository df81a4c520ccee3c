"""-m gpu: the norm fused into the CTA-pair engine (pairnorm.cu; SURVEY.md §8(a) a4+a5 at the cfg4 /
cfg5 sizes, "fuse normalization directly into the GEMM epilogue", Case 2 P:467) against
oracle/linear.py on the dequantized operands the GPU consumed.  Both tile widths (LOKA_PAIRNORM=512:
one accumulator, two N=256 MMAs per K step; =256: double-buffered accumulators), the cross-pair row
record exchange (rows wider than one tile), ragged M / N / K, every output dtype.  Tolerances as
test_gpu_linear.py (D17/D18): FP32 2e-3 guarded; BF16 + one bf16 half-ulp; FP8 codes and
row scales bit-exact vs the oracle's quantize of the GPU's own pre-cast values."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, assert_bytes_equal, assert_scales_equal, f64, guarded_rel_err, to_dev_padded

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None
TOL = 2e-3


@pytest.fixture(params=["512", "256"])
def tn(request):
    old = os.environ.get("LOKA_PAIRNORM")
    os.environ["LOKA_PAIRNORM"] = request.param
    yield int(request.param)
    if old is None:
        del os.environ["LOKA_PAIRNORM"]
    else:
        os.environ["LOKA_PAIRNORM"] = old


def _operands(M, N, K, seed, a_gran="row", b_gran="row", xdist="heavy"):
    x = synth.heavy(M, K, seed) if xdist == "heavy" else synth.gaussian(M, K, seed)
    w = synth.weight(N, K, seed + 1)
    xq, xs = lk.loka_quantize(to_dev_padded(x), "e4m3", a_gran)
    wq, ws = lk.loka_quantize(to_dev_padded(w), "e4m3", b_gran)
    return xq, xs, wq, ws


def _oracle(xq, xs, wq, ws, a_gran="row", b_gran="row", rows=None, **kw):
    a, s = xq.cpu().numpy(), xs.cpu().numpy()
    if rows is not None:
        a = a[rows]
        s = s[rows] if a_gran == "row" else s
    return oracle.linear.linear_norm(a, s, "e4m3", a_gran, wq.cpu().numpy(), ws.cpu().numpy(), "e4m3", b_gran, **kw)


def _check(y, yo, od, base=None):
    if od == "f32":
        assert guarded_rel_err(f64(y), yo) <= TOL
    else:
        b = yo if base is None else base
        guard = np.maximum(np.abs(b), np.sqrt(np.mean(b ** 2, axis=1, keepdims=True)))
        assert np.all(np.abs(f64(y) - yo) <= TOL * guard + 2.0 ** -8 * np.abs(yo))


@pytest.mark.parametrize("M,N,K", [(600, 4096, 1000), (300, 512, 256), (700, 2176, 384), (257, 256, 1152),
                                   (1030, 1280, 520)])
@pytest.mark.parametrize("norm", ["layer", "rms"])
def test_full_row_norm_f32(tn, M, N, K, norm):
    xq, xs, wq, ws = _operands(M, N, K, M + N)
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, out_dtype="f32")
    torch.cuda.synchronize()
    _check(y, _oracle(xq, xs, wq, ws, norm=norm), "f32")


@pytest.mark.parametrize("M,N,K", [(600, 4096, 512), (300, 256, 256), (513, 768, 640)])
def test_blocknorm_hardswish(tn, M, N, K):
    """NEXT-1's fused form (PAPER.md:471-473 BlockNorm-256, P:502 Hard Swish) on the pair engine."""
    xq, xs, wq, ws = _operands(M, N, K, 5)
    for act in ("none", "hardswish"):
        y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="block_rms", norm_block=256, act=act, out_dtype="f32")
        torch.cuda.synchronize()
        yo = _oracle(xq, xs, wq, ws, norm="block_rms", act=act)
        base = _oracle(xq, xs, wq, ws, norm="block_rms")
        guard = np.maximum(np.abs(base), np.sqrt(np.mean(base ** 2, axis=1, keepdims=True)))
        assert np.max(np.abs(f64(y) - yo) / guard) <= TOL, act


@pytest.mark.parametrize("a_gran,b_gran", [("tensor", "tensor"), ("row", "tensor"), ("tensor", "row")])
def test_bias_gamma_beta_bf16_and_scale_grans(tn, a_gran, b_gran):
    M, N, K = 520, 2304, 768
    xq, xs, wq, ws = _operands(M, N, K, 9, a_gran, b_gran)
    g = torch.Generator().manual_seed(2)
    bias = torch.randn(N, generator=g).to(torch.bfloat16)
    gamma = (1 + 0.2 * torch.randn(N, generator=g)).float()
    beta = (0.1 * torch.randn(N, generator=g)).float()
    for act in ("none", "hardswish"):
        y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran=a_gran, b_gran=b_gran, norm="layer", act=act,
                                       bias=bias.to(DEV), gamma=gamma.to(DEV), beta=beta.to(DEV), out_dtype="bf16")
        torch.cuda.synchronize()
        kw = dict(norm="layer", bias=bias.double().numpy(), gamma=gamma.double().numpy(), beta=beta.double().numpy())
        yo = _oracle(xq, xs, wq, ws, a_gran, b_gran, act=act, **kw)
        _check(y, yo, "bf16", base=_oracle(xq, xs, wq, ws, a_gran, b_gran, **kw))


@pytest.mark.parametrize("norm,N", [("layer", 4096), ("rms", 1024), ("block_rms", 4096), ("block_rms", 256),
                                    ("layer", 384)])
@pytest.mark.parametrize("od", ["e4m3", "e5m2"])
def test_fp8_output_bit_exact(tn, norm, N, od):
    """FP8 output with row scales (the next layer's rowwise input): the row amax spans every pair of
    the row (exchanged with the statistics); codes + scales bit-exact vs the oracle's quantize of the
    GPU's own pre-cast values, which are within 2e-3 of the oracle."""
    M, K = 520, 512
    xq, xs, wq, ws = _operands(M, N, K, 13)
    pre = torch.full((M, N), float("nan"), dtype=torch.float32, device=DEV)
    y, ys = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, out_dtype=od, precast=pre)
    torch.cuda.synchronize()
    oq, os_ = oracle.quantize.quantize(f64(pre), od, "row")
    assert_scales_equal(ys, os_)
    assert_bytes_equal(y, oq)
    assert guarded_rel_err(f64(pre), _oracle(xq, xs, wq, ws, norm=norm)) <= TOL


def test_amax_out_producer_side(tn):
    """NEXT-4 producer amax over the stored bf16 values equals max |y| of the output."""
    M, N, K = 600, 4096, 256
    xq, xs, wq, ws = _operands(M, N, K, 21)
    amax = torch.zeros(1, dtype=torch.float32, device=DEV)
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="layer", out_dtype="bf16", amax_out=amax)
    torch.cuda.synchronize()
    assert float(amax) == float(y.float().abs().max())


def test_repeated_launches_and_graph_replay(tn):
    """The exchange state (epoch-tagged flags) across many launches and CUDA-graph replays, where the
    kernel parameters are frozen: every replay must equal the eager result bit for bit."""
    M, N, K = 1100, 4096, 256
    xq, xs, wq, ws = _operands(M, N, K, 31)
    y0, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="layer", out_dtype="f32")
    for _ in range(5):
        y1, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="layer", out_dtype="f32")
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    yg = torch.empty_like(y0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="layer", out_dtype="f32", y=yg, stream=s)  # warm
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="layer", out_dtype="f32", y=yg, stream=s)
    for _ in range(7):
        yg.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(yg, y0)
    _check(y0, _oracle(xq, xs, wq, ws, norm="layer"), "f32")


@pytest.mark.parametrize("M", [32768, 262144])
def test_cfg5_shape_sampled(M):
    """The bench's launch configuration (BJ configs[4] at P=1 and P=8's per-GPU M): heavy-tailed X,
    tensorwise e4m3, K = N = 4096, LayerNorm, default route; 48 sampled rows vs the oracle (bf16 out)
    and the FP32 route on the same rows at 2e-3."""
    K = N = 4096
    x = synth.heavy(M, K, 3, device=DEV)
    w = synth.weight(N, K, 1, device=DEV)
    xq, xs = lk.loka_quantize(x, "e4m3", "tensor")
    wq, ws = lk.loka_quantize(w, "e4m3", "tensor")
    del x
    rows = np.sort(np.random.default_rng(M).choice(M, 48, replace=False))
    yb, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="tensor", b_gran="tensor", norm="layer", out_dtype="bf16")
    torch.cuda.synchronize()
    yo = _oracle(xq, xs, wq, ws, "tensor", "tensor", rows=rows, norm="layer")
    _check(yb[torch.from_numpy(rows).to(DEV)], yo, "bf16")
    del yb
    yf, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="tensor", b_gran="tensor", norm="layer", out_dtype="f32")
    torch.cuda.synchronize()
    _check(yf[torch.from_numpy(rows).to(DEV)], yo, "f32")


@pytest.mark.parametrize("M,N,K,norm", [(600, 4096, 1000, "layer"), (300, 512, 256, "rms"), (520, 768, 384, "block_rms")])
def test_bf16_path_same_epilogue(M, N, K, norm):
    """The library's own BF16 (kind::f16) path with the same fused epilogue (SURVEY.md §8(d)'s secondary
    denominator): y = norm(X W^T) on the bf16 values, against the oracle's FP64 linear + norm at 2e-3."""
    x = synth.heavy(M, K, 2)
    w = synth.weight(N, K, 3)
    y, _ = lk.loka_bf16_linear_norm(to_dev_padded(x), to_dev_padded(w), norm=norm, norm_block=256, out_dtype="f32")
    torch.cuda.synchronize()
    yo = oracle.linear.apply_norm(oracle.linear.fwd(x.double().numpy(), w.double().numpy()), norm, block=256)
    assert guarded_rel_err(f64(y), yo) <= TOL


@pytest.mark.parametrize("norm,N,act,affine", [("layer", 4096, "none", False), ("layer", 2304, "hardswish", True),
                                               ("rms", 1024, "none", True), ("block_rms", 4096, "hardswish", False),
                                               ("block_rms", 768, "none", False)])
@pytest.mark.parametrize("od", ["f32", "bf16"])
def test_norm_backward_on_pair_engine(tn, norm, N, act, affine, od):
    """NEXT-1's norm backward fused into the pair engine's epilogue:
    dh = A . B^T (the next layer's dgrad), g = dh act'(xhat gamma + beta) gamma, dz = rstd (g - mean g
    - xhat mean(g xhat)) (RMS / BlockNorm without mean g), the row sums exchanged like the forward's
    statistics; against oracle.linear.norm_backward on the same saved xhat / rstd at 2e-3."""
    M, K2 = 600, 384
    aq, as_ = lk.loka_quantize(to_dev_padded(synth.grad(M, K2, 3) * 1024), "e5m2", "row")
    bq, bs = lk.loka_quantize(to_dev_padded(synth.weight(N, K2, 4)), "e4m3", "row")
    rng = np.random.default_rng(N)
    xh = torch.tensor(rng.normal(size=(M, N)), dtype=torch.bfloat16)
    nb = N // 256
    rstd = torch.tensor(rng.uniform(0.5, 2.0, size=(M, nb) if norm == "block_rms" else (M,)), dtype=torch.float32)
    gamma = torch.tensor(1 + 0.2 * rng.normal(size=N), dtype=torch.float32) if affine else None
    beta = torch.tensor(0.3 * rng.normal(size=N), dtype=torch.float32) if (affine and norm == "layer") else None
    y, _ = lk.loka_fp8_linear_norm(aq, as_, bq, bs, a_fmt="e5m2", norm=norm, act=act, out_dtype=od,
                                   bwd_xhat=xh.to(DEV), bwd_rstd=rstd.to(DEV), direction="dgrad",
                                   gamma=None if gamma is None else gamma.to(DEV),
                                   beta=None if beta is None else beta.to(DEV))
    torch.cuda.synchronize()
    dh = oracle.linear.linear_norm(aq.cpu().numpy(), as_.cpu().numpy(), "e5m2", "row", bq.cpu().numpy(),
                                   bs.cpu().numpy(), "e4m3", "row")
    dz = oracle.linear.norm_backward(dh, xh.double().numpy(), rstd.double().numpy(), norm,
                                     gamma=None if gamma is None else gamma.double().numpy(),
                                     beta=None if beta is None else beta.double().numpy(), act=act)
    _check(y, dz, od)


@pytest.mark.parametrize("M,N,K,norm", [(600, 4096, 1000, "layer"), (1300, 768, 512, "rms"), (520, 512, 256, "block_rms")])
@pytest.mark.parametrize("given_amax", [False, True])
def test_fused_tensorwise_cast_x_recipe(M, N, K, norm, given_amax, monkeypatch):
    """x_recipe with a tensorwise bf16 A on the pair route: the cast runs inside the GEMM kernel (two
    cast warps per CTA publish per-row-block counters the TMA producers wait on).  Output bit-identical
    to loka_quantize(tensor) + the call on the codes; the codes in the workspace equal the oracle's;
    with x_amax given (the data-parallel all-reduced amax) the cast uses it."""
    import ctypes as C
    monkeypatch.setenv("LOKA_PAIRNORM", "256")  # the pair route also for the small shapes
    monkeypatch.setenv("LOKA_FUSED_CAST", "1")  # (the opt-in route)
    x = to_dev_padded(synth.heavy(M, K, 19))
    wq, ws = lk.loka_quantize(to_dev_padded(synth.weight(N, K, 20)), "e4m3", "row")
    amax = torch.tensor([float(x.float().abs().max()) * (1.5 if given_amax else 1.0)], device=DEV)
    xq, xs = lk.loka_quantize(x, "e4m3", "tensor", phase="cast", amax=amax)
    y_ref, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, a_gran="tensor", norm=norm, out_dtype="f32")
    keep = []
    args, y, _ = lk.make_linear_args(xq, xs, wq, ws, a_gran="tensor", norm=norm, out_dtype="f32", keep=keep)
    args.a = lk._tensor(x, lk.BF16, M, K, None, "tensor")
    if given_amax:
        args.x_amax = amax.data_ptr()
    nws = int(lk._lib.loka_linear_workspace_size(C.byref(args)))
    wsb = torch.empty(nws, dtype=torch.uint8, device=DEV)
    assert lk._lib.loka_fp8_linear_norm(C.byref(args), C.c_void_p(wsb.data_ptr()), nws, None) == 0
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)
    ld = (K + 15) // 16 * 16
    codes = wsb[:M * ld].view(M, ld)[:, :K]
    oq, _ = oracle.quantize.quantize(x.cpu().double().numpy(), "e4m3", "tensor", amax=np.array([float(amax)]))
    assert np.array_equal(codes.cpu().numpy(), oq)


@pytest.mark.parametrize("M,N,K,norm,od", [(4100, 4096, 1000, "layer", "f32"), (2600, 2048, 512, "rms", "f32"),
                                          (3000, 1024, 384, "layer", "e4m3")])
def test_operand_multicast_variant(M, N, K, norm, od, monkeypatch):
    """The opt-in 4-CTA-cluster variant of the pair engine (LOKA_PN_MC=1: two pairs on adjacent column
    tiles of a row block, each CTA's A half multicast to its counterpart): same
    results as the oracle, at shapes with many tiles per pair and an even tile count per row."""
    monkeypatch.setenv("LOKA_PAIRNORM", "256")
    monkeypatch.setenv("LOKA_PN_MC", "1")
    xq, xs, wq, ws = _operands(M, N, K, 29)
    if od == "f32":
        y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, out_dtype="f32")
        torch.cuda.synchronize()
        _check(y, _oracle(xq, xs, wq, ws, norm=norm), "f32")
    else:
        pre = torch.full((M, N), float("nan"), dtype=torch.float32, device=DEV)
        y, ys = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, out_dtype=od, precast=pre)
        torch.cuda.synchronize()
        oq, os_ = oracle.quantize.quantize(f64(pre), od, "row")
        assert_scales_equal(ys, os_)
        assert_bytes_equal(y, oq)
        assert guarded_rel_err(f64(pre), _oracle(xq, xs, wq, ws, norm=norm)) <= TOL


@pytest.mark.parametrize("norm,N", [("layer", 4096), ("rms", 384), ("block_rms", 768), ("layer", 256)])
@pytest.mark.parametrize("od", ["e4m3", "e5m2"])
@pytest.mark.parametrize("M", [520, 64])
def test_fp8_output_1x128_scales(norm, N, od, M):
    """FP8 output with 1x128 scales ("e4m3 + scales (ROW or BLK_1x128)") — the
    pair engine's epilogue thread owns one 128-column granule of its row; its amax comes through the
    same monotone map from the thread's y max / min.  Codes + scales bit-exact vs the oracle's 1x128
    quantize of the GPU's own pre-cast values, which are within 2e-3 of the oracle."""
    K = 512
    xq, xs, wq, ws = _operands(M, N, K, 31)
    pre = torch.full((M, N), float("nan"), dtype=torch.float32, device=DEV)
    y, ys = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, norm_block=256, out_dtype=od, precast=pre,
                                    y_gran="blk_1x128")
    torch.cuda.synchronize()
    assert tuple(ys.shape) == (M, (N + 127) // 128)
    oq, os_ = oracle.quantize.quantize(f64(pre), od, "blk_1x128")
    assert_scales_equal(ys, os_)
    assert_bytes_equal(y, oq)
    assert guarded_rel_err(f64(pre), _oracle(xq, xs, wq, ws, norm=norm)) <= TOL


def test_fp8_output_1x128_only_on_the_fused_norm_route():
    """1x128 output scales exist on the pair engine's norm epilogue; a plain (norm NONE) problem asks
    for them -> LOKA_ERR_UNSUPPORTED, not ROW scales under a 1x128 label."""
    xq, xs, wq, ws = _operands(256, 256, 256, 3)
    with pytest.raises(lk.LokaError) as ei:
        lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="none", out_dtype="e4m3", y_gran="blk_1x128")
    assert ei.value.status == lk.ERR_UNSUPPORTED


@pytest.mark.parametrize("norm,N,act,affine", [("layer", 4096, "none", False), ("layer", 1024, "hardswish", True),
                                               ("rms", 768, "none", True), ("block_rms", 512, "hardswish", False)])
@pytest.mark.parametrize("od", ["e5m2", "e4m3"])
def test_norm_backward_fp8_dz_1x128(norm, N, act, affine, od, monkeypatch):
    """NEXT-1 norm backward with FP8 dz and 1x128 scales (the blockwise recipe's next dgrad operand),
    fused: the granule amax from an extra TMEM pass that computes dz with the same operations as the
    cast pass — codes + scales bit-exact vs the oracle's 1x128 quantize of the GPU's own pre-cast dz,
    which is within 2e-3 of oracle.linear.norm_backward."""
    monkeypatch.setenv("LOKA_PAIRNORM", "256")
    M, K2 = 600, 384
    aq, as_ = lk.loka_quantize(to_dev_padded(synth.grad(M, K2, 5) * 1024), "e5m2", "row")
    bq, bs = lk.loka_quantize(to_dev_padded(synth.weight(N, K2, 6)), "e4m3", "row")
    rng = np.random.default_rng(N + 1)
    xh = torch.tensor(rng.normal(size=(M, N)), dtype=torch.bfloat16)
    nb = N // 256
    rstd = torch.tensor(rng.uniform(0.5, 2.0, size=(M, nb) if norm == "block_rms" else (M,)), dtype=torch.float32)
    gamma = torch.tensor(1 + 0.2 * rng.normal(size=N), dtype=torch.float32) if affine else None
    beta = torch.tensor(0.3 * rng.normal(size=N), dtype=torch.float32) if (affine and norm == "layer") else None
    pre = torch.full((M, N), float("nan"), dtype=torch.float32, device=DEV)
    y, ys = lk.loka_fp8_linear_norm(aq, as_, bq, bs, a_fmt="e5m2", norm=norm, act=act, out_dtype=od,
                                    bwd_xhat=xh.to(DEV), bwd_rstd=rstd.to(DEV), direction="dgrad",
                                    gamma=None if gamma is None else gamma.to(DEV),
                                    beta=None if beta is None else beta.to(DEV), precast=pre, y_gran="blk_1x128")
    torch.cuda.synchronize()
    oq, os_ = oracle.quantize.quantize(f64(pre), od, "blk_1x128")
    assert_scales_equal(ys, os_)
    assert_bytes_equal(y, oq)
    dh = oracle.linear.linear_norm(aq.cpu().numpy(), as_.cpu().numpy(), "e5m2", "row", bq.cpu().numpy(),
                                   bs.cpu().numpy(), "e4m3", "row")
    dz = oracle.linear.norm_backward(dh, xh.double().numpy(), rstd.double().numpy(), norm,
                                     gamma=None if gamma is None else gamma.double().numpy(),
                                     beta=None if beta is None else beta.double().numpy(), act=act)
    assert guarded_rel_err(f64(pre), dz) <= TOL
