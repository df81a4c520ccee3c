"""-m gpu: loka_grouped_fp8_linear (a6) against oracle/linear.py: the cfg3 DHEN-style ensemble
(64 heterogeneous GEMMs over 8 shared inputs, one persistent launch per <= 64 problems) and a
mixed list that also routes norm / FP8-output problems through their own fused launches."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, f64, to_dev_padded

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None
TOL = 2e-3


def _check_bf16(y, yo):
    yg = f64(y)
    rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
    bound = TOL * np.maximum(np.abs(yo), rms) + 2.0 ** -8 * np.abs(yo)
    bad = np.abs(yg - yo) > bound
    assert not bad.any(), (int(bad.sum()), float(np.abs(yg - yo).max()))


def _quant(x):
    return lk.loka_quantize(to_dev_padded(x) if x.device.type == "cpu" else x, "e4m3", "row")


def test_cfg3_ensemble_64_gemms_sampled():
    S = synth.CFG3_DIMS
    M = 2048
    xs = [(synth.heavy(M, k, i, device=DEV) if i % 2 else synth.gaussian(M, k, i, device=DEV)) for i, k in enumerate(S)]
    xq = [_quant(x) for x in xs]
    args, keep, outs = [], [], []
    for i, k in enumerate(S):
        for j, n in enumerate(S):
            wq, ws = _quant(synth.weight(n, k, 1000 + 8 * i + j, device=DEV))
            a, y, _ = lk.make_linear_args(xq[i][0], xq[i][1], wq, ws, out_dtype="bf16", keep=keep)
            args.append(a)
            outs.append((i, wq, ws, y))
    lk.loka_grouped_fp8_linear(args)
    torch.cuda.synchronize()
    rows = torch.randperm(M, generator=torch.Generator().manual_seed(3))[:48].sort().values.to(DEV)
    for i, wq, ws, y in outs:
        q, s = xq[i]
        yo = oracle.linear.linear_norm(q[rows].cpu().numpy(), s[rows].cpu().numpy(), "e4m3", "row",
                                       wq.cpu().numpy(), ws.cpu().numpy(), "e4m3", "row")
        _check_bf16(y[rows], yo)


def test_grouped_mixed_epilogues_and_ragged_shapes():
    """Ragged M/N/K, bias, tensorwise scales, plus problems that need their own fused launch
    (LayerNorm, FP8 output) in the same call."""
    specs = [(300, 200, 208, "none", "bf16", True), (130, 64, 96, "none", "bf16", False),
             (256, 512, 384, "layer", "f32", False), (128, 256, 128, "none", "e4m3", False),
             (1000, 384, 1024, "none", "bf16", True), (64, 136, 16, "none", "bf16", False)]
    args, keep, res = [], [], []
    for t, (M, N, K, norm, od, bias) in enumerate(specs):
        x, w = synth.heavy(M, K, t), synth.weight(N, K, 50 + t)
        gran = "tensor" if t == 1 else "row"
        xq, xs = lk.loka_quantize(to_dev_padded(x), "e4m3", gran)
        wq, ws = lk.loka_quantize(to_dev_padded(w), "e4m3", gran)
        b = torch.randn(N, generator=torch.Generator().manual_seed(t)).to(torch.bfloat16).to(DEV) if bias else None
        a, y, ys = lk.make_linear_args(xq, xs, wq, ws, a_gran=gran, b_gran=gran, norm=norm, out_dtype=od, bias=b,
                                       keep=keep)
        args.append(a)
        res.append((xq, xs, wq, ws, gran, norm, od, b, y, ys))
    lk.loka_grouped_fp8_linear(args)
    torch.cuda.synchronize()
    for xq, xs, wq, ws, gran, norm, od, b, y, ys in res:
        yo = oracle.linear.linear_norm(xq.cpu().numpy(), xs.cpu().numpy(), "e4m3", gran, wq.cpu().numpy(),
                                       ws.cpu().numpy(), "e4m3", gran, norm=norm,
                                       bias=None if b is None else f64(b))
        if od == "bf16":
            _check_bf16(y, yo)
        elif od == "f32":
            rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
            assert np.max(np.abs(f64(y) - yo) / np.maximum(np.abs(yo), rms)) <= TOL
        else:
            deq = oracle.quantize.dequantize(y.cpu().numpy(), ys.cpu().numpy(), "e4m3", "row")
            rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
            assert np.all(np.abs(deq - yo) <= 2.0 ** -4 * np.abs(yo) + TOL * np.maximum(np.abs(yo), rms) + 1e-30)


@pytest.mark.parametrize("od", ["f32", "bf16"])
def test_pair_kernel_ragged_formats_and_many_tiles(od):
    """CTA-pair (256 x 256 tile) grouped engine: ragged M/N/K, e5m2 x e4m3, more tiles than SM
    pairs (persistent walk, both accumulator buffers reused), bias, f32 and bf16 outputs."""
    specs = [(700, 520, 1000, "e5m2", True), (2304, 2048, 256, "e4m3", False), (256, 256, 16, "e4m3", True),
             (130, 1096, 4096, "e4m3", False)]
    args, keep, res = [], [], []
    for t, (M, N, K, af, bias) in enumerate(specs):
        x, w = synth.heavy(M, K, 60 + t), synth.weight(N, K, 70 + t)
        xq, xs = lk.loka_quantize(to_dev_padded(x), af, "row")
        wq, ws = lk.loka_quantize(to_dev_padded(w), "e4m3", "row")
        b = torch.randn(N, generator=torch.Generator().manual_seed(t)).to(DEV) if bias else None
        a, y, _ = lk.make_linear_args(xq, xs, wq, ws, a_fmt=af, out_dtype=od, bias=b, keep=keep)
        args.append(a)
        res.append((xq, xs, wq, ws, af, b, y))
    lk.loka_grouped_fp8_linear(args)
    torch.cuda.synchronize()
    for xq, xs, wq, ws, af, b, y in res:
        M = xq.shape[0]
        rows = torch.randperm(M, generator=torch.Generator().manual_seed(M))[:64].sort().values.to(DEV)
        yo = oracle.linear.linear_norm(xq[rows].cpu().numpy(), xs[rows].cpu().numpy(), af, "row", wq.cpu().numpy(),
                                       ws.cpu().numpy(), "e4m3", "row", bias=None if b is None else f64(b))
        if od == "bf16":
            _check_bf16(y[rows], yo)
        else:
            rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
            assert np.max(np.abs(f64(y[rows]) - yo) / np.maximum(np.abs(yo), rms)) <= TOL


def test_single_cta_grouped_engine_still_correct():
    """LOKA_GROUPED_1CTA=1 selects the single-CTA 128 x 128 grouped kernel (kept for A/B runs)."""
    import subprocess
    import sys
    import os
    code = ("import sys; sys.path.insert(0, 'tests'); import test_gpu_grouped as t; "
            "t.test_grouped_mixed_epilogues_and_ragged_shapes(); print('ok')")
    env = dict(os.environ, LOKA_GROUPED_1CTA="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("M,N,K,od,bias", [(512, 512, 8192, "f32", True), (2048, 1024, 16384, "bf16", False),
                                           (256, 200, 4000, "bf16", True), (96, 1000, 2048, "f32", False)])
def test_split_k_lone_gemm(M, N, K, od, bias):
    """Few 256x256 tiles and a long K (the paper's 2048 x 123200 x 1024 layer, scaled down): the
    CTA-pair engine splits K, writes FP32 partials to the workspace and reduces them in one kernel."""
    x, w = synth.heavy(M, K, 80), synth.weight(N, K, 81)
    xq, xs = lk.loka_quantize(to_dev_padded(x), "e4m3", "row")
    wq, ws = lk.loka_quantize(to_dev_padded(w), "e4m3", "row")
    b = torch.randn(N, generator=torch.Generator().manual_seed(5)).to(DEV) if bias else None
    keep = []
    args, y, _ = lk.make_linear_args(xq, xs, wq, ws, out_dtype=od, bias=b, keep=keep)
    if M % 32 == 0 and N % 4 == 0:
        assert lk.linear_workspace(args) > 0  # split chosen
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, out_dtype=od, bias=b)
    torch.cuda.synchronize()
    rows = torch.randperm(M, generator=torch.Generator().manual_seed(M))[:48].sort().values.to(DEV)
    yo = oracle.linear.linear_norm(xq[rows].cpu().numpy(), xs[rows].cpu().numpy(), "e4m3", "row", wq.cpu().numpy(),
                                   ws.cpu().numpy(), "e4m3", "row", bias=None if b is None else f64(b))
    if od == "bf16":
        _check_bf16(y[rows], yo)
    else:
        rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
        assert np.max(np.abs(f64(y[rows]) - yo) / np.maximum(np.abs(yo), rms)) <= TOL


def test_grouped_bf16_denominator():
    """The library's own BF16 grouped path (loka_grouped_bf16_linear: the kind::f16 instance of the
    CTA-pair engine, SURVEY.md §8(d)'s secondary denominator for the ensemble): 70 problems (two
    launches of <= 64), ragged M / N / K, bias, bf16 and f32 out — y = X W^T (+ b) on the bf16 values
    against the oracle's FP64 product at 2e-3 (bf16 out) / 1e-5 (f32 out)."""
    rng = np.random.default_rng(5)
    probs, keep, ref = [], [], []
    for t in range(70):
        M, N, K = int(rng.integers(1, 700)), int(rng.integers(1, 75)) * 8, int(rng.integers(1, 80)) * 16
        x, w = synth.heavy(M, K, 200 + t), synth.weight(N, K, 300 + t)
        od = "f32" if t % 3 == 0 else "bf16"
        bias = torch.randn(N, generator=torch.Generator().manual_seed(t)) if t % 4 == 1 else None
        xd, wd = to_dev_padded(x), to_dev_padded(w)
        one = torch.ones(1, dtype=torch.float32, device=DEV)
        a, y, _ = lk.make_linear_args(xd, one, wd, one, a_gran="tensor", b_gran="tensor", out_dtype=od,
                                      bias=None if bias is None else bias.to(DEV), keep=keep)
        a.a.dtype = lk.BF16
        a.b.dtype = lk.BF16
        probs.append(a)
        yo = oracle.linear.fwd(x.double().numpy(), w.double().numpy())
        if bias is not None:
            yo = oracle.linear.add_bias(yo, bias.double().numpy())
        ref.append((y, yo, od))
    arr = (lk.loka_linear_args * len(probs))(*probs)
    assert lk._lib.loka_grouped_bf16_linear(len(probs), arr, None) == 0
    torch.cuda.synchronize()
    for y, yo, od in ref:
        if od == "bf16":
            _check_bf16(y, yo)
        else:
            yg = f64(y)
            rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
            assert (np.abs(yg - yo) <= 1e-5 * np.maximum(np.abs(yo), rms)).all(), float(np.abs(yg - yo).max())


def test_grouped_bf16_rejects_epilogues():
    x = to_dev_padded(synth.heavy(64, 64, 1))
    one = torch.ones(1, dtype=torch.float32, device=DEV)
    keep = []
    a, _, _ = lk.make_linear_args(x, one, x, one, a_gran="tensor", b_gran="tensor", norm="layer", out_dtype="f32",
                                  keep=keep)
    a.a.dtype = lk.BF16
    a.b.dtype = lk.BF16
    assert lk._lib.loka_grouped_bf16_linear(1, (lk.loka_linear_args * 1)(a), None) == lk.ERR_UNSUPPORTED
