"""-m gpu: NVFP4 (D35-D38) — the quantize kernel bit-exact with
oracle/nvfp4.py (packed E2M1 codes, E4M3 block-scale codes, FP32 tensor scale), and the
block-scaled GEMM (tcgen05 kind::mxf4nvf4.block_scale.scale_vec::4X) + epilogue against the
oracle's float64 linear on the same codes and scales."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, assert_bytes_equal, assert_scales_equal, f64, guarded_rel_err

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None
TOL = 2e-3


def _q(x, **kw):
    p, sf, st = lk.loka_quantize_nvfp4(x.to(DEV), **kw)
    torch.cuda.synchronize()
    return p, sf, st


@pytest.mark.parametrize("rows,cols", [(1, 16), (7, 64), (256, 1024), (129, 4160), (1000, 512)])
@pytest.mark.parametrize("dist", ["gauss", "heavy"])
def test_quantize_bit_exact(rows, cols, dist):
    x = synth.gaussian(rows, cols, 11) if dist == "gauss" else synth.heavy(rows, cols, 12)
    p, sf, st = _q(x)
    op, osf, ost = oracle.nvfp4.quantize(x.double().numpy())
    assert_bytes_equal(sf, osf, "block scales")
    assert_bytes_equal(p, op, "codes")
    assert_scales_equal(st, ost, "tensor scale")


def test_quantize_f32_input_zero_blocks_and_given_amax():
    x = synth.gaussian(64, 256, 3).float()
    x[5] = 0
    x[6, 16:64] *= 1e-8  # block scales underflow -> signed zeros
    amax = torch.tensor([float(x.abs().max()) * 4.0], device=DEV)  # a (larger) global amax
    p, sf, st = _q(x, amax=amax)
    op, osf, ost = oracle.nvfp4.quantize(x.double().numpy(), amax=np.array([float(amax[0])]))
    assert_bytes_equal(sf, osf, "block scales")
    assert_bytes_equal(p, op, "codes")
    assert_scales_equal(st, ost, "tensor scale")
    p0, sf0, st0 = _q(torch.zeros(32, 64))
    assert not p0.any() and not sf0.any() and float(st0[0]) == 1.0


def test_nonfinite_flagged():
    x = synth.gaussian(32, 64, 1)
    x[3, 7] = float("inf")
    status = torch.zeros(1, dtype=torch.int32, device=DEV)
    _q(x, status=status)
    assert int(status[0]) & 1


def _rand_nvfp4(rows, K, g, emin=-1, emax=1):
    """Random E2M1 codes with power-of-two block scales (E4M3 codes of 2^e) and s_t = 1."""
    codes = torch.randint(0, 16, (rows, K), generator=g).to(torch.uint8)
    packed = (codes[:, 0::2] | (codes[:, 1::2] << 4)).to(torch.uint8)
    e = torch.randint(emin, emax + 1, (rows, K // 16), generator=g)
    sf = ((e + 7) << 3).to(torch.uint8)  # E4M3 code of 2^e (normal range)
    return packed.to(DEV).contiguous(), sf.to(DEV).contiguous(), torch.ones(1, device=DEV)


@pytest.mark.parametrize("M,N,K", [(128, 128, 256), (256, 256, 512), (128, 384, 64), (384, 256, 320)])
def test_block_scales_applied_exactly(M, N, K):
    """Every product and partial sum is exact in FP32 (E2M1 values are multiples of 1/2, scales in
    2^[-1, 1], |sum| < 2^17): the GPU result must equal the float64 oracle bit for bit.  A scale
    applied to the wrong row, column or 16-element block changes the value."""
    g = torch.Generator().manual_seed(M + N + K)
    a = _rand_nvfp4(M, K, g)
    b = _rand_nvfp4(N, K, g)
    y, _ = lk.loka_nvfp4_linear_norm(a, b, out_dtype="f32")
    torch.cuda.synchronize()
    yo = oracle.nvfp4.linear_norm(*(t.cpu().numpy() for t in a), *(t.cpu().numpy() for t in b))
    assert np.array_equal(f64(y), yo), float(np.abs(f64(y) - yo).max())


@pytest.mark.parametrize("M,N,K", [(128, 128, 256), (300, 256, 640), (200, 384, 1024), (512, 1024, 512),
                                   (4096, 256, 2048), (130, 2048, 256)])
@pytest.mark.parametrize("norm", ["none", "layer", "rms"])
def test_linear_norm_vs_oracle(M, N, K, norm):
    x = synth.heavy(M, K, 21)
    w = synth.weight(N, K, 22)
    a, b = _q(x), _q(w)
    y, _ = lk.loka_nvfp4_linear_norm(a, b, norm=norm, out_dtype="f32")
    torch.cuda.synchronize()
    yo = oracle.nvfp4.linear_norm(*(t.cpu().numpy() for t in a), *(t.cpu().numpy() for t in b), norm=norm)
    err = guarded_rel_err(f64(y), yo)
    assert err <= TOL, err


def test_bf16_and_fp8_outputs():
    M, N, K = 256, 512, 1024
    a, b = _q(synth.gaussian(M, K, 31)), _q(synth.weight(N, K, 32))
    yo = oracle.nvfp4.linear_norm(*(t.cpu().numpy() for t in a), *(t.cpu().numpy() for t in b), norm="layer")
    yb, _ = lk.loka_nvfp4_linear_norm(a, b, norm="layer", out_dtype="bf16")
    y8, s8 = lk.loka_nvfp4_linear_norm(a, b, norm="layer", out_dtype="e4m3")
    torch.cuda.synchronize()
    assert guarded_rel_err(f64(yb), yo) <= TOL + 2.0 ** -8
    y8d = oracle.quantize.dequantize(y8.cpu().numpy(), s8.cpu().numpy(), "e4m3", "row")
    assert guarded_rel_err(y8d, yo) <= 2.0 ** -4 + TOL


@pytest.mark.parametrize("M,N,K", [(2560, 2048, 256), (2304, 2304, 320)])
def test_pair_engine_block_scales_exact(M, N, K):
    """>= 74 tiles of 256 x 256 and a plain epilogue: the CTA-pair block-scaled engine
    (cta_group::2, SFB of both column halves in each CTA); exact-product construction as above."""
    g = torch.Generator().manual_seed(M + K)
    a = _rand_nvfp4(M, K, g)
    b = _rand_nvfp4(N, K, g)
    y, _ = lk.loka_nvfp4_linear_norm(a, b, out_dtype="f32")
    torch.cuda.synchronize()
    yo = oracle.nvfp4.linear_norm(*(t.cpu().numpy() for t in a), *(t.cpu().numpy() for t in b))
    assert np.array_equal(f64(y), yo), float(np.abs(f64(y) - yo).max())


@pytest.mark.parametrize("out_dtype", ["f32", "bf16"])
def test_pair_engine_vs_oracle_ragged_bias(out_dtype):
    M, N, K = 2500, 2000, 1088
    a, b = _q(synth.heavy(M, K, 41)), _q(synth.weight(N, K, 42))
    bias = torch.randn(N, device=DEV) * 0.1
    y, _ = lk.loka_nvfp4_linear_norm(a, b, bias=bias, out_dtype=out_dtype)
    torch.cuda.synchronize()
    yo = oracle.nvfp4.linear_norm(*(t.cpu().numpy() for t in a), *(t.cpu().numpy() for t in b),
                                  bias=bias.double().cpu().numpy())
    assert guarded_rel_err(f64(y), yo) <= TOL + (2.0 ** -8 if out_dtype == "bf16" else 0.0)
