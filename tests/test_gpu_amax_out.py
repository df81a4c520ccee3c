"""-m gpu: NEXT-4 producer-side tensor amax: every epilogue engine folds max |y|
over the values it stores into a device word, bit-exactly equal to the amax of the output tensor,
so the next layer's tensorwise quantize can cast with it directly (CAST_WITH_AMAX) and produce the
same bytes as a full quantize (the data-parallel all-reduce then ships this word, a9)."""
import numpy as np
import pytest
import torch

import synth
from gpu_util import DEV, to_dev_padded

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None


def _q(x, gran="row", sf="f32"):
    return lk.loka_quantize(to_dev_padded(x), "e4m3", gran, sf)


CASES = [  # (M, N, K, norm, od, blockwise)      engine
    (300, 512, 256, "layer", "bf16", False),     # fused linear_norm (cluster of 2)
    (256, 1024, 384, "rms", "f32", False),       # fused, cluster of 4
    (4096, 4608, 512, "none", "bf16", False),    # CTA-pair engine
    (512, 512, 8192, "none", "f32", False),      # CTA-pair engine + split-K reduce
    (2048, 2560, 512, "none", "bf16", True),     # UE8M0 block-scaled pair engine
    (1300, 4096, 256, "layer", "bf16", False),   # wide rows: pair GEMM + row-wise norm pass
]


@pytest.mark.parametrize("M,N,K,norm,od,blockwise", CASES)
def test_amax_out_equals_output_amax(M, N, K, norm, od, blockwise):
    x, w = synth.heavy(M, K, 3), synth.weight(N, K, 4)
    if blockwise:
        xq, xs = _q(x, "blk_1x128", "ue8m0")
        wq, ws = _q(w, "blk_128x128", "ue8m0")
        kw = dict(a_gran="blk_1x128", b_gran="blk_128x128", a_scale_fmt="ue8m0", b_scale_fmt="ue8m0")
    else:
        xq, xs = _q(x)
        wq, ws = _q(w)
        kw = {}
    amax = torch.zeros(1, dtype=torch.float32, device=DEV)
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm=norm, out_dtype=od, amax_out=amax, **kw)
    torch.cuda.synchronize()
    ref = y.float().abs().max()
    assert amax.item() == ref.item(), (amax.item(), ref.item())


def test_next_layer_casts_with_the_produced_amax():
    """Layer 1 (LayerNorm, bf16 out, producer amax) -> layer 2's tensorwise quantize CAST_WITH_AMAX
    equals the two-pass FULL quantize of the same tensor, byte for byte."""
    M, K, N = 1024, 512, 768
    xq, xs = _q(synth.heavy(M, K, 5))
    wq, ws = _q(synth.weight(N, K, 6))
    amax = torch.zeros(1, dtype=torch.float32, device=DEV)
    y, _ = lk.loka_fp8_linear_norm(xq, xs, wq, ws, norm="layer", out_dtype="bf16", amax_out=amax)
    q1, s1 = lk.loka_quantize(y, "e4m3", "tensor", phase="cast", amax=amax)
    q2, s2 = lk.loka_quantize(y, "e4m3", "tensor")
    torch.cuda.synchronize()
    assert torch.equal(q1, q2) and torch.equal(s1, s2)
