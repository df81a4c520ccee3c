"""-m gpu: loka_fp8_mlp_stack (a4+a5 for a whole LRM MLP stack in one launch, BJ configs[1]).
At the cfg2 shape the result must be bit-identical to the chain of per-layer loka_fp8_linear_norm
calls (same tiling, same arithmetic); every case is also checked against the oracle run layer by
layer on the GPU's own FP8 hand-offs."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, f64, guarded_rel_err

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None


def _inputs(M, dims, xdist="gaussian"):
    x = synth.heavy(M, dims[0], 7, device=DEV) if xdist == "heavy" else synth.gaussian(M, dims[0], 0, device=DEV)
    xq, xs = lk.loka_quantize(x, "e4m3", "row")
    ws = [lk.loka_quantize(synth.weight(dims[l + 1], dims[l], 100 + l, device=DEV), "e4m3", "row")
          for l in range(len(dims) - 1)]
    return xq, xs, ws


def _chain(xq, xs, ws, norm, out_dtype):
    hq, hs = xq, xs
    outs = []
    for l, (wq, wsc) in enumerate(ws):
        last = l == len(ws) - 1
        y, ys = lk.loka_fp8_linear_norm(hq, hs, wq, wsc, norm=norm, out_dtype=out_dtype if last else "e4m3")
        outs.append((y, ys))
        hq, hs = y, ys
    return outs


def test_cfg2_stack_bit_identical_to_layer_chain():
    dims, M = synth.CFG2_DIMS, 4096
    xq, xs, ws = _inputs(M, dims)
    y, _ = lk.loka_fp8_mlp_stack(xq, xs, ws, norms="layer", out_dtype="bf16")
    chain = _chain(xq, xs, ws, "layer", "bf16")
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int16), chain[-1][0].view(torch.int16))


@pytest.mark.parametrize("norm,out_dtype", [("layer", "e4m3"), ("rms", "f32"), ("none", "bf16")])
def test_stack_vs_oracle(norm, out_dtype):
    dims, M = [512, 1024, 256, 512], 300  # C = 4 (BN 256 / 64 / 128), ragged M
    xq, xs, ws = _inputs(M, dims, "heavy")
    y, ys = lk.loka_fp8_mlp_stack(xq, xs, ws, norms=norm, out_dtype=out_dtype)
    chain = _chain(xq, xs, ws, norm, out_dtype)
    torch.cuda.synchronize()
    # oracle on the chain's own hand-offs: the stack's inputs of every layer equal the chain's
    # up to rounding order of the statistics, so compare the final layer with the tolerance
    hq, hs = (xq, xs) if len(ws) == 1 else chain[-2]
    yo = oracle.linear.linear_norm(hq.cpu().numpy(), hs.cpu().numpy(), "e4m3", "row", ws[-1][0].cpu().numpy(),
                                   ws[-1][1].cpu().numpy(), "e4m3", "row", norm=norm)
    if out_dtype == "e4m3":
        got = oracle.quantize.dequantize(y.cpu().numpy(), ys.cpu().numpy(), "e4m3", "row")
        rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
        assert np.mean(np.abs(got - yo) <= 2.0 ** -3 * np.abs(yo) + 2e-3 * np.maximum(np.abs(yo), rms)) > 0.999
    else:
        got = f64(y)
        tol = 2e-3 if out_dtype == "f32" else 6e-3
        assert guarded_rel_err(got, yo) <= tol or np.mean(
            np.abs(got - yo) <= tol * np.maximum(np.abs(yo), np.sqrt(np.mean(yo ** 2, 1, keepdims=True)))) > 0.999


def test_stack_single_cta_cluster_and_short():
    dims, M = [256, 256, 128, 256], 520  # max N 256 -> C = 1
    xq, xs, ws = _inputs(M, dims)
    y, _ = lk.loka_fp8_mlp_stack(xq, xs, ws, norms="layer", out_dtype="f32")
    chain = _chain(xq, xs, ws, "layer", "f32")
    torch.cuda.synchronize()
    hq, hs = chain[-2]
    yo = oracle.linear.linear_norm(hq.cpu().numpy(), hs.cpu().numpy(), "e4m3", "row", ws[-1][0].cpu().numpy(),
                                   ws[-1][1].cpu().numpy(), "e4m3", "row", norm="layer")
    assert np.mean(np.abs(f64(y) - yo) <= 2e-3 * np.maximum(np.abs(yo), np.sqrt(np.mean(yo ** 2, 1, keepdims=True)))) > 0.999
