"""Pins for oracle/gradcomm.py (D39): exact reconstruction when every gradient is representable
(small integers times per-row powers of two: quantization is exact, so the reduction equals the
float64 sum of the unquantized gradients), P = 1 is dequantization, rank-order invariance of the
float64 sum, and the quantization error bound against the unquantized sum."""
import numpy as np

from oracle import fp8, gradcomm, quantize


def test_exact_when_representable():
    rng = np.random.default_rng(0)
    # |integers| <= 7 times powers of two in [2^-3, 2^3] are E4M3 values (3 mantissa bits, within
    # range), so with row scales 1 the codes carry the gradients exactly
    grads = [rng.integers(-7, 8, (16, 64)) * 2.0 ** rng.integers(-3, 4, (16, 1)) for _ in range(4)]
    codes = [fp8.encode(g, "e4m3") for g in grads]
    scales = [np.ones(16, np.float32) for _ in grads]
    r = gradcomm.reduce_dequantized(codes, scales, "e4m3")
    assert np.array_equal(r, sum(grads))


def test_single_rank_is_dequantize():
    g = np.random.default_rng(1).standard_normal((8, 32))
    r, q, s = gradcomm.quantized_allreduce([g], "e5m2")
    assert np.array_equal(r, quantize.dequantize(q[0], s[0], "e5m2", "row"))


def test_rank_order_invariance_and_error_bound():
    rng = np.random.default_rng(2)
    grads = [rng.standard_normal((32, 128)) * 2.0 ** -10 for _ in range(8)]
    r, q, s = gradcomm.quantized_allreduce(grads, "e5m2")
    r2 = gradcomm.reduce_dequantized(q[::-1], s[::-1], "e5m2")
    assert np.allclose(r, r2, rtol=0, atol=1e-15)
    # rowwise e5m2: |x - x_hat| <= 2^-3 |x| (half of the 2-bit mantissa step) + subnormal floor
    amax = np.stack([np.abs(g).max(axis=1, keepdims=True) for g in grads])
    bound = sum(2.0 ** -3 * np.abs(g) + a * 2.0 ** -16 / 57344 * 2 for g, a in zip(grads, amax))
    assert (np.abs(r - sum(grads)) <= bound).all()
