"""-m gpu: NEXT-2 — LoKA Probe's batched Welford input tracker on the GPU
(loka_probe_track_input: column means, centred bf16 transpose, S_b on the CTA-pair tensor-core
engine with BF16 operands, FP32 merge) against oracle/track.py fed the same bf16 batches."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None


def _batch(rng, b, k, a, shift):
    return torch.tensor(rng.normal(size=(b, k)) @ a + shift, dtype=torch.bfloat16)


@pytest.mark.parametrize("k,batches,shift", [(256, [300, 1000, 77, 512], 0.0), (2048, [4096, 4096], 0.5),
                                             (512, [64, 8, 1, 640], 30.0)])
def test_tracker_matches_oracle(k, batches, shift):
    rng = np.random.default_rng(k)
    a = rng.normal(size=(k, k)) / np.sqrt(k) * (1 + np.arange(k) / k)[None, :]
    tr = lk.InputTracker(k)
    st = oracle.track.init(k)
    for b in batches:
        x = _batch(rng, b, k, a, shift + rng.normal(size=k))
        tr.update(x.cuda())
        st = oracle.track.update(st, x.double().numpy())
    torch.cuda.synchronize()
    assert tr.n == st["n"] == sum(batches)
    mean = tr.mean.double().cpu().numpy()
    assert np.max(np.abs(mean - st["mean"])) <= 1e-5 * max(1.0, np.max(np.abs(st["mean"])))
    cov = tr.covariance().double().cpu().numpy()
    ref = oracle.track.covariance(st)
    # centred values are rounded to bf16 for the tensor cores (2^-9 relative), sums in FP32
    assert np.linalg.norm(cov - ref) <= 5e-3 * np.linalg.norm(ref)
    assert np.max(np.abs(np.diag(cov) - np.diag(ref)) / np.diag(ref)) <= 1e-2
