"""Pins for oracle/track.py (NEXT-2 batched Welford input tracker): the merged
summaries equal numpy's two-pass mean / covariance of the concatenated stream for any partition
(SPEC.md:228, 581), are insensitive to batch order, and the one-batch case reduces
to the textbook scatter."""
import numpy as np
import pytest

from oracle import track as T


def _stream(rng, k, rows):
    a = rng.normal(size=(k, k)) / np.sqrt(k)
    return rng.normal(size=(rows, k)) @ a + rng.normal(size=k) * 3.0


@pytest.mark.parametrize("seed", range(10))
def test_any_partition_equals_two_pass(seed):
    rng = np.random.default_rng(seed)
    k = int(rng.integers(1, 65))
    x = _stream(rng, k, int(rng.integers(2, 3000)))
    cuts = np.sort(rng.choice(np.arange(1, len(x)), size=min(len(x) - 1, int(rng.integers(1, 12))), replace=False))
    st = T.init(k)
    for part in np.split(x, cuts):
        st = T.update(st, part)
    assert st["n"] == len(x)
    assert np.allclose(st["mean"], x.mean(axis=0), rtol=1e-12, atol=1e-12)
    ref = np.cov(x, rowvar=False, ddof=1).reshape(k, k)
    assert np.linalg.norm(T.covariance(st) - ref) <= 1e-10 * max(1.0, np.linalg.norm(ref))


def test_order_insensitive_and_empty_batches():
    rng = np.random.default_rng(1)
    x = _stream(rng, 16, 900)
    parts = np.split(x, [100, 350, 351, 700])
    a, b = T.init(16), T.init(16)
    for p in parts:
        a = T.update(a, p)
    for p in reversed(parts):
        b = T.update(b, p)
    b = T.update(b, x[:0])
    assert a["n"] == b["n"] == 900
    assert np.allclose(a["mean"], b["mean"], atol=1e-12)
    assert np.linalg.norm(a["scatter"] - b["scatter"]) <= 1e-10 * np.linalg.norm(a["scatter"])


def test_single_batch_is_the_centered_gram():
    x = np.array([[1.0, 2.0], [3.0, 6.0], [5.0, 10.0]])
    st = T.update(T.init(2), x)
    assert np.allclose(st["mean"], [3.0, 6.0])
    assert np.allclose(st["scatter"], [[8.0, 16.0], [16.0, 32.0]])  # sum of (x - mu)(x - mu)^T by hand
    assert np.allclose(T.covariance(st), [[4.0, 8.0], [8.0, 16.0]])
