"""Pins for oracle/sample.py and the weight tracker in oracle/track.py (NEXT-3).

* Philox4x64-10 equals numpy's own ``np.random.Philox`` bit generator (an independent
  implementation of the same published function; numpy advances the counter before each block).
* The normals: stream consistency under offsets, moments / tail mass of N(0, 1).
* The jittered Cholesky: closed forms (diagonal, identity, zero covariance), the x10 escalation
  (SPEC.md:262), reconstruction L L^T = a + eps I.
* Sampling: the empirical covariance of T' is Sigma (+ eps I) for a non-diagonal Sigma (a
  transposed factor would give L^T L instead), and vec(W') has covariance V (x) U.
* The weight update: the paper's solves against the explicit-inverse form it started from
  (U' = W_c V^-1 W_c^T), the W_c = 0 case, trace(U) = M, PSD-ness, and
  convergence to a known matrix-normal row covariance.
"""
import numpy as np
import pytest

from oracle import sample as S
from oracle import track as T


@pytest.mark.parametrize("key,ctr", [((0, 0), (1, 0, 0, 0)), ((5, 7), (11, 0, 0, 0)),
                                     ((2**64 - 1, 2**63 + 12345), (2**64 - 1, 3, 9, 2**62)),
                                     ((0x243F6A8885A308D3, 0x13198A2E03707344), (77, 2**40, 0, 1))])
def test_philox_equals_numpy(key, ctr):
    prev = list(ctr)
    prev[0] = (prev[0] - 1) % 2**64  # numpy increments before generating (no borrow needed here)
    bg = np.random.Philox(key=np.array(key, dtype=np.uint64), counter=np.array(prev, dtype=np.uint64))
    ref = bg.random_raw(4)
    got = S.philox4x64_10([ctr], key)[0]
    assert [int(v) for v in got] == [int(v) for v in ref]


def test_philox_stream_matches_numpy_blocks():
    bg = np.random.Philox(key=np.array([9, 0], dtype=np.uint64), counter=np.array([0, 0, 0, 0], dtype=np.uint64))
    ref = bg.random_raw(4 * 50).reshape(50, 4)
    ctr = np.zeros((50, 4), dtype=np.uint64)
    ctr[:, 0] = np.arange(1, 51, dtype=np.uint64)
    assert np.array_equal(S.philox4x64_10(ctr, (9, 0)), ref)


def test_normals_offsets_and_moments():
    z = S.normals(3, 0, 400_000)
    for o in (0, 1, 2, 3, 5, 1001):
        part = S.normals(3, o, 37)
        assert np.array_equal(part, z[o:o + 37])
    assert abs(z.mean()) < 5 * 1 / np.sqrt(len(z))
    assert abs(z.var() - 1.0) < 5 * np.sqrt(2.0 / len(z))
    frac1 = np.mean(np.abs(z) < 1.0)
    assert abs(frac1 - 0.682689492) < 5 * np.sqrt(0.2166 / len(z))
    frac2 = np.mean(np.abs(z) < 2.0)
    assert abs(frac2 - 0.954499736) < 5 * np.sqrt(0.0434 / len(z))
    assert not np.array_equal(S.normals(4, 0, 64), z[:64])
    # the pair (z_even, z_odd) is rotationally symmetric: cov(z_even, z_odd) ~ 0
    pairs = z.reshape(-1, 2)
    assert abs(np.mean(pairs[:, 0] * pairs[:, 1])) < 5 / np.sqrt(len(pairs))


def test_cholesky_closed_forms():
    l, eps = S.cholesky_jittered(np.diag([4.0, 9.0]), eps_rel=1e-12)
    assert np.allclose(l, np.diag([2.0, 3.0]), atol=1e-9)
    assert eps == pytest.approx(1e-12 * 6.5)
    l, eps = S.cholesky_jittered(np.eye(5), eps_rel=1e-6)
    assert eps == pytest.approx(1e-6)
    assert np.allclose(l, np.sqrt(1 + 1e-6) * np.eye(5), rtol=0, atol=1e-15)
    l, eps = S.cholesky_jittered(np.zeros((3, 3)), eps_rel=1e-6)  # constant stream: scale 1 (D30)
    assert eps == pytest.approx(1e-6)
    assert np.allclose(l, 1e-3 * np.eye(3))


def test_cholesky_escalation():
    a = np.diag([1.0, -1e-5])
    l, eps = S.cholesky_jittered(a, eps_rel=1e-6)  # eps0 = 1e-6 * (1 - 1e-5)/2 fails twice
    assert eps == pytest.approx(100 * 1e-6 * (1.0 - 1e-5) / 2)
    assert np.allclose(l @ l.T, a + eps * np.eye(2))
    with pytest.raises(S.NotPositiveDefinite):
        S.cholesky_jittered(np.diag([1.0, -1.0]), eps_rel=1e-6)


def test_cholesky_reconstruction_random_spd():
    rng = np.random.default_rng(0)
    g = rng.normal(size=(16, 16))
    a = g @ g.T + 0.1 * np.eye(16)
    l, eps = S.cholesky_jittered(a, 1e-6)
    assert np.allclose(np.triu(l, 1), 0.0)
    assert np.all(np.diag(l) > 0)
    assert np.linalg.norm(l @ l.T - (a + eps * np.eye(16))) <= 1e-12 * np.linalg.norm(a)


def test_sample_input_covariance_and_mean():
    rng = np.random.default_rng(1)
    k = 6
    g = rng.normal(size=(k, k))
    sigma = g @ g.T / k + 0.2 * np.eye(k)
    mu = rng.normal(size=k) * 3
    l, eps = S.cholesky_jittered(sigma, 1e-6)
    t = S.sample_input(mu, l, 200_000, seed=11)
    assert t.shape == (200_000, k)
    assert np.abs(t.mean(axis=0) - mu).max() < 5 * np.sqrt(np.diag(sigma).max() / len(t))
    emp = np.cov(t, rowvar=False)
    assert np.linalg.norm(emp - sigma) / np.linalg.norm(sigma) < 0.02
    assert np.array_equal(S.sample_input(mu, l, 10, seed=11), t[:10])  # determinism / stream prefix


def test_sample_input_degenerate_covariance():
    mu = np.array([1.0, -2.0, 3.0])
    l, eps = S.cholesky_jittered(np.zeros((3, 3)), 1e-6)
    t = S.sample_input(mu, l, 1000, seed=2)
    assert np.abs(t - mu).max() < 6 * np.sqrt(eps)


def test_sample_weight_vec_covariance():
    """the covariance of vec(W') (column-major vec) is V (x) U."""
    u = np.array([[1.0, 0.6], [0.6, 2.0]])
    v = np.array([[1.0, -0.3, 0.2], [-0.3, 0.5, 0.1], [0.2, 0.1, 1.5]])
    l_u, _ = S.cholesky_jittered(u, 0.0)
    l_v, _ = S.cholesky_jittered(v, 0.0)
    mean = np.arange(6.0).reshape(2, 3)
    draws = 60_000
    # one call per draw would be slow; the stream is consecutive, so draw them as offsets
    z_all = S.normals(5, 0, draws * 6).reshape(draws, 2, 3)
    w = mean[None] + np.einsum("ij,djk,lk->dil", l_u, z_all, l_v)
    assert np.allclose(S.sample_weight(mean, l_u, l_v, seed=5, offset=6 * 17), w[17])
    vec = np.transpose(w - mean[None], (0, 2, 1)).reshape(draws, 6)  # column-major vec
    emp = vec.T @ vec / draws
    ref = np.kron(v, u)
    assert np.linalg.norm(emp - ref) / np.linalg.norm(ref) < 0.05


def _inv_form_update(st, w):
    """The update written with explicit inverses (the form the paper's
    Cholesky solves replace): U' = W_c (V + eps I)^-1 W_c^T / N, V' = W_c^T (U + eps I)^-1 W_c / M."""
    mm, nn = w.shape
    u, v, m, er = st["U"], st["V"], st["m"], st["eps_rel"]
    eu, ev = er * np.trace(u) / mm, er * np.trace(v) / nn
    wc = w - st["mean"]
    u1 = wc @ np.linalg.inv(v + ev * np.eye(nn)) @ wc.T / nn
    v1 = wc.T @ np.linalg.inv(u + eu * np.eye(mm)) @ wc / mm
    u2 = m * u + (1 - m) * u1
    v2 = m * v + (1 - m) * v1
    un = (u2 + u2.T) / 2 + eu * np.eye(mm)
    vn = (v2 + v2.T) / 2 + ev * np.eye(nn)
    s = np.trace(un) / mm
    return un / s, vn * s


def test_weight_update_equals_explicit_inverse_form():
    rng = np.random.default_rng(3)
    mm, nn = 5, 7
    st = T.weight_init(rng.normal(size=(mm, nn)), momentum=0.9, eps_rel=1e-6)
    for it in range(6):  # non-trivial U, V after a few updates (non-diagonal, non-identity)
        w = rng.normal(size=(mm, nn)) * (1 + it) + np.outer(np.arange(mm), np.ones(nn))
        u_ref, v_ref = _inv_form_update(st, w)
        st = T.weight_update(st, w)
        assert np.allclose(st["U"], u_ref, rtol=1e-9, atol=1e-12)
        assert np.allclose(st["V"], v_ref, rtol=1e-9, atol=1e-12)
        assert np.trace(st["U"]) == pytest.approx(mm, rel=1e-12)
        assert np.linalg.eigvalsh(st["U"]).min() > 0 and np.linalg.eigvalsh(st["V"]).min() > 0
    assert st["count"] == 6


def test_weight_update_zero_centered():
    w = np.arange(12.0).reshape(3, 4)
    st = T.weight_init(w, momentum=0.9, eps_rel=1e-6)
    st2 = T.weight_update(st, w)  # W_c = 0 -> U' = V' = 0 -> U = 0.9 I + eps I, renormalised
    assert np.allclose(st2["U"], np.eye(3))
    assert np.allclose(st2["V"], (0.9 + 1e-6) ** 2 * np.eye(4))
    assert np.allclose(st2["mean"], w)
    # V (x) U invariance under the renormalisation: kron equals the unnormalised product
    assert np.allclose(np.kron(st2["V"], st2["U"]), np.kron((0.9 + 1e-6) * np.eye(4), (0.9 + 1e-6) * np.eye(3)))


def test_weight_tracker_recovers_row_covariance():
    """a stream from MN(0, U* = diag(1, 4), V* = I) gives U proportional to U*."""
    rng = np.random.default_rng(4)
    mm, nn = 2, 64
    l_star = np.diag([1.0, 2.0])
    st = T.weight_init(l_star @ rng.normal(size=(mm, nn)), momentum=0.9)
    for _ in range(500):
        st = T.weight_update(st, l_star @ rng.normal(size=(mm, nn)))
    u = st["U"] / st["U"][0, 0]
    assert abs(u[1, 1] - 4.0) / 4.0 < 0.15
    assert abs(u[0, 1]) < 0.15 * 2.0
    assert np.trace(st["U"]) == pytest.approx(mm, rel=1e-12)
