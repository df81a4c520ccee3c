"""-m gpu: NEXT-3 — LoKA Probe's matrix-normal weight tracker and learned-distribution sampling
 on the GPU (linalg.cu: Philox4x64-10 normals, blocked FP32 Cholesky with the
jitter escalation, triangular solves, Gram products, EMA / renormalisation, sampling GEMMs) against
oracle/sample.py and oracle/track.py on the same inputs.

Tolerances: normals — the same 24-bit uniforms on both sides, FP32 log / sincospi
on the GPU: |dz| <= 1e-6 (1 + |z|); factorisations, solves and products — FP32 arithmetic on
well-conditioned inputs: relative Frobenius 1e-5 ... 1e-4 (growing with the size / the number of
chained updates), checked against the FP64 oracle."""
import numpy as np
import pytest
import torch

import oracle
from oracle import sample as S

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None


def _rel(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("seed,offset,n", [(0, 0, 1), (0, 0, 7), (1, 3, 1001), (12345, 2, 4), (2**63 + 5, 1, 33),
                                           (7, 0, 1 << 20), (9, 4 * 10**9 + 1, 999)])
def test_philox_normals_match_oracle(seed, offset, n):
    z = lk.philox_normal(n, seed, offset).double().cpu().numpy()
    ref = S.normals(seed, offset, n)
    assert np.all(np.abs(z - ref) <= 1e-6 * (1.0 + np.abs(ref))), np.max(np.abs(z - ref))


def test_philox_unaligned_output_and_prefix():
    base = lk.philox_normal(1000, 5, 0)
    buf = torch.zeros(1003, device="cuda")
    lk.philox_normal(997, 5, 3, out=buf[3:1000])
    assert torch.equal(buf[3:1000], base[3:1000]) and torch.all(buf[:3] == 0) and torch.all(buf[1000:] == 0)


def _spd(rng, n, shift=1.0):
    g = rng.normal(size=(n, n))
    return g @ g.T / n + shift * np.eye(n)


@pytest.mark.parametrize("n", [1, 5, 64, 65, 130, 200, 513])
def test_cholesky_matches_oracle(n):
    rng = np.random.default_rng(n)
    a = _spd(rng, n)
    a[np.triu_indices(n, 1)] += 1e-3 * rng.normal(size=n * (n - 1) // 2)  # not exactly symmetric: sym() applies
    at = torch.tensor(a, dtype=torch.float32, device="cuda")
    l, eps = lk.cholesky_jittered(at, 1e-6)
    ref, eps_ref = S.cholesky_jittered(at.double().cpu().numpy(), 1e-6)
    assert eps == pytest.approx(eps_ref, rel=1e-6)
    lg = l.double().cpu().numpy()
    assert np.all(np.triu(lg, 1) == 0.0)
    assert _rel(lg, ref) <= 2e-6 * (1 + n / 16)


def test_cholesky_scale_escalation_and_failure():
    a = torch.tensor(np.diag([1.0, -1e-5]), dtype=torch.float32, device="cuda")
    l, eps = lk.cholesky_jittered(a, 1e-6)
    ref, eps_ref = S.cholesky_jittered(np.diag([1.0, np.float32(-1e-5)]), 1e-6)
    assert eps == pytest.approx(eps_ref, rel=1e-5)
    assert np.allclose(l.double().cpu().numpy(), ref, rtol=1e-5, atol=1e-7)
    with pytest.raises(lk.LokaError) as ei:
        lk.cholesky_jittered(torch.tensor(np.diag([1.0, -1.0]), dtype=torch.float32, device="cuda"), 1e-6)
    assert ei.value.status == 7
    z, eps = lk.cholesky_jittered(torch.zeros(3, 3, device="cuda"), 1e-6)  # constant stream (D30)
    assert eps == pytest.approx(1e-6) and torch.allclose(z, 1e-3 * torch.eye(3, device="cuda"))
    rng = np.random.default_rng(2)
    a = _spd(rng, 96) * 50.0
    l, eps = lk.cholesky_jittered(torch.tensor(a, dtype=torch.float32, device="cuda"), 1e-6, a_scale=1 / 49.0)
    ref, eps_ref = S.cholesky_jittered(np.float32(a).astype(np.float64) / 49.0, 1e-6)
    assert eps == pytest.approx(eps_ref, rel=1e-5)
    assert _rel(l.double().cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("m,n,dtype", [(5, 7, torch.float32), (64, 96, torch.bfloat16), (130, 70, torch.float32),
                                       (256, 513, torch.bfloat16)])
def test_weight_tracker_matches_oracle(m, n, dtype):
    rng = np.random.default_rng(m * 1000 + n)
    lu = np.tril(rng.normal(size=(m, m))) / np.sqrt(m) + np.eye(m)
    lv = np.tril(rng.normal(size=(n, n))) / np.sqrt(n) + np.eye(n)
    center = rng.normal(size=(m, n))

    def draw():
        return torch.tensor(center + lu @ rng.normal(size=(m, n)) @ lv.T, dtype=dtype)

    w0 = draw()
    tr = lk.WeightTracker(w0.cuda(), momentum=0.9, eps_rel=1e-6)
    st = oracle.track.weight_init(w0.double().numpy(), momentum=0.9, eps_rel=1e-6)
    for it in range(5):
        w = draw()
        tr.update(w.cuda())
        st = oracle.track.weight_update(st, w.double().numpy())
        torch.cuda.synchronize()
        tol = 2e-5 * (it + 1) * (1 + max(m, n) / 128)
        assert _rel(tr.U.double().cpu().numpy(), st["U"]) <= tol, (it, _rel(tr.U.double().cpu().numpy(), st["U"]))
        assert _rel(tr.V.double().cpu().numpy(), st["V"]) <= tol, (it, _rel(tr.V.double().cpu().numpy(), st["V"]))
        assert _rel(tr.mean.double().cpu().numpy(), st["mean"]) <= 1e-6
    assert tr.count == st["count"] == 5
    assert int(tr.status.item()) == 0
    assert float(torch.trace(tr.U.double())) == pytest.approx(m, rel=1e-5)


@pytest.mark.parametrize("k,b,seed,offset", [(1, 3, 0, 0), (96, 300, 4, 0), (200, 129, 5, 7), (513, 64, 6, 1)])
def test_sample_input_matches_oracle(k, b, seed, offset):
    rng = np.random.default_rng(k)
    l, _ = lk.cholesky_jittered(torch.tensor(_spd(rng, k, 0.5), dtype=torch.float32, device="cuda"), 1e-6)
    mu = torch.tensor(rng.normal(size=k) * 3, dtype=torch.float32, device="cuda")
    t = lk.sample_input(mu, l, b, seed, offset)
    ref = S.sample_input(mu.double().cpu().numpy(), l.double().cpu().numpy(), b, seed, offset)
    scale = np.abs(ref).max()
    assert np.max(np.abs(t.double().cpu().numpy() - ref)) <= 1e-5 * scale * (1 + k / 128)
    tb = lk.sample_input(mu, l, b, seed, offset, out_dtype=torch.bfloat16)
    assert np.max(np.abs(tb.double().cpu().numpy() - ref) / np.maximum(np.abs(ref), 1e-3 * scale)) <= 2 ** -8 + 1e-4


@pytest.mark.parametrize("m,n,seed", [(2, 3, 1), (70, 130, 2), (257, 64, 3)])
def test_sample_weight_matches_oracle(m, n, seed):
    rng = np.random.default_rng(m + n)
    l_u, _ = lk.cholesky_jittered(torch.tensor(_spd(rng, m), dtype=torch.float32, device="cuda"), 1e-6)
    l_v, _ = lk.cholesky_jittered(torch.tensor(_spd(rng, n), dtype=torch.float32, device="cuda"), 1e-6)
    mean = torch.tensor(rng.normal(size=(m, n)), dtype=torch.float32, device="cuda")
    w = lk.sample_weight(mean, l_u, l_v, seed, 11)
    ref = S.sample_weight(mean.double().cpu().numpy(), l_u.double().cpu().numpy(), l_v.double().cpu().numpy(), seed, 11)
    assert np.max(np.abs(w.double().cpu().numpy() - ref)) <= 1e-5 * np.abs(ref).max() * (1 + (m + n) / 128)


def test_input_tracker_sampling_reproduces_covariance():
    """End to end (PAPER.md:282-305 then 374-378): track a stream, sample from the tracked statistics,
    the sample's covariance matches the tracked one (statistical, 100k rows)."""
    rng = np.random.default_rng(9)
    k = 64
    a = rng.normal(size=(k, k)) / np.sqrt(k)
    tr = lk.InputTracker(k)
    for _ in range(4):
        x = torch.tensor(rng.normal(size=(4096, k)) @ a + 2.0, dtype=torch.bfloat16, device="cuda")
        tr.update(x)
    t = tr.sample(100_000, seed=3)
    emp = torch.cov(t.double().T).cpu().numpy()
    cov = tr.covariance().double().cpu().numpy()
    assert _rel(emp, cov) < 0.05
    assert np.max(np.abs(t.double().mean(0).cpu().numpy() - tr.mean.double().cpu().numpy())) < 0.05
