"""Probe cadence and snapshot files: bit-exact round trip,
version / corruption detection, the schedule's invariants.  CPU only (host logic); the GPU
tracker round trip is in test_gpu_snapshot below (-m gpu)."""
import os

import numpy as np
import pytest
import torch

from paper_2605_10886_b200 import snapshot as S


def _snap(rng):
    return {"kind": "weight", "scalars": {"M": 3, "N": 5, "count": 7, "momentum": 0.95, "eps_rel": 1e-6},
            "arrays": {"mean": rng.normal(size=(3, 5)).astype(np.float32),
                       "U": rng.normal(size=(3, 3)).astype(np.float32),
                       "V": np.array(rng.normal(size=(5, 5)), dtype=np.float32)}}


def test_round_trip_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    snap = _snap(rng)
    snap["arrays"]["U"][0, 0] = np.float32(np.nan)  # arbitrary bit patterns survive
    snap["arrays"]["V"][1, 1] = np.float32(-0.0)
    p = str(tmp_path / "w.snap")
    S.save(p, snap)
    back = S.load(p)
    assert back["kind"] == "weight" and back["scalars"] == snap["scalars"]
    for k, a in snap["arrays"].items():
        assert back["arrays"][k].shape == a.shape
        assert np.array_equal(back["arrays"][k].view(np.uint32), a.view(np.uint32))


def test_version_mismatch_and_corruption(tmp_path):
    data = bytearray(S.dumps(_snap(np.random.default_rng(1))))
    bad = bytearray(data)
    bad[8] = 2  # version field
    with pytest.raises(S.FormatVersionMismatch):
        S.loads(bytes(bad))
    with pytest.raises(S.CorruptSnapshot):
        S.loads(bytes(data[:-10]))  # truncated
    flip = bytearray(data)
    flip[len(flip) // 2] ^= 1
    with pytest.raises(S.CorruptSnapshot):
        S.loads(bytes(flip))
    with pytest.raises(S.CorruptSnapshot):
        S.loads(b"not a snapshot at all")


def test_async_save_of_a_copied_snapshot(tmp_path):
    class FakeInput:  # same attributes as InputTracker, host tensors
        def __init__(self):
            self.mean = torch.arange(4, dtype=torch.float32)
            self.scatter = torch.eye(4)
            self.n = 10
    t = FakeInput()
    p = str(tmp_path / "i.snap")
    fut = S.save_async(p, t)
    t.mean.add_(100.0)  # later updates do not leak into the file being written
    assert fut.result(timeout=30) == p
    back = S.load(p)
    assert back["scalars"] == {"n": 10, "K": 4}
    assert np.array_equal(back["arrays"]["mean"], np.arange(4, dtype=np.float32))
    assert not os.path.exists(p + ".tmp")


def test_schedule():
    s = S.ProbeSchedule()
    assert (s.activate_every, s.snapshot_every) == (100, 10_000)
    assert s.should_track(0) and s.should_track(300) and not s.should_track(301)
    assert s.should_snapshot(10_000) and not s.should_snapshot(0) and not s.should_snapshot(15_000)
    with pytest.raises(ValueError):
        S.ProbeSchedule(100, 150)


@pytest.mark.gpu
def test_gpu_tracker_restore(tmp_path):
    lk = pytest.importorskip("paper_2605_10886_b200")
    w = torch.randn(16, 24, device="cuda")
    tr = lk.WeightTracker(w)
    tr.update(torch.randn(16, 24, device="cuda"))
    p = str(tmp_path / "w.snap")
    S.save_async(p, tr).result(timeout=60)
    tr2 = lk.WeightTracker(torch.zeros(16, 24, device="cuda"))
    S.restore(tr2, S.load(p))
    assert torch.equal(tr2.U, tr.U) and torch.equal(tr2.V, tr.V) and torch.equal(tr2.mean, tr.mean)
    assert tr2.count == tr.count == 1
    it = lk.InputTracker(8)
    it.update(torch.randn(64, 8, device="cuda").to(torch.bfloat16))
    S.save(p, S.snapshot(it))
    it2 = lk.InputTracker(8)
    S.restore(it2, S.load(p))
    assert it2.n == 64 and torch.equal(it2.scatter, it.scatter)
