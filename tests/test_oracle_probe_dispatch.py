"""Pins for oracle/probe.py (O11/O12) and oracle/dispatch.py (O13): SPEC worked examples,
brute force on small arrays / random tables, invariants (scaling invariance, monotonicity)."""
import itertools
import json
import math
import os
import random

import numpy as np

from oracle import probe, dispatch

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_mere_spec_examples():
    rng = np.random.default_rng(0)
    ref = rng.standard_normal((13, 17)) + 3.0
    assert probe.mere(ref, ref) == GOLD["mere_equal"]["value"]
    g = GOLD["mere_scaled"]
    assert abs(probe.mere(g["factor"] * ref, ref) - g["value"]) < 1e-12
    ref2 = ref.copy(); ref2[0, 0] = 0.0
    st = probe.mere_stats(ref2 + 0.5, ref2)
    assert math.isfinite(st["mere"]) and st["n_floored"] == 1 and st["count"] == ref.size


def test_mere_bruteforce_and_scaling_invariance():
    rng = np.random.default_rng(1)
    out, ref = rng.standard_normal((6, 9)), rng.standard_normal((6, 9))
    ref[2, 3] = 1e-12  # below the floor
    n = ref.size
    f = 1e-6 * math.fsum(abs(v) for v in ref.reshape(-1)) / n
    rel = [abs(o - r) / max(abs(r), f) for o, r in zip(out.reshape(-1), ref.reshape(-1))]
    st = probe.mere_stats(out, ref)
    assert abs(st["mere"] - sum(rel) / n) < 1e-14 * max(1, st["mere"])
    assert abs(st["max_rel"] - max(rel)) <= 1e-15 * max(rel) and st["n_floored"] == 1
    assert abs(st["sum_abs_ref"] - math.fsum(abs(v) for v in ref.reshape(-1))) < 1e-15
    st2 = probe.mere_stats(4.0 * out, 4.0 * ref)  # SPEC.md:355 invariance (power of two: exact)
    assert st2["mere"] == st["mere"] and st2["n_floored"] == st["n_floored"]


def test_geomean():
    g = GOLD["geomean_1_4"]
    assert abs(probe.geomean(g["values"]) - g["value"]) < 1e-15
    assert abs(probe.geomean([0.0, 1.0]) - math.sqrt(1e-6)) < 1e-18
    assert abs(probe.geomean([0.3]) - 0.3) < 1e-15


def test_dispatch_spec_examples():
    th = GOLD["dispatch_thresholds"]
    for m, sp, kept in GOLD["dispatch_filter"]["cases"]:
        idx = dispatch.select([("c", m, 100.0 / sp)], 100.0, th["mere_budget"], th["min_speedup"])
        assert (idx == 0) == kept
    b = GOLD["dispatch_boundary"]["mere"]
    assert dispatch.select([("c", b, 10.0)], 100.0) == -1
    abc = GOLD["dispatch_abc"]
    cands = [(cid, m, 100.0 / sp) for cid, m, sp in abc["cands"]]
    assert cands[dispatch.select(cands, 100.0)][0] == abc["choice"]
    assert dispatch.select([], 1.0) == -1


def _brute(cands, tb, budget, msp):
    ok = [(t, cid, i) for i, (cid, m, t) in enumerate(cands) if m < budget and t > 0 and tb / t > msp]
    return min(ok)[2] if ok else -1


def test_dispatch_random_tables_bruteforce_and_monotone():
    """SPEC.md:588 acceptance 9: 1,000 random tables incl. ties and all-filtered cases."""
    rnd = random.Random(7)
    for _ in range(1000):
        n = rnd.randint(0, 8)
        ids = rnd.sample(["a", "b", "c", "d", "e", "f", "g", "h", "i"], n)
        cands = [(ids[i], rnd.choice([0.05, 0.1, 0.2, 0.3, rnd.random() * 0.4]),
                  rnd.choice([50.0, 80.0, 95.0, 100.0, rnd.uniform(40, 120)])) for i in range(n)]
        tb = 100.0
        i = dispatch.select(cands, tb)
        assert i == _brute(cands, tb, 0.2, 1.05)
        # monotonicity: tightening thresholds never un-baselines an entry
        if i < 0:
            assert dispatch.select(cands, tb, 0.1, 1.2) == -1


def test_build_plan_per_direction():
    res = {("l0", "fwd"): [("rw", 0.1, 50.0)], ("l0", "wgrad"): [("rw", 0.3, 50.0), ("tw", 0.15, 90.0)]}
    plan = dispatch.build_plan(res, {("l0", "fwd"): 100.0, ("l0", "wgrad"): 100.0})
    assert plan == {("l0", "fwd"): "rw", ("l0", "wgrad"): "tw"}


def test_mere_shard_floor_reading():
    """The data-parallel reading of D10: with the whole tensor's floor passed to each row shard, the
    count-weighted mean of the shards' MEREs equals the whole tensor's MERE (brute force)."""
    rng = np.random.default_rng(3)
    ref = rng.standard_normal((40, 7)) * np.where(rng.random((40, 1)) < 0.3, 1e-9, 1.0)
    out = ref * (1 + 0.01 * rng.standard_normal(ref.shape))
    whole = probe.mere_stats(out, ref)
    f = 1e-6 * np.abs(ref).mean()
    parts = [probe.mere_stats(out[a:b], ref[a:b], floor=f) for a, b in ((0, 13), (13, 29), (29, 40))]
    n = sum(p["count"] for p in parts)
    assert abs(sum(p["mere"] * p["count"] for p in parts) / n - whole["mere"]) <= 1e-12 * whole["mere"]
    assert sum(p["n_floored"] for p in parts) == whole["n_floored"] > 0
    # the same per-element brute force
    den = np.maximum(np.abs(ref), f)
    assert abs(np.mean(np.abs(out - ref) / den) - whole["mere"]) <= 1e-12 * whole["mere"]
