"""-m gpu: loka_probe_error (a7) within 1e-5 relative of oracle/probe.py on the same arrays."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, f64

pytestmark = pytest.mark.gpu
lk = pytest.importorskip("paper_2605_10886_b200") if torch.cuda.is_available() else None


def _check(st, po):
    for k in ("mere", "max_rel", "sum_abs_ref"):
        assert abs(st[k] - po[k]) <= 1e-5 * max(abs(po[k]), 1e-300), (k, st[k], po[k])
    assert st["count"] == po["count"] and st["n_floored"] == po["n_floored"]


@pytest.mark.parametrize("dt_out,dt_ref", [(torch.float32, torch.bfloat16), (torch.bfloat16, torch.bfloat16),
                                           (torch.float32, torch.float32)])
def test_probe_matches_oracle(dt_out, dt_ref):
    shapes = [(256, 256), (300, 130), (2048, 1024), (1, 8), (17, 1000)]
    pairs, ref_np = [], []
    for i, (m, n) in enumerate(shapes):
        ref = synth.heavy(m, n, i).float()
        out = ref * (1 + 0.05 * synth.gaussian(m, n, 50 + i).float())
        if m > 2:
            ref[1, :3] = 0.0  # floored elements
        pairs.append((out.to(dt_out).to(DEV), ref.to(dt_ref).to(DEV)))
    stats = lk.probe_stats_to_dicts(lk.loka_probe_error(pairs))
    for (o, r), st in zip(pairs, stats):
        _check(st, oracle.probe.mere_stats(f64(o), f64(r)))


def test_probe_identical_and_scaled():
    ref = synth.gaussian(512, 512, 1).float().to(DEV) + 3.0
    st = lk.probe_stats_to_dicts(lk.loka_probe_error([(ref, ref), (ref * 1.1, ref)]))
    assert st[0]["mere"] == 0.0 and st[0]["max_rel"] == 0.0
    # 1.1*ref is itself rounded to FP32, so the exact value is the oracle's on the same arrays
    _check(st[1], oracle.probe.mere_stats(f64(ref * 1.1), f64(ref)))
    assert abs(st[1]["mere"] - 0.1) < 1e-4


def test_probe_64_layers_one_call():
    pairs = []
    for g in range(64):
        m, n = 2048, synth.CFG3_DIMS[g % 8]
        ref = synth.gaussian(m, n, g, device=DEV).float()
        pairs.append(((ref + 0.01 * synth.gaussian(m, n, 100 + g, device=DEV).float()).to(torch.bfloat16), ref))
    stats = lk.probe_stats_to_dicts(lk.loka_probe_error(pairs))
    for (o, r), st in list(zip(pairs, stats))[::9]:
        _check(st, oracle.probe.mere_stats(f64(o), f64(r)))


def test_sharded_probe_equals_whole_tensor():
    """The data-parallel probe protocol (dist.probe_error_sharded's two passes) on one GPU with three
    row shards of a layer: pass 1 per shard -> summed (sum |ref|, count) -> loka_probe_error_global per
    shard -> loka_probe_merge: within 1e-5 of the oracle on the whole tensor, floored count exact."""
    g = torch.Generator().manual_seed(4)
    ref = torch.randn(900, 768, generator=g)
    ref[::7] *= 1e-9  # rows that fall under the floor
    out = ref * (1 + 0.02 * torch.randn(900, 768, generator=g))
    o, r = out.to(torch.bfloat16).to(DEV), ref.to(torch.bfloat16).to(DEV)
    shards = [(0, 300), (300, 611), (611, 900)]
    first = [lk.probe_stats_to_dicts(lk.loka_probe_error([(o[a:b], r[a:b])]))[0] for a, b in shards]
    gsum = torch.tensor([[sum(s["sum_abs_ref"] for s in first), float(sum(s["count"] for s in first))]],
                        dtype=torch.float64, device=DEV)
    per = [lk.probe_stats_to_dicts(lk.loka_probe_error([(o[a:b], r[a:b])], global_sum_count=gsum)) for a, b in shards]
    m = lk.probe_merge(per)[0]
    po = oracle.probe.mere_stats(o.cpu().double().numpy(), r.cpu().double().numpy())
    assert m["count"] == po["count"] and m["n_floored"] == po["n_floored"] > 0
    for k in ("mere", "max_rel", "sum_abs_ref"):
        assert abs(m[k] - po[k]) <= 1e-5 * max(abs(po[k]), 1e-30), (k, m[k], po[k])
