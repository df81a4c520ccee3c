"""O13 — LoKA Dispatch constrained selection (TEST INFRASTRUCTURE ONLY).

PAPER.md:541 (§III-C): "candidate implementations are first filtered by accuracy
constraints ... (typically MERE < 0.2) and whose speedup ... exceeds a minimum
improvement factor (typically > 1.05x) ... selects the implementation with the
highest measured throughput."  PAPER.md:547: separate decisions per direction.
Readings (D19): strict inequalities at both
thresholds; speedup = t_baseline / t_candidate (end-to-end time of the same op,
so highest throughput == smallest time); ties -> lexicographically smallest id;
nothing passes -> baseline (returned as -1).
"""
from __future__ import annotations


def select(candidates, baseline_time_us: float, mere_budget: float = 0.2, min_speedup: float = 1.05) -> int:
    """candidates: sequence of (id: str, mere: float, time_us: float). Returns index or -1."""
    best = -1
    for i, (cid, m, t) in enumerate(candidates):
        if not (m < mere_budget):
            continue
        if not (t > 0 and baseline_time_us / t > min_speedup):
            continue
        if best < 0:
            best = i
            continue
        bid, _, bt = candidates[best]
        if t < bt or (t == bt and cid < bid):
            best = i
    return best


def build_plan(results, baseline_times, mere_budget: float = 0.2, min_speedup: float = 1.05) -> dict:
    """results: {(layer, direction): [(id, mere, time_us), ...]}; baseline_times: same keys -> us.
    Returns {(layer, direction): id or "baseline"}."""
    plan = {}
    for key, cands in results.items():
        i = select(cands, baseline_times[key], mere_budget, min_speedup)
        plan[key] = "baseline" if i < 0 else cands[i][0]
    return plan
