"""Summarise ncu captures into profiles/ (committed evidence).

  python tools/ncu_summary.py --launches gpurun_out/launches.csv --full gpurun_out/prof.ncu-rep \
      --out profiles/r01_summary.md [--traffic-json profiles/traffic.json]

* launches: the `--metrics gpu__time_duration.sum --csv` launch list -> per-kernel count, total
  time and share of the profiled steps (cold-cache, serialised: compare SHARES, not absolutes).
* full: one `--set full` capture -> duration, DRAM bytes, tensor-pipe / SM / DRAM utilisation.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess


def read_launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    kn, mv, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) <= mv:
            continue
        name = r[kn].split("(")[0].replace("void ", "")
        val = float(r[mv].replace(",", ""))
        unit = r[mu]
        ns = val * {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}.get(unit, 1.0)
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + ns)
    return agg


def read_full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    d = {k: (v, u) for k, u, v in zip(h, units, vals)}
    return d


def to_bytes(v, u):
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic-json")
    ap.add_argument("--title", default="")
    ap.add_argument("--traffic-key", default="stack_bytes_per_launch")
    a = ap.parse_args()
    lines = [f"# ncu summary {a.title}".rstrip(), ""]
    if a.launches:
        agg = read_launches(a.launches)
        tot = sum(t for _, t in agg.values())
        lines += [f"## Launch list (`{a.launches}`)", "",
                  "gpu__time_duration.sum per launch, `--clock-control none`, cold cache, serialised by ncu.", "",
                  "| kernel | launches | total us | mean us | share of profiled GPU time |", "|---|---|---|---|---|"]
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k[:80]}` | {c} | {t / 1e3:.1f} | {t / c / 1e3:.2f} | {100 * t / tot:.1f}% |")
        lines.append("")
    if a.full:
        d = read_full(a.full)
        name = d.get("Kernel Name", ("?", ""))[0]
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
                "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__cluster_size",
                "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]
        lines += [f"## Full capture (`{a.full}`)", "", f"Kernel: `{name}`", "", "| metric | value | unit |",
                  "|---|---|---|"]
        for k in keys:
            if k in d:
                lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
        if "dram__bytes_read.sum" in d:
            rb = to_bytes(*d["dram__bytes_read.sum"])
            wb = to_bytes(*d.get("dram__bytes_write.sum", ("0", "byte")))
            lines += ["", f"DRAM traffic per launch: {rb + wb:.0f} bytes (read {rb:.0f} + write {wb:.0f})."]
            if a.traffic_json:  # merge: one entry per kernel key
                try:
                    tj = json.load(open(a.traffic_json))
                except (OSError, ValueError):
                    tj = {}
                tj[a.traffic_key] = rb + wb
                tj[a.traffic_key + "_source"] = f"{a.full}: {name}"
                json.dump(tj, open(a.traffic_json, "w"), indent=1)
        lines.append("")
    open(a.out, "w").write("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
