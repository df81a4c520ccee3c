"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            nm = d["Kernel Name"][:70]
            agg[nm][0] += 1
            agg[nm][1] += float(d["Metric Value"].replace(",", ""))
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:5d} {t / 1e3:10.1f} us  mean {t / 1e3 / n:8.2f} us  {k}")
