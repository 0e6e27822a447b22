"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: [0, 0.0])
total = 0.0
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("lrk::<unnamed>::", "")
        v = float(d["Metric Value"]) / 1e3
        agg[name][0] += 1
        agg[name][1] += v
        total += v
print(f"{'kernel':28s} {'launches':>8s} {'total us':>10s} {'share':>6s}")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} {c:8d} {t:10.1f} {100 * t / total:5.1f}%")
print(f"{'all':28s} {sum(c for c, _ in agg.values()):8d} {total:10.1f}")
