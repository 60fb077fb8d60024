"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count,
average and share of the summed launch time."""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    name = re.sub(r"\(.*", "", r[ki]).split("::")[-1]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(t for _, t in agg.values())
print(f"| kernel | launches | avg us | share |\n|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {n} | {t / n:.1f} | {t / tot:.3f} |")
