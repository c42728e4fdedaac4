"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = start = None
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr, start = r, i + 1
        break
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[start:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("ppgpu::", "")
    v = float(r[vi].replace(",", ""))
    v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[ui], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':28s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'avg us':>9s}")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} {c:8d} {t / 1e3:10.3f} {t / tot * 100:6.1f}% {t / c:9.2f}")
print(f"{'total':28s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.3f}")
