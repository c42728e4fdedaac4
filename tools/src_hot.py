"""Hot source lines of an ncu source-page CSV (ncu -i rep --page source --csv --print-source cuda,sass)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 45
cur, hdr = None, None
agg = collections.defaultdict(lambda: [0, 0, ""])
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Function Name":
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        ln = int(r[0])
        s = int(r[hdr.index("# Samples")] or 0)
        ins = int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    a = agg[(cur, ln)]
    a[0] += s
    a[1] += ins
    a[2] = r[1][:90]
tot_s = sum(a[0] for a in agg.values())
tot_i = sum(a[1] for a in agg.values())
print("total samples", tot_s, "warp instructions", tot_i)
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:5d} {100 * a[0] / tot_s:5.1f}% samp {100 * a[1] / tot_i:5.1f}% inst  {a[2]}")
