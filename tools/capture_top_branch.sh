#!/usr/bin/env bash
# Capture the longest k_branch_x launch of a workload with ncu --set full.
# usage: tools/capture_top_branch.sh <workload> <out-prefix>
set -e
W=$1; OUT=$2
python tools/profile_run.py $W > gpurun_out/${OUT}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${KRE:-k_branch_x} --csv \
    --log-file gpurun_out/${OUT}_branch_launches.csv python tools/profile_run.py $W > /dev/null 2>&1
IDX=$(python - "$OUT" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/{sys.argv[1]}_branch_launches.csv")))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h = r; body = rows[i + 1:]; break
vi = h.index("Metric Value"); ii = h.index("ID")
vals = [(float(r[vi].replace(",", "")), k) for k, r in enumerate(body) if len(r) > vi]
print(max(vals)[1])
PY
)
echo "top launch index $IDX"
# --kernel-id invocation numbers count launches of the matching kernel, 1-based
ncu --set full --clock-control none --import-source on --kernel-id ::regex:${KRE:-k_branch_x}:$((IDX + 1)) \
    -o gpurun_out/${OUT} python tools/profile_run.py $W > /dev/null 2>&1
