# eps0 > 0 profile: launch list of the config-2 shape and one full capture of the longest k_branch_sublayer launch
mkdir -p gpurun_out/eps
P=gpurun_out/eps
W=${W:-config2_pi4_eps1e-4_t8}
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_$W.csv python tools/profile_run.py $W --warm > $P/run.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py $P/launches_$W.csv > $P/launches_${W}_summary.txt; cat $P/launches_${W}_summary.txt | head -30
IDX=$(python - "$P/launches_$W.csv" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h = r; body = rows[i + 1:]; break
vi = h.index("Metric Value"); ki = h.index("Kernel Name")
n = 0; best = (0, 0)
for r in body:
    if len(r) > vi and "k_branch_sublayer" in r[ki]:
        v = float(r[vi].replace(",", ""))
        if v > best[0]: best = (v, n)
        n += 1
print(best[1])
PY
)
echo "top k_branch_sublayer launch index $IDX"
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_branch_sublayer --launch-skip $IDX --launch-count 1 -o $P/full_spec_$W python tools/profile_run.py $W --warm > /dev/null 2>&1; echo "full rc=$?"
python tools/ncu_summary.py $P/full_spec_$W.ncu-rep > $P/full_spec_${W}_summary.txt; cat $P/full_spec_${W}_summary.txt
