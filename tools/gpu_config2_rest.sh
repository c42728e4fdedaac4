# BASELINE config 2, theta_h = k pi/16 for the k in $KS (default 5 6 7 8): one
# process per k under its own timeout, first eps0 = $EPS0 (default 1e-4)
mkdir -p gpurun_out
for k in ${KS:-5 6 7 8}; do
  timeout ${TMO:-600} python tools/config2_search.py --k $k --eps0 ${EPS0:-1e-4} --budget ${BUDGET:-400} >> gpurun_out/config2_rest.jsonl 2>> gpurun_out/config2_rest.err; echo "k=$k rc=$?"
done
grep summary gpurun_out/config2_rest.jsonl | cut -c1-220
tail -5 gpurun_out/config2_rest.err
