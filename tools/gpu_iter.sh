# one development iteration on the GPU: parity tests, then the default bench
# (no CPU leg) with the dense kernel and, for comparison, with the dense path
# inside k_branch_sublayer (PP_NO_DENSE_KERNEL=1); extra workloads in $WL
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
for W in config0_t10 ${WL:-}; do
  timeout 600 python bench.py --workload $W --no-cpu-baseline --steps 5 > gpurun_out/iter_$W.json 2> gpurun_out/iter_$W.err; echo "bench $W rc=$?"
  python - <<PY
import json
d=json.load(open("gpurun_out/iter_$W.json"))
r=d["roofline"]
print("$W", "ms/step", round(d["ms_per_step"],3), "e2e ms", round(d["e2e"]["ms_per_step"],3), "branch ms", round(r["branch_ms_per_step"],3), "frac", round(r["frac"],4), "launches", d["gpu_launches"])
PY
done
if [ -n "${COMPARE:-}" ]; then
  PP_NO_DENSE_KERNEL=1 timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/iter_nodk.json 2> gpurun_out/iter_nodk.err; echo "bench nodk rc=$?"
  python -c "
import json
d=json.load(open('gpurun_out/iter_nodk.json')); r=d['roofline']
print('no dense kernel: ms/step', round(d['ms_per_step'],3), 'branch ms', round(r['branch_ms_per_step'],3), 'frac', round(r['frac'],4))"
fi
