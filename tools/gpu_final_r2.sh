# round-2 final refresh: GPU suite, bench lines (default + config1 + config2 shape), reference arm,
# DRAM traffic, launch list and one full ncu capture of the top dense launch; outputs in gpurun_out/final/
mkdir -p gpurun_out/final
P=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > $P/gpu.txt
timeout 1800 python -m pytest tests -m gpu -x -q > $P/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $P/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $P/smoke.log
timeout 900 python tools/traffic.py config0_t10 config1 config2_pi4_eps1e-4_t8 > $P/traffic.log 2>&1; echo "traffic rc=$?"; cp profiles/branch_traffic.json $P/
timeout 900 python bench.py > $P/bench_config0_t10.json 2> $P/bench_config0_t10.err; echo "bench default rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $P/bench_ref_config0_t10.json 2> $P/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --workload config1 --steps 20 > $P/bench_config1.json 2> $P/bench_config1.err; echo "bench config1 rc=$?"
timeout 900 python bench.py --workload config2_pi4_eps1e-4_t8 --steps 5 > $P/bench_config2_pi4_eps1e-4_t8.json 2> $P/bench_c2.err; echo "bench config2 shape rc=$?"
for W in config0_t10; do
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_${W}.csv python tools/profile_run.py $W --warm > /dev/null 2>&1; echo "launches $W rc=$?"
  python tools/launch_summary.py $P/launches_${W}.csv > $P/launches_${W}_summary.txt
done
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_dense_sublayer --launch-skip 9 --launch-count 1 -o $P/full_dense_config0_t10 python tools/profile_run.py config0_t10 --warm > /dev/null 2>&1; echo "full rc=$?"
python tools/ncu_summary.py $P/full_dense_config0_t10.ncu-rep > $P/full_dense_config0_t10_summary.txt
python - <<'PY'
import json
for f in ["bench_config0_t10","bench_ref_config0_t10","bench_config1","bench_config2_pi4_eps1e-4_t8"]:
    try:
        d=json.load(open(f"gpurun_out/final/{f}.json")); r=d.get("roofline") or {}
        print(f, "ms/step", round(d["ms_per_step"],3), "value %.3e"%d["value"], "e2e %.3e"%d["e2e"]["value"], "branch ms", r.get("branch_ms_per_step"), "frac", r.get("frac"), "traffic", r.get("traffic"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e: print(f, "ERR", e)
PY
