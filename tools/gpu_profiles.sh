# round profile refresh: bench lines, reference arm, launch lists, traffic, full captures
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/prof_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/prof_smoke.log | tail -2
mkdir -p gpurun_out/prof
P=gpurun_out/prof
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > $P/gpu.txt
timeout 600 python bench.py > $P/bench_config1.json 2> $P/bench_config1.err; echo "bench1 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $P/bench_ref_config1.json 2> $P/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --workload config0_t10 --no-cpu-baseline --steps 5 > $P/bench_config0_t10.json 2> $P/bench_c0.err; echo "bench0 rc=$?"
timeout 900 python bench.py --workload config2_pi4_eps1e-4_t8 --steps 5 > $P/bench_config2_pi4_eps1e-4_t8.json 2> $P/bench_c2.err; echo "bench2 rc=$?"
timeout 900 python tools/traffic.py config1 config0_t10 config2_pi4_eps1e-4_t8 > $P/traffic.log 2>&1; echo "traffic rc=$?"; cp profiles/branch_traffic.json $P/
for W in config1 config0_t10; do
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_${W}.csv python tools/profile_run.py $W --warm > /dev/null 2>&1; echo "launches $W rc=$?"
  python tools/launch_summary.py $P/launches_${W}.csv > $P/launches_${W}_summary.txt
done
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_branch_sublayer --launch-skip 4 --launch-count 1 -o $P/full_sublayer_config1 python tools/profile_run.py config1 --warm > /dev/null 2>&1; echo "full1 rc=$?"
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_branch_sublayer --launch-skip 9 --launch-count 1 -o $P/full_sublayer_config0_t10 python tools/profile_run.py config0_t10 --warm > /dev/null 2>&1; echo "full0 rc=$?"
