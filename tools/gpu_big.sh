mkdir -p gpurun_out
timeout 900 python bench.py --workload config0_t10 --no-cpu-baseline --steps 5 > gpurun_out/bench_c0t10.json 2> gpurun_out/bench_c0t10.err; echo "bench0 rc=$?"
cat gpurun_out/bench_c0t10.json; tail -3 gpurun_out/bench_c0t10.err
timeout 900 python bench.py --workload config2_pi4_eps1e-4_t8 --no-cpu-baseline --steps 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench2 rc=$?"
cat gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c0t10_warm.csv python tools/profile_run.py config0_t10 --warm > gpurun_out/ncu0.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_c0t10_warm.csv
