set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_config1.json 2> gpurun_out/bench_config1.err; echo "bench rc=$?"
cat gpurun_out/bench_config1.json; tail -3 gpurun_out/bench_config1.err
PP_TRACE=1 timeout 600 python tools/profile_run.py config1 --warm
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_config1_warm.csv python tools/profile_run.py config1 --warm > gpurun_out/ncu1.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_config1_warm.csv
