mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_native_sharded.py tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q --timeout 500 --tb=short -rf -k "native or scale or ledgers or speculative or deferred or truncated" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error|assert" gpurun_out/pytest_gpu.log | tail -24
PP_NO_SPECULATE=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_eps_pergate.csv python tools/eps_profile.py --eps 2e-5 --t 8 > gpurun_out/ncu_pergate.log 2>&1; echo "ncu pergate rc=$?"
python tools/launch_summary.py gpurun_out/launches_eps_pergate.csv | head -25
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_eps_spec.csv python tools/eps_profile.py --eps 2e-5 --t 8 > gpurun_out/ncu_spec.log 2>&1; echo "ncu spec rc=$?"
python tools/launch_summary.py gpurun_out/launches_eps_spec.csv | head -25
