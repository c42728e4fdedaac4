mkdir -p gpurun_out
python tools/_dbg_batches.py 2>&1 | tail -12
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q --timeout 400 --tb=short -rf -k "many_terms or random or speculative or tracked or shards or reinit or scale or ledgers" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error|assert" gpurun_out/pytest_gpu.log | tail -20
T=9 EPS=2e-5 timeout 1200 bash tools/gpu_eps.sh 2>&1 | head -40
