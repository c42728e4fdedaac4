# One GPU pass (gpurun): the -m gpu suite, the default bench line, the
# reference arm.  Outputs land in gpurun_out/.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ -n "${REF_ARM:-}" ]; then
  timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
  cat gpurun_out/bench_ref.json
fi
