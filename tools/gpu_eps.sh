# eps0 > 0 fused-run measurements (gpurun): default vs per-gate launches, and
# the config-0 dense work shape.  Outputs in gpurun_out/.
mkdir -p gpurun_out
T=${T:-10}; EPS=${EPS:-2e-5}
PP_DEBUG=1 timeout 900 python tools/eps_profile.py --eps $EPS --t $T > gpurun_out/eps_spec.jsonl 2> gpurun_out/eps_spec.err; echo "spec rc=$?"
grep -c "discovery round" gpurun_out/eps_spec.err; grep "speculative run" gpurun_out/eps_spec.err | tail -3
PP_NO_SPECULATE=1 timeout 900 python tools/eps_profile.py --eps $EPS --t $T > gpurun_out/eps_pergate.jsonl 2> gpurun_out/eps_pergate.err; echo "pergate rc=$?"
cat gpurun_out/eps_spec.jsonl gpurun_out/eps_pergate.jsonl

