# repro: config 2, theta_h = 5 pi/16, eps0 = 1.5e-5 ran for 50 minutes without an answer
mkdir -p gpurun_out
PP_DEBUG=1 timeout ${TMO:-240} python tools/config2_search.py --k 5 --eps0 1.5e-5 --budget 1 > gpurun_out/repro_k5.jsonl 2> gpurun_out/repro_k5.err; echo "rc=$?"
grep -c . gpurun_out/repro_k5.err; grep "k=5" gpurun_out/repro_k5.err | tail -4; tail -30 gpurun_out/repro_k5.err | cut -c1-220
