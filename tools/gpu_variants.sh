# A/B of prebuilt libppgpu.so variants under _var/<name>/ (LD_PRELOAD), bench config0_t10 without the CPU leg
mkdir -p gpurun_out
for v in ${VARS:-A C D}; do
  LD_PRELOAD=$PWD/_var/$v/libppgpu.so PP_DEBUG=1 timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  grep -m1 "dense CTAs" gpurun_out/var_$v.err
  python -c "
import json
d=json.load(open('gpurun_out/var_$v.json')); r=d['roofline']
print('$v', 'ms/step', round(d['ms_per_step'],3), 'branch ms', round(r['branch_ms_per_step'],3), 'frac', round(r['frac'],4))"
done
