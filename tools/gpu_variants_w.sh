# A/B of prebuilt libppgpu.so variants under _var/<name>/ (LD_PRELOAD) on a workload ($WLV, default the config-2 shape)
mkdir -p gpurun_out
for v in ${VARS:-D}; do
  LD_PRELOAD=$PWD/_var/$v/libppgpu.so timeout 600 python bench.py --workload ${WLV:-config2_pi4_eps1e-4_t8} --no-cpu-baseline --steps 5 > gpurun_out/varw_$v.json 2> gpurun_out/varw_$v.err
  python -c "
import json
d=json.load(open('gpurun_out/varw_$v.json')); r=d['roofline']
print('$v', 'ms/step', round(d['ms_per_step'],3), 'branch ms', round(r['branch_ms_per_step'],3))"
done
