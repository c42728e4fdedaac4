for v in "" "PP_NO_DENSE_KERNEL=1" "PP_DENSE_CAREFUL=1" "PP_NO_DENSE_KERNEL=1 PP_DENSE_CAREFUL=1"; do
  env $v timeout 300 python bench.py --workload config1 --no-cpu-baseline --steps 10 > gpurun_out/c1.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/c1.json')); r=d['roofline']
print('$v', 'ms/step', round(d['ms_per_step'],3), 'branch ms', round(r['branch_ms_per_step'],3), 'launches', d['gpu_launches'])"
done
