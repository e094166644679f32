for pl in 0 1; do
  SD_ISECT_PLAN=$pl timeout 600 python bench.py --workload c2 --no-cpu --steps 5 > gpurun_out/plan_$pl.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/plan_$pl.json').read().strip().splitlines()[-1])
print('plan=$pl', {k:round(v['ms_per_step'],3) for k,v in d['per_metric'].items()}, d['roofline']['kernel_ms'])"
done
