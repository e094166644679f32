mkdir -p gpurun_out
for f in 0 1; do for w in c2 c3 c5 c4; do
  SD_ISECT_FLAT=$f timeout 600 python bench.py --workload $w --no-cpu --steps 5 > gpurun_out/ab_${w}_$f.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_${w}_$f.json').read().strip().splitlines()[-1])
print('flat=$f $w', {k:round(v['ms_per_step'],3) for k,v in d['per_metric'].items()})"
done; done
