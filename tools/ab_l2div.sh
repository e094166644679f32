for dv in 1 5; do for w in c2 c3 c5; do
  SD_ISECT_L2_DIV=$dv timeout 600 python bench.py --workload $w --no-cpu --no-extra --steps 5 > gpurun_out/div_${dv}_$w.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/div_${dv}_$w.json').read().strip().splitlines()[-1])
print('div=$dv $w', round(d['ms_per_step'],3))"
done; done
