for b in 25 60 123 245; do
  SD_ISECT_BAND=$b timeout 600 python bench.py --workload c5 --no-cpu --no-extra --steps 5 > gpurun_out/kb_$b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/kb_$b.json').read().strip().splitlines()[-1])
print('kband=$b', round(d['ms_per_step'],3))"
done
