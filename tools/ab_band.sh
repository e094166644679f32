for b in ${BANDS:-5 10 20 40}; do
  SD_ISECT_BAND=$b timeout 600 python bench.py --workload c2 --no-cpu --no-extra --steps 5 > gpurun_out/band_$b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/band_$b.json').read().strip().splitlines()[-1])
print('band=$b', round(d['ms_per_step'],3), d['roofline']['kernel_ms'])"
done
