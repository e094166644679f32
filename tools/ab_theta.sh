for th in ${THETAS:-2000 3690 6000 10000}; do
  SD_HEAVY_DEG=$th timeout 600 python bench.py --workload c2 --no-cpu --no-extra --steps 5 > gpurun_out/th_$th.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/th_$th.json').read().strip().splitlines()[-1])
print('theta=$th', round(d['ms_per_step'],3), d['roofline']['kernel_ms'])"
done
