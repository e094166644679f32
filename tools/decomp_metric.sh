#!/bin/bash
# sweep-kernel time decomposition per metric (C2): full, epilogue only (1), intersections only (2)
mkdir -p gpurun_out
for m in ${METRICS:-cosine manhattan}; do for d in 0 1 2; do
  SD_ISECT_DEBUG=$d timeout 600 python bench.py --workload ${WL:-c2} --metric $m --no-cpu --no-extra --no-check --steps 5 > gpurun_out/decm_${m}_$d.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/decm_${m}_$d.json').read().strip().splitlines()[-1])
print('$m debug=$d step', round(d['ms_per_step'],3), 'kernel', (d.get('roofline') or {}).get('kernel_ms'))"
done; done
