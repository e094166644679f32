#!/bin/bash
# time decomposition of the fused kernel: full, sweep only, epilogue only
mkdir -p gpurun_out
for w in ${WL:-c2 c5}; do for d in ${DBG:-0 1 2}; do
  SD_ISECT_DEBUG=$d timeout 600 python bench.py --workload $w --no-cpu --no-extra --steps 5 > gpurun_out/dec_${w}_$d.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/dec_${w}_$d.json').read().strip().splitlines()[-1])
print('$w debug=$d', round(d['ms_per_step'],3), (d.get('roofline') or {}).get('kernel_ms'))"
done; done
python tools/host_overhead.py 2>&1 | tail -3
