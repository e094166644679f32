#!/bin/bash
# A/B of the dense gather's rows in flight per lane (SD_HGATHER_UNROLL): 8 (default) vs 4
mkdir -p gpurun_out
for v in hgu4 default hgu4 default; do
  if [ "$v" = default ]; then unset SD_LIB; else export SD_LIB=$PWD/paper_2104_06357_b200/libsemidist_b200_$v.so; fi
  for w in c2 c5; do
    timeout 600 python bench.py --workload $w --no-cpu --no-extra --steps 5 > gpurun_out/hgu_${v}_$w.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/hgu_${v}_$w.json').read().strip().splitlines()[-1])
a=d.get('agreement',{}); print('$v $w', round(d['ms_per_step'],3), a.get('parity_rule_cells_failed', a.get('mismatches_outside_ties')))"
  done
done
