#!/bin/bash
# A/B of the straight-line epilogue's 128-cell groups in flight (SD_ISECT_EPF)
mkdir -p gpurun_out
for v in default epf2 epf8 default; do
  if [ "$v" = default ]; then unset SD_LIB; else export SD_LIB=$PWD/paper_2104_06357_b200/libsemidist_b200_$v.so; fi
  for spec in c2:cosine c2:manhattan c5:cosine; do
    w=${spec%%:*}; m=${spec##*:}
    timeout 600 python bench.py --workload $w --metric $m --no-cpu --no-extra --steps 5 > gpurun_out/epf_${v}_$w$m.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/epf_${v}_$w$m.json').read().strip().splitlines()[-1])
a=d.get('agreement',{}); print('$v $w $m', round(d['ms_per_step'],3), a.get('parity_rule_cells_failed', a.get('mismatches_outside_ties')))"
  done
done
