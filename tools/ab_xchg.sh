#!/bin/bash
# A/B: epilogue load-and-zero as ld+st (default) vs 16-byte shared exchange (SD_ISECT_XCHG=1)
mkdir -p gpurun_out
for v in default xchg default xchg; do
  if [ "$v" = default ]; then unset SD_LIB; else export SD_LIB=$PWD/paper_2104_06357_b200/libsemidist_b200_$v.so; fi
  for spec in c2:cosine c2:manhattan c5:cosine; do
    w=${spec%%:*}; m=${spec##*:}
    timeout 600 python bench.py --workload $w --metric $m --no-cpu --no-extra --steps 5 > gpurun_out/x_${v}_$w$m.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/x_${v}_$w$m.json').read().strip().splitlines()[-1])
print('$v $w $m', round(d['ms_per_step'],3), (d.get('roofline') or {}).get('kernel_ms'), d.get('agreement',{}).get('parity_rule_cells_failed', d.get('agreement',{}).get('mismatches_outside_ties')))"
  done
done
