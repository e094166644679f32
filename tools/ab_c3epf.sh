#!/bin/bash
# pairwise epilogue groups in flight on C3: 4 (default) vs 2
mkdir -p gpurun_out
for v in e2 default; do
  if [ "$v" = default ]; then unset SD_LIB; else export SD_LIB=$PWD/paper_2104_06357_b200/libsemidist_b200_$v.so; fi
  for m in jensenshannon canberra kl; do
    timeout 600 python bench.py --workload c3 --metric $m --no-cpu --no-extra --steps 5 > gpurun_out/c3e_${v}_$m.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/c3e_${v}_$m.json').read().strip().splitlines()[-1])
print('$v $m', round(d['ms_per_step'],3), d.get('agreement',{}).get('parity_rule_cells_failed'))"
  done
done
