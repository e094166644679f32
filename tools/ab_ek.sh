#!/bin/bash
# kNN epilogue groups in flight: 2 (default) vs 1
mkdir -p gpurun_out
for v in ek1 default ek1 default; do
  if [ "$v" = default ]; then unset SD_LIB; else export SD_LIB=$PWD/paper_2104_06357_b200/libsemidist_b200_$v.so; fi
  timeout 600 python bench.py --workload c5 --no-cpu --no-extra --steps 5 > gpurun_out/ek_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ek_$v.json').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],3), d.get('agreement',{}).get('mismatches_outside_ties'))"
done
