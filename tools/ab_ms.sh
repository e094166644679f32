#!/bin/bash
# A/B of the min-sum block's CTA shape (consumer warps x heavy rows per warp)
mkdir -p gpurun_out
for v in ms22; do
  SD_LIB=$PWD/paper_2104_06357_b200/libsemidist_b200_$v.so timeout 600 python -m pytest tests -q -m gpu -x -k "manhattan or minsum" > gpurun_out/ms_$v.log 2>&1; echo "$v tests: $(tail -1 gpurun_out/ms_$v.log)"
done
for v in ms20 ms22; do
  if [ "$v" = default ]; then unset SD_LIB; else export SD_LIB=$PWD/paper_2104_06357_b200/libsemidist_b200_$v.so; fi
  for dt in float32 float64; do
    timeout 600 python bench.py --workload c2 --metric manhattan --dtype $dt --no-cpu --no-extra --steps 5 > gpurun_out/ms_${v}_$dt.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ms_${v}_$dt.json').read().strip().splitlines()[-1])
print('$v $dt', round(d['ms_per_step'],3), d.get('agreement',{}).get('parity_rule_cells_failed'))"
  done
  timeout 300 python tools/timeline.py --metric manhattan 2>/dev/null | grep -E "hminsum"
done
