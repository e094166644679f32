#!/bin/bash
# ncu --set full of ONE launch of a kernel per (workload, metric[, dtype]) —
# the timed launch of a 1-step bench run — exported on the box to text (raw
# metrics, source-level SASS counters) so gpurun_out/ stays small.
#   NCU_SPECS="c2:cosine c3:canberra c2:cosine:float64" NCU_KERNEL=isect_kernel bash tools/gpu_ncu.sh
mkdir -p gpurun_out
K=${NCU_KERNEL:-isect_kernel}
for spec in ${NCU_SPECS:-c2:cosine}; do
  IFS=: read -r w m dt <<< "$spec"
  dt=${dt:-float32}
  tag=${w}_${m}_${dt}_${K}
  rep=/tmp/prof_${tag}
  rm -f $rep.ncu-rep
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$K -s ${NCU_SKIP:-1} -c 1 \
    -o $rep python bench.py --workload $w --metric $m --dtype $dt --steps 1 --warmup 1 --no-cpu --no-extra \
    --no-check > gpurun_out/ncu_${tag}.log 2>&1
  echo "ncu $tag rc=$?"
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/raw_${tag}.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${tag}.csv 2>/dev/null
  rm -f $rep.ncu-rep
done
