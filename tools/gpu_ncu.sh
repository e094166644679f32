#!/bin/bash
# ncu full captures (one launch each) of the fused kernel on selected workloads,
# exported on the box to text (raw metrics, source-level SASS counters) so the
# merged gpurun_out/ stays under the copy-back limit.
mkdir -p gpurun_out
for spec in ${NCU_SPECS:-c2:cosine}; do
  w=${spec%%:*}; m=${spec##*:}
  rep=/tmp/prof_${w}_${m}_${NCU_KERNEL:-isect}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-isect_kernel} -s ${NCU_SKIP:-1} -c 1 \
    -o $rep python bench.py --workload $w --metric $m --steps 1 --warmup 1 --no-cpu --no-extra \
    > gpurun_out/ncu_${w}_${m}.log 2>&1
  tail -1 gpurun_out/ncu_${w}_${m}.log
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/raw_${w}_${m}_${NCU_KERNEL:-isect}.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${w}_${m}_${NCU_KERNEL:-isect}.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_${w}_${m}_${NCU_KERNEL:-isect}.csv 2>/dev/null
  ls -la gpurun_out/*_${w}_${m}.csv
done
