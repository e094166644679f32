#!/bin/bash
# ncu full captures (one launch each) of the fused kernel on selected workloads.
mkdir -p gpurun_out
for spec in ${NCU_SPECS:-c2:cosine}; do
  w=${spec%%:*}; m=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:isect_kernel -s 1 -c 1 \
    -o gpurun_out/prof_${w}_${m} python bench.py --workload $w --metric $m --steps 1 --warmup 1 --no-cpu --no-extra \
    > gpurun_out/ncu_${w}_${m}.log 2>&1
  tail -2 gpurun_out/ncu_${w}_${m}.log
done
