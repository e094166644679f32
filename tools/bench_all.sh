#!/bin/bash
# Every BASELINE config on one GPU (JSON lines under gpurun_out/bench_<wl>.json).
mkdir -p gpurun_out
for wl in c1 c2 c3 c4 c5; do
  extra=""
  case $wl in c3|c4) extra="--no-cpu";; esac
  timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --ref-budget 10 $extra > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
  echo "$wl rc=$? $(tail -c 300 gpurun_out/bench_$wl.json | head -c 0)"; tail -2 gpurun_out/bench_$wl.err
done
