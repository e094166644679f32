#!/bin/bash
# ncu launch list (per-kernel durations) of one bench configuration
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG:-x}.csv \
  python bench.py ${BENCH_ARGS:---steps 2 --warmup 1 --no-cpu --no-extra} > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_${TAG:-x}.csv | head -25
