#!/bin/bash
# One gpurun call: tests, bench (JSON line), ncu launch list and a full capture
# of the fused kernel.  Output under gpurun_out/ (scratch); summaries are copied
# into profiles/ by tools/summarize_ncu.py.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --extra > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:isect_kernel -s 1 -c 1 -o gpurun_out/prof_isect python bench.py --steps 1 --warmup 1 --no-cpu --extra > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
