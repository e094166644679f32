#!/bin/bash
# One gpurun call producing the round's evidence: GPU tests, smoke, the default
# bench line + every BASELINE workload, the reference arm, the ncu launch list
# of the default bench, and ncu --set full text exports of the fused kernel and
# the hybrid kernels.  Output under gpurun_out/ (scratch); copy summaries into
# profiles/ with tools/summarize_evidence.py.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for w in c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w --no-cpu > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1
for k in isect_kernel hgemm hgather heavy_rows; do NCU_KERNEL=$k bash tools/gpu_ncu.sh > /dev/null 2>&1; done
ls gpurun_out
