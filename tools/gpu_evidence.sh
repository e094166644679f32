#!/bin/bash
# One gpurun call producing a round's evidence (scratch under gpurun_out/;
# copy into profiles/ with `python tools/summarize_evidence.py <tag>`):
# GPU tests, smoke, the default bench line + every BASELINE workload (CPU
# baseline and oracle agreement included), the reference arm, the ncu launch
# list of the default bench, ncu --set full of the sweep kernel for every
# workload/metric, and of the hybrid kernels on C2.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > gpurun_out/smi.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
fi
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -1 gpurun_out/bench_c2.err
for w in ${WORKLOADS:-c1 c3 c4 c5}; do
  timeout 1200 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  tail -1 gpurun_out/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-check > /dev/null 2>&1
if [ -z "$SKIP_NCU" ]; then
  NCU_SPECS=${NCU_SPECS:-"c2:cosine c2:euclidean c2:manhattan c2:cosine:float64 c3:canberra c3:chebyshev c3:jensenshannon c3:kl c5:cosine"} \
    bash tools/gpu_ncu.sh
  for k in dense_tc hgather heavy_rows; do NCU_SPECS=c2:cosine NCU_KERNEL=$k bash tools/gpu_ncu.sh; done
  for k in hminsum hgather; do NCU_SPECS=c2:manhattan NCU_KERNEL=$k bash tools/gpu_ncu.sh; done
  NCU_SPECS="c4:hellinger c4:jaccard" NCU_KERNEL=dense_tc bash tools/gpu_ncu.sh
  # compute-sanitizer is closed on this pool since r02e (runs under it left GPUs needing a reset); last logs: profiles/r02d_sanitize_*.txt
  timeout 120 python tools/hbm_probe.py > gpurun_out/hbm_probe.json 2>&1
fi
for m in cosine manhattan; do timeout 300 python tools/timeline.py --metric $m 2>/dev/null | grep -v "^ *[0-9.]* *[0-9.]* *[0-9.]* *[0-9]* *step$" > gpurun_out/timeline_c2_$m.txt; done
timeout 300 python tools/timeline.py --metric cosine --queries 1250 2>/dev/null | grep -v "^ *[0-9.]* *[0-9.]* *[0-9.]* *[0-9]* *step$" > gpurun_out/timeline_c2_cosine_q1250.txt
timeout 300 python tools/timeline.py --workload c5 --steps 2 2>/dev/null | grep -v "^ *[0-9.]* *[0-9.]* *[0-9.]* *[0-9]* *step$" > gpurun_out/timeline_c5_cosine.txt
ls gpurun_out | wc -l
