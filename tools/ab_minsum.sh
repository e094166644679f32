mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "manhattan or minsum or hybrid or coo" > gpurun_out/ms_pytest.log 2>&1; tail -2 gpurun_out/ms_pytest.log
timeout 600 python bench.py --workload c2 --metric manhattan --no-cpu --no-extra > gpurun_out/ms_bench.json 2>gpurun_out/ms_bench.err; tail -1 gpurun_out/ms_bench.json | cut -c1-300
timeout 300 python tools/timeline.py --metric manhattan 2>/dev/null | grep -v "^ *[0-9.]* *[0-9.]* *[0-9.]* *[0-9]* *step$" > gpurun_out/ms_timeline.txt; grep -E "hminsum|isect|span" gpurun_out/ms_timeline.txt
