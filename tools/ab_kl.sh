#!/bin/bash
# 16-bit KL counts: GPU tests on KL / chebyshev / C3 + the C3 lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -k "kl or chebyshev or c3 or golden or namm" > gpurun_out/kl_pytest.log 2>&1; tail -2 gpurun_out/kl_pytest.log
for spec in c3:kl c3:chebyshev; do
  w=${spec%%:*}; m=${spec##*:}
  timeout 900 python bench.py --workload $w --metric $m --no-cpu --no-extra --steps 5 > gpurun_out/kl_$m.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/kl_$m.json').read().strip().splitlines()[-1])
print('$m', round(d['ms_per_step'],3), (d.get('roofline') or {}).get('kernel_ms'), d.get('agreement'))"
done
timeout 900 python bench.py --workload c3 --metric kl --dtype float64 --no-cpu --no-extra --steps 3 > gpurun_out/kl_f64.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/kl_f64.json').read().strip().splitlines()[-1])
print('kl f64', round(d['ms_per_step'],3), d.get('agreement'))"
