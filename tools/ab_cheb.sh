#!/bin/bash
# 16-bit chebyshev masks: GPU tests + the C3 chebyshev lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -k "chebyshev or c3 or golden or namm or kl" > gpurun_out/cheb_pytest.log 2>&1; tail -2 gpurun_out/cheb_pytest.log
for spec in c3:chebyshev; do
  w=${spec%%:*}; m=${spec##*:}
  timeout 900 python bench.py --workload $w --metric $m --no-cpu --no-extra --steps 5 > gpurun_out/cheb_$m.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/cheb_$m.json').read().strip().splitlines()[-1])
print('$m', round(d['ms_per_step'],3), (d.get('roofline') or {}).get('kernel_ms'), d.get('agreement'))"
done
timeout 900 python bench.py --workload c3 --metric chebyshev --dtype float64 --no-cpu --no-extra --steps 3 > gpurun_out/cheb_f64.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/cheb_f64.json').read().strip().splitlines()[-1])
print('cheb f64', round(d['ms_per_step'],3), d.get('agreement'))"
