#!/bin/bash
# fp64 epilogue layout check: GPU tests + C2 fp64 lines + the fp32 headline
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/f64_pytest.log 2>&1; tail -2 gpurun_out/f64_pytest.log
for m in cosine manhattan; do
  timeout 600 python bench.py --workload c2 --metric $m --dtype float64 --no-cpu --no-extra > gpurun_out/f64_$m.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/f64_$m.json').read().strip().splitlines()[-1])
print('f64 $m', round(d['ms_per_step'],3), d['roofline'].get('kernel_ms'), d.get('agreement',{}).get('parity_rule_cells_failed'))"
done
timeout 600 python bench.py --workload c2 --no-cpu --no-extra > gpurun_out/f32_cos.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/f32_cos.json').read().strip().splitlines()[-1])
print('f32 cosine', round(d['ms_per_step'],3), d['roofline'].get('kernel_ms'), d.get('agreement',{}).get('parity_rule_cells_failed'))"
