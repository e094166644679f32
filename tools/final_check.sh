#!/bin/bash
# full GPU suite + smoke + the C2 lines (manhattan included) after the last change
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/final_pytest.log 2>&1; tail -1 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
python -c "
import json; d=json.loads(open('gpurun_out/final_c2.json').read().strip().splitlines()[-1])
print('c2', round(d['ms_per_step'],3), d['roofline'].get('frac'), d.get('agreement',{}).get('parity_rule_cells_failed'))
for k,v in d['per_metric'].items(): print('  ',k, round(v['ms_per_step'],3))
for k,v in d['per_metric_f64'].items(): print('   f64',k, round(v['ms_per_step'],3))"
