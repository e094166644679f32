#!/bin/bash
# kNN change check: GPU tests (kNN / cosine) + the C5 bench line + timeline
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -k "knn or kneighbors or topk or c5 or cosine or sharded" > gpurun_out/knn_pytest.log 2>&1; tail -2 gpurun_out/knn_pytest.log
timeout 900 python bench.py --workload c5 --no-cpu > gpurun_out/knn_c5.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/knn_c5.json').read().strip().splitlines()[-1])
print('c5', round(d['ms_per_step'],3), d['value'], (d.get('roofline') or {}).get('kernel_ms'), d.get('agreement'))"
timeout 300 python tools/timeline.py --workload c5 --steps 2 2>/dev/null | grep -E "isect|span"
