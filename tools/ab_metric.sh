for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset SD_LIB; else export SD_LIB=$PWD/paper_2104_06357_b200/libsemidist_b200_$v.so; fi
  for m in ${METRICS:-euclidean manhattan}; do
    timeout 600 python bench.py --workload c2 --metric $m --no-cpu --no-extra --steps 5 > gpurun_out/abm_${v}_$m.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/abm_${v}_$m.json').read().strip().splitlines()[-1])
print('$v $m', round(d['ms_per_step'],3), (d.get('roofline') or {}).get('kernel_ms'))"
  done
done
