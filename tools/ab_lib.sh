# A/B the default library against variants (SD_LIB) on the c2 cosine bench
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset SD_LIB; else export SD_LIB=$PWD/paper_2104_06357_b200/libsemidist_b200_$v.so; fi
  for w in ${WL:-c2}; do
    timeout 600 python bench.py --workload $w --no-cpu --no-extra --steps 5 > gpurun_out/ab_${v}_$w.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ab_${v}_$w.json').read().strip().splitlines()[-1])
print('$v $w', round(d['ms_per_step'],3), (d.get('roofline') or {}).get('kernel_ms'))"
  done
done
