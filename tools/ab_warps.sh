export SD_LIB=$PWD/paper_2104_06357_b200/libsemidist_b200_w16.so
for t in 3584 4096; do for w in c2 c3 c5; do
  SD_TILE=$t timeout 900 python bench.py --workload $w --no-cpu --no-extra --steps 5 > gpurun_out/w16_${t}_$w.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/w16_${t}_$w.json').read().strip().splitlines()[-1])
print('w16 tile=$t $w', round(d['ms_per_step'],3))"
done; done
