for t in 2048 8192; do for w in c5 c3; do
  SD_TILE=$t timeout 900 python bench.py --workload $w --no-cpu --no-extra --steps 3 > gpurun_out/tile_${t}_$w.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/tile_${t}_$w.json').read().strip().splitlines()[-1])
print('tile=$t $w', round(d['ms_per_step'],3))"
done; done
