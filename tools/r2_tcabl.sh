# TC kernel ablations at C4 (timing only; results are wrong when KDE_TC5_ABL is set)
for v in 0 1 2 3 4 5 6 7; do
  KDE_TC5_ABL=$v timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/abl.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/abl.json').read().strip().splitlines()[-1]); print('abl $v main_ms', d['phases_ms']['main_ms'])
" 2>/dev/null || echo "abl $v failed"
done
