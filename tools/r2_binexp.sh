# binning A/B experiments at C4 (bench phases); args: list of "ENV=VAL" settings ("-" = none)
for v in "$@"; do
  if [ "$v" = "-" ]; then e=""; else e="$v"; fi
  env $e timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/be.json 2> gpurun_out/be.err
  python -c "
import json
try:
    d=json.loads(open('gpurun_out/be.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['phases_ms'])
except Exception as ex: print('$v FAILED', ex, open('gpurun_out/be.err').read()[-800:])
"
done
