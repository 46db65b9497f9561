# round-2 iteration on the GPU: tools/r2_iter.sh "<pytest -k expr>" "<bench configs>" "<paths>"
sel=$1; cfgs=${2:-"C2 C4"}; paths=${3:-"tensor"}
if [ -n "$sel" ]; then timeout 900 python -m pytest tests -x -q -m gpu -k "$sel" > gpurun_out/it_pytest.log 2>&1; tail -3 gpurun_out/it_pytest.log; fi
for c in $cfgs; do for p in $paths; do
  timeout 240 python bench.py --config $c --path $p --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/it_${c}_$p.json 2> gpurun_out/it_${c}_$p.err
  python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/it_${c}_$p.json').read().strip().splitlines()[-1]); r=d['roofline']
    print('$c $p step', d['ms_per_step'], d['phases_ms'], 'frac', r['frac'])
except Exception as e: print('$c $p FAILED', e); print(open('gpurun_out/it_${c}_$p.err').read()[-1500:])
"
done; done
