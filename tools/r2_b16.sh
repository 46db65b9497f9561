for b in 8 16; do for p in tensor direct; do
KDE_BUCKET=$b timeout 200 python bench.py --config C4 --path $p --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B=$b $p', d['ms_per_step'], d['phases_ms'])"
done; done
