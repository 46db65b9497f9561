for st in 520 1100; do for r in 0; do for c in C4 C5; do
KDE_RS_STAGED=$st KDE_RS_ROUNDS=$r timeout 200 python bench.py --config $c --path tensor --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('staged<=$st rounds=$r $c bin', d['phases_ms']['bin_ms'])"
done; done; done
