timeout 300 python -m pytest tests -x -q -m gpu -k "binning" 2>&1 | tail -1
for c in C2 C4 C5; do echo "$c $(timeout 200 python bench.py --config $c --path tensor --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['phases_ms']['bin_ms'])")"; done
