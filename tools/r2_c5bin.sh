timeout 300 python -m pytest tests -x -q -m gpu -k "binning" 2>&1 | tail -1
for h in 1 4 8; do echo "C5 h=$h $(timeout 200 python bench.py --config C5 --hpx $h --path tensor --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['phases_ms'])")"; done
echo "C4 $(timeout 200 python bench.py --path tensor --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['phases_ms'])")"
