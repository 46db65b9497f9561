for b in 8 16; do for c in C2 C4; do
echo "B=$b $c $(KDE_BUCKET=$b timeout 200 python bench.py --config $c --path tensor --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phases_ms'])")"
done; done
