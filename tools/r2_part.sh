for pp in 128 256 512 1024; do for c in C2 C4; do
echo "part=$pp $c $(KDE_PART_PTS=$pp timeout 200 python bench.py --config $c --path direct --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phases_ms'])")"
done; done
