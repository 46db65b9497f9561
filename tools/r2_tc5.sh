export KDE_DEBUG=1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
unset KDE_DEBUG
timeout 600 python -m pytest tests -x -q -m gpu -k "tensor or cutoff9 or C5" > gpurun_out/it_pytest.log 2>&1; tail -2 gpurun_out/it_pytest.log
for c in C2 C4; do for t5 in 1 0; do echo "tc5=$t5 $c $(KDE_TC5=$t5 timeout 200 python bench.py --config $c --path tensor --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phases_ms'])")"; done; done
