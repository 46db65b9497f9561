python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for sc in 0 1 0 1; do
  for cfg in C2 C4; do
    KDE_SEG_HALF=$sc python bench.py --config $cfg --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$cfg half=$sc', d['ms_per_step'], d['phases_ms'])"
  done
done
echo done
