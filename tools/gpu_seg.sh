python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for sc in 1 2 4; do
  for cfg in C2 C4; do
    KDE_SEG_SCALE=$sc python bench.py --config $cfg --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$cfg seg x$sc', d['ms_per_step'], d['phases_ms'])"
  done
done
echo done
