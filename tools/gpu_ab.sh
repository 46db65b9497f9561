# A/B: radix-sort knobs on C2/C4/C5 (tensor path), snap C2, segreduce change; launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "bin or hot or shard" > gpurun_out/pytest_ab.log 2>&1; echo pytest $?; tail -2 gpurun_out/pytest_ab.log
timeout 300 python -m pytest tests/test_gpu_snap.py -x -q > gpurun_out/pytest_snap.log 2>&1; echo pytest_snap $?; tail -2 gpurun_out/pytest_snap.log
rm -f gpurun_out/ab.txt
for cfg in C2 C4; do
for v in "8 256" "16 256" "8 512" "16 512" "16 1024"; do
  set -- $v
  KDE_RS_ROUNDS=$1 KDE_RS_STAGED=$2 python bench.py --config $cfg --path tensor --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$cfg rounds=$1 staged<=$2', 'step', d['ms_per_step'], 'bin', d['phases_ms']['bin_ms'], 'combine', d['phases_ms']['combine_ms'])" >> gpurun_out/ab.txt
done; done
python bench.py --path snap --steps 20 --warmup 3 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('snap C2 step', d['ms_per_step'])" >> gpurun_out/ab.txt
cat gpurun_out/ab.txt
