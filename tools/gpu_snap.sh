python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_snap.py -x -q > gpurun_out/pytest_snap.log 2>&1; echo pytest_snap $?
tail -3 gpurun_out/pytest_snap.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor" > gpurun_out/pytest_tc.log 2>&1; echo pytest_tc $?
tail -3 gpurun_out/pytest_tc.log
rm -f gpurun_out/bench_tc.jsonl
for p in tensor tensor_split; do
  timeout 300 python bench.py --path $p --no-cpu-baseline --steps 20 --warmup 3 >> gpurun_out/bench_tc.jsonl 2>>gpurun_out/bench_tc.err
done
echo done
