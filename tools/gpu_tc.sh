# tensor-core kernel iteration: parity + C2 bench + ncu full of the TC kernel
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor" > gpurun_out/pytest_tc.log 2>&1; echo pytest_tc $?
tail -3 gpurun_out/pytest_tc.log
rm -f gpurun_out/bench_tc.jsonl
for p in tensor tensor_split; do
  timeout 300 python bench.py --path $p --no-cpu-baseline --steps 20 --warmup 3 >> gpurun_out/bench_tc.jsonl 2>>gpurun_out/bench_tc.err
done
timeout 300 python bench.py --config C3 --path tensor --no-cpu-baseline --steps 10 --warmup 3 >> gpurun_out/bench_tc.jsonl 2>>gpurun_out/bench_tc.err
timeout 300 python bench.py --config C4 --path tensor --no-cpu-baseline --steps 10 --warmup 3 >> gpurun_out/bench_tc.jsonl 2>>gpurun_out/bench_tc.err
ncu --set full --clock-control none --import-source on -k regex:tc_splat_kernel -c 1 -o gpurun_out/c2_tensor -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
