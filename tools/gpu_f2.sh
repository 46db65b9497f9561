# F2 (all product kernels on the tensor-core path) + sub-window TC (C5 large h)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor" > gpurun_out/pytest_tc.log 2>&1; echo pytest_tc $?
tail -3 gpurun_out/pytest_tc.log
rm -f gpurun_out/bench_c3_kernels.jsonl
for kn in uniform triangular epanechnikov quartic triweight tricube gaussian cosine; do
  for p in tensor direct; do
    timeout 300 python bench.py --config C3 --kernel $kn --path $p --no-cpu-baseline --steps 10 --warmup 3 >> gpurun_out/bench_c3_kernels.jsonl 2>>gpurun_out/bench_c3.err
  done
done
rm -f gpurun_out/bench_c5.jsonl
for h in 1 2 4 8 16 32; do
  for p in tensor direct; do
    timeout 600 python bench.py --config C5 --hpx $h --path $p --no-cpu-baseline --steps 5 --warmup 3 >> gpurun_out/bench_c5.jsonl 2>>gpurun_out/bench_c5.err
  done
done
echo done
