# split-fp16 accuracy mode + warp-private downsweep
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -5 gpurun_out/pytest_gpu.log
rm -f gpurun_out/bench_split.jsonl
for p in tensor tensor_split direct; do
  timeout 300 python bench.py --path $p --no-cpu-baseline --steps 20 --warmup 3 >> gpurun_out/bench_split.jsonl 2>>gpurun_out/bench_split.err
done
timeout 300 python bench.py --config C4 --path tensor --no-cpu-baseline --steps 10 --warmup 3 >> gpurun_out/bench_split.jsonl 2>>gpurun_out/bench_split.err
timeout 300 python bench.py --config C5 --hpx 1 --path tensor --no-cpu-baseline --steps 5 --warmup 3 >> gpurun_out/bench_split.jsonl 2>>gpurun_out/bench_split.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_tensor.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
