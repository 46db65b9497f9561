set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench $?
python bench.py --path direct --no-cpu-baseline > gpurun_out/bench_c2_direct.json 2>&1
for c in C3 C4; do for p in tensor direct; do python bench.py --config $c --path $p --no-cpu-baseline --steps 10 --warmup 3 >> gpurun_out/bench_configs.jsonl 2>>gpurun_out/bench_configs.err; done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_tensor.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_direct.csv python bench.py --path direct --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:splat_kernel -c 2 -o gpurun_out/c2_tensor -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:splat_kernel -c 2 -o gpurun_out/c2_direct -f python bench.py --path direct --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
