# quick state check at HEAD: smoke, full GPU suite, default bench, C4 launch list with DRAM bytes
mkdir -p gpurun_out/head; F=gpurun_out/head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo smoke $?; tail -1 $F/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > $F/pytest_gpu.log 2>&1; echo pytest $?; tail -3 $F/pytest_gpu.log
timeout 600 python bench.py --cpu-seconds 5 > $F/bench_default.json 2> $F/bench_default.err; echo bench $?; cut -c1-600 $F/bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $F/launches_c4_tensor.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu $?
