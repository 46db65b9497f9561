set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --config C4 --path tensor --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2base_c4_tensor.json 2> gpurun_out/r2base_c4_tensor.err
timeout 600 python bench.py --config C4 --path direct --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2base_c4_direct.json 2> gpurun_out/r2base_c4_direct.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2base_launches_c4_tensor.csv python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_splat_kernel -c 1 -o gpurun_out/r2base_c4_tensor -f python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"rs_downsweep|bin_convert|gather_kernel|offsets_kernel|rs_upsweep" -c 8 -o gpurun_out/r2base_c4_bin -f python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
