# Round-2 evidence on one B200: build + smoke, the GPU test suite, bench lines (default C4 with
# cpu_baseline; every config x path; DP-compressed C4), the reference arm, band projection,
# ncu launch lists + full captures of the dominant kernels at C4, SASS instruction counts.
set -x
mkdir -p gpurun_out/final
F=gpurun_out/final
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $F/smoke.log 2>&1; echo smoke $?
tail -1 $F/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $F/pytest_gpu.log 2>&1; echo pytest $?
tail -3 $F/pytest_gpu.log
python bench.py > $F/bench_default.json 2> $F/bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > $F/bench_reference.json 2>&1
rm -f $F/bench_all.jsonl
for p in direct tensor_split; do timeout 600 python bench.py --path $p --cpu-seconds 5 >> $F/bench_all.jsonl 2>>$F/bench_all.err; done
for e in 0.5 1.0 5.0; do for p in tensor direct; do timeout 600 python bench.py --dp-eps $e --path $p --cpu-seconds 5 >> $F/bench_all.jsonl 2>>$F/bench_all.err; done; done
for c in C1 C2 C3; do for p in tensor direct; do timeout 300 python bench.py --config $c --path $p --cpu-seconds 5 --steps 10 --warmup 3 >> $F/bench_all.jsonl 2>>$F/bench_all.err; done; done
for h in 1 4 16 32; do for p in tensor direct; do timeout 600 python bench.py --config C5 --hpx $h --path $p --cpu-seconds 5 --steps 5 --warmup 3 >> $F/bench_all.jsonl 2>>$F/bench_all.err; done; done
for c in C2 C4; do timeout 300 python bench.py --config $c --path snap --steps 10 --warmup 3 >> $F/bench_all.jsonl 2>>$F/bench_all.err; done
timeout 900 python tools/band_projection.py --config C4 --path tensor > $F/band_projection_c4.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $F/launches_c4_tensor.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $F/launches_c4_direct.csv python bench.py --path direct --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc5_kernel|combine_strip_kernel|combine_kernel|os_pass_kernel|bin_convert|gather_offsets" -c 6 -o $F/c4_tensor -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^splat_kernel|segreduce" -c 2 -o $F/c4_direct -f python bench.py --path direct --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for f in paper_2004_13653_b200/build/*.o; do echo "== $f"; cuobjdump -sass $f | grep -oE "UTCHMMA|UTCBAR|LDTM|UTMALDG|UBLKCP|FFMA2|FMUL2|FFMA |MUFU.EX2|SYNCS[.A-Z]*" | sort | uniq -c; done > $F/sass_counts.txt 2>&1
ls -la $F
echo done
