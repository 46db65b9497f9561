# binning profile at C4: launch list with DRAM bytes + one full capture of convert / pass / gather
mkdir -p gpurun_out/bp; F=gpurun_out/bp
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $F/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"os_pass|bin_convert|gather_offsets|os_scan" -c 5 -o $F/bin -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $F/full.log 2>&1; echo ncu2 $?
