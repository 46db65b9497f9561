# ncu full capture (+source) of one kernel at C4 -> gpurun_out/<name>.ncu-rep ; args: regex name [bench args]
k=$1; o=$2; shift 2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" $NCU_EXTRA -c 1 -o gpurun_out/$o -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/$o.log 2>&1; echo ncu $?
