# ncu capture of one kernel: tools/r2_prof.sh <regex> <out-name> <bench args...>
set -x
k=$1; o=$2; shift 2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -c 1 -o gpurun_out/$o -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/$o.log 2>&1
tail -3 gpurun_out/$o.log
