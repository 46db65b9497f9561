# os_pass kernel times (ncu launch list) under env settings
for v in "$@"; do
  if [ "$v" = "-" ]; then e=""; else e="$v"; fi
  env $e timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"os_pass|bin_convert|gather" -c 8 --csv python bench.py --no-cpu-baseline --steps 1 --warmup 3 2>/dev/null | grep -E "os_pass|bin_convert|gather" | awk -F'","' -v v="$v" '{print v, $5, $(NF-2), $NF}' | tail -8
done
