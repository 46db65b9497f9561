python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py -x -q -k "bin or shard or C1 or hot or stats" > gpurun_out/pytest_bin.log 2>&1; echo pytest $?
tail -2 gpurun_out/pytest_bin.log
rm -f gpurun_out/check.jsonl
python bench.py --no-cpu-baseline >> gpurun_out/check.jsonl 2>/dev/null
python bench.py --config C4 --no-cpu-baseline --steps 10 >> gpurun_out/check.jsonl 2>/dev/null
python bench.py --config C5 --hpx 1 --no-cpu-baseline --steps 5 >> gpurun_out/check.jsonl 2>/dev/null
python - <<'PY'
import json
for l in open("gpurun_out/check.jsonl"):
    d = json.loads(l)
    print(d["config"]["config"], d["config"]["path"], d["ms_per_step"], d.get("phases_ms"))
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_tensor.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
