python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -2 gpurun_out/pytest_gpu.log
rm -f gpurun_out/check.jsonl
python bench.py --no-cpu-baseline >> gpurun_out/check.jsonl 2>/dev/null
python bench.py --path direct --no-cpu-baseline >> gpurun_out/check.jsonl 2>/dev/null
python bench.py --config C3 --no-cpu-baseline --steps 10 >> gpurun_out/check.jsonl 2>/dev/null
python bench.py --config C3 --path direct --no-cpu-baseline --steps 10 >> gpurun_out/check.jsonl 2>/dev/null
python bench.py --config C4 --no-cpu-baseline --steps 10 >> gpurun_out/check.jsonl 2>/dev/null
python bench.py --config C4 --path direct --no-cpu-baseline --steps 10 >> gpurun_out/check.jsonl 2>/dev/null
python - <<'PY'
import json
for l in open("gpurun_out/check.jsonl"):
    d = json.loads(l)
    print(d["config"]["config"], d["config"]["path"], d["ms_per_step"], d["step_ms_rank0"], d["phases_ms"])
PY
echo done
