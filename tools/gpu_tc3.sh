python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
tail -1 gpurun_out/smoke.log
rm -f gpurun_out/check.jsonl
for i in 1 2; do python bench.py --no-cpu-baseline >> gpurun_out/check.jsonl 2>/dev/null; done
python bench.py --config C4 --no-cpu-baseline --steps 10 >> gpurun_out/check.jsonl 2>/dev/null
python bench.py --config C3 --no-cpu-baseline --steps 10 >> gpurun_out/check.jsonl 2>/dev/null
python - <<'PY'
import json
for l in open("gpurun_out/check.jsonl"):
    d = json.loads(l)
    print(d["config"]["config"], d["config"]["path"], d["ms_per_step"], d.get("phases_ms"))
PY
echo done
