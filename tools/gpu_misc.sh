python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo pytest_dist $?
tail -3 gpurun_out/pytest_dist.log
rm -f gpurun_out/bench_radial.jsonl
for kn in gaussian epanechnikov cosine; do timeout 300 python bench.py --config C3 --kernel $kn --radial --path direct --no-cpu-baseline --steps 10 >> gpurun_out/bench_radial.jsonl 2>>gpurun_out/bench_radial.err; done
python - <<'PY'
import json
for l in open("gpurun_out/bench_radial.jsonl"):
    d = json.loads(l); r = d["roofline"]
    print(d["config"]["kernel"], d["config"]["form"], d["ms_per_step"], "%.3g" % d["value"], r["bound"], r["achieved"], r["peak"], r["unit"], r["frac"])
PY
tail -3 gpurun_out/bench_radial.err
echo done
