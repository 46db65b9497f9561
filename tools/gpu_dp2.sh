python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1200 python -m pytest tests/test_gpu_dp.py tests/test_gpu_parity.py -x -q -k "dp or bin or C1 or hot" > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -2 gpurun_out/pytest_gpu.log
python - > gpurun_out/dp_timing.txt 2>&1 <<'PY'
import time, numpy as np, torch, aisgen
from paper_2004_13653_b200 import kde_dp
c = aisgen.generate("islands", 20_000_000, aisgen.SEED_BASE + 3)
x, y, o = (torch.from_numpy(a).cuda() for a in (c.x, c.y, np.asarray(c.traj_offsets, np.int64)))
for eps in (0.5, 1.0, 5.0):
    kde_dp(x, y, o, eps); torch.cuda.synchronize()
    t = time.perf_counter(); _, nk, r = kde_dp(x, y, o, eps); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"kde_dp eps={eps} m: {dt*1e3:.2f} ms wall, 20M points ({len(c.traj_offsets)-1} trajectories), kept {nk} (compression {100*(1-nk/20e6):.2f}%), {r} rounds")
import oracle
t = time.perf_counter(); oracle.dp_compress(c.x, c.y, c.traj_offsets, 1.0)
print(f"oracle serial DP eps=1.0 m: {(time.perf_counter()-t)*1e3:.1f} ms (1 host core)")
PY
cat gpurun_out/dp_timing.txt
rm -f gpurun_out/check.jsonl
python bench.py --no-cpu-baseline >> gpurun_out/check.jsonl 2>/dev/null
python bench.py --config C4 --no-cpu-baseline --steps 10 >> gpurun_out/check.jsonl 2>/dev/null
python - <<'PY'
import json
for l in open("gpurun_out/check.jsonl"):
    d = json.loads(l)
    print(d["config"]["config"], d["config"]["path"], d["ms_per_step"], d.get("phases_ms"))
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_tensor.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
