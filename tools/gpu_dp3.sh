python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/pytest_dp.log 2>&1; echo pytest_dp $?
tail -3 gpurun_out/pytest_dp.log
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
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dp.csv python tools/dp_prof.py > gpurun_out/dp_prof.log 2>&1
echo done
