# round-end evidence: full GPU suite, bench lines for every config/path, reference arm,
# DP timing, ncu launch lists + full captures of the dominant kernels
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c2_default.json 2> gpurun_out/bench_c2_default.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_c2_reference.json 2>&1
rm -f gpurun_out/bench_all.jsonl
for p in direct tensor_split; do python bench.py --path $p --no-cpu-baseline >> gpurun_out/bench_all.jsonl 2>>gpurun_out/bench_all.err; done
for c in C1 C3 C4; do for p in tensor direct; do timeout 300 python bench.py --config $c --path $p --no-cpu-baseline --steps 10 --warmup 3 >> gpurun_out/bench_all.jsonl 2>>gpurun_out/bench_all.err; done; done
for h in 1 4 16 32; do for p in tensor direct; do timeout 600 python bench.py --config C5 --hpx $h --path $p --no-cpu-baseline --steps 5 --warmup 3 >> gpurun_out/bench_all.jsonl 2>>gpurun_out/bench_all.err; done; done
for c in C2 C4; do timeout 300 python bench.py --config $c --path snap --steps 10 --warmup 3 >> gpurun_out/bench_all.jsonl 2>>gpurun_out/bench_all.err; done
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
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_tensor.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_direct.csv python bench.py --path direct --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_snap.csv python bench.py --path snap --steps 5 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_splat_kernel -c 1 -o gpurun_out/c2_tensor -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^splat_kernel|segreduce|combine|rs_downsweep|bin_convert|gather_kernel" -c 8 -o gpurun_out/c2_direct -f python bench.py --path direct --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dp.csv python tools/dp_prof.py > /dev/null 2>&1
ls gpurun_out
echo done
