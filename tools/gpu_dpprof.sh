python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dp.csv python tools/dp_prof.py > gpurun_out/dp_prof.log 2>&1
tail -2 gpurun_out/dp_prof.log
echo done
