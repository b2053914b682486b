set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/gputests17.log 2>&1; tail -6 gpurun_out/gputests17.log
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) 2>&1 | tail -5
( time timeout 1200 python bench.py > gpurun_out/bench_c4_r17.json ) 2>&1 | tail -4
# ncu: launch list of the same bench command (shares), then one full capture of the ring V_n-only step
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file gpurun_out/launches_c4_r17.csv python bench.py --steps 1 --warmup 3 > gpurun_out/ncu_launches.log 2>&1; tail -2 gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ring -c 2 -o gpurun_out/ring_recur_c4_final -f python tools/prof_recur.py --launches 3 > gpurun_out/ncu_ring.log 2>&1; tail -2 gpurun_out/ncu_ring.log
