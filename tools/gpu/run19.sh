set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/gputests19.log 2>&1; tail -4 gpurun_out/gputests19.log
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) 2>&1 | tail -3
( time timeout 1200 python bench.py > gpurun_out/bench_c4_r19.json ) 2>&1 | tail -4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ring -c 4 -o gpurun_out/ring_recur_c3_256 -f python tools/prof_recur.py --lattice 128 128 64 --nb 256 --launches 1 > gpurun_out/ncu_ring_c3.log 2>&1; tail -2 gpurun_out/ncu_ring_c3.log
