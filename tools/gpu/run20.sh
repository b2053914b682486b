set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/gputests20.log 2>&1; tail -4 gpurun_out/gputests20.log
( time timeout 1500 python tools/c3.py --kernels lanczos2 > gpurun_out/c3_solve_r20.jsonl ) 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ring -c 2 -o gpurun_out/ring_recur_c4_r20 -f python tools/prof_recur.py --launches 3 > gpurun_out/ncu_ring.log 2>&1; tail -2 gpurun_out/ncu_ring.log
( time timeout 1200 python bench.py > gpurun_out/bench_c4_r20.json ) 2>&1 | tail -3
