set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:step_|gram|gemm|Kernel2" -c 900 --csv --log-file gpurun_out/launches_c4_r18.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; tail -2 gpurun_out/ncu_launches.log
( time timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref_r18.json ) 2>&1 | tail -4
( time timeout 600 python bench.py --workload c2 > gpurun_out/bench_c2_r18.json ) 2>&1 | tail -4
( time timeout 1500 python tools/c3.py --kernels lanczos2 > gpurun_out/c3_solve_r18.jsonl ) 2>&1 | tail -4
