set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
# final-code evidence (r02e): plain bench first (exit 0 without ncu), then the launch list of the
# same command and one --set full capture of the dominant kernel
( time timeout 900 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02e_bench_short.json ) 2>&1 | tail -3
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:step_|gram|gemm|Kernel2' -c 900 --csv --log-file gpurun_out/r02e_launches_c4.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02e_ncu_launches.log 2>&1; tail -2 gpurun_out/r02e_ncu_launches.log
timeout 900 python tools/prof_recur.py --launches 3 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ring -c 2 -o gpurun_out/r02e_ring_recur_c4 -f python tools/prof_recur.py --launches 3 > gpurun_out/r02e_ncu_ring.log 2>&1; tail -2 gpurun_out/r02e_ncu_ring.log
