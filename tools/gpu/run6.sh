set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo rc=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rc=$?
timeout 300 python tools/prof_recur.py && \
ncu --set full --clock-control none --import-source on -k regex:step_tma -s 5 -c 1 -o gpurun_out/r02_c4_recur python tools/prof_recur.py --launches 5 > gpurun_out/ncu_full.log 2>&1
timeout 300 python tools/prof_recur.py --lattice 64 64 64 --nb 32 && \
ncu --set full --clock-control none --import-source on -k regex:step_tma -s 5 -c 1 -o gpurun_out/r02_c2_recur python tools/prof_recur.py --lattice 64 64 64 --nb 32 --launches 5 >> gpurun_out/ncu_full.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
