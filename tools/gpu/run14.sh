set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo rc=$?
