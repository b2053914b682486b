set -x
export PYTHONUNBUFFERED=1
( time timeout 2400 python -m pytest tests -m gpu -x -q ) 2>&1 | tail -6
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) 2>&1 | tail -5
( time timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4_full.json ) 2>&1 | tail -4
( time timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_full.json ) 2>&1 | tail -4
