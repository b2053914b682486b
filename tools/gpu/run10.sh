set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_vgroup.py -x -q 2>&1 | tail -3
timeout 1500 python tests/golden/make_c3s_golden.py --out gpurun_out/c3s_solve.json 2>&1 | tail -5
cp gpurun_out/c3s_solve.json tests/golden/c3s_solve.json
timeout 1800 python -m pytest tests/test_gpu_c3.py -x -q -rA 2>&1 | tail -15
timeout 1200 python tools/vgroup_bench.py --ranks 1,2,4 --deg 60 --reps 3
