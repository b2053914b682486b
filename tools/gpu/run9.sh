set -x
export PYTHONUNBUFFERED=1
timeout 1200 python tools/vgroup_bench.py --ranks 1,2,4 --deg 60 --reps 3
timeout 600 python tools/vgroup_bench.py --ranks 2 --deg 60 --reps 3 --compact 0
