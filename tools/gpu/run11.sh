set -x
export PYTHONUNBUFFERED=1
timeout 900 python tools/gram_exp.py --reps 5
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -4
