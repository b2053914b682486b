set -x
export PYTHONUNBUFFERED=1
timeout 900 python tools/gram_exp.py --tsgemm
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3
timeout 900 python tools/c3.py --kernels lanczos2 2>&1 | tail -1 | cut -c1-900
