set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_dmma.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3
