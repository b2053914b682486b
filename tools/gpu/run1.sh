set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python tools/band_exp.py --cases c4,c3_256,c3_32,c2 --bytes 0,4,8,16,32,64 2>&1
