set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3
CHEBFD_B200_LIB=$PWD/build/ab/libchebfd_r01.so timeout 600 python tools/band_exp.py --cases c2,c4,c3_256 --bytes -1 --deg 60
timeout 1200 python tools/band_exp.py --cases c4,c3_256,c3_32,c2 --bytes 0,16,32 --dyn 0,1,2,4 --deg 60
CHEBFD_B200_LIB=$PWD/build/ab/libchebfd_r01.so timeout 600 python tools/band_exp.py --cases c2,c4 --bytes -1 --deg 60
