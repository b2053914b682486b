#!/bin/bash
# A/B builds: recompile the given translation units with extra nvcc flags and link a variant
# library from them plus the default build's other objects.
#   tools/build_variant.sh NAME "-DCFD_FOO=1" step_gc.cu [more.cu]   -> variants/NAME.so
# Use with CHEBFD_B200_LIB=variants/NAME.so.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; FLAGS=$2; shift 2
SRC=$ROOT/paper_1510_04895_b200/csrc
OBJ=$ROOT/build/obj
VOBJ=$ROOT/build/var_$NAME
mkdir -p "$VOBJ" "$ROOT/variants"
OBJS=""
for f in "$OBJ"/*.o; do
  b=$(basename "$f" .o); skip=0
  for t in "$@"; do [ "$b" = "${t%.cu}" ] && skip=1; done
  [ $skip = 0 ] && OBJS="$OBJS $f"
done
for t in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -DCFD_EXPERIMENTAL=0 -std=c++20 -O3 -lineinfo \
    -ccbin /usr/bin/g++ -Xcompiler -fPIC --expt-relaxed-constexpr $FLAGS -c "$SRC/$t" -o "$VOBJ/${t%.cu}.o" &
done
wait
for t in "$@"; do OBJS="$OBJS $VOBJ/${t%.cu}.o"; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o "$ROOT/variants/$NAME.so" $OBJS \
  -L/usr/local/cuda/lib64 -lcublas -lcusolver -lnccl -lpthread -Xlinker -rpath,/usr/local/cuda/lib64
echo "built variants/$NAME.so"
