#!/bin/bash
# tools/variant.sh NAME SRC "-DFLAGS..."  -> build/libpicgpu_NAME.so with SRC recompiled under FLAGS
set -e
cd "$(dirname "$0")/.."
python paper_2601_08277_b200/build.py > /dev/null
NAME=$1; SRC=$2; shift 2
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I include -I paper_2601_08277_b200/csrc"
$NVCC $ARCH $FL "$@" -c paper_2601_08277_b200/csrc/$SRC.cu -o build/${SRC}_$NAME.o
OBJS=""
for s in $(python -c "from paper_2601_08277_b200 import build; print(' '.join(x[:-3] for x in build.SOURCES))"); do
  if [ $s == $SRC ]; then OBJS="$OBJS build/${SRC}_$NAME.o"; else OBJS="$OBJS build/$s.o"; fi
done
$NVCC $ARCH -shared --cudart static -o build/libpicgpu_$NAME.so $OBJS
echo build/libpicgpu_$NAME.so
