#!/bin/bash
# Build a variant of libfastnorm_b200.so for A/B timing (tools/ab_lib.py):
#   bash tools/build_ab.sh NAME [-DFLAG=V ...]   ->  tools/ab/lib_NAME.so
set -e
NAME=$1; shift
SRC=paper_1606_06508_b200/csrc
OBJ=/tmp/fnb_ab_$NAME; mkdir -p $OBJ tools/ab
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="$ARCH -O3 -lineinfo -std=c++17 -fmad=false -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-O2"
pids=()
for f in fastnorm_kernels workloads selftest bounds; do
  nvcc $FLAGS "$@" -DFNB_BUILD_FLAGS="\"ab $NAME $*\"" -c $SRC/$f.cu -o $OBJ/$f.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
nvcc $ARCH -shared -o tools/ab/lib_$NAME.so $OBJ/*.o -lcudart_static -lrt -lpthread -ldl
echo tools/ab/lib_$NAME.so
