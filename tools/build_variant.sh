#!/bin/bash
# Build a variant of libpmorb200.so with extra nvcc defines (A/B experiments):
#   tools/build_variant.sh NAME -DFOO=1 ...   -> build/variants/libpmorb200_NAME.so
# select it at run time with PMP_LIB=build/variants/libpmorb200_NAME.so
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
FLAGS="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I include $*"
SRC=paper_1809_06574_b200/csrc
OUT=build/variants/$NAME
mkdir -p $OUT
objs=()
pids=()
for f in structure assemble ls blockops orth cycle solve gcro_host peak cplx; do
  nvcc $FLAGS -c $SRC/$f.cu -o $OUT/$f.o &
  pids+=($!)
  objs+=($OUT/$f.o)
done
for f in hostls comm; do
  nvcc $FLAGS -c $SRC/$f.cpp -o $OUT/$f.o &
  pids+=($!)
  objs+=($OUT/$f.o)
done
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/libpmorb200_$NAME.so "${objs[@]}" -ldl
echo build/variants/libpmorb200_$NAME.so
