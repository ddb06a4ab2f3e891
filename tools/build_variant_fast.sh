#!/bin/bash
# Variant of libpmorb200.so that differs from the in-tree build only in
# solve.cu's compile flags (k_solve experiments): compiles solve.cu with the
# extra defines and links it with the main build's other objects.
#   tools/build_variant_fast.sh NAME -DFOO=1 ...  -> build/variants/libpmorb200_NAME.so
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
FLAGS="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I include $*"
mkdir -p build/variants/$NAME
nvcc $FLAGS -c paper_1809_06574_b200/csrc/solve.cu -o build/variants/$NAME/solve.o
objs=()
for f in structure assemble ls blockops orth cycle gcro_host peak cplx hostls comm; do objs+=(build/$f.o); done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/libpmorb200_$NAME.so build/variants/$NAME/solve.o "${objs[@]}" -ldl
echo build/variants/libpmorb200_$NAME.so
