#!/bin/bash
# Build libpmorb200.so in-tree for sm_100a (called by __graft_entry__.build()).
# Sources compile in parallel into build/, then link into the package.
set -e
cd "$(dirname "$0")"
NVCC=${NVCC:-nvcc}
FLAGS="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I include"
SRC=paper_1809_06574_b200/csrc
mkdir -p build
objs=()
pids=()
for f in structure assemble ls blockops orth cycle solve gcro_host peak cplx; do
  $NVCC $FLAGS -c $SRC/$f.cu -o build/$f.o &
  pids+=($!)
  objs+=(build/$f.o)
done
for f in hostls comm; do
  $NVCC $FLAGS -c $SRC/$f.cpp -o build/$f.o &
  pids+=($!)
  objs+=(build/$f.o)
done
for p in "${pids[@]}"; do wait $p; done
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o paper_1809_06574_b200/libpmorb200.so "${objs[@]}" -ldl
