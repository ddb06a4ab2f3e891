#!/bin/bash
# Build libpmorb200.so in-tree for sm_100a (called by __graft_entry__.build()).
# Sources compile in parallel into build/, then link into the package.  An
# object is rebuilt when its source, any csrc header or the public header is
# newer (PMP_REBUILD=1 forces everything).
set -e
cd "$(dirname "$0")"
NVCC=${NVCC:-nvcc}
FLAGS="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I include"
SRC=paper_1809_06574_b200/csrc
mkdir -p build
stale() {  # stale OBJ SRC
  [ -n "$PMP_REBUILD" ] && return 0
  [ ! -f "$1" ] && return 0
  [ "$2" -nt "$1" ] && return 0
  for h in $SRC/*.cuh include/*.h build.sh; do [ "$h" -nt "$1" ] && return 0; done
  return 1
}
objs=()
pids=()
for f in structure assemble ls blockops orth cycle solve gcro_host peak cplx; do
  if stale build/$f.o $SRC/$f.cu; then
    $NVCC $FLAGS -c $SRC/$f.cu -o build/$f.o &
    pids+=($!)
  fi
  objs+=(build/$f.o)
done
for f in hostls comm; do
  if stale build/$f.o $SRC/$f.cpp; then
    $NVCC $FLAGS -c $SRC/$f.cpp -o build/$f.o &
    pids+=($!)
  fi
  objs+=(build/$f.o)
done
for p in "${pids[@]}"; do wait $p; done
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o paper_1809_06574_b200/libpmorb200.so "${objs[@]}" -ldl
