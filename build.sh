#!/bin/bash
# Build libpmorb200.so in-tree for sm_100a (called by __graft_entry__.build()).
set -e
cd "$(dirname "$0")"
NVCC=${NVCC:-nvcc}
$NVCC -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 \
  -Xcompiler -fPIC -shared -I include \
  -o paper_1809_06574_b200/libpmorb200.so \
  paper_1809_06574_b200/csrc/structure.cu paper_1809_06574_b200/csrc/assemble.cu \
  paper_1809_06574_b200/csrc/ls.cu paper_1809_06574_b200/csrc/blockops.cu paper_1809_06574_b200/csrc/orth.cu \
  paper_1809_06574_b200/csrc/hostls.cpp
