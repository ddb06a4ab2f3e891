#!/bin/bash
# Streaming kernels at c4 size: event-timed GB/s, then ncu --set full of one
# k_assemble_multi and one k_spmm launch (reports in gpurun_out/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/stream_kernels.py --config 4 > gpurun_out/stream_c4.txt 2>&1; echo "plain rc=$?"; cat gpurun_out/stream_c4.txt | tail -3
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_assemble_multi -s 1 -c 1 -f \
  -o gpurun_out/k_assemble_multi_c4 python tools/stream_kernels.py --config 4 > gpurun_out/ncu_asm.log 2>&1; echo "ncu asm rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_spmm -s 1 -c 1 -f \
  -o gpurun_out/k_spmm_c4 python tools/stream_kernels.py --config 4 > gpurun_out/ncu_spmm.log 2>&1; echo "ncu spmm rc=$?"
