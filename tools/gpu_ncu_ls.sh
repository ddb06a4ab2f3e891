#!/bin/bash
# ncu --set full captures (with source) of the least-squares kernels: the
# 128-thread team tier on c3 (k_ls) and the segmented register tier on c2
# (k_ls_seg), one launch each; reports in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_ls -s 6 -c 1 -f \
  -o gpurun_out/k_ls_team_c3 python tools/build_timing.py --config 3 --systems 2 > gpurun_out/ncu_ls_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_ls_seg -s 2 -c 1 -f \
  -o gpurun_out/k_ls_seg_c2 python tools/build_timing.py --config 2 --systems 16 > gpurun_out/ncu_ls_c2.log 2>&1; echo "ncu c2 rc=$?"
