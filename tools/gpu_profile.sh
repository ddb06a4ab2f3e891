#!/bin/bash
# Profiling session: cold-path host profile, per-phase stamps of k_solve at
# c4 and c2 (stamps variant), launch list + one ncu --set full of k_solve at
# c4 (6 systems).  Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/cold_profile.py --config 2 > gpurun_out/cold_c2.txt 2>&1; echo "cold c2 rc=$?"
timeout 900 python tools/cold_profile.py --config 4 > gpurun_out/cold_c4.txt 2>&1; echo "cold c4 rc=$?"
if [ -f build/variants/libpmorb200_stamps.so ]; then
  PMP_LIB=build/variants/libpmorb200_stamps.so timeout 600 python tools/solve_phases.py --config 4 --groups 6 > gpurun_out/phases_c4_g6.txt 2>&1; echo "phases c4 rc=$?"
  PMP_LIB=build/variants/libpmorb200_stamps.so timeout 600 python tools/solve_phases.py --config 2 --groups 6 > gpurun_out/phases_c2_g6.txt 2>&1; echo "phases c2 rc=$?"
fi
if [ "$NCU" = 1 ]; then
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_solve -c 1 \
    -o gpurun_out/k_solve_c4 python tools/solve_phases.py --config 4 --groups 6 > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"
fi
