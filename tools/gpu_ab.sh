#!/bin/bash
# A/B of library variants on the persistent solve: per-phase stamps of one
# 6-system batch (tools/solve_phases.py).
#   tools/gpu_ab.sh "4 2" stamps_stage stamps_nostage   (configs, variant names)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cfgs=$1; shift
for v in "$@"; do
  for c in $cfgs; do
    PMP_LIB=build/variants/libpmorb200_$v.so timeout 900 python tools/solve_phases.py --config $c --groups 6 > gpurun_out/ab_${v}_c$c.txt 2>&1
    echo "$v c$c rc=$? $(head -1 gpurun_out/ab_${v}_c$c.txt)"
  done
done
