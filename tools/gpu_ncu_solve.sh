#!/bin/bash
# One ncu --set full capture (with source) of k_solve for a 6-system batch of
# config $1 (default 4); report in gpurun_out/k_solve_c$1.ncu-rep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
c=${1:-4}
timeout 600 python tools/solve_phases.py --config $c --groups 6 > gpurun_out/plain_phases_c$c.txt 2>&1; echo "plain rc=$? $(head -1 gpurun_out/plain_phases_c$c.txt)"
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:k_solve -s 2 -c 1 -f \
  -o gpurun_out/k_solve_c$c python tools/solve_phases.py --config $c --groups 6 > gpurun_out/ncu_c$c.log 2>&1; echo "ncu rc=$?"
