#!/bin/bash
# One ncu --set full capture (with source) of k_solve for a 6-system batch of
# config $1 (default 4).  The report stays on the GPU box (it exceeds what
# gpurun copies back); its details page, DRAM / duration metrics and the
# per-source-line aggregation come back as text in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
c=${1:-4}
rep=/tmp/k_solve_c$c
timeout 600 python tools/solve_phases.py --config $c --groups 6 > gpurun_out/plain_phases_c$c.txt 2>&1; echo "plain rc=$? $(head -2 gpurun_out/plain_phases_c$c.txt | tr '\n' ' ')"
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:k_solve -s 2 -c 1 -f \
  -o $rep python tools/solve_phases.py --config $c --groups 6 > gpurun_out/ncu_c$c.log 2>&1; echo "ncu rc=$?"
ncu -i $rep.ncu-rep --page details 2>/dev/null | grep -v "^\s*$" > gpurun_out/ncu_full_k_solve_c$c.txt
ncu -i $rep.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,smsp__inst_executed.sum 2>/dev/null | tail -3 >> gpurun_out/ncu_full_k_solve_c$c.txt
ncu -i $rep.ncu-rep --page source --csv --print-source cuda,sass > /tmp/k_solve_c${c}_src.csv 2>/dev/null
python tools/ncu_lines.py /tmp/k_solve_c${c}_src.csv 40 > gpurun_out/ncu_k_solve_c${c}_lines.txt 2>&1
rm -f $rep.ncu-rep /tmp/k_solve_c${c}_src.csv
