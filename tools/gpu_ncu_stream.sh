#!/bin/bash
# Streaming kernels at c4 size: event-timed GB/s, then ncu --set full of one
# k_assemble_multi and one k_spmm launch; text summaries in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/stream_kernels.py --config 4 > gpurun_out/stream_c4.txt 2>&1; echo "plain rc=$?"; tail -3 gpurun_out/stream_c4.txt
for k in k_assemble_multi k_spmm; do
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -f \
    -o /tmp/${k}_c4 python tools/stream_kernels.py --config 4 > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
  ncu -i /tmp/${k}_c4.ncu-rep --page details 2>/dev/null | grep -v "^\s*$" > gpurun_out/ncu_full_${k}_c4.txt
  ncu -i /tmp/${k}_c4.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum 2>/dev/null | tail -3 >> gpurun_out/ncu_full_${k}_c4.txt
  rm -f /tmp/${k}_c4.ncu-rep
done
