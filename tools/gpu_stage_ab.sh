#!/bin/bash
# staged-ring A/B: phases (stamps build), sequence goldens, short c4 bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 4 3 2; do
  PMP_LIB=build/variants/libpmorb200_stamps_stage.so timeout 600 python tools/solve_phases.py --config $c --groups 6 > gpurun_out/st_phases_c$c.txt 2>&1; echo "phases c$c rc=$?"
done
timeout 1200 python -m pytest tests/test_gpu_sequence.py -x -q > gpurun_out/st_seq.log 2>&1; echo "seq tests rc=$?"
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-warm > gpurun_out/st_bench_c4.json 2> gpurun_out/st_bench_c4.err; echo "bench c4 rc=$?"
