#!/bin/bash
# staged ring (cp.async) A/B + complex tests + sequence tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 4 3; do
  PMP_LIB=build/variants/libpmorb200_stamps_stage.so timeout 600 python tools/solve_phases.py --config $c --groups 6 > gpurun_out/st2_phases_c$c.txt 2>&1; echo "phases c$c rc=$?"
done
if [ -f build/variants/libpmorb200_stamps_rpt4.so ]; then
  PMP_LIB=build/variants/libpmorb200_stamps_rpt4.so timeout 600 python tools/solve_phases.py --config 4 --groups 6 > gpurun_out/rpt4_phases_c4.txt 2>&1; echo "rpt4 rc=$?"
fi
timeout 900 python -m pytest tests/test_gpu_complex.py -x -q > gpurun_out/cx_tests.log 2>&1; echo "cx tests rc=$?"
timeout 1200 python -m pytest tests/test_gpu_sequence.py -x -q > gpurun_out/st2_seq.log 2>&1; echo "seq tests rc=$?"
