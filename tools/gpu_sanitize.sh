#!/bin/bash
# compute-sanitizer over the benchmarked composition on a small sequence
# (memcheck / synccheck / racecheck; logs in gpurun_out/sanitize_*.log).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py 16 > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'ERROR SUMMARY' gpurun_out/sanitize_$tool.log) $(grep 'ERROR SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
