#!/bin/bash
# A/B of library variants: per-phase stamps (stamps_<v>) and c2 bench lines.
# usage: tools/ab_phases.sh v1 v2 ...   (build/variants/libpmorb200_<v>.so)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  if [ -f build/variants/libpmorb200_stamps_$v.so ]; then
    for c in 4 2; do
      PMP_LIB=build/variants/libpmorb200_stamps_$v.so timeout 600 python tools/solve_phases.py --config $c --groups 6 > gpurun_out/ab_phases_${v}_c$c.txt 2>&1
    done
  fi
  if [ -f build/variants/libpmorb200_$v.so ]; then
    PMP_LIB=build/variants/libpmorb200_$v.so timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_bench_${v}_c2.json 2>gpurun_out/ab_bench_${v}_c2.err
  fi
  echo "$v done"
done
