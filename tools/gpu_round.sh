#!/bin/bash
# One GPU session: GPU tests, smoke, c2 + c4 bench lines (logs in gpurun_out/).
# usage: tools/gpu_round.sh [tests|smoke|c2|c4|all]...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
what=${@:-all}
for w in $what; do
  case $w in
    tests|all) timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" ;;
  esac
  case $w in
    smoke|all) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" ;;
  esac
  case $w in
    c2|all) timeout 900 python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?" ;;
  esac
  case $w in
    c4|all) timeout 1800 python bench.py --config 4 --steps 2 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?" ;;
  esac
done
