#!/bin/bash
# A/B of library variants on the bench (c2 sequence): LIBS="name=path ..."
# ("main" = the in-tree library).  Two repetitions each, interleaved.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
  for kv in ${LIBS:-main=}; do
    name=${kv%%=*}; path=${kv#*=}
    if [ -n "$path" ]; then L="PMP_LIB=$path"; else L=""; fi
    env $L python bench.py --no-cpu-baseline --no-e2e --steps 5 ${BENCH_ARGS} > gpurun_out/ab_${name}_$rep.log 2>&1
    echo $name rep$rep $(tail -1 gpurun_out/ab_${name}_$rep.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); k=d['kernels']; print('ms', round(d['ms_per_step'],2), 'solve', round(d['phases_s']['solve']*1e3,2), 'build', round(d['phases_s']['build']*1e3,3), 'ls_multi', round(k.get('pmp_ls_columns_multi',{}).get('total_ms',0),3), 'iters', d['iterations']['mean'])" 2>&1 | tail -1)
  done
done
