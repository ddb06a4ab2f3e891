for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then L=""; else L="PMP_LIB=build/variants/libpmorb200_$v.so"; fi
  for rep in 1 2; do
    env $L python bench.py --batch 6 --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/ab_$v.log 2>&1
    echo $v $(tail -1 gpurun_out/ab_$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['phases_s']['solve']*1e3,2))")
  done
done
