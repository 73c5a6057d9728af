#!/bin/bash
# Round 2: LOW-path regression A/B (variants) + ncu --set full of the MID k_tc_rows on c5.
T=${1:-r2d}
mkdir -p gpurun_out
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), [ (k['kernel'], round(k['ms'],3)) for k in d['roofline']['kernels']])" $1 "$2" 2>&1 | tail -1; }
for c in c2 c3 c5s; do
  for v in r2base main npos chunk both; do
    if [ $v = main ]; then unset PGABB_LIB_VARIANT; else export PGABB_LIB_VARIANT=$v; fi
    timeout 900 python bench.py --config $c --orient low --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${c}_${v}_$T.json 2> gpurun_out/bench_${c}_${v}_$T.err
    summ gpurun_out/bench_${c}_${v}_$T.json "$c $v"
  done
  unset PGABB_LIB_VARIANT
done
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:"k_tc_rows" -c 1 -o gpurun_out/prof_c5mid$T -f python bench.py --config c5 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full_c5mid$T.log 2>&1
tail -n 2 gpurun_out/ncu_full_c5mid$T.log
