#!/bin/bash
# Round 2: full GPU tests with R25 auto rule, then A/B bench lines: round-1 library
# (variant r2base) vs this build in auto / low / mid orientation.
T=${1:-r2c}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; tail -n 5 gpurun_out/pytest_gpu_$T.log
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), [ (k['kernel'], round(k['ms'],3)) for k in d['roofline']['kernels']], d['roofline'].get('items'))" $1 "$2" 2>&1 | tail -1; }
for c in c2 c3 c4 c5; do
  PGABB_LIB_VARIANT=r2base timeout 900 python bench.py --config $c --orient low --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${c}_base_$T.json 2> gpurun_out/bench_${c}_base_$T.err
  summ gpurun_out/bench_${c}_base_$T.json "$c base"
  for o in auto low mid; do
    timeout 900 python bench.py --config $c --orient $o --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${c}_${o}_$T.json 2> gpurun_out/bench_${c}_${o}_$T.err
    summ gpurun_out/bench_${c}_${o}_$T.json "$c $o"
  done
done
