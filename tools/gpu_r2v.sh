#!/bin/bash
# Round 2: heavy-kernel small-held path A/B (main vs nosmall) + parity tests.
T=${1:-r2v}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_orient.py tests/test_gpu_parity.py tests/test_gpu_vertex.py -q -x -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; tail -n 2 gpurun_out/pytest_$T.log
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), [ (k['kernel'], round(k['ms'],3)) for k in d['roofline']['kernels']])" $1 "$2" 2>&1 | tail -1; }
for c in c2 c3 c5; do
  for v in main nosmall; do
    if [ $v = main ]; then unset PGABB_LIB_VARIANT; else export PGABB_LIB_VARIANT=$v; fi
    timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${c}_${v}_$T.json 2> gpurun_out/bench_${c}_${v}_$T.err
    summ gpurun_out/bench_${c}_${v}_$T.json "$c $v"
  done
  unset PGABB_LIB_VARIANT
done
