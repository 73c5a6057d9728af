#!/bin/bash
# Round 2: full GPU tests + auto bench lines of every config.
T=${1:-r2o}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; tail -n 3 gpurun_out/pytest_gpu_$T.log
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), [ (k['kernel'], round(k['ms'],3)) for k in d['roofline']['kernels']])" $1 "$2" 2>&1 | tail -1; }
for c in c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${c}_$T.json 2> gpurun_out/bench_${c}_$T.err
  summ gpurun_out/bench_${c}_$T.json "$c auto"
done
