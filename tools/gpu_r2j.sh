#!/bin/bash
# Round 2: multi-rank library tests, rule parity; c3/c4 p sweeps (LOW/auto).
T=${1:-r2j}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/pytest_dist_$T.log 2>&1; tail -n 3 gpurun_out/pytest_dist_$T.log
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), [ (k['kernel'], round(k['ms'],3)) for k in d['roofline']['kernels']])" $1 "$2" 2>&1 | tail -1; }
for p in 4 8 12 16 24 32; do
  timeout 600 python bench.py --config c3 --p $p --orient low --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c3_p${p}_$T.json 2> gpurun_out/bench_c3_p${p}_$T.err
  summ gpurun_out/bench_c3_p${p}_$T.json "c3 p=$p low"
done
for p in 1 2 3 4 6; do
  timeout 600 python bench.py --config c4 --p $p --orient low --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c4_p${p}_$T.json 2> gpurun_out/bench_c4_p${p}_$T.err
  summ gpurun_out/bench_c4_p${p}_$T.json "c4 p=$p low"
done
