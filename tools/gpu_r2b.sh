#!/bin/bash
# Round 2: orientation (R25) validation -- GPU tests, then per-config bench lines (auto, low).
T=${1:-r2b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_orient.py -x -q -p no:cacheprovider > gpurun_out/pytest_orient_$T.log 2>&1; tail -n 15 gpurun_out/pytest_orient_$T.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_orient.py > gpurun_out/pytest_gpu_$T.log 2>&1; tail -n 15 gpurun_out/pytest_gpu_$T.log
for c in c2 c3 c4 c5; do
  for o in auto low; do
    timeout 900 python bench.py --config $c --orient $o --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${c}_${o}_$T.json 2> gpurun_out/bench_${c}_${o}_$T.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], d.get('ms_per_step'), d.get('parity',{}).get('match'), [ (k['kernel'], round(k['ms'],3)) for k in d['roofline']['kernels']], d['roofline'].get('items'))" gpurun_out/bench_${c}_${o}_$T.json $c $o 2>&1 | tail -1
  done
done
