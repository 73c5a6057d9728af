#!/bin/bash
# quick iteration: all GPU tests + device-only bench lines for the given configs.
# usage: bash tools/gpu_quick.sh <tag> [configs...]   (extra bench args in $BARGS)
T=${1:-v}; shift
CFGS=${@:-c2 c3 c4 c5}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; tail -4 gpurun_out/pytest_$T.log
for c in $CFGS; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e $BARGS > gpurun_out/bench_$c$T.json 2> gpurun_out/bench_$c$T.err
  python - "$c" "gpurun_out/bench_$c$T.json" <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[2]) if l.startswith('{')][-1])
    r=d['roofline']; print(sys.argv[1], 'ms %.3f'%d['ms_per_step'], 'Eps %.3e'%d['value'], 'frac %.3f'%r['frac'], 'T', d['config']['triangles'], d.get('parity',{}).get('match'))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
  tail -1 gpurun_out/bench_$c$T.err
done
