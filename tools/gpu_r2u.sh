#!/bin/bash
# Round 2: collaborative CPU+GPU (NEXT-3) -- tests + e2e lines at several host shares.
T=${1:-r2u}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_collab.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_collab_$T.log 2>&1; tail -n 3 gpurun_out/pytest_collab_$T.log
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e=d.get('e2e') or {}; print(sys.argv[2], 'dev', round(d.get('ms_per_step'),3), 'e2e', round(e.get('ms_per_step',0),3), 'h2d', e.get('h2d_bytes_per_step'), 'host_ms', e.get('ms_host_share'), d.get('parity',{}).get('match'))" $1 "$2" 2>&1 | tail -1; }
for c in c4 c3; do
  for h in 0 20 50 100 200; do
    timeout 900 python bench.py --config $c --host-permille $h --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_${c}_h${h}_$T.json 2> gpurun_out/bench_${c}_h${h}_$T.err
    summ gpurun_out/bench_${c}_h${h}_$T.json "$c host=$h"
  done
done
