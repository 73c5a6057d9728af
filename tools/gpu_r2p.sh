#!/bin/bash
# Round 2: NEXT-row paths with the R25 orientation: per-vertex t(v), components,
# streamed c5 through a budget; default bench line with e2e + cpu baseline.
T=${1:-r2p}
mkdir -p gpurun_out
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), (d.get('e2e') or {}).get('ms_per_step'), d.get('roofline',{}).get('kernel'))" $1 "$2" 2>&1 | tail -1; }
for c in c2 c5; do
  for o in auto low; do
    timeout 900 python bench.py --config $c --path vertex --orient $o --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_vtx_${c}_${o}_$T.json 2> gpurun_out/bench_vtx_${c}_${o}_$T.err
    summ gpurun_out/bench_vtx_${c}_${o}_$T.json "vertex $c $o"
  done
done
timeout 900 python bench.py --config c5 --budget-gb 16 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c5b16_$T.json 2> gpurun_out/bench_c5b16_$T.err
summ gpurun_out/bench_c5b16_$T.json "c5 budget 16GB auto"
timeout 900 python bench.py --config c5 --budget-gb 16 --orient low --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c5b16low_$T.json 2> gpurun_out/bench_c5b16low_$T.err
summ gpurun_out/bench_c5b16low_$T.json "c5 budget 16GB low"
timeout 900 python bench.py > gpurun_out/bench_default_$T.json 2> gpurun_out/bench_default_$T.err
summ gpurun_out/bench_default_$T.json "default"
