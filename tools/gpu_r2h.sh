#!/bin/bash
# Round 2: c5 with small p (fewer (edge, x) visits, wider held sets) in MID / auto.
T=${1:-r2h}
mkdir -p gpurun_out
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), [ (k['kernel'], round(k['ms'],3)) for k in d['roofline']['kernels']])" $1 "$2" 2>&1 | tail -1; }
for p in 1 2 4 8; do
  for o in mid auto; do
    timeout 600 python bench.py --config c5 --p $p --orient $o --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_c5_p${p}${o}_$T.json 2> gpurun_out/bench_c5_p${p}${o}_$T.err
    summ gpurun_out/bench_c5_p${p}${o}_$T.json "c5 p=$p $o"
  done
done
