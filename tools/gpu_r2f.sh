#!/bin/bash
# Round 2: c5 p / cut-rule sweep in the auto orientation + per-task stats (times, blocks).
T=${1:-r2f}
mkdir -p gpurun_out
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), [ (k['kernel'], round(k['ms'],3)) for k in d['roofline']['kernels']])" $1 "$2" 2>&1 | tail -1; }
timeout 900 python tools/task_stats.py c5 16 auto > gpurun_out/tasks_c5_p16_$T.json 2> gpurun_out/tasks_c5_p16_$T.err
for p in 16 24 32 48; do
  for r in 0 1; do
    timeout 900 python bench.py --config c5 --p $p --cut-rule $r --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_c5_p${p}r${r}_$T.json 2> gpurun_out/bench_c5_p${p}r${r}_$T.err
    summ gpurun_out/bench_c5_p${p}r${r}_$T.json "c5 p=$p rule=$r"
  done
done
